#!/bin/bash
# Round-2 bench lines (one B200): every config, both arms of the default config.
# usage: tools/gpu_round2.sh TAG   -> gpurun_out/bench_<cfg>_<TAG>.json
tag=${1:-r2}
mkdir -p gpurun_out
timeout 600 python bench.py --steps 200 --warmup 10 > gpurun_out/bench_default_$tag.json 2> gpurun_out/bench_default_$tag.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference_c2_$tag.json 2> /dev/null
for cfg in "c3 f64" "c4 f64" "c5 f64" "c5 f32"; do
  set -- $cfg
  timeout 900 python bench.py --config $1 --dtype $2 --steps 50 --warmup 5 > gpurun_out/bench_$1_$2_$tag.json 2> gpurun_out/bench_$1_$2_$tag.err
done
python tools/bench_brief.py gpurun_out/bench_*_$tag.json
