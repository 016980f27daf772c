#!/bin/bash
# A/B of alternative in-tree builds: tools/ab_lib.sh CFG:DT NAME=LIBPATH ... (run under gpurun; NAME=default
# for the in-tree library)
cd_=$1; shift
cfg=${cd_%%:*}; dt=${cd_##*:}
mkdir -p gpurun_out
for rep in 1 2; do
  for spec in "$@"; do
    name=${spec%%=*}; lib=${spec#*=}
    if [ "$lib" = "default" ]; then unset RIMDP_B200_LIB; else export RIMDP_B200_LIB=$lib; fi
    timeout 600 python bench.py --config $cfg --dtype $dt --steps 30 --warmup 5 --no-cpu > gpurun_out/ablib_${cfg}_${dt}_$name.json 2>/dev/null
    python tools/bench_brief.py gpurun_out/ablib_${cfg}_${dt}_$name.json | tail -1 | sed "s/^/$name /"
  done
done
unset RIMDP_B200_LIB
