#!/bin/bash
# A/B of an engine env switch on C5: tools/ab_env.sh VAR VALUE_A VALUE_B [configs...] (run under gpurun)
var=$1; a=$2; b=$3; shift 3
cfgs=${@:-"c5:f64 c5:f32"}
mkdir -p gpurun_out
for rep in 1 2; do
 for val in "$a" "$b"; do
  for cd in $cfgs; do
   cfg=${cd%%:*}; dt=${cd##*:}
   env $var=$val timeout 600 python bench.py --config $cfg --dtype $dt --steps 30 --warmup 5 --no-cpu > gpurun_out/ab_${cfg}_${dt}_$val.json 2>/dev/null
   python tools/bench_brief.py gpurun_out/ab_${cfg}_${dt}_$val.json | tail -1 | sed "s/^/$var=$val /"
  done
 done
done
