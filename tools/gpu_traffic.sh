#!/bin/bash
# ncu launch lists with DRAM bytes for every config -> profiles/ncu_traffic.json (run under gpurun)
# usage: tools/gpu_traffic.sh TAG   (CONFIGS="c5:f64 c5:f32" to restrict)
tag=${1:-r2}
mkdir -p gpurun_out/launch
for cd in ${CONFIGS:-c2:f64 c3:f64 c5:f64 c5:f32 c4:f64}; do
  cfg=${cd%%:*}; dt=${cd##*:}
  n=300; [ "$cfg" = "c4" ] && n=40
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -c $n --csv --log-file gpurun_out/launch/launches_${cfg}_${dt}_$tag.csv \
      python bench.py --config $cfg --dtype $dt --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
  python tools/traffic_update.py ${cfg}_${dt} gpurun_out/launch/launches_${cfg}_${dt}_$tag.csv
  python tools/launch_summary.py gpurun_out/launch/launches_${cfg}_${dt}_$tag.csv > gpurun_out/launch/launches_${cfg}_${dt}_$tag.txt
done
cp profiles/ncu_traffic.json gpurun_out/launch/ncu_traffic.json
