#!/bin/bash
# ncu launch lists with DRAM bytes for every config -> profiles/ncu_traffic.json (run under gpurun)
tag=${1:-r2}
mkdir -p gpurun_out/launch
for cfg in "c2 f64" "c3 f64" "c5 f64" "c5 f32" "c4 f64"; do
  set -- $cfg
  n=300; [ "$1" = "c4" ] && n=40
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -c $n --csv --log-file gpurun_out/launch/launches_$1_$2_$tag.csv \
      python bench.py --config $1 --dtype $2 --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
  python tools/traffic_update.py $1_$2 gpurun_out/launch/launches_$1_$2_$tag.csv
  python tools/launch_summary.py gpurun_out/launch/launches_$1_$2_$tag.csv > gpurun_out/launch/launches_$1_$2_$tag.txt
done
cp profiles/ncu_traffic.json gpurun_out/launch/ncu_traffic.json
