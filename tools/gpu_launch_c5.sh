#!/bin/bash
# ncu launch lists (time + DRAM bytes) of C5 f64 and f32 only (run under gpurun)
tag=${1:-r2}
mkdir -p gpurun_out/launch
for dt in f64 f32; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -c 300 --csv --log-file gpurun_out/launch/launches_c5_${dt}_$tag.csv \
      python bench.py --config c5 --dtype $dt --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/launch/launches_c5_${dt}_$tag.csv > gpurun_out/launch/launches_c5_${dt}_$tag.txt
done
