# per-launch device time and DRAM bytes for the bench command of each config (cold-cache, serialised)
set -x
for c in ${CONFIGS:-c2:f64 c3:f64 c4:f64 c5:f64 c5:f32}; do
  cfg=${c%%:*}; dt=${c#*:}
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c ${NLAUNCH:-60} --csv --log-file gpurun_out/launches_${cfg}_${dt}.csv python bench.py --config $cfg --dtype $dt --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/launches_${cfg}_${dt}.csv | head -20
done
