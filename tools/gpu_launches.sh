# ncu launch lists (per-kernel durations) for the listed configs, plus optional full captures
set -x
for c in ${CONFIGS:-c5:f64 c3:f64 c4:f64}; do
  cfg=${c%%:*}; dt=${c#*:}
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NLAUNCH:-80} --csv --log-file gpurun_out/launches_${cfg}_${dt}.csv python bench.py --config $cfg --dtype $dt --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_l_${cfg}.log 2>&1; tail -2 gpurun_out/ncu_l_${cfg}.log
done
for spec in ${FULL}; do
  cfg=${spec%%:*}; rest=${spec#*:}; dt=${rest%%:*}; kern=${rest#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kern -s ${SKIP:-4} -c 1 -o gpurun_out/prof_${cfg}_${kern} python bench.py --config $cfg --dtype $dt --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_f_${cfg}.log 2>&1; tail -2 gpurun_out/ncu_f_${cfg}.log
done
