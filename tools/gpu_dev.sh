# development loop: smoke, selected GPU tests, bench lines (no cpu baseline), optional launch lists
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest ${TESTS:-tests -m gpu} -x -q 2>&1 | tail -15
for c in ${CONFIGS:-c2:f64}; do
  cfg=${c%%:*}; dt=${c#*:}
  timeout ${BENCH_TIMEOUT:-900} python bench.py --config $cfg --dtype $dt --steps ${STEPS:-50} --warmup 5 --no-cpu ${BENCH_ARGS} > gpurun_out/bench_${cfg}_${dt}.json 2> gpurun_out/bench_${cfg}_${dt}.err
  tail -2 gpurun_out/bench_${cfg}_${dt}.err
  python tools/bench_brief.py gpurun_out/bench_${cfg}_${dt}.json
done
for c in ${LAUNCHES}; do
  cfg=${c%%:*}; dt=${c#*:}
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NLAUNCH:-80} --csv --log-file gpurun_out/launches_${cfg}_${dt}.csv python bench.py --config $cfg --dtype $dt --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/launches_${cfg}_${dt}.csv
done
