# parity tests, then bench lines for the listed configs (no ncu)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
if [ -z "$SKIP_TESTS" ]; then timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} 2>&1 | tail -15; fi
for c in ${CONFIGS:-c2}; do
  cfg=${c%%:*}; dt=${c#*:}; [ "$dt" = "$c" ] && dt=f64
  timeout ${BENCH_TIMEOUT:-900} python bench.py --config $cfg --dtype $dt --steps ${STEPS:-200} --warmup 10 ${BENCH_ARGS} > gpurun_out/bench_${cfg}_${dt}.json 2> gpurun_out/bench_${cfg}_${dt}.err
  tail -4 gpurun_out/bench_${cfg}_${dt}.err
  python tools/bench_brief.py gpurun_out/bench_${cfg}_${dt}.json
done
