# smoke, full GPU parity suite, reference arm, bench lines for every config (no ncu)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS} 2>&1 | tail -25
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -2 gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
for c in ${CONFIGS:-c2 c3 c5:f64 c5:f32 c4}; do
  cfg=${c%%:*}; dt=${c#*:}; [ "$dt" = "$c" ] && dt=f64
  timeout ${BENCH_TIMEOUT:-900} python bench.py --config $cfg --dtype $dt --steps ${STEPS:-100} --warmup 5 ${BENCH_ARGS} > gpurun_out/bench_${cfg}_${dt}.json 2> gpurun_out/bench_${cfg}_${dt}.err
  tail -4 gpurun_out/bench_${cfg}_${dt}.err
  python tools/bench_brief.py gpurun_out/bench_${cfg}_${dt}.json
done
