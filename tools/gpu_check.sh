# sanity: smoke, GPU parity tests, default bench line
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 600 python bench.py > gpurun_out/bench_check.json 2> gpurun_out/bench_check.err; tail -3 gpurun_out/bench_check.err
cat gpurun_out/bench_check.json
