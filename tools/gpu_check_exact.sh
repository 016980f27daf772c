mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu -k "c5 or long or workloads or sharded or engine or f32 or float32" 2>&1 | tail -3
for i in 1 2; do timeout 600 python bench.py --config c5 --dtype f32 --steps 30 --warmup 5 --no-cpu > gpurun_out/cut_c5_f32.json 2>/dev/null; python tools/bench_brief.py gpurun_out/cut_c5_f32.json | tail -1; done
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_run.py 2>&1 | tail -3
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_run.py 2>&1 | tail -3
