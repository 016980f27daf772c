mkdir -p gpurun_out
for pk in 0 1 0 1; do
 for dt in f64 f32; do
  RIMDP_TINY_PACK=$pk timeout 600 python bench.py --config c5 --dtype $dt --steps 30 --warmup 5 > gpurun_out/ab_c5_${dt}_pk$pk.json 2>/dev/null
  python tools/bench_brief.py gpurun_out/ab_c5_${dt}_pk$pk.json | tail -1 | sed "s/^/pk=$pk /"
 done
done
timeout 900 python -m pytest tests -q -x -m gpu -k "c5 or tiny or long or workloads or engine" 2>&1 | tail -3
