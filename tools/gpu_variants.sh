# parity + bench under several engine variants (env), no ncu
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in ${VARIANTS:-"RIMDP_SHORT_BLOCKS=4" "RIMDP_SHORT_BLOCKS=5"}; do
  env $v timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu ${BENCH_ARGS} > gpurun_out/var.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/var.json'));r=d['roofline'];print('$v', 'ms/step %.4f'%d['ms_per_step'], 'kernel %.4f'%r['launch_ms'], 'frac %.3f'%r['frac'], 'e2e %.3fs'%d['e2e']['seconds_to_convergence'], 'exact', d['e2e']['values_bit_exact_vs_reference'])"
done
