# experiment: engine variants (env) per config, bench lines only; optional ncu capture
# usage: EXPS="c5:f64:RIMDP_STREAMS=4 c4:f64:RIMDP_MEDIUM_BLOCKS=4" bash tools/gpu_exp.sh
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
if [ -n "$TESTS" ]; then timeout 1200 python -m pytest tests -m gpu -x -q $TESTS 2>&1 | tail -3; fi
for x in $EXPS; do
  cfg=$(echo $x | cut -d: -f1); dt=$(echo $x | cut -d: -f2); envs=$(echo $x | cut -d: -f3- | tr ',' ' ')
  env $envs timeout ${BENCH_TIMEOUT:-600} python bench.py --config $cfg --dtype $dt --steps ${STEPS:-100} --warmup 5 --no-cpu ${NOE2E:+--no-e2e} > gpurun_out/exp.json 2> gpurun_out/exp.err || tail -5 gpurun_out/exp.err
  echo -n "$x  "; python tools/bench_brief.py gpurun_out/exp.json | cut -c1-200
done
if [ -n "$NCU_KERNEL" ]; then
  env $NCU_ENV timeout 900 ncu --set full --clock-control none --import-source on -k regex:$NCU_KERNEL -s ${NCU_SKIP:-6} -c 1 -o gpurun_out/prof_${NCU_TAG:-x} python bench.py --config ${NCU_CFG:-c5} --dtype ${NCU_DT:-f64} --steps 10 --warmup 3 --no-cpu > gpurun_out/ncu_${NCU_TAG:-x}.log 2>&1; tail -2 gpurun_out/ncu_${NCU_TAG:-x}.log
fi
