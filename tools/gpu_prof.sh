# GPU tests (optional) then full ncu captures: FULL="cfg:dtype:kernel_regex ..."
set -x
if [ -n "$TESTS" ]; then timeout 1500 python -m pytest $TESTS -x -q 2>&1 | tail -15; fi
IFS=";" read -ra SPECS <<< "$FULL"
for spec in "${SPECS[@]}"; do
  cfg=${spec%%:*}; rest=${spec#*:}; dt=${rest%%:*}; kern=${rest#*:}
  tag=$(echo $kern | tr -c 'a-zA-Z0-9_' '_')
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$kern" -s ${SKIP:-2} -c 1 -o gpurun_out/prof_${cfg}_${tag} python bench.py --config $cfg --dtype $dt --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_f_${cfg}_${tag}.log 2>&1; tail -2 gpurun_out/ncu_f_${cfg}_${tag}.log
done
