# quick iteration: parity tests, bench, launch list, one full ncu capture of the top kernel
TAG=${TAG:-x}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 600 python bench.py --steps 200 --warmup 10 ${BENCH_ARGS} > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -2 gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 20 --warmup 3 --no-cpu ${BENCH_ARGS} > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KERNEL:-omax_short} -s 6 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 10 --warmup 3 --no-cpu ${BENCH_ARGS} > gpurun_out/ncu_$TAG.log 2>&1; tail -2 gpurun_out/ncu_$TAG.log
