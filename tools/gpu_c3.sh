set -x
timeout 900 python bench.py --config c3 --steps 50 --warmup 5 --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -3 gpurun_out/bench_c3.err
cat gpurun_out/bench_c3.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 10 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:omax_long -s 4 -c 1 -o gpurun_out/prof_c3long python bench.py --config c3 --steps 10 --warmup 3 --no-cpu > gpurun_out/ncu_c3.log 2>&1; tail -2 gpurun_out/ncu_c3.log
