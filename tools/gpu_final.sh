# round-end evidence: launch lists (+ DRAM) -> ncu_traffic.json, smoke, GPU tests, reference arm, bench lines,
# one ncu --set full capture of the default config's column kernel.  TAG names the files under profiles/round1/.
set -x
TAG=${TAG:-final}
P=gpurun_out/final; mkdir -p $P
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
for c in ${LCONFIGS:-c2:f64 c3:f64 c5:f64 c5:f32}; do
  cfg=${c%%:*}; dt=${c#*:}
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c ${NLAUNCH:-60} --csv --log-file $P/launches_${cfg}_${dt}_${TAG}.csv python bench.py --config $cfg --dtype $dt --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
  python tools/launch_summary.py $P/launches_${cfg}_${dt}_${TAG}.csv > $P/launches_${cfg}_${dt}_${TAG}.txt
  python tools/traffic_update.py ${cfg}_${dt} $P/launches_${cfg}_${dt}_${TAG}.csv
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -5
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $P/bench_reference_c2_${TAG}.json 2> gpurun_out/bench_ref.err; cat $P/bench_reference_c2_${TAG}.json
timeout 600 python bench.py > $P/bench_default_${TAG}.json 2> gpurun_out/bench_default.err; python tools/bench_brief.py $P/bench_default_${TAG}.json
for c in ${CONFIGS:-c2 c3 c5:f64 c5:f32 c4}; do
  cfg=${c%%:*}; dt=${c#*:}; [ "$dt" = "$c" ] && dt=f64
  timeout 900 python bench.py --config $cfg --dtype $dt --steps 100 --warmup 5 > $P/bench_${cfg}_${dt}_${TAG}.json 2> gpurun_out/bench_${cfg}_${dt}.err
  python tools/bench_brief.py $P/bench_${cfg}_${dt}_${TAG}.json
done
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:omax_short -s 6 -c 1 -o gpurun_out/prof_c2_short_${TAG} python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_c2.log 2>&1; tail -2 gpurun_out/ncu_c2.log
python tools/ncu_summary.py gpurun_out/prof_c2_short_${TAG}.ncu-rep > $P/ncu_c2_omax_short_${TAG}.txt 2>&1
python tools/ncu_lines.py gpurun_out/prof_c2_short_${TAG}.ncu-rep >> $P/ncu_c2_omax_short_${TAG}.txt 2>&1
cp profiles/ncu_traffic.json $P/; ls $P
