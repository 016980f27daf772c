#!/bin/bash
# Round-end evidence on one B200: GPU tests, smoke, every bench line (tools/gpu_round2.sh TAG),
# and the 2-rank bench path with both ranks on device 0.
tag=${1:-v4}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -4 | tee gpurun_out/pytest_gpu_$tag.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
bash tools/gpu_round2.sh $tag
RIMDP_BENCH_DEVICE_MAP=0,0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 \
    > gpurun_out/bench_n2_shared_$tag.json 2> gpurun_out/bench_n2_shared_$tag.err
python tools/bench_brief.py gpurun_out/bench_n2_shared_$tag.json | tail -1
