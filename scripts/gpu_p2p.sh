#!/bin/bash
# Peer-board exchanges: in-process parity tests, then the N>1 bench paths with two processes
# sharing the one GPU (gloo for the host plumbing; --exchange p2p and collective).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_p2p.py -x -q > gpurun_out/pytest_p2p.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_p2p.log
tail -15 gpurun_out/pytest_p2p.log
for ex in p2p collective; do for m in L C; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
  bench.py --gpus 2 --mode $m --backend gloo --exchange $ex --same-device --steps 20 --warmup 5 --no-cpu-baseline --no-secondary \
  > gpurun_out/bench_mode${m}_${ex}.json 2> gpurun_out/bench_mode${m}_${ex}.err
echo "mode $m exchange $ex rc=$?"; head -c 400 gpurun_out/bench_mode${m}_${ex}.json; echo; grep -v "^\*\|OMP_NUM" gpurun_out/bench_mode${m}_${ex}.err | tail -4
done; done
