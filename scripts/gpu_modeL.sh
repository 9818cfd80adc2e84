#!/bin/bash
# Functional check of the N>1 bench paths (Mode L and Mode C) on a 1-GPU box: 2 ranks, gloo, same device.
mkdir -p gpurun_out
for m in L C; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
  bench.py --gpus 2 --mode $m --backend gloo --same-device --steps 20 --warmup 5 --no-cpu-baseline --no-secondary \
  > gpurun_out/bench_mode${m}_gloo.json 2> gpurun_out/bench_mode${m}_gloo.err
echo "mode $m rc=$?"; head -c 700 gpurun_out/bench_mode${m}_gloo.json; echo; grep -v "^\*\|OMP_NUM" gpurun_out/bench_mode${m}_gloo.err | tail -5
done
