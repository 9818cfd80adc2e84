#!/bin/bash
# Functional check of the N>1 (Mode L) bench path on a 1-GPU box: 2 ranks, gloo, same device.
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --backend gloo --same-device --steps 20 --warmup 5 --no-cpu-baseline --no-secondary \
  > gpurun_out/bench_modeL_gloo.json 2> gpurun_out/bench_modeL_gloo.err
echo "modeL rc=$?"; cat gpurun_out/bench_modeL_gloo.json | head -c 1500; tail -5 gpurun_out/bench_modeL_gloo.err
