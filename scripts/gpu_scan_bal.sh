#!/bin/bash
# Balanced scan schedule: parity tests, then the size sweep (default variant) and PPO.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_returns.py -x -q > gpurun_out/pytest_returns.log 2>&1; tail -3 gpurun_out/pytest_returns.log
SHAPES=${SHAPES:-128x4096,1024x4096,2048x4096,2048x4736,1024x16384,1024x18944,512x65536,128x65536} VARIANTS="${VARIANTS:-0}" bash scripts/gpu_scan_ab.sh
