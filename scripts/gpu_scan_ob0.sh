#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_returns.py -x -q > gpurun_out/pytest_returns.log 2>&1; tail -2 gpurun_out/pytest_returns.log
SHAPES=${SHAPES:-128x4096,1024x4096,2048x4736,1024x16384,512x65536,128x65536} VARIANTS="${VARIANTS:-0 18 19 20 21}" bash scripts/gpu_scan_ab.sh
VARIANTS=0,21,18,0 timeout 600 python scripts/scan_variants.py | tr -d '\n '; echo
