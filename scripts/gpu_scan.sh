#!/bin/bash
# Scan kernel variants: parity, then PPO timing per variant.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_returns.py -x -q > gpurun_out/pytest_returns.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_returns.log
timeout 600 python scripts/scan_variants.py > gpurun_out/scan_variants.json 2> gpurun_out/scan_variants.err
tail -3 gpurun_out/pytest_returns.log; cat gpurun_out/scan_variants.json; tail -5 gpurun_out/scan_variants.err
