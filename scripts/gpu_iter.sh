#!/bin/bash
# Iteration call: build, GPU tests, PPO scan variants (grouped TMA 7/8/9 vs default).
python paper_1909_01500_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
VARIANTS=0,7,8,9,0,7,8,9 timeout 300 python scripts/scan_variants.py > gpurun_out/scan_variants.json 2>&1
tail -2 gpurun_out/pytest_gpu.log; cat gpurun_out/scan_variants.json
