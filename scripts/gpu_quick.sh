#!/bin/bash
# Quick iteration call: GPU tests (or a subset), gather probe, bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/gather_probe.py > gpurun_out/gather_probe.json 2> gpurun_out/gather_probe.err
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/gather_probe.json; cat gpurun_out/bench.json | head -c 1500
