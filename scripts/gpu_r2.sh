#!/bin/bash
# Round-2 iteration call: GPU tests, the driver's bench command, the default bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench_k20.json 2> gpurun_out/bench_k20.err
if [ -z "$QUICK" ]; then
timeout 900 python bench.py --no-secondary --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_k1000.json 2> gpurun_out/bench_k1000.err
fi
tail -3 gpurun_out/pytest_gpu.log; head -c 600 gpurun_out/bench_k20.json; tail -2 gpurun_out/bench_k20.err
