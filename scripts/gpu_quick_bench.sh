#!/bin/bash
# Quick: selected GPU tests (PYTEST_K) then one bench without secondaries / baseline.
mkdir -p gpurun_out
K=${1:-"sumtree or gather"}
timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-secondary --no-cpu-baseline --steps 400 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
tail -2 gpurun_out/pytest_gpu.log; python -c "
import json; d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step']*1e3, d['step_us_stats']['replays_200'], d['roofline']['avg_launch_ms'], d['e2e']['value'])"
tail -2 gpurun_out/bench_q.err
