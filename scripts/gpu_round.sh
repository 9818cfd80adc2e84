#!/bin/bash
# Standard iteration call: GPU tests, gather limiter probe, full bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
VARIANTS=${VARIANTS:-0} DIAGS=${DIAGS:-0,1,2,3,16,19} timeout 600 python scripts/gather_diag.py > gpurun_out/gather_diag.json 2> gpurun_out/gather_diag.err
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/pytest_gpu.log; python -c "
import json; print(json.dumps(json.load(open('gpurun_out/gather_diag.json'))))"; tail -3 gpurun_out/gather_diag.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('step_us', d['ms_per_step']*1e3, 'gather_us', d['roofline']['avg_launch_ms']*1e3, 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value']); print(json.dumps(d.get('secondary')))"; tail -3 gpurun_out/bench.err
