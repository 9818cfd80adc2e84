#!/bin/bash
# A/B: bench with and without programmatic dependent launch, plus GPU tests.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
RPL_PDL=0 timeout 600 python bench.py --no-cpu-baseline --no-secondary > gpurun_out/bench_nopdl.json 2> gpurun_out/bench_nopdl.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_pdl.json 2> gpurun_out/bench_pdl.err
tail -2 gpurun_out/pytest_gpu.log; for f in nopdl pdl; do python -c "
import json; d=json.load(open('gpurun_out/bench_$f.json')); print('$f', d['ms_per_step']*1e3, d['roofline']['avg_launch_ms']*1e3, d['e2e']['value'], d.get('secondary'))"; tail -2 gpurun_out/bench_$f.err; done
