#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gather.py -x -q -k "sample" > gpurun_out/pytest_fs.log 2>&1; tail -2 gpurun_out/pytest_fs.log
for r in 1 2; do for fs in 0 1; do
  timeout 600 python bench.py --no-cpu-baseline --no-secondary --steps 400 --fused-sample $fs > gpurun_out/fs_$fs.json 2> gpurun_out/fs_$fs.err
  python -c "import json;d=json.load(open('gpurun_out/fs_$fs.json'));print('fused=$fs', round(d['ms_per_step']*1e3,3), round(d['roofline']['avg_launch_ms']*1e3,3), round(d['e2e']['value']))" || tail -3 gpurun_out/fs_$fs.err
done; done
RPL_NVCC_EXTRA="-DRPL_TRACE" python paper_1909_01500_b200/build.py --force > /dev/null 2>&1
STEP=fused python scripts/step_trace.py
python scripts/step_trace.py
python paper_1909_01500_b200/build.py --force > /dev/null 2>&1
