#!/bin/bash
# Round-end evidence: build, GPU suite, smoke, full bench, launch list + ncu full of the gather.
mkdir -p gpurun_out
python paper_1909_01500_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
bash scripts/gpu_profile_all.sh > /dev/null 2>&1
python scripts/ncu_summary.py launches gpurun_out/launches.csv > gpurun_out/ncu_launches_step.json 2> gpurun_out/ncu_sum.err
python scripts/ncu_summary.py full gpurun_out/prof_gather.ncu-rep > gpurun_out/ncu_full_gather.json 2>> gpurun_out/ncu_sum.err
python scripts/ncu_summary.py full gpurun_out/prof_small.ncu-rep > gpurun_out/ncu_full_small.json 2>> gpurun_out/ncu_sum.err
tail -2 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log
python -c "
import json; d=json.load(open('gpurun_out/bench_full.json')); r=d['roofline']; print('step_us', d['ms_per_step']*1e3, 'gather_us', r['avg_launch_ms']*1e3, 'frac', r['frac'], 'e2e', d['e2e']['value'], 'cpu', d['cpu_baseline']['value'])"
head -c 300 gpurun_out/bench_reference.json; echo
cat gpurun_out/ncu_launches_step.json
