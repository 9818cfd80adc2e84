#!/bin/bash
# Round evidence: build, full bench (in-graph gather timing), launch list + ncu full captures.
python paper_1909_01500_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python -c "
import json; d=json.load(open('gpurun_out/bench_full.json')); r=d['roofline']; print('step_us', d['ms_per_step']*1e3, 'gather_us', r['avg_launch_ms']*1e3, 'eager', r['avg_launch_ms_eager']*1e3, 'frac', r['frac'], 'e2e', d['e2e']['value'])"
tail -3 gpurun_out/bench_full.err
bash scripts/gpu_profile_all.sh > /dev/null 2>&1
python scripts/ncu_summary.py launches gpurun_out/launches.csv > gpurun_out/ncu_launches_step.json 2> gpurun_out/ncu_sum.err
python scripts/ncu_summary.py full gpurun_out/prof_gather.ncu-rep > gpurun_out/ncu_full_gather.json 2>> gpurun_out/ncu_sum.err
python scripts/ncu_summary.py full gpurun_out/prof_small.ncu-rep > gpurun_out/ncu_full_small.json 2>> gpurun_out/ncu_sum.err
cat gpurun_out/ncu_launches_step.json | head -60; tail -5 gpurun_out/ncu_sum.err
