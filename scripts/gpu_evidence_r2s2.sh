#!/bin/bash
# Round-2 session-2 evidence: smoke, driver-shaped and default bench, reference arm, ncu launch list of
# the step, ncu --set full of the sequence gather / the scans / the tree kernels, source lines.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_k20.json 2> gpurun_out/bench_k20.err
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
bash scripts/gpu_profile_all.sh > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_scan_pipe -c 2 -o gpurun_out/prof_scan_large python scripts/scan_one.py 1024 16384 > gpurun_out/prof_scan_large.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/launches.csv > gpurun_out/ncu_launches_step.json 2> gpurun_out/ncu_sum.err
python scripts/ncu_summary.py full gpurun_out/prof_gather.ncu-rep > gpurun_out/ncu_full_gather.json 2>> gpurun_out/ncu_sum.err
python scripts/ncu_summary.py full gpurun_out/prof_small.ncu-rep > gpurun_out/ncu_full_small.json 2>> gpurun_out/ncu_sum.err
python scripts/ncu_summary.py full gpurun_out/prof_scan_large.ncu-rep > gpurun_out/ncu_full_scan_large.json 2>> gpurun_out/ncu_sum.err
python scripts/ncu_lines.py gpurun_out/prof_gather.ncu-rep > gpurun_out/ncu_lines_gather.txt 2>> gpurun_out/ncu_sum.err
tail -1 gpurun_out/smoke.log
for f in bench_k20 bench_full; do python -c "
import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', 'step_us', round(d['ms_per_step']*1e3,2), 'gather_us', round(r['avg_launch_ms']*1e3,2), 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value']), 'cpu', d.get('cpu_baseline',{}).get('value'), 'clocks', d['clocks'])"; done
head -c 300 gpurun_out/bench_reference.json; echo
head -c 1500 gpurun_out/ncu_launches_step.json
python scripts/ncu_summary.py full gpurun_out/prof_small.ncu-rep > /dev/null 2>&1
ncu -i gpurun_out/prof_gather.ncu-rep --page raw --csv > gpurun_out/prof_gather_raw.csv 2>/dev/null
