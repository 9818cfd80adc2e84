#!/bin/bash
# Full GPU suite, smoke, default bench (1000 steps) and the driver-shaped bench.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_k20.json 2> gpurun_out/bench_k20.err
for f in bench_full bench_k20; do python -c "
import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', 'step_us', round(d['ms_per_step']*1e3,2), 'value', round(d['value']), 'gather_us', round(r['avg_launch_ms']*1e3,2), 'frac', round(r['frac'],3), 'marg', round(r.get('frac_marginal') or 0,3), 'e2e', round(d['e2e']['value']), 'clocks', d['clocks'], 'ret', {k: round(v,2) for k,v in d['returns'].items() if 'us_per_call' in k})" || tail -5 gpurun_out/$f.err; done
