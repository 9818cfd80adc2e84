#!/bin/bash
# Fused update+sample: parity, step breakdown, bench A/B.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sumtree.py -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_sumtree.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sumtree.log
timeout 300 python scripts/step_breakdown.py > gpurun_out/step_breakdown.json 2> gpurun_out/step_breakdown.err
for f in 0 1 0 1; do
  timeout 300 python bench.py --no-secondary --no-cpu-baseline --tree-fused $f > gpurun_out/bench_f$f.json 2> gpurun_out/bench_f$f.err
  python -c "import json;d=json.load(open('gpurun_out/bench_f$f.json'));print('fused=$f', d['ms_per_step'], d['e2e']['value'] if d.get('e2e') else None)"
done
tail -3 gpurun_out/pytest_sumtree.log; cat gpurun_out/step_breakdown.json
