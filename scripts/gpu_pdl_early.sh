#!/bin/bash
# A/B: dependents launched right after each step kernel's griddepcontrol.wait (librpl_early.so)
# against the default (trigger at the end / implicit at exit).  The early variant was built
# with pdl_trigger() after pdl_wait() in k_tree_update, k_tree_sample, k_gather_seq_pipe_lsu
# and k_nstep (RPL_NVCC_EXTRA=-D... build); measured slower and removed.
mkdir -p gpurun_out
cp paper_1909_01500_b200/librpl.so /tmp/librpl_default.so
for v in default early default early; do
  if [ $v = early ]; then cp paper_1909_01500_b200/librpl_early.so paper_1909_01500_b200/librpl.so; else cp /tmp/librpl_default.so paper_1909_01500_b200/librpl.so; fi
  timeout 300 python scripts/step_breakdown.py > gpurun_out/sb_$v.json 2>/dev/null
  timeout 300 python bench.py --no-secondary --no-cpu-baseline > gpurun_out/bench_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bench_$v.json'));s=json.load(open('gpurun_out/sb_$v.json'));print('$v', round(d['ms_per_step']*1e3,2), round(d['e2e']['value']), {k:v for k,v in s.items() if k.startswith('stacked')})"
done
cp /tmp/librpl_default.so paper_1909_01500_b200/librpl.so
cp paper_1909_01500_b200/librpl_early.so paper_1909_01500_b200/librpl.so
timeout 600 python -m pytest tests/test_gpu_sumtree.py tests/test_gpu_gather.py tests/test_gpu_returns.py -x -q 2>&1 | tail -2
cp /tmp/librpl_default.so paper_1909_01500_b200/librpl.so
