#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_gather_dyn.py tests/test_gpu_step.py -x -q > gpurun_out/pytest_dyn.log 2>&1; tail -3 gpurun_out/pytest_dyn.log
STEP=fused SETTINGS="${SET1:--1,10,10 88,10,10 80,16,8 70,16,8 80,16,4 70,24,6 88,16,10 80,12,6}" python scripts/ab_dyn_sweep.py
RPL_NVCC_EXTRA="-DRPL_TRACE" python paper_1909_01500_b200/build.py --force > /dev/null 2>&1
for st in ${TRACE_SET:-80,16,8 70,16,6}; do
  DYN=$st STEADY=1 STEP=fused python scripts/step_trace.py > gpurun_out/tr_$st.json 2>&1
  python -c "
import json; t=open('gpurun_out/tr_$st.json').read(); d=json.loads(t[t.index('{'):t.rindex('}')+1])['ns_from_update_entry_median']
print('$st', {k: d.get(k) for k in ('graph_us_per_step', 'gather_end', 'dyn_units_total', 'cta_end_us_percentiles_p0_p10_p50_p90_p100_last', 'dyn_slowest8_end_static_units', 'dyn_slowest4_grabs_t_rows_queued')})" || tail -3 gpurun_out/tr_$st.json
done
python paper_1909_01500_b200/build.py --force > /dev/null 2>&1
