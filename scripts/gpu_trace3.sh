#!/bin/bash
for v in "-DRPL_PDL_EARLY=0" "-DRPL_PDL_EARLY=1 -DRPL_UPD_TRIGGER_AT=3"; do
  for tr in "" "-DRPL_TRACE"; do
    RPL_NVCC_EXTRA="$tr $v" python paper_1909_01500_b200/build.py --force > /dev/null 2>&1
    echo "== $tr $v"
    STEADY=1 STEP=fused python scripts/step_trace.py | python -c "import json,sys; d=json.load(sys.stdin); print('trace-script steady us/step', round(d['ns_from_update_entry_median']['graph_us_per_step'],3))"
    timeout 600 python bench.py --no-cpu-baseline --no-secondary --steps 400 > gpurun_out/t3.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/t3.json'));print('bench us/step', round(d['ms_per_step']*1e3,3))"
  done
done
python paper_1909_01500_b200/build.py --force > /dev/null 2>&1
