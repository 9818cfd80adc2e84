#!/bin/bash
for v in "-DRPL_PDL_EARLY=0" "-DRPL_PDL_EARLY=1 -DRPL_UPD_TRIGGER_AT=3"; do
  RPL_NVCC_EXTRA="-DRPL_TRACE $v" python paper_1909_01500_b200/build.py --force > /dev/null 2>&1
  echo "$v"; STEADY=1 STEP=fused python scripts/step_trace.py | tr -d '\n '; echo
  STEP=fused python scripts/step_trace.py | tr -d '\n '; echo
done
python paper_1909_01500_b200/build.py --force > /dev/null 2>&1
