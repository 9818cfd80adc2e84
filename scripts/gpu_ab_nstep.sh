#!/bin/bash
# Build-flag A/B of the n-step kernel's outputs per thread (RPL_NSTEP_U).
mkdir -p gpurun_out
for u in ${US:-1 2 4 8}; do
  RPL_NVCC_EXTRA="-DRPL_NSTEP_U=$u" python paper_1909_01500_b200/build.py --force > gpurun_out/abn_build_$u.log 2>&1 || tail -3 gpurun_out/abn_build_$u.log
  for r in 1 2; do echo "U=$u $(timeout 120 python scripts/nstep_time.py)"; done
done
python paper_1909_01500_b200/build.py --force > /dev/null 2>&1
