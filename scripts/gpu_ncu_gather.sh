#!/bin/bash
# ncu --set full of the default sequence gather: skeleton (diag 19) and normal (diag 0).
mkdir -p gpurun_out
for d in ${DIAGS:-19 0}; do
  DIAGS=$d timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather_seq -s 6 -c 1 \
    -o gpurun_out/prof_gather_d$d python scripts/gather_diag.py > gpurun_out/prof_gather_d$d.log 2>&1
done
ls gpurun_out
