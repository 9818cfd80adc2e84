#!/bin/bash
mkdir -p gpurun_out
for v in ${VARIANTS:-7 9}; do
  RPL_SCAN_VARIANT=$v timeout 600 ncu --set full --clock-control none -k regex:k_scan -c 2 -o gpurun_out/ncu_scan_v$v -f python scripts/scan_one.py ${SIZE:-2048 4096} > gpurun_out/ncu_scan_v$v.log 2>&1
  tail -3 gpurun_out/ncu_scan_v$v.log
done
