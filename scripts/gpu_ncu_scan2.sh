#!/bin/bash
# ncu --set full of the default GAE scan at one size (source + instruction mix), for the scan rework.
mkdir -p gpurun_out
SZ=${SIZE:-1024 16384}
RPL_SCAN_VARIANT=${VAR:-0} timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_scan -c 1 -o gpurun_out/ncu_scan_gae -f python scripts/scan_one.py $SZ > gpurun_out/ncu_scan_gae.log 2>&1
tail -2 gpurun_out/ncu_scan_gae.log
python scripts/ncu_lines.py gpurun_out/ncu_scan_gae.ncu-rep 40 > gpurun_out/ncu_scan_gae_lines.txt 2>&1
ncu -i gpurun_out/ncu_scan_gae.ncu-rep --page details --csv > gpurun_out/ncu_scan_gae_details.csv 2>&1
ncu -i gpurun_out/ncu_scan_gae.ncu-rep --page raw --csv > gpurun_out/ncu_scan_gae_raw.csv 2>&1
ncu -i gpurun_out/ncu_scan_gae.ncu-rep --page source --csv --print-source=sass > gpurun_out/ncu_scan_gae_sass.csv 2>&1
head -30 gpurun_out/ncu_scan_gae_lines.txt
