#!/bin/bash
# Scan shape A/B: the size sweep under several RPL_SCAN_VARIANT values (no tests).
mkdir -p gpurun_out
for v in ${VARIANTS:-0 10 11 12}; do
  RPL_SCAN_VARIANT=$v timeout 600 python scripts/scan_sweep.py > gpurun_out/scan_sweep_v$v.json 2> gpurun_out/scan_sweep_v$v.err
  python -c "
import json; d=json.load(open('gpurun_out/scan_sweep_v$v.json'))
for r in d['sweep']: print('v$v', r['T'], r['B'], 'gae %.2f us %.2f' % (r['gae_us'], r['gae_frac']), 'disc %.2f us %.2f' % (r['disc_us'], r['disc_frac']))
" || tail -3 gpurun_out/scan_sweep_v$v.err
done
