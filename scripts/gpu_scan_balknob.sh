#!/bin/bash
mkdir -p gpurun_out
for k in 0 1 2 3; do
  RPL_SCAN_BAL=$k SHAPES=${SHAPES:-1024x16384,1024x18944,512x65536,2048x4736} timeout 600 python scripts/scan_sweep.py > gpurun_out/scan_bal$k.json 2> gpurun_out/scan_bal$k.err
  python -c "
import json; d=json.load(open('gpurun_out/scan_bal$k.json'))
for r in d['sweep']: print('bal$k', r['T'], r['B'], 'gae %.2f us %.2f' % (r['gae_us'], r['gae_frac']), 'disc %.2f us %.2f' % (r['disc_us'], r['disc_frac']))
" || tail -3 gpurun_out/scan_bal$k.err
done
