#!/bin/bash
mkdir -p gpurun_out
for k in 1 0 1; do
  RPL_SCAN_SPREAD=$k SHAPES=${SHAPES:-1024x4096,2048x4096,2048x4736,1024x16384,512x65536,128x4096,128x65536} timeout 600 python scripts/scan_sweep.py > gpurun_out/scan_spread$k.json 2> gpurun_out/scan_spread$k.err
  python -c "
import json; d=json.load(open('gpurun_out/scan_spread$k.json'))
for r in d['sweep']: print('spread$k', r['T'], r['B'], 'gae %.2f us %.2f' % (r['gae_us'], r['gae_frac']), 'disc %.2f us %.2f' % (r['disc_us'], r['disc_frac']))
" || tail -3 gpurun_out/scan_spread$k.err
done
