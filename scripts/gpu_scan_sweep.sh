#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_returns.py -x -q --durations=5 > gpurun_out/pytest_returns.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_returns.log
for v in ${VARIANTS:-0 7 8}; do
  RPL_SCAN_VARIANT=$v timeout 600 python scripts/scan_sweep.py > gpurun_out/scan_sweep_v$v.json 2> gpurun_out/scan_sweep_v$v.err
done
tail -3 gpurun_out/pytest_returns.log
for v in ${VARIANTS:-0 7 8}; do python -c "
import json,sys; d=json.load(open('gpurun_out/scan_sweep_v$v.json'))
for r in d['sweep']: print('v$v', r['T'], r['B'], 'gae %.2f us %.2f' % (r['gae_us'], r['gae_frac']), 'disc %.2f us %.2f' % (r['disc_us'], r['disc_frac']), 'floor %.2f us %.2f' % (r['floor_stream_us'], r['floor_frac']))
"; done
