#!/bin/bash
# Same-box A/B: R2D2 step with update + sample as two launches (0) or one (1, single-CTA kernel).
mkdir -p gpurun_out
for round in 1 2 3; do
  for f in 0 1; do
    timeout 300 python bench.py --no-secondary --no-cpu-baseline --steps 800 --tree-fused $f > gpurun_out/ab_fused_${f}_$round.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/ab_fused_${f}_$round.json').read().strip().splitlines()[-1])
print('fused=$f round=$round', round(d['ms_per_step']*1e3,2), 'median', round(d['step_us_stats']['replays_200']['median_us'],2), 'launches', d['gpu_launches'])"
  done
done
