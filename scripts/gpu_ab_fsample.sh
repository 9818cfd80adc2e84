#!/bin/bash
# Same-box A/B: R2D2 step with sampling inside the gather (1) or a separate sampler launch (0).
mkdir -p gpurun_out
for round in 1 2 3; do
  for f in 0 1; do
    timeout 300 python bench.py --no-secondary --no-cpu-baseline --steps 800 --fused-sample $f > gpurun_out/ab_fsample_${f}_$round.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/ab_fsample_${f}_$round.json').read().strip().splitlines()[-1])
print('fused_sample=$f round=$round', round(d['ms_per_step']*1e3,2), 'median', round(d['step_us_stats']['replays_200']['median_us'],2), 'launches', d['gpu_launches'], 'e2e', round(d['e2e']['value']))"
  done
done
