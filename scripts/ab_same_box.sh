#!/bin/bash
# Same-box A/B of the default bench: variant A = the sources in scripts/ab/ (copies of older
# csrc files), variant B = the working tree.  Alternates A B A B A B.  Measurement only.
set -u
mkdir -p gpurun_out
CS=paper_1909_01500_b200/csrc
mkdir -p /tmp/ab_b
for f in scripts/ab/*.cu; do cp $CS/$(basename $f) /tmp/ab_b/; cp $f $CS/; done
python paper_1909_01500_b200/build.py --force > gpurun_out/ab_build_a.log 2>&1; cp paper_1909_01500_b200/librpl.so /tmp/librpl_A.so
for f in scripts/ab/*.cu; do cp /tmp/ab_b/$(basename $f) $CS/; done
python paper_1909_01500_b200/build.py --force > gpurun_out/ab_build_b.log 2>&1; cp paper_1909_01500_b200/librpl.so /tmp/librpl_B.so
for v in A B A B A B; do
  cp /tmp/librpl_$v.so paper_1909_01500_b200/librpl.so
  if [ "${MODE:-r2d2}" = dqn ]; then  # the DQN secondary alone (bs 32 / 128 / 512 step us)
    timeout 600 python -c "
import torch, bench, paper_1909_01500_b200 as rpl
d = bench.bench_dqn(torch.device('cuda:0'), rpl)
print('$v', *[round(d[f'bs{b}']['us_per_step'], 3) for b in (32, 128, 512)])" 2> gpurun_out/ab_$v.err
  else
    timeout 600 python bench.py --no-cpu-baseline --no-secondary ${BENCH_ARGS:-} > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
    python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));print('$v', round(d['ms_per_step']*1e3,3), round(d['roofline']['avg_launch_ms']*1e3,3), round(d['e2e']['value']))"
  fi
done
cp /tmp/librpl_B.so paper_1909_01500_b200/librpl.so
