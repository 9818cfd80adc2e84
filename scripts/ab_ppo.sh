#!/bin/bash
# Same-box A/B of build flags on the PPO secondary (bench.bench_ppo): VARIANTS as ab_flags.sh.
set -u
mkdir -p gpurun_out
names=()
for v in ${VARIANTS}; do
  name=${v%%=*}; flags=${v#*=}; flags=${flags//,/ }
  RPL_NVCC_EXTRA="$flags" python paper_1909_01500_b200/build.py --force > gpurun_out/abp_build_$name.log 2>&1 || { echo "build $name failed"; tail -5 gpurun_out/abp_build_$name.log; }
  cp paper_1909_01500_b200/librpl.so /tmp/librpl_$name.so; names+=($name)
done
for r in $(seq ${ROUNDS:-3}); do for name in "${names[@]}"; do
  cp /tmp/librpl_$name.so paper_1909_01500_b200/librpl.so
  timeout 600 python -c "
import json, torch, bench, paper_1909_01500_b200 as rpl
d = bench.bench_ppo(torch.device('cuda:0'), rpl)
print('$name', round(d['gae_us_per_call'], 3), round(d['disc_us_per_call'], 3))" 2> gpurun_out/abp_$name.err || tail -3 gpurun_out/abp_$name.err
done; done
python paper_1909_01500_b200/build.py --force > /dev/null 2>&1
