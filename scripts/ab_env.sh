#!/bin/bash
# Same-box A/B of environment knobs: VARIANTS="name1=VAR=val name2=VAR=val ..." (one VAR=val
# per name; "base=" for none).  ROUNDS rounds over all variants of the default bench.
set -u
mkdir -p gpurun_out
python paper_1909_01500_b200/build.py > gpurun_out/abe_build.log 2>&1
for r in $(seq ${ROUNDS:-3}); do for v in ${VARIANTS}; do
  name=${v%%=*}; kv=${v#*=}
  env $kv timeout 600 python bench.py --no-cpu-baseline --no-secondary ${BENCH_ARGS:-} > gpurun_out/abe_$name.json 2> gpurun_out/abe_$name.err
  python -c "import json;d=json.load(open('gpurun_out/abe_$name.json'));print('$name', round(d['ms_per_step']*1e3,3), round(d['roofline']['avg_launch_ms']*1e3,3), round(d['e2e']['value']))" || tail -3 gpurun_out/abe_$name.err
done; done
