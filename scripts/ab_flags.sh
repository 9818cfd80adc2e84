#!/bin/bash
# Same-box A/B of build flags: VARIANTS="name1=-DX=1 name2=-DX=2 ..." (names without spaces;
# flags joined with commas for several).  Builds each, then runs the default bench
# (BENCH_ARGS) in ROUNDS rounds over all variants.  Measurement only.
set -u
mkdir -p gpurun_out
names=()
for v in ${VARIANTS}; do
  name=${v%%=*}; flags=${v#*=}; flags=${flags//,/ }
  RPL_NVCC_EXTRA="$flags" python paper_1909_01500_b200/build.py --force > gpurun_out/abf_build_$name.log 2>&1 || { echo "build $name failed"; tail -5 gpurun_out/abf_build_$name.log; }
  cp paper_1909_01500_b200/librpl.so /tmp/librpl_$name.so; names+=($name)
done
for r in $(seq ${ROUNDS:-3}); do for name in "${names[@]}"; do
  cp /tmp/librpl_$name.so paper_1909_01500_b200/librpl.so
  timeout 600 python bench.py --no-cpu-baseline --no-secondary ${BENCH_ARGS:-} > gpurun_out/abf_$name.json 2> gpurun_out/abf_$name.err
  python -c "import json;d=json.load(open('gpurun_out/abf_$name.json'));print('$name', round(d['ms_per_step']*1e3,3), round(d['roofline']['avg_launch_ms']*1e3,3), round(d['e2e']['value']))" || tail -3 gpurun_out/abf_$name.err
done; done
python paper_1909_01500_b200/build.py --force > /dev/null 2>&1
