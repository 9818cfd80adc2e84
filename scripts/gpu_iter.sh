#!/bin/bash
# Iteration call: build, GPU tests, tree latency with staging on/off, bench.
python paper_1909_01500_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for st in 1 0 1 0; do
RPL_TREE_STAGE=$st python - <<'PY' >> gpurun_out/tree_lat.txt 2>&1
import json, os, torch, bench, paper_1909_01500_b200 as rpl
r = bench.tree_latency(torch.device("cuda:0"), rpl)
print(os.environ["RPL_TREE_STAGE"], json.dumps(r))
PY
RPL_TREE_STAGE=$st timeout 300 python bench.py --no-secondary --no-cpu-baseline --steps 1000 --warmup 50 > gpurun_out/bench_st$st.json 2> gpurun_out/bench_st$st.err
python -c "import json;d=json.load(open('gpurun_out/bench_st$st.json'));print('stage=$st', d['ms_per_step']*1e3, d['e2e']['value'], d['roofline']['frac'])" >> gpurun_out/tree_lat.txt
done
tail -2 gpurun_out/pytest_gpu.log; cat gpurun_out/tree_lat.txt
