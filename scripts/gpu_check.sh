#!/bin/bash
# One gpurun call: GPU parity tests, smoke, sequence-gather variant probe, bench,
# ncu launch list of the bench step and one --set full capture of the gather.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python scripts/gather_probe.py > gpurun_out/gather_probe.json 2> gpurun_out/gather_probe.err
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 40 --csv \
  --log-file gpurun_out/launches.csv python bench.py --profile --no-graph --steps 20 --warmup 50 --no-secondary --no-cpu-baseline > gpurun_out/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gather -s 60 -c 2 \
  -o gpurun_out/prof_gather python bench.py --profile --no-graph --steps 4 --warmup 30 --no-secondary --no-cpu-baseline > gpurun_out/prof_gather.log 2>&1
fi
ls -la gpurun_out
