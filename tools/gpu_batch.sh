#!/bin/bash
# Verification batch for one gpurun call (run from the repo root on the GPU
# box: gpurun -- 'bash tools/gpu_batch.sh'): smoke, the -m gpu suite, the
# bench line, and the ncu launch list of a short bench run.  Outputs land in
# gpurun_out/ (merged back by gpurun); copy what should be judged to profiles/.
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "rc=$?" >> gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  --no-e2e --no-3d --no-sweep --no-traffic > /dev/null 2>&1
