set -x; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/f3_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f3_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/f3_gputest.log
timeout 900 python bench.py > gpurun_out/f3_bench.json 2> gpurun_out/f3_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f3_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-3d --no-sweep --no-traffic > /dev/null 2>&1
