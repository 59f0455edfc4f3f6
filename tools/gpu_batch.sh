set -x; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/f_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/f_gputest.log
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-3d --no-sweep --no-traffic > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream2d -s 1 -c 1 -o gpurun_out/f_stream2d_j2d5pt_t8 python tools/prof_run.py j2d5pt 8192 1000 8 > gpurun_out/f_ncu1.log 2>&1
