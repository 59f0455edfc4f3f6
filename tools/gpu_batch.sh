set -x; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f4_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/f4_smoke.log
timeout 900 python bench.py > gpurun_out/f4_bench.json 2> gpurun_out/f4_bench.err
