set -x; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "resident or j1d3pt" > gpurun_out/gen_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gen_tests.log
EBISU_GEN_CTAS=2 timeout 900 python tools/gen_bench.py 64 > gpurun_out/gen_bench2.log 2>&1
EBISU_GEN_CTAS=1 timeout 900 python tools/gen_bench.py 64 > gpurun_out/gen_bench1.log 2>&1
