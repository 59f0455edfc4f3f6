set -x; mkdir -p gpurun_out
timeout 600 python tools/e2e_breakdown.py > gpurun_out/e2e.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "golden or concurrent or purity or odd_width or fp32_within" > gpurun_out/host_tests.log 2>&1; echo "rc=$?" >> gpurun_out/host_tests.log
