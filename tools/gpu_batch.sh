set -x; mkdir -p gpurun_out
timeout 300 python tools/e2e_breakdown.py > gpurun_out/staging2.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "host_entry or concurrent or golden or purity or reference_suite" > gpurun_out/host_tests2.log 2>&1; echo "rc=$?" >> gpurun_out/host_tests2.log
