set -x; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "host_entry or concurrent or golden or purity" > gpurun_out/host_tests.log 2>&1; echo "rc=$?" >> gpurun_out/host_tests.log
