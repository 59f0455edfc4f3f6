set -x; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "cluster or device_tiles or reference_suite or integration or halo" > gpurun_out/clu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/clu_tests.log
