set -x; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_reference_suite.py -x -q -k cli > gpurun_out/cli_test.log 2>&1; echo "rc=$?" >> gpurun_out/cli_test.log
