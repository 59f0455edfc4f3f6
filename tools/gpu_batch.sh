set -x; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "3d" > gpurun_out/t3dcl.log 2>&1; echo "rc=$?" >> gpurun_out/t3dcl.log
