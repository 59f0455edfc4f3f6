set -x; mkdir -p gpurun_out
for i in 1 2 3; do timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cluster or device_tiles or halo or odd_width" > gpurun_out/clu_tests$i.log 2>&1; echo "rc=$?" >> gpurun_out/clu_tests$i.log; done
