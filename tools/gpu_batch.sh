set -x; mkdir -p gpurun_out
(cd scratch/r01 && timeout 300 python ../../tools/ab3d.py) >> gpurun_out/ab3d4.log 2>&1
timeout 300 python tools/ab3d.py >> gpurun_out/ab3d4.log 2>&1
timeout 600 python tools/tune_depths.py j3d7pt j3d27pt j3d17pt poisson j3d13pt >> gpurun_out/ab3d4.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "3d or config4 or config5 or odd or reassoc or fp32" > gpurun_out/t3d.log 2>&1; echo "rc=$?" >> gpurun_out/t3d.log
