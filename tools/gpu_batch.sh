set -x; mkdir -p gpurun_out
for i in 1 2; do
(cd scratch/r01 && timeout 300 python ../../tools/ab2d.py) >> gpurun_out/ab2d.log 2>&1
timeout 300 python tools/ab2d.py >> gpurun_out/ab2d.log 2>&1
done
