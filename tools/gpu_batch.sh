set -x; mkdir -p gpurun_out
EBISU_LIB_PATH=$PWD/scratch/libebisu_exp.so timeout 300 python tools/clu_bench.py > gpurun_out/clu_exp.log 2>&1
