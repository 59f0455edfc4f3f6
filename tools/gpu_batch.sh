set -x; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "slab or distributed or multi_rank or output_plane or reserve" > gpurun_out/dist_tests.log 2>&1; echo "rc=$?" >> gpurun_out/dist_tests.log
