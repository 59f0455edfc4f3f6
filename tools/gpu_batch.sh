set -x; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "reserve or host_entry or distributed or slab" > gpurun_out/r02_gputest5.log 2>&1; echo "rc=$?" >> gpurun_out/r02_gputest5.log
