set -x; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/f2_bench.json 2> gpurun_out/f2_bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream3d -s 1 -c 1 -o gpurun_out/f2_stream3d_j3d7pt_t4 python tools/prof_run.py j3d7pt 512 500 4 > gpurun_out/f2_ncu.log 2>&1
