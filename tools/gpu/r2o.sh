set -x
timeout 600 tools/c5_lab 10 > gpurun_out/r2o_lab.txt 2>&1
PDCS_TIMING=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2o_c5.json 2> gpurun_out/r2o_c5.err
