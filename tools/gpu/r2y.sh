export PYTHONUNBUFFERED=1
PDCS_TIMING=1 timeout 600 python tools/e2e_var.py 4 > gpurun_out/r2y_a.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_scale_parity.py -q -x > gpurun_out/r2y_pt.log 2>&1
PDCS_TIMING=1 timeout 600 python tools/e2e_var.py 4 > gpurun_out/r2y_b.txt 2>&1
free -g > gpurun_out/r2y_mem.txt; nproc >> gpurun_out/r2y_mem.txt
