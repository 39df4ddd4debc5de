export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py tests/test_gpu_sharded.py -q -x > gpurun_out/r4j_pt.log 2>&1; echo rc=$? >> gpurun_out/r4j_pt.log
PDCS_TIMING=1 timeout 600 python tools/e2e_var.py 5 > gpurun_out/r4j_var.txt 2>&1
