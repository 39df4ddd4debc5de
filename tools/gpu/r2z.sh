export PYTHONUNBUFFERED=1
PDCS_TIMING=1 timeout 600 python tools/e2e_var.py 6 > gpurun_out/r2z_a.txt 2>&1
