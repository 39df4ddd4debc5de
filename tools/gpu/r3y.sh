export PYTHONUNBUFFERED=1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r3y_pytest.log 2>&1; echo rc=$? >> gpurun_out/r3y_pytest.log
PDCS_TIMING=1 timeout 600 python tools/e2e_var.py 5 > gpurun_out/r3y_var.txt 2>&1
