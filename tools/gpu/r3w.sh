export PYTHONUNBUFFERED=1
timeout 600 python tools/profile_e2e.py C5 20 > gpurun_out/r3w_prof.txt 2>&1
timeout 600 python tools/e2e_var.py 6 > gpurun_out/r3w_var.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "solve or box or c5 or C5" > gpurun_out/r3w_pt.log 2>&1; echo rc=$? >> gpurun_out/r3w_pt.log
