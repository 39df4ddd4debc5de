set -x
export PYTHONUNBUFFERED=1
PDCS_TIMING=1 timeout 300 python tools/profile_e2e.py C5 20 cold > gpurun_out/r2n_prof_e2e_cold.txt 2>&1
PDCS_TIMING=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2n_c5.json 2> gpurun_out/r2n_c5.err
timeout 1200 python -m pytest tests/test_gpu_batch.py tests/test_gpu_sharded.py -q > gpurun_out/r2n_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2n_pytest.log
