set -x
export PYTHONUNBUFFERED=1
for t in "" "pgrid=148" "pgrid=74" "pgrid=18"; do
  PDCS_TUNE=$t timeout 300 python bench.py --config C1 --batch 64 --steps 2000 --warmup 50 --no-cpu-baseline --no-e2e --profile-reps 0 >> gpurun_out/r2r_c1.jsonl 2>> gpurun_out/r2r_c1.err
done
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_parity.py -q -k "batch or solve_many or solve_matches or determin or nan or time_limit or step_level" > gpurun_out/r2r_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2r_pytest.log
