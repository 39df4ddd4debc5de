set -x
export PYTHONUNBUFFERED=1
for t in "" "vec=0"; do
  PDCS_TUNE=$t timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-ttt-c1 --no-e2e >> gpurun_out/r2k_c5.jsonl 2>> gpurun_out/r2k_c5.err
  PDCS_TUNE=$t timeout 300 python bench.py --config C1 --steps 2000 --warmup 50 --no-cpu-baseline --no-ttt-c1 --no-e2e >> gpurun_out/r2k_c1.jsonl 2>> gpurun_out/r2k_c1.err
done
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2k_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2k_pytest.log
