export PYTHONUNBUFFERED=1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r4x_pytest.log 2>&1; echo rc=$? >> gpurun_out/r4x_pytest.log
for t in "" "halfw=8" "halfw=2"; do
  PDCS_TUNE="$t" timeout 300 python bench.py --config C2 --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r4x_cfg.jsonl 2>> gpurun_out/r4x_cfg.err
done
for t in "" "xhalfw=8" "xhalfw=2"; do
  PDCS_TUNE="$t" timeout 300 python bench.py --config C2p --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r4x_cfg.jsonl 2>> gpurun_out/r4x_cfg.err
done
