export PYTHONUNBUFFERED=1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r3s_pytest.log 2>&1; echo rc=$? >> gpurun_out/r3s_pytest.log
for c in C2 C2p; do
  timeout 300 python bench.py --config $c --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r3s_cfg.jsonl 2>> gpurun_out/r3s_cfg.err
done
