set -x
export PYTHONUNBUFFERED=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2p_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2p_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2p_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2p_pytest.log
for c in C1 C2 C3 C4 C3p C2p; do
  timeout 300 python bench.py --config $c --steps 2000 --warmup 50 --no-cpu-baseline --no-ttt-c1 --no-e2e >> gpurun_out/r2p_cfg.jsonl 2>> gpurun_out/r2p_cfg.err
done
timeout 300 python bench.py --config C1 --batch 64 --steps 2000 --warmup 50 --no-cpu-baseline --no-ttt-c1 --no-e2e --no-sustained --profile-reps 0 >> gpurun_out/r2p_batch.jsonl 2>> gpurun_out/r2p_batch.err
