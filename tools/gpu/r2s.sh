set -x
export PYTHONUNBUFFERED=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2s_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2s_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2s_pytest.log
timeout 300 python bench.py --config C1 --batch 64 --steps 2000 --warmup 50 --no-cpu-baseline --no-e2e --profile-reps 0 >> gpurun_out/r2s_c1.jsonl 2>> gpurun_out/r2s_c1.err
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r2s_c5.json 2> gpurun_out/r2s_c5.err
