set -x
export PYTHONUNBUFFERED=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2m_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2m_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2m_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2m_pytest.log
for t in "" "expminb=2" "expminb=3"; do
  PDCS_TUNE=$t timeout 300 python bench.py --config C3 --steps 2000 --warmup 50 --no-cpu-baseline --no-ttt-c1 --no-e2e >> gpurun_out/r2m_c3.jsonl 2>> gpurun_out/r2m_c3.err
done
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r2m_c5.json 2> gpurun_out/r2m_c5.err
for t in "" "persist=0"; do
  PDCS_TUNE=$t timeout 300 python bench.py --config C1 --steps 2000 --warmup 50 --no-cpu-baseline --no-e2e --profile-reps 0 >> gpurun_out/r2m_c1.jsonl 2>> gpurun_out/r2m_c1.err
done
timeout 300 python tools/profile_e2e.py C5 20 > gpurun_out/r2m_prof_e2e.txt 2>&1
