set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2b_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2b_pytest.log
for t in "" "expminb=3" "expminb=4" "expsplit=0"; do
  PDCS_TUNE=$t timeout 300 python bench.py --config C3 --steps 2000 --warmup 50 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r2b_c3.jsonl 2>> gpurun_out/r2b_c3.err
done
timeout 300 tools/c5_lab 10 > gpurun_out/r2b_lab.txt 2>&1
