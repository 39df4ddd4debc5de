set -x
export PYTHONUNBUFFERED=1
for t in "" "ubox=0" "split=1" "split=1,hs=1" "hs=1"; do
  PDCS_TUNE=$t timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-ttt-c1 --no-e2e >> gpurun_out/r2e_c5.jsonl 2>> gpurun_out/r2e_c5.err
done
PDCS_TUNE=split=1,hs=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py -x -q -k "c5 or C5 or solve_matches_reference" > gpurun_out/r2e_pytest_split.log 2>&1; echo rc=$? >> gpurun_out/r2e_pytest_split.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c5 or C5 or solve_matches_reference or step_level" > gpurun_out/r2e_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2e_pytest.log
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_blk_exp<2" -s 3 -c 1 -o gpurun_out/r2e_c3exp python bench.py --config C3 --steps 40 --warmup 10 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained --profile-reps 0 > gpurun_out/r2e_ncu.log 2>&1
