set -x
export PYTHONUNBUFFERED=1
for t in "" "ubox=0" "split=1" "split=1,hs=1" "hs=1"; do
  PDCS_TUNE=$t timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-ttt-c1 --no-e2e >> gpurun_out/r2f_c5.jsonl 2>> gpurun_out/r2f_c5.err
done
PDCS_TIMING=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ttt-c1 --no-sustained > gpurun_out/r2f_e2e.json 2> gpurun_out/r2f_e2e.err
timeout 300 tools/c5_lab 10 > gpurun_out/r2f_lab.txt 2>&1
PDCS_TUNE=split=1,hs=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py -x -q -k "c5 or C5 or solve_matches_reference" > gpurun_out/r2f_pytest_split.log 2>&1; echo rc=$? >> gpurun_out/r2f_pytest_split.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2f_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2f_pytest.log
timeout 300 python bench.py --config C3 --steps 40 --warmup 10 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained --profile-reps 0 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_blk_exp<2" -s 3 -c 1 -o gpurun_out/r2f_c3exp python bench.py --config C3 --steps 40 --warmup 10 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained --profile-reps 0 > gpurun_out/r2f_ncu.log 2>&1
