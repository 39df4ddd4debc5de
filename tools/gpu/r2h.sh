set -x
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests/test_gpu_scale_parity.py -x -q > gpurun_out/r2h_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2h_pytest.log
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_blk_exp<\(int\)2" -s 3 -c 1 -o gpurun_out/r2h_c3exp python bench.py --config C3 --steps 40 --warmup 10 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained --profile-reps 0 > gpurun_out/r2h_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --launch-skip 200 --launch-count 60 --csv --log-file gpurun_out/r2h_c5_launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ttt-c1 --no-e2e --no-sustained --profile-reps 0 > gpurun_out/r2h_c5_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_lane_pass|k_y_epi|k_t_epi|k_step_x" --launch-skip 40 --launch-count 8 -o gpurun_out/r2h_c5full python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ttt-c1 --no-e2e --no-sustained --profile-reps 0 > gpurun_out/r2h_c5full.log 2>&1
for c in C3p C2p; do
  timeout 600 python bench.py --config $c --steps 2000 --warmup 50 --no-cpu-baseline --no-ttt-c1 --no-e2e >> gpurun_out/r2h_primal.jsonl 2>> gpurun_out/r2h_primal.err
done
