set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py tests/test_gpu_acceptance.py tests/test_gpu_batch.py -x -q -k "c2 or C2 or solve_matches_reference or batch or socp or ball" > gpurun_out/r2i_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2i_pytest.log
for t in "" "socfuse=0"; do
  PDCS_TUNE=$t timeout 300 python bench.py --config C2 --steps 2000 --warmup 50 --no-cpu-baseline --no-ttt-c1 --no-e2e >> gpurun_out/r2i_c2.jsonl 2>> gpurun_out/r2i_c2.err
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --launch-skip 1500 --launch-count 80 --csv --log-file gpurun_out/r2i_c5_launches.csv python bench.py --steps 400 --warmup 5 --no-cpu-baseline --no-ttt-c1 --no-e2e --no-sustained --profile-reps 0 > gpurun_out/r2i_c5_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_lane_pass|k_y_epi|k_t_epi|k_step_x" --launch-skip 400 --launch-count 8 -o gpurun_out/r2i_c5full python bench.py --steps 400 --warmup 5 --no-cpu-baseline --no-ttt-c1 --no-e2e --no-sustained --profile-reps 0 > gpurun_out/r2i_c5full.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --launch-skip 1500 --launch-count 80 --csv --log-file gpurun_out/r2i_c2_launches.csv python bench.py --config C2 --steps 400 --warmup 5 --no-cpu-baseline --no-ttt-c1 --no-e2e --no-sustained --profile-reps 0 > gpurun_out/r2i_c2_ncu.log 2>&1
