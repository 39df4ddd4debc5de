set -x
export PYTHONUNBUFFERED=1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct --clock-control none --launch-skip 3000 --launch-count 60 --csv --log-file gpurun_out/r2u_c2_launches.csv python bench.py --config C2 --steps 600 --warmup 5 --no-cpu-baseline --no-ttt-c1 --no-e2e --no-sustained --profile-reps 0 > gpurun_out/r2u_c2_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_rows_pass|k_y_epi|k_t_epi|k_blk" --launch-skip 300 --launch-count 8 -o gpurun_out/r2u_c2full python bench.py --config C2 --steps 400 --warmup 5 --no-cpu-baseline --no-ttt-c1 --no-e2e --no-sustained --profile-reps 0 > gpurun_out/r2u_c2full.log 2>&1
