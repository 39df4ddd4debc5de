export PYTHONUNBUFFERED=1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_ctrl_ls" --launch-skip 300 --launch-count 1 -o gpurun_out/r4c_ctrl python bench.py --config C2 --steps 400 --warmup 5 --no-cpu-baseline --no-ttt-c1 --no-e2e --no-sustained --profile-reps 0 > gpurun_out/r4c.log 2>&1
