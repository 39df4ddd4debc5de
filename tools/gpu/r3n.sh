export PYTHONUNBUFFERED=1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_blk_exp" --launch-skip 200 --launch-count 1 -o gpurun_out/r3n_c3exp python bench.py --config C3 --steps 400 --warmup 5 --no-cpu-baseline --no-ttt-c1 --no-e2e --no-sustained --profile-reps 0 > gpurun_out/r3n.log 2>&1
