set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2c_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2c_pytest.log
timeout 300 tools/c5_lab 10 > gpurun_out/r2c_lab.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_blk_exp -s 6 -c 1 -o gpurun_out/r2c_c3exp python bench.py --config C3 --steps 40 --warmup 10 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained --profile-reps 0 > gpurun_out/r2c_ncu.log 2>&1
