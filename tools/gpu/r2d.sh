set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_sanitizer.py tests/test_gpu_sharded.py -x -q > gpurun_out/r2d_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2d_pytest.log
PDCS_TIMING=1 timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2d_bench_c5.json 2> gpurun_out/r2d_bench_c5.err
timeout 600 python bench.py --sharded --selfcheck --steps 200 --warmup 20 --no-cpu-baseline --no-ttt-c1 > gpurun_out/r2d_sharded.json 2> gpurun_out/r2d_sharded.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2d_ref.json 2> gpurun_out/r2d_ref.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_blk_exp -s 30 -c 6 -o gpurun_out/r2d_c3exp python bench.py --config C3 --steps 40 --warmup 10 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained --profile-reps 0 > gpurun_out/r2d_ncu.log 2>&1
