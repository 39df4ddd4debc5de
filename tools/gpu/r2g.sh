set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_parity.py -x -q -k "batch or solve_many" > gpurun_out/r2g_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2g_pytest.log
for b in 8 32 64; do
  timeout 600 python bench.py --config C1 --batch $b --steps 2000 --warmup 50 --no-cpu-baseline --no-ttt-c1 --no-e2e --no-sustained --profile-reps 0 >> gpurun_out/r2g_batch.jsonl 2>> gpurun_out/r2g_batch.err
done
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r2g_c5.json 2> gpurun_out/r2g_c5.err
for c in C1 C2 C3 C4; do
  timeout 300 python bench.py --config $c --steps 2000 --warmup 50 --no-cpu-baseline --no-ttt-c1 --no-e2e >> gpurun_out/r2g_cfg.jsonl 2>> gpurun_out/r2g_cfg.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_blk_exp<\(int\)2" -s 3 -c 1 -o gpurun_out/r2g_c3exp python bench.py --config C3 --steps 40 --warmup 10 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained --profile-reps 0 > gpurun_out/r2g_ncu.log 2>&1
