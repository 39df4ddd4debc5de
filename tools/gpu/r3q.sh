export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_variants.py -q > gpurun_out/r3q_var.log 2>&1; echo rc=$? >> gpurun_out/r3q_var.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py tests/test_gpu_batch.py -q -k "C2 or c2 or batch or socp or ball or solve_matches" > gpurun_out/r3q_par.log 2>&1; echo rc=$? >> gpurun_out/r3q_par.log
for t in "" "yblkfuse=0" "" "yblkfuse=0"; do
  PDCS_TUNE="$t" timeout 300 python bench.py --config C2 --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r3q_cfg.jsonl 2>> gpurun_out/r3q_cfg.err
done
