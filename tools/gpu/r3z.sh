export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_variants.py -q > gpurun_out/r3z_var.log 2>&1; echo rc=$? >> gpurun_out/r3z_var.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py -q -k "exp or c3 or C3 or dexp or expc" > gpurun_out/r3z_par.log 2>&1; echo rc=$? >> gpurun_out/r3z_par.log
for t in "" "expfuse=0" "" "expfuse=0"; do
  PDCS_TUNE="$t" timeout 300 python bench.py --config C3 --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r3z_cfg.jsonl 2>> gpurun_out/r3z_cfg.err
done
