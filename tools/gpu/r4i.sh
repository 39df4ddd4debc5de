export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_variants.py -q > gpurun_out/r4i_var.log 2>&1; echo rc=$? >> gpurun_out/r4i_var.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py tests/test_gpu_acceptance.py -q -k "prim or c3p or exp or nan" > gpurun_out/r4i_par.log 2>&1; echo rc=$? >> gpurun_out/r4i_par.log
for t in "" "texpfuse=0" "" "texpfuse=0"; do
  PDCS_TUNE="$t" timeout 300 python bench.py --config C3p --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r4i_cfg.jsonl 2>> gpurun_out/r4i_cfg.err
done
