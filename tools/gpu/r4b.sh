export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_variants.py -q > gpurun_out/r4b_var.log 2>&1; echo rc=$? >> gpurun_out/r4b_var.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py -q -k "c4 or C4 or rsoc or giant or long" > gpurun_out/r4b_par.log 2>&1; echo rc=$? >> gpurun_out/r4b_par.log
for t in "" "runs=0" "" "runs=0"; do
  PDCS_TUNE="$t" timeout 300 python bench.py --config C4 --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r4b_cfg.jsonl 2>> gpurun_out/r4b_cfg.err
done
