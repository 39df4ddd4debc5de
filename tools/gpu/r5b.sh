export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py tests/test_gpu_variants.py tests/test_gpu_acceptance.py -q -k "giant or c4 or C4 or rsoc or markowitz" > gpurun_out/r5b_pt.log 2>&1; echo rc=$? >> gpurun_out/r5b_pt.log
for t in "" "giantfuse=0" "" "giantfuse=0"; do
  PDCS_TUNE="$t" timeout 300 python bench.py --config C4 --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r5b_cfg.jsonl 2>> gpurun_out/r5b_cfg.err
done
