export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_variants.py -q > gpurun_out/r4w_var.log 2>&1; echo rc=$? >> gpurun_out/r4w_var.log
for t in "" "thread_max=4,halfw=4" "thread_max=4"; do
  PDCS_TUNE="$t" timeout 300 python bench.py --config C2 --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r4w_cfg.jsonl 2>> gpurun_out/r4w_cfg.err
done
for t in "" "xhalfw=4"; do
  PDCS_TUNE="$t" timeout 300 python bench.py --config C2p --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r4w_cfg.jsonl 2>> gpurun_out/r4w_cfg.err
done
