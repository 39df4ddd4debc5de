export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_variants.py -q > gpurun_out/r3i_var.log 2>&1; echo rc=$? >> gpurun_out/r3i_var.log
for c in C2 C2p C3 C3p C4 C5s; do
  timeout 300 python bench.py --config $c --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r3i_cfg.jsonl 2>> gpurun_out/r3i_cfg.err
done
