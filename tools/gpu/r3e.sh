export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py -q -x -k "long or C4 or c4 or giant" > gpurun_out/r3e_pt.log 2>&1; echo rc=$? >> gpurun_out/r3e_pt.log
for c in C4 C3; do
  timeout 300 python bench.py --config $c --steps 300 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r3e_cfg.jsonl 2>> gpurun_out/r3e_cfg.err
done
