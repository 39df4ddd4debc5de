export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_variants.py -q > gpurun_out/r3h_var.log 2>&1; echo rc=$? >> gpurun_out/r3h_var.log
timeout 900 python -m pytest tests/test_gpu_scale_parity.py -q -k "c2p or c3p or c4" > gpurun_out/r3h_par.log 2>&1; echo rc=$? >> gpurun_out/r3h_par.log
for c in C2p C3p C4 C5s; do
  timeout 300 python bench.py --config $c --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r3h_cfg.jsonl 2>> gpurun_out/r3h_cfg.err
done
