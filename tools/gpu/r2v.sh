set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_variants.py -q -x > gpurun_out/r2v_var.log 2>&1; echo rc=$? >> gpurun_out/r2v_var.log
for t in "" "cls_vw=8" "cls_vw=16" "cls_vw=32" "cls=0"; do
  PDCS_TUNE="$t" timeout 300 python bench.py --config C2 --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r2v_c2.jsonl 2>> gpurun_out/r2v_c2.err
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "C2 or c2s" > gpurun_out/r2v_par.log 2>&1; echo rc=$? >> gpurun_out/r2v_par.log
timeout 900 python -m pytest tests/test_gpu_scale_parity.py -q -k "c2" >> gpurun_out/r2v_par.log 2>&1; echo rc=$? >> gpurun_out/r2v_par.log
