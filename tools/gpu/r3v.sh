export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_batch.py tests/test_gpu_parity.py -q -x > gpurun_out/r3v_pt.log 2>&1; echo rc=$? >> gpurun_out/r3v_pt.log
for t in "pool_gb=4" "pool_gb=64" "pool_gb=4" "pool_gb=64"; do
  echo "$t" >> gpurun_out/r3v.txt
  PDCS_TUNE=$t PDCS_TIMING=1 timeout 600 python tools/e2e_var.py 6 > gpurun_out/r3v_tmp.txt 2>&1
  grep -E "^rep .*wall" gpurun_out/r3v_tmp.txt | cut -c1-140 >> gpurun_out/r3v.txt
done
