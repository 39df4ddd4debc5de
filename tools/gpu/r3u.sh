export PYTHONUNBUFFERED=1
for t in "pool_gb=4" "pool_gb=64" "pool_gb=4" "pool_gb=64"; do
  echo "$t" >> gpurun_out/r3u.txt
  PDCS_TUNE=$t PDCS_TIMING=1 timeout 600 python tools/e2e_var.py 5 > gpurun_out/r3u_tmp.txt 2>&1
  grep -E "^rep .*wall|create transpose|create panels|row ids" gpurun_out/r3u_tmp.txt | cut -c1-120 >> gpurun_out/r3u.txt
done
