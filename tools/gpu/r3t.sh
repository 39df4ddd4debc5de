export PYTHONUNBUFFERED=1
for t in 4 8 12 4 8 12; do
  echo "threads $t" >> gpurun_out/r3t.txt
  PDCS_COPY_THREADS=$t timeout 600 python tools/e2e_var.py 4 2>/dev/null | grep rep >> gpurun_out/r3t.txt
done
