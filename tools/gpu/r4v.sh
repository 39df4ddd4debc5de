export PYTHONUNBUFFERED=1
for cfg in "32 2" "32 3" "64 3" "16 4" "32 2"; do
  set -- $cfg
  echo "stage_mb=$1 stages=$2" >> gpurun_out/r4v.txt
  PDCS_STAGE_MB=$1 PDCS_STAGES=$2 timeout 600 python tools/e2e_var.py 5 2>/dev/null | grep "^rep" | sed 's/engine init.*precondition/ .. precondition/' | cut -c1-120 >> gpurun_out/r4v.txt
done
