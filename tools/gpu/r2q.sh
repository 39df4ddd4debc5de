set -x
export PYTHONUNBUFFERED=1
for t in "" "pt=1" "py=2" "py=4" "pt=3" "pt=1,py=4"; do
  PDCS_TUNE=$t timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-ttt-c1 --no-e2e >> gpurun_out/r2q_c5.jsonl 2>> gpurun_out/r2q_c5.err
done
