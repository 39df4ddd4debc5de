export PYTHONUNBUFFERED=1
for t in "" "halfminb=3" "halfminb=4"; do
  PDCS_TUNE="$t" timeout 300 python bench.py --config C2 --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r3l_cfg.jsonl 2>> gpurun_out/r3l_cfg.err
done
