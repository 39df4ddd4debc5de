export PYTHONUNBUFFERED=1
for t in "" "cls=0" "" "cls=0"; do
  PDCS_TUNE="$t" timeout 300 python bench.py --config C3 --steps 300 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r3b_cfg.jsonl 2>> gpurun_out/r3b_cfg.err
done
