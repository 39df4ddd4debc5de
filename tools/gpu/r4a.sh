export PYTHONUNBUFFERED=1
for t in "" "expminb=3" "expminb=2" ""; do
  PDCS_TUNE="$t" timeout 300 python bench.py --config C3 --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r4a_cfg.jsonl 2>> gpurun_out/r4a_cfg.err
done
