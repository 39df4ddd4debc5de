export PYTHONUNBUFFERED=1
for t in "" "gpass=4" "gpass=6" "gy=6" "gt=6" "gx=4" ""; do
  PDCS_TUNE="$t" timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r4n_cfg.jsonl 2>> gpurun_out/r4n_cfg.err
done
