export PYTHONUNBUFFERED=1
for t in "" "vwy=32" "vwt=32" "vwy=32,vwt=32" "vwy=1,vwt=1" ""; do
  PDCS_TUNE="$t" timeout 300 python bench.py --config C1 --steps 2000 --warmup 50 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained --profile-reps 0 >> gpurun_out/r4z_cfg.jsonl 2>> gpurun_out/r4z_cfg.err
done
