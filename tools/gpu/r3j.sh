export PYTHONUNBUFFERED=1
for c in C4 C2; do
for t in "" "cls_vw=4"; do
  PDCS_TUNE="$t" timeout 300 python bench.py --config $c --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r3j_cfg.jsonl 2>> gpurun_out/r3j_cfg.err
done
done
