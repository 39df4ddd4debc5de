export PYTHONUNBUFFERED=1
for c in C2 C2p C3 C3p C4 C5s; do
for t in "" "cls=0"; do
  PDCS_TUNE="$t" timeout 300 python bench.py --config $c --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r3g_cfg.jsonl 2>> gpurun_out/r3g_cfg.err
done
done
