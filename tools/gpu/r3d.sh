export PYTHONUNBUFFERED=1
for c in C4 C3; do
for t in "" "chunk=2048" "chunk=4096" "chunk=16384"; do
  PDCS_TUNE="$t" timeout 300 python bench.py --config $c --steps 300 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r3d_cfg.jsonl 2>> gpurun_out/r3d_cfg.err
done
done
