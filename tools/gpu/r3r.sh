export PYTHONUNBUFFERED=1
for t in "" "thread_max=16" "" "thread_max=16"; do
  PDCS_TUNE="$t" timeout 300 python bench.py --config C2 --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r3r_cfg.jsonl 2>> gpurun_out/r3r_cfg.err
done
for t in "" "thread_max=16"; do
  PDCS_TUNE="$t" timeout 300 python bench.py --config C2p --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r3r_cfg.jsonl 2>> gpurun_out/r3r_cfg.err
done
