export PYTHONUNBUFFERED=1
for c in C1 C2 C3 C4 C2p C3p; do
  timeout 400 python bench.py --config $c --steps 2000 --warmup 50 --no-cpu-baseline --no-ttt-c1 --no-e2e >> gpurun_out/r3p_cfg.jsonl 2>> gpurun_out/r3p_cfg.err
done
timeout 600 python bench.py --steps 200 --warmup 20 > gpurun_out/r3p_c5.json 2> gpurun_out/r3p_c5.err
for c in C1 C2 C3 C4; do
  timeout 300 python tools/ttt.py $c 1e-6 250 >> gpurun_out/r3p_ttt.jsonl 2>> gpurun_out/r3p_ttt.err
done
timeout 300 python bench.py --config C1 --batch 64 --steps 2000 --warmup 50 --no-cpu-baseline --no-e2e --profile-reps 0 > gpurun_out/r3p_c1b.json 2>> gpurun_out/r3p_c1b.err
