export PYTHONUNBUFFERED=1
cp paper_2603_15504_b200/libpdcs.so /tmp/new.so
for v in new old new old; do
  if [ $v = old ]; then cp tools/old_libpdcs.so paper_2603_15504_b200/libpdcs.so; else cp /tmp/new.so paper_2603_15504_b200/libpdcs.so; fi
  touch -d '2030-01-01' paper_2603_15504_b200/libpdcs.so
  echo $v >> gpurun_out/r3c_cfg.jsonl
  timeout 300 python bench.py --config C3 --steps 300 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r3c_cfg.jsonl 2>> gpurun_out/r3c_cfg.err
done
nvidia-smi -q -d CLOCK,POWER,PERFORMANCE > gpurun_out/r3c_smi.txt
