export PYTHONUNBUFFERED=1
cp paper_2603_15504_b200/libpdcs.so /tmp/new.so
for v in new old new old; do
  if [ $v = old ]; then cp tools/old_libpdcs.so paper_2603_15504_b200/libpdcs.so; else cp /tmp/new.so paper_2603_15504_b200/libpdcs.so; fi
  touch -d '2030-01-01' paper_2603_15504_b200/libpdcs.so
  echo $v >> gpurun_out/r4g_cfg.jsonl
  timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r4g_cfg.jsonl 2>> gpurun_out/r4g_cfg.err
done
cp /tmp/new.so paper_2603_15504_b200/libpdcs.so; touch -d '2030-01-01' paper_2603_15504_b200/libpdcs.so
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "c5 or C5 or box" > gpurun_out/r4g_pt.log 2>&1; echo rc=$? >> gpurun_out/r4g_pt.log
