export PYTHONUNBUFFERED=1
for t in "" "cls_cv=-1" "cls_cv=-1,cls_vw=8" "cls_cv=-1,cls_vw=16"; do
  PDCS_TUNE="$t" timeout 300 python bench.py --config C4 --steps 300 --warmup 20 --no-cpu-baseline --no-e2e --no-ttt-c1 --no-sustained >> gpurun_out/r3f_cfg.jsonl 2>> gpurun_out/r3f_cfg.err
done
