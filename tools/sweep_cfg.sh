# per-config launch sweep: CFG=C4 SWEEP="default tile_t=1 ..." bash tools/sweep_cfg.sh (under gpurun)
mkdir -p gpurun_out
for T in ${SWEEP:-default}; do
  [ "$T" = "default" ] && T=""
  PDCS_TUNE="$T" timeout 300 python bench.py --config ${CFG:-C5} --steps ${STEPS:-600} --warmup 50 --no-cpu-baseline --no-e2e --profile-reps 3 > gpurun_out/sw.json 2>gpurun_out/sw.err || { echo "FAIL $T"; tail -3 gpurun_out/sw.err; continue; }
  python -c "
import json; d=json.load(open('gpurun_out/sw.json')); s=d['stages_ms']
print('%s %-24s %8.1f it/s  ' % ('${CFG:-C5}', '$T' or 'default', d['value']) + ' '.join('%s=%.3f' % (k, v) for k, v in s.items()))"
done
