# C5 launch-configuration sweep (bench.py per PDCS_TUNE variant); run under gpurun
mkdir -p gpurun_out
for T in ${SWEEP:-"" "py=1,pt=1" "py=2,pt=1" "py=3,pt=1" "py=4,pt=2" "py=3,pt=2" "py=6,pt=3"}; do
  [ "$T" = "default" ] && T=""
  PDCS_TUNE="$T" timeout 300 python bench.py --steps 600 --warmup 50 --no-cpu-baseline --no-e2e --profile-reps 3 > gpurun_out/sw.json 2>gpurun_out/sw.err || { echo "FAIL $T"; tail -3 gpurun_out/sw.err; continue; }
  python -c "
import json; d=json.load(open('gpurun_out/sw.json')); s=d['stages_ms']; L=d['config']['launch']
print('%-22s %7.1f it/s  x=%.3f y=%.3f t=%.3f  panels=%d/%d vw=%d/%d grids=%d/%d/%d' % ('$T' or 'default', d['value'], s['step_x'], s['step_y_spmv'], s['step_t_spmv'], L['panels_g'], L['panels_gt'], L['step_vw_g'], L['step_vw_gt'], L['grid_step_x'], L['grid_step_y'], L['grid_step_t']))"
done
