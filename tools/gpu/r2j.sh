set -x
export PYTHONUNBUFFERED=1
PDCS_TIMING=1 timeout 300 python tools/profile_e2e.py C5 20 > gpurun_out/r2j_prof_e2e.txt 2>&1
timeout 1000 python tools/ttt.py C5 1e-4 900 >> gpurun_out/r2j_ttt.jsonl 2>> gpurun_out/r2j_ttt.err
timeout 1000 python tools/ttt.py C5planted 1e-6 900 >> gpurun_out/r2j_ttt.jsonl 2>> gpurun_out/r2j_ttt.err
for c in C2 C3 C4; do timeout 900 python tools/ttt.py $c 1e-6 800 >> gpurun_out/r2j_ttt.jsonl 2>> gpurun_out/r2j_ttt.err; done
