set -x
for mb in 48 160; do timeout 120 tools/tma_gather_probe $mb >> gpurun_out/r2l_tma.txt 2>&1; done
