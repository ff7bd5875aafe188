#!/bin/bash
# ncu evidence for the headline kernels (run under gpurun, 1 GPU).
# 1) launch list of one bench-like pyramid (per-launch durations, cold, serialised)
# 2) one --set full capture of the level-1 kernel (16384^2, TMA-staged rows)
# 3) one --set full capture of the fused level-pair kernel (levels 1+2 of 16384^2)
set -e
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches.csv python scripts/prof_level.py --pyramid 8 --iters 2 > /dev/null
ncu --set full --clock-control none --import-source on -k regex:level_kernel -s 2 -c 1 \
    -o gpurun_out/prof_level1 -f python scripts/prof_level.py --iters 3 > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 1 -c 1 \
    -o gpurun_out/prof_pair -f python scripts/prof_pair.py --iters 3 > gpurun_out/ncu_pair.log 2>&1
