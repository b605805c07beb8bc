#!/bin/bash
# r02 pass L: warps per CTA of the packed build on a 50k-scenario configs[3] slice (25 000 warp jobs:
# 6.5 rounds at 26 warps x 148 SMs) and configs[2] FIFO (50 000 jobs, 14.1 rounds at 24), and the
# branch-free due vote (liburg_dp)
mkdir -p gpurun_out
P=paper_2509_12207_b200
for W in 26 25 24 22; do echo "== jitter urgengo 50k, $W warps/CTA"; URG_WARPS_PER_CTA=$W timeout 600 python tools/ab.py jitter urgengo 50000 $P/liburg.so 2>&1; done | tee gpurun_out/ab_l.txt
for W in 24 23 22; do echo "== usweep fifo 100k, $W warps/CTA"; URG_WARPS_PER_CTA=$W timeout 600 python tools/ab.py usweep fifo 100000 $P/liburg.so 2>&1; done | tee -a gpurun_out/ab_l.txt
echo "== jitter dp"; timeout 900 python tools/ab.py jitter urgengo 50000 $P/liburg.so $P/liburg_dp.so 2>&1 | tee -a gpurun_out/ab_l.txt
echo "== scaleout dp"; timeout 600 python tools/ab.py scaleout urgengo 300000 $P/liburg.so $P/liburg_dp.so 2>&1 | tee -a gpurun_out/ab_l.txt
echo "== paper11 dp"; timeout 600 python tools/ab.py paper11 urgengo 0 $P/liburg.so $P/liburg_dp.so 2>&1 | tee -a gpurun_out/ab_l.txt
