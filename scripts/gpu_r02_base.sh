#!/bin/bash
# r02 baseline: timings of the r01 kernels on the round-2 headline slice and the regression cases
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_base.txt 2>&1
L=paper_2509_12207_b200/liburg.so
echo "== jitter 50k (configs[3] slice)"; timeout 600 python tools/ab.py jitter urgengo 50000 $L 2>&1 | tee gpurun_out/base.txt
echo "== jitter fifo 50k"; timeout 600 python tools/ab.py jitter fifo 50000 $L 2>&1 | tee -a gpurun_out/base.txt
echo "== usweep fifo 100k"; timeout 600 python tools/ab.py usweep fifo 100000 $L 2>&1 | tee -a gpurun_out/base.txt
echo "== usweep static 100k"; timeout 600 python tools/ab.py usweep static 100000 $L 2>&1 | tee -a gpurun_out/base.txt
echo "== scaleout 300k"; timeout 600 python tools/ab.py scaleout urgengo 300000 $L 2>&1 | tee -a gpurun_out/base.txt
