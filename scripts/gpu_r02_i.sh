#!/bin/bash
# r02 A/B I: cold state in shared memory (88 regs at 640 threads) vs base; 768 / 832-thread packed CTAs
mkdir -p gpurun_out
P=paper_2509_12207_b200
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_i.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_i.log
tail -3 gpurun_out/pytest_i.log
echo "== jitter urgengo 50k"; timeout 1500 python tools/ab.py jitter urgengo 50000 $P/liburg_base.so $P/liburg.so $P/liburg_pk768.so $P/liburg_pk832.so 2>&1 | tee gpurun_out/ab_i.txt
echo "== scaleout urgengo 300k"; timeout 900 python tools/ab.py scaleout urgengo 300000 $P/liburg_base.so $P/liburg.so $P/liburg_pk768.so $P/liburg_pk832.so 2>&1 | tee -a gpurun_out/ab_i.txt
echo "== usweep fifo 100k"; timeout 600 python tools/ab.py usweep fifo 100000 $P/liburg_base.so $P/liburg.so $P/liburg_pk768.so 2>&1 | tee -a gpurun_out/ab_i.txt
echo "== paper11 urgengo"; timeout 600 python tools/ab.py paper11 urgengo 0 $P/liburg_base.so $P/liburg.so 2>&1 | tee -a gpurun_out/ab_i.txt
