#!/bin/bash
# r02 A/B 1: packed FIFO/STATIC regression fix (oldc = r01 behaviour) and the per-kernel Philox block cache (nokq = r01)
mkdir -p gpurun_out
P=paper_2509_12207_b200
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_ab1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ab1.log
tail -3 gpurun_out/pytest_ab1.log
echo "== jitter urgengo 50k"; timeout 900 python tools/ab.py jitter urgengo 50000 $P/liburg.so $P/liburg_nokq.so $P/liburg_oldc.so 2>&1 | tee gpurun_out/ab1.txt
echo "== jitter fifo 50k"; timeout 900 python tools/ab.py jitter fifo 50000 $P/liburg.so $P/liburg_oldc.so 2>&1 | tee -a gpurun_out/ab1.txt
echo "== usweep fifo 100k"; timeout 600 python tools/ab.py usweep fifo 100000 $P/liburg.so $P/liburg_oldc.so 2>&1 | tee -a gpurun_out/ab1.txt
echo "== usweep static 100k"; timeout 600 python tools/ab.py usweep static 100000 $P/liburg.so $P/liburg_oldc.so 2>&1 | tee -a gpurun_out/ab1.txt
echo "== scaleout urgengo 300k"; timeout 600 python tools/ab.py scaleout urgengo 300000 $P/liburg.so $P/liburg_oldc.so 2>&1 | tee -a gpurun_out/ab1.txt
echo "== paper11 urgengo"; timeout 600 python tools/ab.py paper11 urgengo 0 $P/liburg.so $P/liburg_oldc.so 2>&1 | tee -a gpurun_out/ab1.txt
