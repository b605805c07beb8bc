#!/bin/bash
# r02 A/B F: base vs +lb/32-bit constants vs +fast-step budget
mkdir -p gpurun_out
P=paper_2509_12207_b200
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_f.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f.log
tail -3 gpurun_out/pytest_f.log
echo "== jitter urgengo 50k"; timeout 1200 python tools/ab.py jitter urgengo 50000 $P/liburg_base.so $P/liburg_lb.so $P/liburg.so 2>&1 | tee gpurun_out/ab_f.txt
echo "== scaleout urgengo 300k"; timeout 900 python tools/ab.py scaleout urgengo 300000 $P/liburg_base.so $P/liburg_lb.so $P/liburg.so 2>&1 | tee -a gpurun_out/ab_f.txt
echo "== usweep fifo 100k"; timeout 600 python tools/ab.py usweep fifo 100000 $P/liburg_base.so $P/liburg.so 2>&1 | tee -a gpurun_out/ab_f.txt
echo "== usweep static 100k"; timeout 600 python tools/ab.py usweep static 100000 $P/liburg_base.so $P/liburg.so 2>&1 | tee -a gpurun_out/ab_f.txt
echo "== paper11 urgengo"; timeout 600 python tools/ab.py paper11 urgengo 0 $P/liburg_base.so $P/liburg_lb.so $P/liburg.so 2>&1 | tee -a gpurun_out/ab_f.txt
