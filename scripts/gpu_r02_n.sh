#!/bin/bash
# r02 pass N: packed CTAs UrgenGo 1024 / ASYNC 896 (default) vs 832 / 768 (base, = pass M's nopre2);
# ASYNC 1024 variant; GPU tests on the default
mkdir -p gpurun_out
P=paper_2509_12207_b200
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_n.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_n.log
tail -2 gpurun_out/pytest_n.log
echo "== jitter urgengo 50k"; timeout 900 python tools/ab.py jitter urgengo 50000 $P/liburg_base.so $P/liburg.so 2>&1 | tee gpurun_out/ab_n.txt
echo "== scaleout urgengo 300k"; timeout 600 python tools/ab.py scaleout urgengo 300000 $P/liburg_base.so $P/liburg.so 2>&1 | tee -a gpurun_out/ab_n.txt
echo "== usweep fifo 100k"; timeout 600 python tools/ab.py usweep fifo 100000 $P/liburg_base.so $P/liburg.so $P/liburg_a1024.so 2>&1 | tee -a gpurun_out/ab_n.txt
echo "== usweep static 100k"; timeout 600 python tools/ab.py usweep static 100000 $P/liburg_base.so $P/liburg.so $P/liburg_a1024.so 2>&1 | tee -a gpurun_out/ab_n.txt
echo "== paper11 urgengo"; timeout 600 python tools/ab.py paper11 urgengo 0 $P/liburg_base.so $P/liburg.so 2>&1 | tee -a gpurun_out/ab_n.txt
