#!/bin/bash
# r02 pass M: branch-free due vote + (latency core build) the kernel behind the head drawn ahead, vs
# base; packed CTAs of 896 / 1024 threads (UrgenGo) and 896 (FIFO)
mkdir -p gpurun_out
P=paper_2509_12207_b200
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_m.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_m.log
tail -2 gpurun_out/pytest_m.log
echo "== paper11 urgengo"; timeout 600 python tools/ab.py paper11 urgengo 0 $P/liburg_base.so $P/liburg_nopre2.so $P/liburg.so 2>&1 | tee gpurun_out/ab_m.txt
echo "== jitter urgengo 50k"; timeout 1200 python tools/ab.py jitter urgengo 50000 $P/liburg_base.so $P/liburg.so $P/liburg_t896.so $P/liburg_t1024.so 2>&1 | tee -a gpurun_out/ab_m.txt
echo "== scaleout urgengo 300k"; timeout 600 python tools/ab.py scaleout urgengo 300000 $P/liburg_base.so $P/liburg.so $P/liburg_t896.so 2>&1 | tee -a gpurun_out/ab_m.txt
echo "== usweep fifo 100k"; timeout 600 python tools/ab.py usweep fifo 100000 $P/liburg_base.so $P/liburg.so $P/liburg_a896.so 2>&1 | tee -a gpurun_out/ab_m.txt
echo "== usweep static 100k"; timeout 600 python tools/ab.py usweep static 100000 $P/liburg_base.so $P/liburg.so $P/liburg_a896.so 2>&1 | tee -a gpurun_out/ab_m.txt
