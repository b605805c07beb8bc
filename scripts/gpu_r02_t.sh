#!/bin/bash
# r02 pass T: launch counts kept per instance in the lane's record slot instead of a per-launch counter
# (liburg_nl) vs the pass-S default; GPU parity tests on the nl build (URG_LIB)
mkdir -p gpurun_out
P=paper_2509_12207_b200
URG_LIB=$PWD/$P/liburg_nl.so timeout 1200 python -m pytest tests -m gpu -q -x -k "not debug" > gpurun_out/pytest_t.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_t.log
tail -2 gpurun_out/pytest_t.log
echo "== jitter urgengo 50k"; timeout 1200 python tools/ab.py jitter urgengo 50000 $P/liburg.so $P/liburg_nl.so 2>&1 | tee gpurun_out/ab_t.txt
echo "== scaleout urgengo 300k"; timeout 600 python tools/ab.py scaleout urgengo 300000 $P/liburg.so $P/liburg_nl.so 2>&1 | tee -a gpurun_out/ab_t.txt
echo "== usweep fifo 100k"; timeout 600 python tools/ab.py usweep fifo 100000 $P/liburg.so $P/liburg_nl.so 2>&1 | tee -a gpurun_out/ab_t.txt
echo "== paper11 urgengo"; timeout 600 python tools/ab.py paper11 urgengo 0 $P/liburg.so $P/liburg_nl.so 2>&1 | tee -a gpurun_out/ab_t.txt
