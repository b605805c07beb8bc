#!/bin/bash
# r02 pass V: all GPU tests on the default (pass-U kernels); per-half utilisation sums packed in one
# REDUX (hs) and, for packed UrgenGo, any-retire / any-due from one REDUX.OR (rohs)
mkdir -p gpurun_out
P=paper_2509_12207_b200
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_v.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_v.log
tail -2 gpurun_out/pytest_v.log
URG_LIB=$PWD/$P/liburg_rohs.so timeout 1200 python -m pytest tests -m gpu -q -x -k "not debug" > gpurun_out/pytest_v_rohs.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_v_rohs.log
tail -2 gpurun_out/pytest_v_rohs.log
echo "== jitter urgengo 50k"; timeout 1200 python tools/ab.py jitter urgengo 50000 $P/liburg.so $P/liburg_hs.so $P/liburg_rohs.so 2>&1 | tee gpurun_out/ab_v.txt
echo "== scaleout urgengo 300k"; timeout 900 python tools/ab.py scaleout urgengo 300000 $P/liburg.so $P/liburg_hs.so $P/liburg_rohs.so 2>&1 | tee -a gpurun_out/ab_v.txt
echo "== usweep fifo 100k"; timeout 600 python tools/ab.py usweep fifo 100000 $P/liburg.so $P/liburg_hs.so 2>&1 | tee -a gpurun_out/ab_v.txt
echo "== usweep static 100k"; timeout 600 python tools/ab.py usweep static 100000 $P/liburg.so $P/liburg_hs.so 2>&1 | tee -a gpurun_out/ab_v.txt
