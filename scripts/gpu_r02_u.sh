#!/bin/bash
# r02 pass U: on top of nl (per-instance launch count), the any-multi test read off the fit ballot
# (nlam) and the fast-step budget kept as a fixed end point (nlamb); GPU parity tests on nlamb
mkdir -p gpurun_out
P=paper_2509_12207_b200
URG_LIB=$PWD/$P/liburg_nlamb.so timeout 1200 python -m pytest tests -m gpu -q -x -k "not debug" > gpurun_out/pytest_u.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_u.log
tail -2 gpurun_out/pytest_u.log
echo "== jitter urgengo 50k"; timeout 1200 python tools/ab.py jitter urgengo 50000 $P/liburg.so $P/liburg_nl.so $P/liburg_nlam.so $P/liburg_nlamb.so 2>&1 | tee gpurun_out/ab_u.txt
echo "== scaleout urgengo 300k"; timeout 900 python tools/ab.py scaleout urgengo 300000 $P/liburg.so $P/liburg_nl.so $P/liburg_nlam.so $P/liburg_nlamb.so 2>&1 | tee -a gpurun_out/ab_u.txt
echo "== usweep fifo 100k"; timeout 600 python tools/ab.py usweep fifo 100000 $P/liburg.so $P/liburg_nlamb.so 2>&1 | tee -a gpurun_out/ab_u.txt
echo "== paper11 urgengo"; timeout 600 python tools/ab.py paper11 urgengo 0 $P/liburg.so $P/liburg_nl.so $P/liburg_nlamb.so 2>&1 | tee -a gpurun_out/ab_u.txt
