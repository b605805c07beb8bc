#!/bin/bash
# r02 pass W: on top of the pass-U kernels, the warp index through a lane-0 shuffle (uniform register for the
# warp's slot base, no per-use rematerialisation) in the packed UrgenGo build (uw); parity tests on uw
mkdir -p gpurun_out
P=paper_2509_12207_b200
URG_LIB=$PWD/$P/liburg_uwall.so timeout 1200 python -m pytest tests -m gpu -q -x -k "not debug" > gpurun_out/pytest_w.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_w.log
tail -2 gpurun_out/pytest_w.log
echo "== jitter urgengo 50k"; timeout 1200 python tools/ab.py jitter urgengo 50000 $P/liburg.so $P/liburg_uw.so $P/liburg_uwall.so 2>&1 | tee gpurun_out/ab_w.txt
echo "== scaleout urgengo 300k"; timeout 900 python tools/ab.py scaleout urgengo 300000 $P/liburg.so $P/liburg_uw.so $P/liburg_uwall.so 2>&1 | tee -a gpurun_out/ab_w.txt
echo "== usweep fifo 100k"; timeout 600 python tools/ab.py usweep fifo 100000 $P/liburg.so $P/liburg_uwall.so 2>&1 | tee -a gpurun_out/ab_w.txt
echo "== usweep static 100k"; timeout 600 python tools/ab.py usweep static 100000 $P/liburg.so $P/liburg_uwall.so 2>&1 | tee -a gpurun_out/ab_w.txt
echo "== paper11 urgengo"; timeout 600 python tools/ab.py paper11 urgengo 0 $P/liburg.so $P/liburg_uwall.so 2>&1 | tee -a gpurun_out/ab_w.txt
