#!/bin/bash
# r02 pass AB: lambda from the parameter bank only in the packed FIFO / STATIC / classical builds (bl2;
# the packed UrgenGo kernel's SASS is unchanged); parity tests on bl2
mkdir -p gpurun_out
P=paper_2509_12207_b200
URG_LIB=$PWD/$P/liburg_bl2.so timeout 1200 python -m pytest tests -m gpu -q -x -k "not debug" > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ab.log
tail -2 gpurun_out/pytest_ab.log
echo "== usweep fifo 100k"; timeout 600 python tools/ab.py usweep fifo 100000 $P/liburg.so $P/liburg_bl2.so 2>&1 | tee gpurun_out/ab_ab.txt
echo "== usweep static 100k"; timeout 600 python tools/ab.py usweep static 100000 $P/liburg.so $P/liburg_bl2.so 2>&1 | tee -a gpurun_out/ab_ab.txt
echo "== jitter fifo 50k"; timeout 900 python tools/ab.py jitter fifo 50000 $P/liburg.so $P/liburg_bl2.so 2>&1 | tee -a gpurun_out/ab_ab.txt
echo "== paper11 urgengo"; timeout 600 python tools/ab.py paper11 urgengo 0 $P/liburg.so $P/liburg_bl2.so 2>&1 | tee -a gpurun_out/ab_ab.txt
