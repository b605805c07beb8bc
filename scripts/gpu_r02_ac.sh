#!/bin/bash
# r02 pass AC: packed UrgenGo with the new-head vote instead of the every-step fit ballot (nca)
mkdir -p gpurun_out
P=paper_2509_12207_b200
URG_LIB=$PWD/$P/liburg_nca.so timeout 1200 python -m pytest tests -m gpu -q -x -k "not debug" > gpurun_out/pytest_ac.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ac.log
tail -2 gpurun_out/pytest_ac.log
echo "== jitter urgengo 50k"; timeout 1200 python tools/ab.py jitter urgengo 50000 $P/liburg.so $P/liburg_nca.so 2>&1 | tee gpurun_out/ab_ac.txt
echo "== scaleout urgengo 300k"; timeout 900 python tools/ab.py scaleout urgengo 300000 $P/liburg.so $P/liburg_nca.so 2>&1 | tee -a gpurun_out/ab_ac.txt
