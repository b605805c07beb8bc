#!/bin/bash
# r02 pass P: lane index / lane bit from the special registers (liburg_lid) and, on top, the per-lane
# slots at shared offset 0 with the blob after them (liburg_sfirst), vs base (= pass O kernels);
# GPU parity tests run on the sfirst build (URG_LIB)
mkdir -p gpurun_out
P=paper_2509_12207_b200
URG_LIB=$PWD/$P/liburg_sfirst.so timeout 1200 python -m pytest tests -m gpu -q -x -k "not debug" > gpurun_out/pytest_p.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_p.log
tail -2 gpurun_out/pytest_p.log
echo "== jitter urgengo 50k"; timeout 1200 python tools/ab.py jitter urgengo 50000 $P/liburg_base.so $P/liburg_lid.so $P/liburg_sfirst.so 2>&1 | tee gpurun_out/ab_p.txt
echo "== scaleout urgengo 300k"; timeout 600 python tools/ab.py scaleout urgengo 300000 $P/liburg_base.so $P/liburg_lid.so $P/liburg_sfirst.so 2>&1 | tee -a gpurun_out/ab_p.txt
echo "== usweep fifo 100k"; timeout 600 python tools/ab.py usweep fifo 100000 $P/liburg_base.so $P/liburg_lid.so $P/liburg_sfirst.so 2>&1 | tee -a gpurun_out/ab_p.txt
echo "== paper11 urgengo"; timeout 600 python tools/ab.py paper11 urgengo 0 $P/liburg_base.so $P/liburg_lid.so $P/liburg_sfirst.so 2>&1 | tee -a gpurun_out/ab_p.txt
