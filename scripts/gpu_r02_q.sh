#!/bin/bash
# r02 pass Q: lane special registers in the packed UrgenGo build only (default) vs base (pass O);
# the duration clamp on 32-bit halves (liburg_clamp); GPU tests on the default
mkdir -p gpurun_out
P=paper_2509_12207_b200
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log
tail -2 gpurun_out/pytest_q.log
echo "== jitter urgengo 50k"; timeout 1200 python tools/ab.py jitter urgengo 50000 $P/liburg_base.so $P/liburg.so $P/liburg_clamp.so 2>&1 | tee gpurun_out/ab_q.txt
echo "== scaleout urgengo 300k"; timeout 600 python tools/ab.py scaleout urgengo 300000 $P/liburg_base.so $P/liburg.so $P/liburg_clamp.so 2>&1 | tee -a gpurun_out/ab_q.txt
echo "== usweep fifo 100k"; timeout 600 python tools/ab.py usweep fifo 100000 $P/liburg_base.so $P/liburg.so $P/liburg_clamp.so 2>&1 | tee -a gpurun_out/ab_q.txt
echo "== paper11 urgengo"; timeout 600 python tools/ab.py paper11 urgengo 0 $P/liburg_base.so $P/liburg.so $P/liburg_clamp.so 2>&1 | tee -a gpurun_out/ab_q.txt
