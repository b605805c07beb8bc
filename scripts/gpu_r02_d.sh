#!/bin/bash
# r02 pass D: all GPU tests incl. the full-size ones, A/B of the flag change, a profile of the packed build
mkdir -p gpurun_out
P=paper_2509_12207_b200
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_d.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_d.log
tail -4 gpurun_out/pytest_d.log
grep -E "passed|failed" gpurun_out/pytest_d.log | tail -2
echo "== jitter urgengo 50k"; timeout 1200 python tools/ab.py jitter urgengo 50000 $P/liburg_base.so $P/liburg.so 2>&1 | tee gpurun_out/ab_d.txt
echo "== scaleout urgengo 300k"; timeout 900 python tools/ab.py scaleout urgengo 300000 $P/liburg_base.so $P/liburg.so 2>&1 | tee -a gpurun_out/ab_d.txt
echo "== paper11 urgengo"; timeout 600 python tools/ab.py paper11 urgengo 0 $P/liburg_base.so $P/liburg.so 2>&1 | tee -a gpurun_out/ab_d.txt
bash scripts/gpu_r02_prof.sh d
