#!/bin/bash
# r02 pass R: GPU tests on the default (lane registers + 32-bit-half clamp); latency build with the
# 32-bit step counter flushed on the rare path (liburg_ns) on configs[1]
mkdir -p gpurun_out
P=paper_2509_12207_b200
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r.log
tail -2 gpurun_out/pytest_r.log
echo "== paper11 urgengo"; timeout 600 python tools/ab.py paper11 urgengo 0 $P/liburg_base.so $P/liburg.so $P/liburg_ns.so 2>&1 | tee gpurun_out/ab_r.txt
echo "== paper11 fifo"; timeout 600 python tools/ab.py paper11 fifo 0 $P/liburg.so $P/liburg_ns.so 2>&1 | tee -a gpurun_out/ab_r.txt
echo "== paper11 urgengo again"; timeout 600 python tools/ab.py paper11 urgengo 0 $P/liburg.so $P/liburg_ns.so 2>&1 | tee -a gpurun_out/ab_r.txt
