#!/bin/bash
# r02 A/B G: base (lb everywhere + budget) vs +rare-branch hints (lb everywhere) vs +hints, lb throughput-only
mkdir -p gpurun_out
P=paper_2509_12207_b200
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_debug.py -m gpu -q -x > gpurun_out/pytest_g.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_g.log
tail -3 gpurun_out/pytest_g.log
echo "== jitter urgengo 50k"; timeout 1200 python tools/ab.py jitter urgengo 50000 $P/liburg_base.so $P/liburg_rare.so $P/liburg.so 2>&1 | tee gpurun_out/ab_g.txt
echo "== scaleout urgengo 300k"; timeout 900 python tools/ab.py scaleout urgengo 300000 $P/liburg_base.so $P/liburg_rare.so $P/liburg.so 2>&1 | tee -a gpurun_out/ab_g.txt
echo "== paper11 urgengo"; timeout 600 python tools/ab.py paper11 urgengo 0 $P/liburg_base.so $P/liburg_rare.so $P/liburg.so 2>&1 | tee -a gpurun_out/ab_g.txt
echo "== paper11 fifo"; timeout 600 python tools/ab.py paper11 fifo 0 $P/liburg_base.so $P/liburg.so 2>&1 | tee -a gpurun_out/ab_g.txt
