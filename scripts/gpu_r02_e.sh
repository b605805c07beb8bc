#!/bin/bash
# r02 pass E: packed 768-thread A/B; every BASELINE.json configuration at full size with clocks
mkdir -p gpurun_out
P=paper_2509_12207_b200
echo "== jitter urgengo 50k"; timeout 900 python tools/ab.py jitter urgengo 50000 $P/liburg.so $P/liburg_pk768.so 2>&1 | tee gpurun_out/ab_e.txt
echo "== scaleout urgengo 300k"; timeout 600 python tools/ab.py scaleout urgengo 300000 $P/liburg.so $P/liburg_pk768.so 2>&1 | tee -a gpurun_out/ab_e.txt
timeout 3000 python tools/run_configs.py r02 > gpurun_out/run_configs_r02.log 2>&1; echo "run_configs rc=$?"
cp profiles/r02_configs.* gpurun_out/ 2>/dev/null
tail -40 gpurun_out/run_configs_r02.log
