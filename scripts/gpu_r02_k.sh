#!/bin/bash
# r02 pass K: per-lane slot layout (one base register) + cold 64-bit values of the packed build in
# shared memory + zero-cost wake index + 32-bit step counter in every build, vs base (pass J default);
# 1024-thread and ASYNC-832 variants; source-level ncu of the packed UrgenGo build
mkdir -p gpurun_out
P=paper_2509_12207_b200
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_k.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_k.log
tail -2 gpurun_out/pytest_k.log
echo "== jitter urgengo 50k"; timeout 900 python tools/ab.py jitter urgengo 50000 $P/liburg_base.so $P/liburg.so $P/liburg_t1024.so 2>&1 | tee gpurun_out/ab_k.txt
echo "== scaleout urgengo 300k"; timeout 600 python tools/ab.py scaleout urgengo 300000 $P/liburg_base.so $P/liburg.so $P/liburg_t1024.so 2>&1 | tee -a gpurun_out/ab_k.txt
echo "== usweep fifo 100k"; timeout 600 python tools/ab.py usweep fifo 100000 $P/liburg_base.so $P/liburg.so $P/liburg_a832.so $P/liburg_t1024.so 2>&1 | tee -a gpurun_out/ab_k.txt
echo "== paper11 urgengo"; timeout 600 python tools/ab.py paper11 urgengo 0 $P/liburg_base.so $P/liburg.so 2>&1 | tee -a gpurun_out/ab_k.txt
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:urg_sim_kernel -s 0 -c 1 \
    -o gpurun_out/prof_jitter_k python bench.py --steps 1 --warmup 0 --scenarios 24000 --horizon-ms 3000 --no-cpu-baseline \
    --no-regimes --e2e-steps 1 > gpurun_out/ncu_full_jitter_k.log 2>&1; echo "ncu jitter rc=$?"
python tools/ncu_summary.py gpurun_out/prof_jitter_k.ncu-rep gpurun_out/r02_ncu_key_metrics_jitter_k.json > /dev/null
