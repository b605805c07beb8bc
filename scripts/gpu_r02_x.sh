#!/bin/bash
# r02 pass X: sync costs in 32 bits (sc32; host: sync_hi_ns < 2^32 - 1) vs the default (pass-W kernels);
# parity tests on sc32; --set full capture of the default's headline kernel
mkdir -p gpurun_out
P=paper_2509_12207_b200
URG_LIB=$PWD/$P/liburg_sc32.so timeout 1200 python -m pytest tests -m gpu -q -x -k "not debug" > gpurun_out/pytest_x.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_x.log
tail -2 gpurun_out/pytest_x.log
echo "== jitter urgengo 50k"; timeout 1200 python tools/ab.py jitter urgengo 50000 $P/liburg.so $P/liburg_sc32.so 2>&1 | tee gpurun_out/ab_x.txt
echo "== scaleout urgengo 300k"; timeout 900 python tools/ab.py scaleout urgengo 300000 $P/liburg.so $P/liburg_sc32.so 2>&1 | tee -a gpurun_out/ab_x.txt
echo "== usweep fifo 100k"; timeout 600 python tools/ab.py usweep fifo 100000 $P/liburg.so $P/liburg_sc32.so 2>&1 | tee -a gpurun_out/ab_x.txt
echo "== paper11 urgengo"; timeout 600 python tools/ab.py paper11 urgengo 0 $P/liburg.so $P/liburg_sc32.so 2>&1 | tee -a gpurun_out/ab_x.txt
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:urg_sim_kernel -s 0 -c 1 \
    -o gpurun_out/prof_jitter_x python bench.py --steps 1 --warmup 0 --scenarios 24000 --horizon-ms 3000 --no-cpu-baseline \
    --no-regimes --e2e-steps 1 > gpurun_out/ncu_full_jitter_x.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py gpurun_out/prof_jitter_x.ncu-rep gpurun_out/r02_ncu_key_metrics_jitter_x.json > /dev/null
