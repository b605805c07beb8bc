#!/bin/bash
# r02 pass C: all GPU tests (incl. the debug-build trace diff), smem histogram A/B + DRAM bytes,
# one --set full capture of the configs[3] bench kernel instantiation (short horizon)
mkdir -p gpurun_out
P=paper_2509_12207_b200
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_c.log
tail -5 gpurun_out/pytest_c.log
echo "== jitter urgengo 50k: smem hist / global hist"
timeout 600 python tools/ab.py jitter urgengo 50000 $P/liburg.so 2>&1 | tee gpurun_out/ab_c.txt
URG_SMEM_HIST=0 timeout 600 python tools/ab.py jitter urgengo 50000 $P/liburg.so 2>&1 | tee -a gpurun_out/ab_c.txt
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:urg_sim_kernel -s 0 -c 1 -o gpurun_out/traffic_jitter_c python bench.py --steps 1 --warmup 0 --scenarios 50000 \
    --no-cpu-baseline --no-regimes --e2e-steps 1 > gpurun_out/ncu_traffic_c.log 2>&1; echo "ncu traffic rc=$?"
python tools/ncu_summary.py gpurun_out/traffic_jitter_c.ncu-rep gpurun_out/r02_traffic_jitter_c.json --traffic jitter urgengo
cp profiles/traffic.json gpurun_out/traffic_c.json
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:urg_sim_kernel -s 0 -c 1 \
    -o gpurun_out/prof_jitter_c python bench.py --steps 1 --warmup 0 --scenarios 8192 --horizon-ms 4000 --no-cpu-baseline \
    --no-regimes --e2e-steps 1 > gpurun_out/ncu_full_c.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py gpurun_out/prof_jitter_c.ncu-rep gpurun_out/r02_ncu_key_metrics_jitter.json > /dev/null
echo done
