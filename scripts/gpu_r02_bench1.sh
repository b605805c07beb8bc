#!/bin/bash
# r02: the new default bench (configs[3] whole), the reference arm, DRAM traffic of one bench step's
# kernel, one --set full capture of the same instantiation (8192 scenarios), and the launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_b1.txt 2>&1
nproc > gpurun_out/nproc_b1.txt
timeout 1500 python bench.py > gpurun_out/bench_b1.json 2> gpurun_out/bench_b1.err; echo "bench rc=$?"
cut -c1-600 gpurun_out/bench_b1.json
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_b1.json 2> gpurun_out/bench_ref_b1.err; echo "ref rc=$?"
cut -c1-300 gpurun_out/bench_ref_b1.json
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:urg_sim_kernel -s 0 -c 1 -o gpurun_out/traffic_jitter python bench.py --steps 1 --warmup 0 --scenarios 50000 \
    --no-cpu-baseline --no-regimes --e2e-steps 1 > gpurun_out/ncu_traffic_b1.log 2>&1; echo "ncu traffic rc=$?"
python tools/ncu_summary.py gpurun_out/traffic_jitter.ncu-rep gpurun_out/r02_traffic_jitter.json --traffic jitter urgengo
cp profiles/traffic.json gpurun_out/traffic.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:urg_sim_kernel -s 0 -c 1 \
    -o gpurun_out/prof_jitter_b1 python bench.py --steps 1 --warmup 0 --scenarios 8192 --no-cpu-baseline --no-regimes \
    --e2e-steps 1 > gpurun_out/ncu_full_b1.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py gpurun_out/prof_jitter_b1.ncu-rep gpurun_out/r02_ncu_key_metrics_jitter.json > /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b1.csv \
    python bench.py --steps 2 --warmup 1 --scenarios 20000 --no-cpu-baseline --no-regimes --e2e-steps 1 > gpurun_out/bench_under_ncu_b1.log 2>&1
echo done
