#!/bin/bash
# r02 bench pass 3 (kernels of pass N): DRAM traffic of one bench step's kernel first (so the bench line
# carries roofline.traffic), the bench line, the reference arm, the launch list, one --set full capture
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_o.txt 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:urg_sim_kernel -s 0 -c 1 -o gpurun_out/traffic_jitter_o python bench.py --steps 1 --warmup 0 --scenarios 50000 \
    --no-cpu-baseline --no-regimes --e2e-steps 1 > gpurun_out/ncu_traffic_o.log 2>&1; echo "ncu traffic rc=$?"
python tools/ncu_summary.py gpurun_out/traffic_jitter_o.ncu-rep gpurun_out/r02_traffic_jitter_o.json --traffic jitter urgengo | tail -1
cp profiles/traffic.json gpurun_out/traffic.json
timeout 1500 python bench.py > gpurun_out/bench_o.json 2> gpurun_out/bench_o.err; echo "bench rc=$?"
cut -c1-700 gpurun_out/bench_o.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_o.json 2> gpurun_out/bench_ref_o.err; echo "ref rc=$?"
cut -c1-300 gpurun_out/bench_ref_o.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_o.csv \
    python bench.py --steps 2 --warmup 1 --scenarios 20000 --no-cpu-baseline --no-regimes --e2e-steps 1 > gpurun_out/bench_under_ncu_o.log 2>&1
echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:urg_sim_kernel -s 0 -c 1 \
    -o gpurun_out/prof_jitter_o python bench.py --steps 1 --warmup 0 --scenarios 24000 --horizon-ms 3000 --no-cpu-baseline \
    --no-regimes --e2e-steps 1 > gpurun_out/ncu_full_jitter_o.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py gpurun_out/prof_jitter_o.ncu-rep gpurun_out/r02_ncu_key_metrics_jitter_o.json > /dev/null
echo done
