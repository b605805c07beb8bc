#!/bin/bash
# r02 bench pass 5 (final kernels: pass-X build): DRAM traffic of one bench
# launch, the bench line, the launch list, one --set full capture, then every BASELINE.json
# configuration at full size with the BASELINE.md oracle sample (tools/run_configs.py)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_y.txt 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:urg_sim_kernel -s 0 -c 1 -o gpurun_out/traffic_jitter_y python bench.py --steps 1 --warmup 0 --scenarios 50000 \
    --no-cpu-baseline --no-regimes --e2e-steps 1 > gpurun_out/ncu_traffic_y.log 2>&1; echo "ncu traffic rc=$?"
python tools/ncu_summary.py gpurun_out/traffic_jitter_y.ncu-rep gpurun_out/r02_traffic_jitter_y.json --traffic jitter urgengo | tail -1
cp profiles/traffic.json gpurun_out/traffic.json
timeout 1500 python bench.py > gpurun_out/bench_y.json 2> gpurun_out/bench_y.err; echo "bench rc=$?"
cut -c1-400 gpurun_out/bench_y.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_y.csv \
    python bench.py --steps 2 --warmup 1 --scenarios 20000 --no-cpu-baseline --no-regimes --e2e-steps 1 > gpurun_out/bench_under_ncu_y.log 2>&1
echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:urg_sim_kernel -s 0 -c 1 \
    -o gpurun_out/prof_jitter_y python bench.py --steps 1 --warmup 0 --scenarios 24000 --horizon-ms 3000 --no-cpu-baseline \
    --no-regimes --e2e-steps 1 > gpurun_out/ncu_full_jitter_y.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py gpurun_out/prof_jitter_y.ncu-rep gpurun_out/r02_ncu_key_metrics_jitter_y.json > /dev/null
timeout 2400 python tools/run_configs.py r02final2 > gpurun_out/run_configs_y.log 2>&1; echo "configs rc=$?"
cp profiles/r02final2_configs.json gpurun_out/ 2>/dev/null
tail -5 gpurun_out/run_configs_y.log
echo done
