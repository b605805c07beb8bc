#!/bin/bash
# r02: ncu --set full captures (source-level) of the packed build on configs[3] and configs[4] workloads
mkdir -p gpurun_out
TAG=${1:-p1}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:urg_sim_kernel -s 0 -c 1 \
    -o gpurun_out/prof_jitter_$TAG python bench.py --steps 1 --warmup 0 --scenarios 24000 --horizon-ms 3000 --no-cpu-baseline \
    --no-regimes --e2e-steps 1 > gpurun_out/ncu_full_jitter_$TAG.log 2>&1; echo "ncu jitter rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:urg_sim_kernel -s 0 -c 1 \
    -o gpurun_out/prof_scaleout_$TAG python bench.py --config scaleout --steps 1 --warmup 0 --scenarios 40000 --no-cpu-baseline \
    --no-regimes --e2e-steps 1 > gpurun_out/ncu_full_scaleout_$TAG.log 2>&1; echo "ncu scaleout rc=$?"
python tools/ncu_summary.py gpurun_out/prof_jitter_$TAG.ncu-rep gpurun_out/r02_ncu_key_metrics_jitter_$TAG.json > /dev/null
python tools/ncu_summary.py gpurun_out/prof_scaleout_$TAG.ncu-rep gpurun_out/r02_ncu_key_metrics_scaleout_$TAG.json > /dev/null
echo done
