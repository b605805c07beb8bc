#!/bin/bash
# Round evidence: parity tests, smoke, one --set full capture of the bench's simulation kernel
# (its DRAM bytes feed bench.py's roofline.traffic), bench (+reference arm), ncu launch list,
# NEXT-row measurements, the packed-build capture, sanitizers, design-option studies.
# usage: bash scripts/gpu_full.sh TAG
TAG=${1:-r01}
mkdir -p gpurun_out profiles
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:urg_sim_kernel -s 1 -c 1 \
    -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-throughput > gpurun_out/ncu_full_$TAG.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_$TAG.ncu-rep gpurun_out/${TAG}_ncu_key_metrics_bench.json --traffic paper11 urgengo \
    > gpurun_out/ncu_summary_$TAG.log 2>&1; cp profiles/traffic.json gpurun_out/
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-throughput > gpurun_out/bench_under_ncu_$TAG.log 2>&1
tail -2 gpurun_out/pytest_$TAG.log; cat gpurun_out/smoke_$TAG.log; cut -c1-300 gpurun_out/bench_$TAG.json
timeout 900 python tools/measure_next.py $TAG > gpurun_out/next_$TAG.log 2>&1; cp profiles/${TAG}_next.json gpurun_out/ 2>/dev/null
# throughput regime: one --set full capture of the packed (two scenarios per warp) kernel
timeout 900 ncu --set full --clock-control none --import-source on -k regex:urg_sim_kernel -s 1 -c 1 \
    -o gpurun_out/prof_pk_$TAG python bench.py --config scaleout --scenarios 40000 --steps 1 --warmup 1 \
    --no-cpu-baseline --no-throughput > gpurun_out/ncu_pk_$TAG.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_pk_$TAG.ncu-rep gpurun_out/${TAG}_ncu_key_metrics_pk.json > /dev/null 2>&1
timeout 900 bash scripts/sanitize.sh > gpurun_out/sanitize_$TAG.log 2>&1
timeout 900 python tools/run_studies.py $TAG > gpurun_out/studies_$TAG.log 2>&1; cp profiles/${TAG}_studies.* gpurun_out/ 2>/dev/null
echo done
