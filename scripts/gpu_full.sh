#!/bin/bash
# Round evidence: parity tests, smoke, bench (+reference arm), ncu launch list and one
# --set full capture of the bench's simulation kernel, NEXT-row measurements.
# usage: bash scripts/gpu_full.sh TAG
TAG=${1:-r01}
mkdir -p gpurun_out profiles
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-throughput > gpurun_out/bench_under_ncu_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:urg_sim_kernel -s 1 -c 1 \
    -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-throughput > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 600 python tools/measure_next.py $TAG > gpurun_out/next_$TAG.log 2>&1; cp profiles/${TAG}_next.json gpurun_out/ 2>/dev/null
tail -2 gpurun_out/pytest_$TAG.log; cat gpurun_out/smoke_$TAG.log; cut -c1-300 gpurun_out/bench_$TAG.json
# throughput regime: one --set full capture of the packed (two scenarios per warp) kernel
timeout 900 ncu --set full --clock-control none --import-source on -k regex:urg_sim_kernel -s 1 -c 1 \
    -o gpurun_out/prof_pk_$TAG python bench.py --config scaleout --scenarios 40000 --steps 1 --warmup 1 \
    --no-cpu-baseline --no-throughput > gpurun_out/ncu_pk_$TAG.log 2>&1
timeout 600 bash scripts/sanitize.sh > gpurun_out/sanitize_$TAG.log 2>&1
