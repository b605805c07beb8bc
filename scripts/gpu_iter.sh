#!/bin/bash
# Fast iteration pass: parity tests, one bench line, one ncu --set full capture of urg_sim_kernel.
# usage: bash scripts/gpu_iter.sh TAG [extra bench args]
TAG=${1:-iter}; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 600 python bench.py "$@" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:urg_sim_kernel -s 1 -c 1 \
    -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 1 --no-cpu-baseline "$@" > gpurun_out/ncu_$TAG.log 2>&1
tail -3 gpurun_out/pytest_$TAG.log; cat gpurun_out/bench_$TAG.json
