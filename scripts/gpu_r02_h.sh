#!/bin/bash
# r02 pass H: bench line of the current kernels, latency-build check, packed-build profiles
mkdir -p gpurun_out
P=paper_2509_12207_b200
timeout 1500 python bench.py > gpurun_out/bench_h.json 2> gpurun_out/bench_h.err; echo "bench rc=$?"
cut -c1-400 gpurun_out/bench_h.json
echo "== paper11 urgengo"; timeout 600 python tools/ab.py paper11 urgengo 0 $P/liburg_base.so $P/liburg.so 2>&1 | tee gpurun_out/ab_h.txt
bash scripts/gpu_r02_prof.sh h
