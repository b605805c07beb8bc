#!/bin/bash
# A/B pass for a kernel change: GPU parity tests on the default build, then tools/ab.py timing of
# the default build against experiment builds (liburg_<name>.so) on the headline and throughput
# workloads.  usage: bash scripts/gpu_ab.sh TAG lib1 lib2 ...   (libs relative to the package dir)
TAG=${1:-ab}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -2 gpurun_out/pytest_$TAG.log
L=""; for l in "$@"; do L="$L paper_2509_12207_b200/$l"; done
echo "== paper11 (configs[1], latency build)"; timeout 600 python tools/ab.py paper11 urgengo 0 $L $L 2>&1 | tee gpurun_out/ab_$TAG.txt
echo "== scaleout 300k (throughput build)"; timeout 600 python tools/ab.py scaleout urgengo 300000 $L 2>&1 | tee -a gpurun_out/ab_$TAG.txt
