#!/bin/bash
# r02 pass J: per-policy packed CTA sizes (UrgenGo 832, FIFO/STATIC 768) vs base; ASYNC 832 variant;
# source-level ncu captures of the packed UrgenGo build (configs[3] workload) and the latency build (configs[1])
mkdir -p gpurun_out
P=paper_2509_12207_b200
echo "== jitter urgengo 50k"; timeout 900 python tools/ab.py jitter urgengo 50000 $P/liburg_base.so $P/liburg.so 2>&1 | tee gpurun_out/ab_j.txt
echo "== usweep fifo 100k"; timeout 600 python tools/ab.py usweep fifo 100000 $P/liburg_base.so $P/liburg.so $P/liburg_asy832.so 2>&1 | tee -a gpurun_out/ab_j.txt
echo "== usweep static 100k"; timeout 600 python tools/ab.py usweep static 100000 $P/liburg_base.so $P/liburg.so $P/liburg_asy832.so 2>&1 | tee -a gpurun_out/ab_j.txt
bash scripts/gpu_r02_prof.sh j
timeout 900 ncu --set full --clock-control none --import-source on -k regex:urg_sim_kernel -s 1 -c 1 \
    -o gpurun_out/prof_paper11_j python tools/ab.py paper11 urgengo 0 $P/liburg.so > gpurun_out/ncu_full_paper11_j.log 2>&1; echo "ncu paper11 rc=$?"
python tools/ncu_summary.py gpurun_out/prof_paper11_j.ncu-rep gpurun_out/r02_ncu_key_metrics_paper11_j.json > /dev/null
ls -la gpurun_out
