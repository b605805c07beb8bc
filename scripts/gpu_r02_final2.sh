#!/bin/bash
# r02 final check 2 (after the FIFO / STATIC parameter-bank change): every GPU test, smoke(), and
# configs[2] at full size with the oracle sample
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_final2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_final2.log
tail -3 gpurun_out/pytest_final2.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final2.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_final2.log
tail -2 gpurun_out/smoke_final2.log
timeout 1200 python tools/run_configs.py r02final3 --configs usweep > gpurun_out/run_configs_final2.log 2>&1; echo "configs rc=$?"
cp profiles/r02final3_configs.json gpurun_out/ 2>/dev/null
tail -26 gpurun_out/run_configs_final2.log
