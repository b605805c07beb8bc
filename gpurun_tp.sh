set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for W in 8 16; do URG_WARPS_PER_CTA=$W python bench.py --config scaleout --scenarios 300000 --steps 3 --warmup 1 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('W=$W', d['value']/1e9, 'G/s', d['kernel_ms'], 'ms', d['roofline']['frac'])"; done
python bench.py --config jitter --scenarios 20000 --horizon-ms 10000 --steps 2 --warmup 1 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('jitter', d['value']/1e9, 'G/s', d['kernel_ms'], 'ms')"
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_v8.json; python -c "import json; d=json.load(open('gpurun_out/bench_v8.json')); print('paper11', d['value']/1e9, d['kernel_ms'], d['parity_sample'])"
