#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout=1200 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu_tests.log
for c in 3 2 4 1; do python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('config $c', round(d['value']/1e9,3), 'G samples/s', {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()}, 'nif', (d['nif']['inferences_per_s'] or 0)/1e9, d['nif']['roofline']['frac'], 'e2e', round(d['e2e']['value']/1e9,3))"; done > gpurun_out/bench_cfgs.log 2>&1
