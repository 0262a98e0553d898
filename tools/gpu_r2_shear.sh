#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_adversarial.py tests/test_gpu_aov.py -q -x -p no:cacheprovider > gpurun_out/shear_tests.log 2>&1; echo "rc $?" >> gpurun_out/shear_tests.log
for c in 3 4 2 1; do python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('config=$c', round(d['value']/1e9,3), 'G samples/s', {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()}, 'e2e', round(d['e2e']['value']/1e9,3), round(d['e2e']['scene_create_ms_median'],1))"; done > gpurun_out/shear.log 2>&1
PT_BVH_TIMING=1 python tools/bvh_time.py > gpurun_out/bvh_phases.txt 2>&1
