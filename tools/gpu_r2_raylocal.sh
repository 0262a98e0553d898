#!/bin/bash
mkdir -p gpurun_out build/variants
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_adversarial.py -q -x -p no:cacheprovider > gpurun_out/rl_tests.log 2>&1; echo "rc $?" >> gpurun_out/rl_tests.log
for v in "PT_RAY_LOCAL=1" "PT_RAY_LOCAL=0"; do
  python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_$v.so', defines=['$v'])" > /dev/null 2>&1 || { echo "build $v failed"; continue; }
  for c in 3 4 2 1; do
    PT_B200_LIB=build/variants/libpt_$v.so python bench.py --config $c --steps 8 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v config=$c', round(d['value']/1e9,3), 'G samples/s', {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})"
  done
done > gpurun_out/raylocal.log 2>&1
