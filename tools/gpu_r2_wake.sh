#!/bin/bash
# dynamic-replacement path kernel: parity (frames) and PT_TRACE_WAKE variants on configs 3, 4, 1
mkdir -p gpurun_out build/variants
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_divergence.py -q -x -p no:cacheprovider -k "render or furnace or divergence or deterministic" > gpurun_out/wake_tests.log 2>&1; echo "rc $?" >> gpurun_out/wake_tests.log
for w in ${WAKES:-4 8 12 16 24 32}; do
  python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_w$w.so', defines=['PT_TRACE_WAKE=$w'])" > /dev/null 2>&1 || { echo "build $w failed"; continue; }
  for c in 3 4 1; do
    PT_B200_LIB=build/variants/libpt_w$w.so python bench.py --config $c --steps ${STEPS:-8} --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('wake=$w config=$c', round(d['value']/1e9,3), 'G samples/s', {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})"
  done
done > gpurun_out/wake.log 2>&1
