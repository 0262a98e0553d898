#!/bin/bash
# Round 2: builder timings, the GPU suite (with the new parity tests), short-stack depth variants on configs 3 and 4
mkdir -p gpurun_out build/variants
python tools/bvh_time.py --sweep > gpurun_out/bvh_time.jsonl 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q --timeout=900 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu_tests.log
for D in ${DEPTHS:-8 12 16 24}; do
  python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_ss$D.so', defines=['PT_SSTACK=$D'])" > /dev/null 2>&1 || { echo "build $D failed"; continue; }
  for c in 3 4; do
    PT_B200_LIB=build/variants/libpt_ss$D.so python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sstack=$D config=$c', round(d['value']/1e9,3), 'G samples/s', {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()}, 'e2e', round(d['e2e']['value']/1e9,3), 'create', round(d['e2e']['scene_create_ms_median'],1))"
  done
done > gpurun_out/sstack.log 2>&1
