#!/bin/bash
# Round 2 session 3: GPU suite; short-stack / carveout variants (configs 3, 1); NIF schedule change in the bench
mkdir -p gpurun_out build/variants
timeout 1800 python -m pytest tests -m gpu -q --timeout=900 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu_tests.log
for v in "0 -1" "8 -1" "8 25" "8 50" "16 50" "16 100"; do
  set -- $v; D=$1; C=$2
  python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_ss${D}_c${C}.so', defines=['PT_SSTACK=$D','PT_TRACE_CARVEOUT=$C'])" > /dev/null 2>&1 || { echo "build $D $C failed"; continue; }
  for c in 3 1; do
    PT_B200_LIB=build/variants/libpt_ss${D}_c${C}.so python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sstack=$D carveout=$C config=$c', round(d['value']/1e9,3), 'G samples/s', {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()}, 'nif', round(d['nif']['inferences_per_s']/1e9,3), 'G/s frac', round(d['nif']['roofline']['frac'],3))"
  done
done > gpurun_out/variants.log 2>&1
