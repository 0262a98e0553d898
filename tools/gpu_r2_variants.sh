#!/bin/bash
# bench frame rate of build variants (comma-separated define lists in PT_VARIANTS) on configs PT_CFGS
mkdir -p gpurun_out build/variants
for v in ${PT_VARIANTS}; do
  python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_$v.so', defines='$v'.split(','))" > /dev/null 2>&1 || { echo "build $v failed"; continue; }
  for c in ${PT_CFGS:-3}; do
    PT_B200_LIB="build/variants/libpt_$v.so" timeout 600 python bench.py --config $c --steps ${PT_STEPS:-10} --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v config=$c', round(d['value']/1e9,4), 'G samples/s', {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})"
  done
done > gpurun_out/variants.log 2>&1
cat gpurun_out/variants.log
