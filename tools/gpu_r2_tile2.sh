#!/bin/bash
mkdir -p gpurun_out build/variants
for v in "PT_TILE_W=4" "PT_TILE_W=16" "PT_TILE_W=8"; do
  python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_$v.so', defines=['$v'])" > /dev/null 2>&1 || { echo "build $v failed"; continue; }
  for c in 3 4; do
    PT_B200_LIB=build/variants/libpt_$v.so python bench.py --config $c --steps 8 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v config=$c', round(d['value']/1e9,3), 'G samples/s', {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})"
  done
done > gpurun_out/tile2.log 2>&1
