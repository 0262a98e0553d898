#!/bin/bash
# SFU/FMA sine split variants timed inside the render (bench.py config 1) and on the NIF microbenchmark
mkdir -p gpurun_out build/variants
for m in ${MUFU_PAIRS:-8 9 10}; do
  python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_m$m.so', defines=['PT_NIF_MUFU_PAIRS=$m'])" > /dev/null 2>&1 || { echo "build m=$m failed"; continue; }
  PT_B200_LIB=build/variants/libpt_m$m.so python bench.py --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mufu_pairs=$m', round(d['value']/1e9,3), 'G samples/s; nif', round(d['kernels_ms_per_step']['nif'],4), 'ms', round(d['nif']['inferences_per_s']/1e9,3), 'G inf/s')"
  PT_B200_LIB=build/variants/libpt_m$m.so python tools/nif_bench.py --tag "mufu_pairs=$m" | cut -c1-120
done
