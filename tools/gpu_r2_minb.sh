#!/bin/bash
mkdir -p gpurun_out build/variants
for v in "PT_FB_MINB=6" "PT_FB_MINB=8" "PT_TS_MINB=6 PT_FB_MINB=7" "PT_TS_MINB=8 PT_FB_MINB=7" "PT_TRACE_WAKE=16" "PT_TRACE_WAKE=10"; do
  tag=$(echo $v | tr ' =' '__')
  defs=$(python -c "import sys; print(repr(sys.argv[1].split()))" "$v")
  python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_$tag.so', defines=$defs)" > /dev/null 2>&1 || { echo "build $v failed"; continue; }
  for c in 3 4; do
    PT_B200_LIB=build/variants/libpt_$tag.so python bench.py --config $c --steps 8 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v config=$c', round(d['value']/1e9,3), 'G samples/s', {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})"
  done
done > gpurun_out/minb.log 2>&1
python bench.py --config 3 --steps 8 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('default config=3', round(d['value']/1e9,3), 'G samples/s', {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})" >> gpurun_out/minb.log
