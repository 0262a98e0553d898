#!/bin/bash
mkdir -p gpurun_out build/variants
for v in "PT_MBAR_BACKOFF=0" "PT_MBAR_BACKOFF=1" "PT_MBAR_BACKOFF=2 PT_MBAR_NS=20" "PT_MBAR_BACKOFF=2 PT_MBAR_NS=100" "PT_MBAR_BACKOFF=1 PT_MBAR_SPIN=1"; do
  tag=$(echo $v | tr ' =' '__')
  defs=$(python -c "import sys; print(repr(sys.argv[1].split()))" "$v")
  python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_$tag.so', defines=$defs)" > /dev/null 2>&1 || { echo "build $v failed"; continue; }
  PT_B200_LIB=build/variants/libpt_$tag.so python tools/nif_bench.py --tag "$v" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['tag'], round(d['inferences_per_s']/1e9,3), 'G inf/s', round(d['frac_burst'],3))"
  PT_B200_LIB=build/variants/libpt_$tag.so python bench.py --config 3 --steps 8 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('   $v config=3', round(d['value']/1e9,3), 'G samples/s', {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()}, 'nif frac', round(d['nif']['roofline']['frac'],3))"
done > gpurun_out/backoff.log 2>&1
