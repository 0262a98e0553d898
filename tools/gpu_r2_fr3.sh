#!/bin/bash
# paper-NIF (kind 1) microbenchmark of build variants (PT_VARIANTS, default: producer-warp counts)
mkdir -p gpurun_out build/variants
for v in ${PT_VARIANTS:-PT_FR3_PRODUCERS=4 PT_FR3_PRODUCERS=6 PT_FR3_PRODUCERS=8}; do
  python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_$v.so', defines=['$v'])" > /dev/null 2>&1 || { echo "build $v failed"; continue; }
  PT_B200_LIB=build/variants/libpt_$v.so timeout 120 python tools/nif_bench.py --kind 1 --check --tag $v | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['tag'], round(d['inferences_per_s']/1e9,3), 'G inf/s', round(d['frac_burst'],3), d['max_abs_dy'])"
done
