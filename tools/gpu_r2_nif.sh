#!/bin/bash
# SIREN schedule variants: NIF microbenchmark + bench (config 3) per variant
mkdir -p gpurun_out build/variants
for v in "PT_NIF_OUT_EARLY=0" "PT_NIF_OUT_EARLY=1"; do
  python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_$v.so', defines=['$v'])" > /dev/null 2>&1 || { echo "build $v failed"; continue; }
  PT_B200_LIB=build/variants/libpt_$v.so python tools/nif_bench.py --tag "$v" | cut -c1-200
  PT_B200_LIB=build/variants/libpt_$v.so python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v config 3', round(d['value']/1e9,3), 'G samples/s', {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()}, 'nif', round(d['nif']['inferences_per_s']/1e9,3), 'G/s frac', round(d['nif']['roofline']['frac'],3))"
done > gpurun_out/nif_variants.log 2>&1
# the round-1 schedule (output layer behind the D buffer, bias step) for reference
cp paper_2305_20061_b200/csrc/siren_kernel.cu /tmp/siren_cur.cu
cp tools/variants/siren_kernel_r1.cu paper_2305_20061_b200/csrc/siren_kernel.cu
python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_r1sched.so')" > /dev/null 2>&1
cp /tmp/siren_cur.cu paper_2305_20061_b200/csrc/siren_kernel.cu
PT_B200_LIB=build/variants/libpt_r1sched.so python tools/nif_bench.py --tag "r1 schedule" | cut -c1-200 >> gpurun_out/nif_variants.log 2>&1
PT_B200_LIB=build/variants/libpt_r1sched.so python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('r1 schedule config 3', round(d['value']/1e9,3), 'G samples/s', {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()}, 'nif', round(d['nif']['inferences_per_s']/1e9,3), 'G/s frac', round(d['nif']['roofline']['frac'],3))" >> gpurun_out/nif_variants.log 2>&1
