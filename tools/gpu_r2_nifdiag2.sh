#!/bin/bash
mkdir -p gpurun_out build/variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/mma_shapes tools/mma_shapes.cu && ./build/mma_shapes > gpurun_out/mma_shapes_r2.txt 2>&1
for v in "PT_NIF_DIAG=0" "PT_NIF_DIAG=1" "PT_NIF_DIAG=2"; do
  python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_$v.so', defines=['$v'])" > /dev/null 2>&1 || { echo "build $v failed"; continue; }
  PT_B200_LIB=build/variants/libpt_$v.so python tools/nif_bench.py --tag "transposed $v" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['tag'], round(d['inferences_per_s']/1e9,3), 'G inf/s', round(d['frac_burst'],3))"
done > gpurun_out/nif_diag2.log 2>&1
for k in 4 8 16 32; do python bench.py --config 3 --wave-samples $k --steps 10 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('wave_samples=$k', round(d['value']/1e9,3), 'G samples/s', {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})"; done > gpurun_out/wave_k.log 2>&1
