#!/bin/bash
mkdir -p gpurun_out build/variants
for v in "PT_NIF_DIAG=0" "PT_NIF_DIAG=1" "PT_NIF_DIAG=3" "PT_NIF_DIAG=4"; do
  python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_$v.so', defines=['$v'])" > /dev/null 2>&1 || { echo "build $v failed"; continue; }
  PT_B200_LIB=build/variants/libpt_$v.so python tools/nif_bench.py --tag "$v" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['tag'], round(d['inferences_per_s']/1e9,3), 'G inf/s', round(d['frac_burst'],3), 'cycles/tile at 1965 MHz', round(148*1.965e9*128/d['inferences_per_s']))"
done > gpurun_out/nif_diag3.log 2>&1
