#!/bin/bash
# SIREN diagnostics: spin vs suspend waits; no TMEM store; no sine (microbenchmark only, wrong results)
mkdir -p gpurun_out build/variants
for v in "PT_MBAR_SPIN=0" "PT_MBAR_SPIN=1" "PT_NIF_DIAG=1" "PT_NIF_DIAG=2" "PT_NIF_MUFU_PAIRS=8" "PT_NIF_MUFU_PAIRS=10"; do
  python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_$v.so', defines=['$v'])" > /dev/null 2>&1 || { echo "build $v failed"; continue; }
  PT_B200_LIB=build/variants/libpt_$v.so python tools/nif_bench.py --tag "$v" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['tag'], round(d['inferences_per_s']/1e9,3), 'G inf/s', round(d['frac_burst'],3))"
done > gpurun_out/nif_diag.log 2>&1
