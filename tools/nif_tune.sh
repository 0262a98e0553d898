#!/bin/bash
# Build NIF variants (SFU/FMA sine split) and microbenchmark each on the B200.
mkdir -p gpurun_out build/variants
for m in ${MUFU_PAIRS:-16 12 10 9 8 6}; do
  python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_m$m.so', defines=['PT_NIF_MUFU_PAIRS=$m'])" > /dev/null 2>&1 || { echo "build m=$m failed"; continue; }
  PT_B200_LIB=build/variants/libpt_m$m.so python tools/nif_bench.py --check --tag "mufu_pairs=$m"
done
