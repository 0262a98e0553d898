#!/bin/bash
mkdir -p gpurun_out build/variants
for ns in 2 3; do
python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_trace$ns.so', defines=['PT_NIF_TRACE', 'PT_NIF_SLOTS=$ns'])" > /dev/null 2>&1
PT_TRACE_SLOTS=$ns PT_B200_LIB=build/variants/libpt_trace$ns.so timeout 120 python tools/nif_trace.py > gpurun_out/nif_trace_s$ns.txt 2>&1
done
python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_trace4.so', defines=['PT_NIF_TRACE', 'PT_NIF_DIAG=4'])" > /dev/null 2>&1
PT_TRACE_SLOTS=3 PT_B200_LIB=build/variants/libpt_trace4.so timeout 120 python tools/nif_trace.py > gpurun_out/nif_trace_d4.txt 2>&1
