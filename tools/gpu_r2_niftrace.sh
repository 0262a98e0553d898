#!/bin/bash
mkdir -p gpurun_out build/variants
python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_trace.so', defines=['PT_NIF_TRACE'])" > /dev/null 2>&1
python tools/nif_trace.py > gpurun_out/nif_trace_r2.txt 2>&1
