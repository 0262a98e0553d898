#!/bin/bash
# trace builds (PT_NIF_TRACE + each comma-separated define list in PT_TRACE_VARIANTS)
mkdir -p gpurun_out build/variants
for v in ${PT_TRACE_VARIANTS:-"PT_NIF_DIAG=0"}; do
python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_trace_$v.so', defines=['PT_NIF_TRACE'] + '$v'.split(','))" > /dev/null 2>&1 || echo "build $v failed"
PT_TRACE_SLOTS=3 PT_B200_LIB="build/variants/libpt_trace_$v.so" timeout 120 python tools/nif_trace.py > "gpurun_out/nif_trace_$v.txt" 2>&1
echo "== $v"; tail -24 "gpurun_out/nif_trace_$v.txt"
done
