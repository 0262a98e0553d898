#!/bin/bash
# SIREN slots in flight / accumulator load variants (comma-separated define lists), NIF GPU tests, a short
# config-3 bench, the 3-slot trace
mkdir -p gpurun_out build/variants
python -c "from paper_2305_20061_b200 import _build; _build.build()" > /dev/null 2>&1 || echo "default build failed"
for v in ${PT_VARIANTS:-"PT_NIF_SLOTS=2" "PT_NIF_SLOTS=3" "PT_NIF_LD32=0" "PT_NIF_SLOTS=2,PT_NIF_LD32=0"}; do
  python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_$v.so', defines='$v'.split(','))" > /dev/null 2>&1 || { echo "build $v failed"; continue; }
  PT_B200_LIB="build/variants/libpt_$v.so" timeout 120 python tools/nif_bench.py --check --tag "$v" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['tag'], round(d['inferences_per_s']/1e9,3), 'G inf/s', round(d['frac_burst'],3), 'cycles/tile at 1965 MHz', round(148*1.965e9*128/d['inferences_per_s']), {k: v for k, v in d.items() if k.startswith('max')})"
done > gpurun_out/nif_slots.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "nif or siren or render or smoke" > gpurun_out/slots_tests.log 2>&1; tail -3 gpurun_out/slots_tests.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-also > gpurun_out/slots_bench.json 2> gpurun_out/slots_bench.err
cat gpurun_out/nif_slots.log
python -c "import json; d=json.load(open('gpurun_out/slots_bench.json')); print(d['value'], d['nif']['inferences_per_s'], d['nif']['roofline']['frac'])" 2>&1 | tail -2
python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_trace3.so', defines=['PT_NIF_TRACE'])" > /dev/null 2>&1
PT_TRACE_SLOTS=3 PT_B200_LIB=build/variants/libpt_trace3.so timeout 120 python tools/nif_trace.py > gpurun_out/nif_trace_s3.txt 2>&1
tail -24 gpurun_out/nif_trace_s3.txt
