#!/bin/bash
mkdir -p gpurun_out build/variants
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "nif" -p no:cacheprovider > gpurun_out/nif_tests.log 2>&1; echo "rc $?" >> gpurun_out/nif_tests.log
for v in "PT_NIF_DEFER_ST=1" "PT_NIF_DEFER_ST=0"; do
  python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_$v.so', defines=['$v'])" > /dev/null 2>&1 || { echo "build $v failed"; continue; }
  PT_B200_LIB=build/variants/libpt_$v.so python tools/nif_bench.py --tag "$v" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['tag'], round(d['inferences_per_s']/1e9,3), 'G inf/s', round(d['frac_burst'],3))"
done > gpurun_out/nif_defer.log 2>&1
for c in 3 2 4; do python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('config $c', round(d['value']/1e9,3), 'G samples/s', {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()}, 'nif', (d['nif']['inferences_per_s'] or 0)/1e9, d['nif']['roofline']['frac'], 'e2e', round(d['e2e']['value']/1e9,3))"; done > gpurun_out/bench_cfgs.log 2>&1
for m in 6 7 8; do
  python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_ts$m.so', defines=['PT_TS_MINB=$m'])" > /dev/null 2>&1 || { echo "build $m failed"; continue; }
  PT_B200_LIB=build/variants/libpt_ts$m.so python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('minb=$m', round(d['value']/1e9,3), 'G samples/s', {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})"
done > gpurun_out/ts_minb_c3.log 2>&1
