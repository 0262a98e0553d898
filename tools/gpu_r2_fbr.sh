#!/bin/bash
mkdir -p gpurun_out build/variants
python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_fbr.so', defines=['PT_FB_REPLACE=1'])" > /dev/null 2>&1
PT_B200_LIB=build/variants/libpt_fbr.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "render or primary" > gpurun_out/fbr_tests.log 2>&1; echo "rc $?" >> gpurun_out/fbr_tests.log
for lib in build/variants/libpt_fbr.so paper_2305_20061_b200/libpt_b200.so; do
  for c in 3 4; do PT_B200_LIB=$lib python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib config=$c', round(d['value']/1e9,3), 'G samples/s', {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})"; done
done > gpurun_out/fbr.log 2>&1
