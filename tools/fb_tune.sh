# first_bounce_kernel register-cap variants (PT_FB_MINB) with the path kernel at its default cap
mkdir -p gpurun_out build/variants
for m in ${FB_MINB:-6 8}; do
  python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_fb$m.so', defines=['PT_FB_MINB=$m'])" > /dev/null 2>&1 || { echo "build $m failed"; continue; }
  PT_B200_LIB=build/variants/libpt_fb$m.so python bench.py --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fb_minb=$m', round(d['value']/1e9,3), 'G samples/s', d['kernels_ms_per_step'])"
done
