# NIF iteration: variants + trace + gpu tests (nif only)
mkdir -p gpurun_out
bash tools/nif_tune.sh > gpurun_out/nif_tune.log 2>&1
python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_trace.so', defines=['PT_NIF_TRACE'])" > /dev/null 2>&1
python tools/nif_trace.py > gpurun_out/nif_trace.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -k nif -q --timeout=300 -p no:cacheprovider > gpurun_out/gpu_nif_tests.log 2>&1
