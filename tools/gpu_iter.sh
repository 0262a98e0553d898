# iteration: gpu tests (all), bench, NIF timeline trace + microbench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --timeout=400 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu_tests.log
python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.err
python tools/nif_bench.py --check --tag cur > gpurun_out/nif_bench.jsonl 2>&1
python -c "from paper_2305_20061_b200 import _build; _build.build(out='build/variants/libpt_trace.so', defines=['PT_NIF_TRACE'])" > /dev/null 2>&1
python tools/nif_trace.py > gpurun_out/nif_trace.txt 2>&1
MUFU_PAIRS="${MUFU_PAIRS:-7 8 9}" bash tools/nif_tune.sh > gpurun_out/nif_tune.log 2>&1
