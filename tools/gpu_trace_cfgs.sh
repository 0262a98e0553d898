# traversal iteration: all gpu tests, counting build (fp64 fallback rates), bench configs 1, 3, 4
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --timeout=400 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu_tests.log
python tools/trace_count.py > gpurun_out/trace_count.json 2> gpurun_out/trace_count.err
for c in ${CONFIGS:-1 3 4}; do timeout 900 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.log 2> gpurun_out/bench_c$c.err; done
