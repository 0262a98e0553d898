mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --timeout=400 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu_tests.log
python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2> gpurun_out/bench.err
for c in 3 4; do python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c$c.log 2> gpurun_out/bench_c$c.err; done
python tools/trace_count.py > gpurun_out/trace_count.json 2> gpurun_out/trace_count.err
TS_MINB="6 7 8" bash tools/ts_tune.sh > gpurun_out/ts_tune.log 2>&1
