# traversal iteration: gpu tests (all), bench, register-cap variants, ncu of trace_shade bounces 1-3
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --timeout=400 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu_tests.log
python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.err
TS_MINB="${TS_MINB:-6 7 8}" bash tools/ts_tune.sh > gpurun_out/ts_tune.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"trace_shade" -s 0 -c 3 -o gpurun_out/prof_ts python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_ts.log 2>&1
echo "ncu ts rc $?" >> gpurun_out/bench.err
