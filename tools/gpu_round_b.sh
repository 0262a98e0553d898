# full GPU check: gpu tests, bench (with cpu baseline), launch list, full captures of trace_shade + NIF
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout=400 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu_tests.log
python bench.py --steps 50 --warmup 5 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu launch rc $?" >> gpurun_out/bench.err
ncu --set full --clock-control none --import-source on -k regex:"trace_shade" -s 0 -c 2 -o gpurun_out/prof_ts python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_ts.log 2>&1
echo "ncu ts rc $?" >> gpurun_out/bench.err
ncu --set full --clock-control none --import-source on -k regex:"nif_fused" -s 0 -c 1 -o gpurun_out/prof_nif python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_nif.log 2>&1
echo "ncu nif rc $?" >> gpurun_out/bench.err
