# tests, bench (config 1 + cpu baseline), counting build, DRAM traffic capture, launch list, full captures,
# configs 2-4 bench lines
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --timeout=400 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu_tests.log
python tools/trace_count.py > gpurun_out/trace_count.json 2> gpurun_out/trace_count.err
mkdir -p profiles/round1 && cp gpurun_out/trace_count.json profiles/round1/trace_count.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:"first_bounce|path_kernel|siren|accumulate" --csv --log-file gpurun_out/traffic_c1.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_traffic.log 2>&1
python tools/ncu_traffic.py gpurun_out/traffic_c1.csv > gpurun_out/ncu_traffic_c1.json && cp gpurun_out/ncu_traffic_c1.json profiles/round1/
python bench.py --steps 50 --warmup 5 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"first_bounce|path_kernel" -s 0 -c 2 -o gpurun_out/prof_ts python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_ts.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"siren" -s 0 -c 1 -o gpurun_out/prof_nif python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_nif.log 2>&1
for c in 2 3 4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.log 2> gpurun_out/bench_c$c.err; done
