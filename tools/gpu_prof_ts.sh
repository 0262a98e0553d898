mkdir -p gpurun_out
python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"trace_shade" -s 0 -c 4 -o gpurun_out/prof_ts2 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_ts2.log 2>&1
