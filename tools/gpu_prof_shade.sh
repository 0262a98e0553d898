mkdir -p gpurun_out
python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"shade|traverse" -s 0 -c 2 -o gpurun_out/prof_ts python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_ts.log 2>&1
