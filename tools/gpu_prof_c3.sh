mkdir -p gpurun_out
python tools/trace_bench.py --config 3 --iters 1 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:primary -s 2 -c 1 -o gpurun_out/prof_prim3 python tools/trace_bench.py --config 3 --iters 1 > gpurun_out/ncu_prim3.log 2>&1
