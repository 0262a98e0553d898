mkdir -p gpurun_out
for c in 1 2 3; do python tools/trace_bench.py --config $c; done > gpurun_out/trace_bench.txt 2>&1
python tools/trace_bench.py --config 1 --iters 1 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:primary -s 2 -c 1 -o gpurun_out/prof_prim python tools/trace_bench.py --config 1 --iters 1 > gpurun_out/ncu_prim.log 2>&1
python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:traverse -s 0 -c 1 -o gpurun_out/prof_trav1 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_trav1.log 2>&1
