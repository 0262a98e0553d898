#!/bin/bash
# ncu --set full captures of the path kernels and the SIREN kernel on the headline workload (config 3)
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"first_bounce|path_kernel" -s 2 -c 2 -o gpurun_out/prof_ts_c3 -f python bench.py --config 3 --steps 1 --warmup 0 --no-cpu-baseline --no-also > gpurun_out/ncu_ts_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"siren" -s 1 -c 1 -o gpurun_out/prof_nif_c3 -f python bench.py --config 3 --steps 1 --warmup 0 --no-cpu-baseline --no-also > gpurun_out/ncu_nif_c3.log 2>&1
