#!/bin/bash
# profiles of the current build on the headline workload (config 3): counting build, per-kernel DRAM /
# instruction / local-memory / SIMT capture of one step, launch list, full ncu captures of the path kernels
# and the SIREN kernel
mkdir -p gpurun_out
rm -f build/variants/libpt_count.so
timeout 900 python tools/trace_count.py > gpurun_out/trace_count.json 2> gpurun_out/trace_count.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum,smsp__thread_inst_executed.sum --clock-control none -k regex:"first_bounce|path_kernel|siren|accumulate" --csv --log-file gpurun_out/traffic_c3.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-also > gpurun_out/ncu_traffic.log 2>&1
python tools/ncu_traffic.py gpurun_out/traffic_c3.csv trace > gpurun_out/ncu_traffic_c3.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-also > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"first_bounce|path_kernel" -s 2 -c 2 -o gpurun_out/prof_ts_c3b -f python bench.py --config 3 --steps 1 --warmup 0 --no-cpu-baseline --no-also > gpurun_out/ncu_ts_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"siren" -s 1 -c 1 -o gpurun_out/prof_nif_c3b -f python bench.py --config 3 --steps 1 --warmup 0 --no-cpu-baseline --no-also > gpurun_out/ncu_nif_c3.log 2>&1
