#!/bin/bash
# Round-2 baseline on the headline workload (config 3): bench line, counting build, DRAM/instruction capture
# of one step, launch list, then the GPU test suite.
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.err
timeout 900 python tools/trace_count.py > gpurun_out/trace_count.json 2> gpurun_out/trace_count.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum,smsp__thread_inst_executed.sum --clock-control none -k regex:"first_bounce|path_kernel|siren|accumulate" --csv --log-file gpurun_out/traffic_c3.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-also > gpurun_out/ncu_traffic.log 2>&1
python tools/ncu_traffic.py gpurun_out/traffic_c3.csv trace > gpurun_out/ncu_traffic_c3.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-also > gpurun_out/ncu_launch.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q --timeout=600 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu_tests.log
