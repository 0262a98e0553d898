set -x
python bench.py --steps 50 --warmup 5 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc $?"
timeout 900 python -m pytest tests -m gpu -q --timeout=300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/gpu_tests.log
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc $?"
ncu --set full --clock-control none --import-source on -k regex:nif_fused -s 2 -c 1 -o gpurun_out/prof_nif python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_nif.log 2>&1; echo "ncu2 rc $?"
ncu --set full --clock-control none --import-source on -k regex:traverse -s 4 -c 2 -o gpurun_out/prof_trav python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_trav.log 2>&1; echo "ncu3 rc $?"
