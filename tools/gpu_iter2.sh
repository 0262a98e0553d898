# iteration: all gpu tests, bench config 1 (+ config 3), spp sweep
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --timeout=400 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu_tests.log
python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2> gpurun_out/bench.err
python bench.py --config 3 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c3.log 2> gpurun_out/bench_c3.err
timeout 300 python tools/spp_sweep.py > gpurun_out/spp_sweep.jsonl 2> gpurun_out/spp_sweep.err
