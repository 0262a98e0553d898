set -x
mkdir -p gpurun_out
bash tools/nif_tune.sh > gpurun_out/nif_tune.log 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout=300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc $?"
python bench.py --steps 50 --warmup 5 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc $?"
