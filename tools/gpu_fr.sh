# paper NIF (kind 1): parity tests + microbench for both kinds
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout=300 -p no:cacheprovider -k "nif" > gpurun_out/fr_tests.log 2>&1; echo "pytest rc $?" >> gpurun_out/fr_tests.log
for k in 0 1; do timeout 120 python tools/nif_bench.py --kind $k --check --tag kind$k >> gpurun_out/fr_bench.jsonl 2>> gpurun_out/fr_bench.err; done
