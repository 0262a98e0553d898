mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nif_family.py -x -q --timeout=600 -p no:cacheprovider > gpurun_out/family_tests.log 2>&1; echo "pytest rc $?" >> gpurun_out/family_tests.log
timeout 600 python tools/nif_sweep.py > gpurun_out/nif_sweep.jsonl 2> gpurun_out/nif_sweep.err
