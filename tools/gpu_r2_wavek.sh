#!/bin/bash
# wave size per config under the sample-group order (bench --wave-samples)
mkdir -p gpurun_out
for cw in "4 8" "4 16" "4 32" "2 32" "2 64" "3 16" "3 32"; do
  set -- $cw
  timeout 600 python bench.py --config $1 --wave-samples $2 --steps 8 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('config=$1 wave_samples=$2', round(d['value']/1e9,4), 'G samples/s', {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})"
done > gpurun_out/wavek.log 2>&1
cat gpurun_out/wavek.log
