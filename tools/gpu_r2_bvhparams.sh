#!/bin/bash
# BVH build parameters (env knobs read by pt_scene_create): configs 3 and 4
mkdir -p gpurun_out
for v in "PT_BVH_BINS=16" "PT_BVH_BINS=32" "PT_BVH_NODE_COST=1.0" "PT_BVH_NODE_COST=2.0" "PT_BVH_MAX_LEAF=3" "PT_BVH_MAX_LEAF=2"; do
  for c in 3 4; do
    env $v python bench.py --config $c --steps 8 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v config=$c', round(d['value']/1e9,3), 'G samples/s', {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})"
  done
done > gpurun_out/bvhparams.log 2>&1
