#!/bin/bash
mkdir -p gpurun_out
for v in "PT_BVH_BINS=16" "PT_BVH_NODE_COST=1.0 PT_BVH_MAX_LEAF=2" "PT_BVH_NODE_COST=1.0 PT_BVH_MAX_LEAF=2 PT_BVH_BINS=32" "PT_BVH_NODE_COST=0.75 PT_BVH_MAX_LEAF=2 PT_BVH_BINS=32" "PT_BVH_NODE_COST=1.0 PT_BVH_MAX_LEAF=1 PT_BVH_BINS=32" "PT_BVH_NODE_COST=0.5 PT_BVH_MAX_LEAF=2 PT_BVH_BINS=32"; do
  for c in 3 4 2; do
    env $v python bench.py --config $c --steps 8 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v config=$c', round(d['value']/1e9,3), 'G samples/s', {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})"
  done
done > gpurun_out/bvhparams2.log 2>&1
