#!/bin/bash
# LSU copy-kernel variants (N=1 Config 2; 16 requests = 1 wave): plain, .cs stores,
# next-item prefetch, both.  Then peer_ce N=2 gather with each variant.
for v in ${VARIANTS:-0 1 2 3}; do
  KVX_LSU_VARIANT=$v timeout 300 python bench.py --requests 16 --steps 8 --no-match --no-cpu-baseline --no-e2e > gpurun_out/lsuv$v.json 2>/dev/null
  echo "variant=$v $(python profiles/show.py gpurun_out/lsuv$v.json | head -2 | tr '\n' ' ')"
done
