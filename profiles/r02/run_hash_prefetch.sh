#!/bin/bash
# K1b token prefetch depth (sub-rounds in flight), rebuilt per value
cd "$(dirname "$0")/../.."
for PF in 2 3 4 5; do
  make -C paper_2407_00079_b200/csrc -j8 EXTRA_NVFLAGS="-DKVX_HASH_PREFETCH=$PF" -B > /dev/null 2>&1 || echo "build failed"
  timeout 60 python tests/perf/hash_phase.py 2>&1 | tail -1 | sed "s/^/prefetch=$PF /"
done | tee gpurun_out/hash_prefetch.txt
make -C paper_2407_00079_b200/csrc -j8 -B > /dev/null 2>&1
