#!/bin/bash
# r02: half-warp hash with warp-priority first claims (KVX_HASH_PRIO) x warps per SM
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for P in 0 1; do for W in 8 12 16 20; do
  KVX_HASH_PRIO=$P KVX_HASH_HW_WARPS=$W timeout 300 python tests/perf/hash_phase.py 2>&1 | tail -1
done; done | tee gpurun_out/hash_prio.txt
