#!/bin/bash
# r02: high-word shifts on the FMA pipe (KVX_HASH_FMA) x warps; lone-request latency
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for F in 0 1; do for W in 12 16; do
  KVX_HASH_FMA=$F KVX_HASH_HW_WARPS=$W timeout 300 python tests/perf/hash_phase.py 2>&1 | tail -1 | sed "s/^/fma=$F /"
done; done | tee gpurun_out/hash_fma.txt
for F in 0 1; do KVX_HASH_FMA=$F HL_TOKENS=24576 timeout 300 python tests/perf/hash_latency.py 2>&1 | head -1 | sed "s/^/fma=$F /"; done | tee -a gpurun_out/hash_fma.txt
