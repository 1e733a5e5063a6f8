#!/bin/bash
# r02: match -- next-wave query-key prefetch, slot vs sector probing
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for S in 0 1; do for GC in "2 2" "4 2" "4 1" "2 4"; do set -- $GC
  KVX_MATCH_SECTOR=$S KVX_MATCH_GROUP=$1 KVX_MATCH_CHAINS=$2 MP_PIN=0 timeout 300 python tests/perf/match_phase.py 2>&1 | grep after_hash=1 | sed "s/^/prefetch sector=$S /"
done; done | tee gpurun_out/match_sweep5.txt
for S in 0 1; do KVX_MATCH_SECTOR=$S MP_NREQ=148 MP_PIN=0 timeout 300 python tests/perf/match_phase.py 2>&1 | grep after_hash=1 | sed "s/^/prefetch sector=$S /"; done | tee -a gpurun_out/match_sweep5.txt
timeout 600 python -m pytest tests/test_gpu_hash_match.py tests/test_gpu_conductor.py tests/test_gpu_xmatch.py -x -q 2>&1 | tail -2
