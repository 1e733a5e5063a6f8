#!/bin/bash
# r02: match -- sector probing (256-bit sector loads) vs slot probing
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for S in 0 1; do for GC in "2 2" "2 1" "4 1" "2 4" "4 2" "8 1"; do set -- $GC
  KVX_MATCH_SECTOR=$S KVX_MATCH_GROUP=$1 KVX_MATCH_CHAINS=$2 MP_PIN=0 timeout 300 python tests/perf/match_phase.py 2>&1 | grep after_hash=1 | sed "s/^/sector=$S /"
done; done | tee gpurun_out/match_sweep4.txt
for N in 148 4096; do KVX_MATCH_SECTOR=1 MP_NREQ=$N MP_PIN=0 timeout 300 python tests/perf/match_phase.py 2>&1 | grep after_hash=1 | sed "s/^/sector=1 /"; done | tee -a gpurun_out/match_sweep4.txt
timeout 600 python -m pytest tests/test_gpu_hash_match.py tests/test_gpu_conductor.py tests/test_gpu_xmatch.py -x -q 2>&1 | tail -2
