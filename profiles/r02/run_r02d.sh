#!/bin/bash
# r02d: match (warps x chains) sweep, drop-in latency with pool recycling, hash ncu (pipelined)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for GC in "1 4" "2 4" "2 2" "2 1" "4 2" "4 1" "8 1" "8 2"; do
  set -- $GC
  KVX_MATCH_GROUP=$1 KVX_MATCH_CHAINS=$2 timeout 300 python tests/perf/match_phase.py 2>&1 | grep "after_hash=1" | sed "s/^/chains=$2 /"
done | tee gpurun_out/match_sweep2.txt
bash profiles/r02/run_dropin.sh 2>&1 | tee gpurun_out/dropin_latency2.txt
timeout 900 python -m pytest tests/test_gpu_dropin.py tests/test_gpu_dropin_engine.py tests/test_gpu_hash_match.py -x -q 2>&1 | tail -2
bash profiles/r02/run_hash_ncu.sh
