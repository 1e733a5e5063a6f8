#!/bin/bash
# r02: match kernel -- warps per task x L2 pin x after-hash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for G in 1 2 4 8; do KVX_MATCH_GROUP=$G timeout 300 python tests/perf/match_phase.py 2>&1 | grep -v "^$" | tail -4; done | tee gpurun_out/match_sweep.txt
