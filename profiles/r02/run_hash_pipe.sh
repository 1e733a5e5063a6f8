#!/bin/bash
# r02: software-pipelined half-warp hash (KVX_HASH_PIPE=1) vs the r01 loop
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_hash_match.py -x -q 2>&1 | tail -2
for P in 0 1; do for W in 12 16; do
  KVX_HASH_PIPE=$P KVX_HASH_HW_WARPS=$W timeout 300 python tests/perf/hash_phase.py 2>&1 | tail -1 | sed "s/^/pipe=$P /"
done; done | tee gpurun_out/hash_pipe.txt
for P in 0 1; do KVX_HASH_PIPE=$P HL_NS=1,592,3552 timeout 300 python tests/perf/hash_latency.py 2>&1 | sed "s/^/pipe=$P /"; done | tee -a gpurun_out/hash_pipe.txt
bash profiles/r02/run_dropin.sh 2>&1 | tee gpurun_out/dropin_latency.txt
KVX_MATCH_GROUP=2 timeout 300 python tests/perf/match_phase.py > gpurun_out/mp.txt 2>&1 && \
KVX_MATCH_GROUP=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:match_group -s 6 -c 1 \
  -o gpurun_out/prof_match_g2_r02 python tests/perf/match_phase.py > gpurun_out/ncu_mp.log 2>&1
echo "ncu match rc=$?"
