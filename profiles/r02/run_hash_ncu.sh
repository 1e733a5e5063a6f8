#!/bin/bash
# r02: source-level ncu of the half-warp hash kernel on ONE 1,536-block request
# (the lone key chain's per-step latency) and on the Config 4 batch
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
HL_NS=1 timeout 300 python tests/perf/hash_latency.py > gpurun_out/hl1.txt 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:halfwarp_hash -s 3 -c 1 \
  -o gpurun_out/prof_hash_lone_r02 env HL_NS=1 python tests/perf/hash_latency.py > gpurun_out/ncu_hl.log 2>&1
echo "ncu lone rc=$?"
timeout 300 python tests/perf/hash_phase.py > gpurun_out/hp.txt 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:halfwarp_hash -s 3 -c 1 \
  -o gpurun_out/prof_hash_batch_r02 python tests/perf/hash_phase.py > gpurun_out/ncu_hp.log 2>&1
echo "ncu batch rc=$?"
