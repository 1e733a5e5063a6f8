#!/bin/bash
# r02: hash issue path -- lazy (rare-branch partial rows) vs per-chunk sizes every sub-round
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_hash_match.py -x -q 2>&1 | tail -2
for I in 0 1; do for r in 1 2; do KVX_HASH_ISSUE=$I timeout 300 python tests/perf/hash_phase.py 2>&1 | tail -1 | sed "s/^/issue=$I /"; done; done | tee gpurun_out/hash_issue.txt
for I in 0 1; do KVX_HASH_ISSUE=$I HL_NS=1 timeout 300 python tests/perf/hash_latency.py 2>&1 | sed "s/^/issue=$I /"; done | tee -a gpurun_out/hash_issue.txt
# the default bench line once more (DRAM-tier fix)
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/n1_c2_r02i.json 2> gpurun_out/n1_c2_r02i.err; echo "bench rc=$?"
