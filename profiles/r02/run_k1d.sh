#!/bin/bash
# K1d (per-SM producers + fold lanes) vs K1b (half-warp): parity, batch time, latency
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
make -C paper_2407_00079_b200/csrc -j8 > /dev/null 2>&1 || echo "build failed"
KVX_HASH_KERNEL=fold timeout 300 python -m pytest tests/test_gpu_hash_match.py -x -q 2>&1 | tail -3
(
for P in 12 16 20 23 24; do
  KVX_HASH_KERNEL=fold KVX_HASH_PRODUCERS=$P timeout 120 python tests/perf/hash_phase.py 2>&1 | tail -1 | sed "s/^/fold producers=$P /"
done
timeout 120 python tests/perf/hash_phase.py 2>&1 | tail -1 | sed "s/^/halfwarp /"
KVX_HASH_KERNEL=fold HL_NS=1,148,592,3552 timeout 200 python tests/perf/hash_latency.py 2>&1 | sed "s/^/fold /"
) | tee gpurun_out/k1d.txt
