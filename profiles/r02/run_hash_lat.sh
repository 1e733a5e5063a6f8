#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
KVX_HASH_PRIO=1 timeout 600 python tests/perf/hash_latency.py 2>&1 | tee gpurun_out/hash_lat.txt
