#!/bin/bash
# r02: stage 1 fused (hash + queue-fed match) -- parity tests, default bench line
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hash_match.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/n1_c2_r02j.json 2> gpurun_out/n1_c2_r02j.err; echo "bench rc=$?"; tail -c 400 gpurun_out/n1_c2_r02j.err
