#!/bin/bash
cd "$(dirname "$0")/../.."
make -C paper_2407_00079_b200/csrc -j8 > /dev/null 2>&1 || echo "build failed"
mkdir -p gpurun_out
HP_TRACE=gpurun_out/k1d_trace_c4.npy timeout 120 python tests/perf/hash_profile.py 2>&1 | tail -4
HP_EQUAL=148 HP_TRACE=gpurun_out/k1d_trace_148.npy timeout 120 python tests/perf/hash_profile.py 2>&1 | tail -4
