#!/bin/bash
# Config 5 at N=1 (local fused, programmatic dependent launch between layer units)
mkdir -p gpurun_out/c5_r01j
for bs in 16 32 64 128 256 512; do
  for dt in 2 1; do
    timeout 300 python bench.py --block-size $bs --dtype-bytes $dt --steps 3 --no-match --no-cpu-baseline --no-e2e \
      > gpurun_out/c5_r01j/n1_bs${bs}_dt${dt}.json 2>/dev/null; echo "n1 bs=$bs dt=$dt rc=$?"
  done
done
