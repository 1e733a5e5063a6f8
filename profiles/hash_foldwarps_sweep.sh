#!/bin/bash
# Stage-1 hash: folding warps per reserved SM (1 per sub-partition = 4, 2 per = 8); rebuilds on the box.
for w in 4 8; do
  touch paper_2407_00079_b200/csrc/kvx_hash.cu
  make -s -C paper_2407_00079_b200/csrc EXTRA_NVFLAGS=-DKVX_HASH_FOLD_WARPS=$w > /dev/null 2>&1
  echo "fold_warps=$w $(python tests/perf/hash_phase.py) $(python tests/perf/hash_phase.py)"
done
touch paper_2407_00079_b200/csrc/kvx_hash.cu; make -s -C paper_2407_00079_b200/csrc > /dev/null 2>&1
