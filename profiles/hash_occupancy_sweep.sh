#!/bin/bash
# Stage-1 hash: registers/occupancy (min CTAs per SM) sweep; rebuilds libkvx on the box.
for m in 3 4 5; do
  touch paper_2407_00079_b200/csrc/kvx_hash.cu
  make -s -C paper_2407_00079_b200/csrc EXTRA_NVFLAGS=-DKVX_HASH_MIN_CTAS=$m > /dev/null 2>&1
  echo "min_ctas=$m $(python tests/perf/hash_phase.py) | produce-only: $(KVX_HASH_FOLD_SMS=-1 python tests/perf/hash_phase.py)"
done
touch paper_2407_00079_b200/csrc/kvx_hash.cu; make -s -C paper_2407_00079_b200/csrc > /dev/null 2>&1
