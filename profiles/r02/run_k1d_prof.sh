#!/bin/bash
cd "$(dirname "$0")/../.."
make -C paper_2407_00079_b200/csrc -j8 > /dev/null 2>&1 || echo "build failed"
KVX_HASH_KERNEL=fold timeout 200 python -m pytest tests/test_gpu_hash_match.py -x -q 2>&1 | tail -1
(
for CFG in "32 1 0" "32 0 0"; do set -- $CFG
  echo "== pass=$1 share=$2 key=$3"
  KVX_HASH_FOLD_PASS=$1 KVX_HASH_FOLD_SHARE=$2 KVX_HASH_PRIO_KEY=$3 timeout 60 python tests/perf/hash_profile.py 2>&1 | tail -4
  KVX_HASH_FOLD_PASS=$1 KVX_HASH_FOLD_SHARE=$2 KVX_HASH_PRIO_KEY=$3 KVX_HASH_KERNEL=fold timeout 60 python tests/perf/hash_phase.py 2>&1 | tail -1
done
KVX_HASH_FOLD_SHARE=0 HP_EQUAL=148 timeout 60 python tests/perf/hash_profile.py 2>&1 | tail -4
) | tee gpurun_out/k1d_prof2.txt
