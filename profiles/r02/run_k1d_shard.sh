#!/bin/bash
# K1d vs K1b on the sharded stage-1 hash (one rank's token-balanced shard of Config 4)
cd "$(dirname "$0")/../.."
make -C paper_2407_00079_b200/csrc -j8 > /dev/null 2>&1 || echo "build failed"
(
for SH in "0/1" "0/2" "1/2" "0/4" "3/4"; do
  HASH_SHARD=$SH timeout 60 python tests/perf/hash_phase.py 2>&1 | tail -1
  HASH_SHARD=$SH KVX_HASH_KERNEL=fold timeout 60 python tests/perf/hash_phase.py 2>&1 | tail -1
  HASH_SHARD=$SH KVX_HASH_KERNEL=fold KVX_HASH_FOLD_SHARE=0 timeout 60 python tests/perf/hash_phase.py 2>&1 | tail -1 | sed 's/^/share0 /'
done
) | tee gpurun_out/k1d_shard.txt
