cd /root/repo
make -C paper_2407_00079_b200/csrc -j8 >/dev/null 2>&1
for SH in 0/1 0/2 0/4 0/8; do for W in 6 8 10 12 16; do
  HASH_SHARD=$SH KVX_HASH_HW_WARPS=$W timeout 60 python tests/perf/hash_phase.py 2>&1 | tail -1 | sed "s/^/W=$W /"
done; done | tee gpurun_out/hw_sweep.txt
