# half-warp block-hash kernel: parity + (chains per lane x warps per SM) sweep + the old fused kernel (Config 4 batch)
timeout 300 python -m pytest tests/test_gpu_hash_match.py -x -q 2>&1 | tail -2
for c in ${CHAINS:-1 2}; do for w in ${WARPS:-4 8 12}; do
  echo "chains=$c warps=$w $(KVX_HASH_HW_CHAINS=$c KVX_HASH_HW_WARPS=$w timeout 120 python tests/perf/hash_phase.py)"; done; done
echo "fused: $(KVX_HASH_KERNEL=fused timeout 120 python tests/perf/hash_phase.py)"
