timeout 300 python -m pytest tests/test_gpu_hash_match.py -x -q 2>&1 | tail -1
for v in 1 2 0; do for w in 4 8 12; do echo "variant=$v warps=$w $(KVX_HASH_HW_VARIANT=$v KVX_HASH_HW_WARPS=$w timeout 120 python tests/perf/hash_phase.py)"; done; done
for v in 1 2; do echo "variant=$v parity: $(KVX_HASH_HW_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_hash_match.py -x -q 2>&1 | tail -1)"; done
