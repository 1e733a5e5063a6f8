"""CPU oracle for the KVCache hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  It is the checker, never the
thing measured as the product and never a fallback for it.

Two libraries sit behind it:

* ``liboracle.so`` -- this repo's plain-C restatement (``kvx_oracle.c``) of
  chain_hash (proj/src/kvcache.cpp:14-23), match_prefix
  (proj/src/kvcache.cpp:150-158), find_best_prefix_match
  (proj/src/conductor.cpp:57-73) and the build-defined byte stages
  (gather / scatter / paged copy, synthetic KV content, decode allocator).
* ``_ref/libkvref.so`` -- the reference's own kvcache.cpp / conductor.cpp /
  perf_model.cpp compiled in place (oracle/Makefile) behind ``ref_shim.cpp``.
  Only present where /root/reference was available at build time; the
  committed fixtures under tests/golden/ carry its outputs to the GPU box.
"""
from .oracle import *  # noqa: F401,F403
from .oracle import Oracle, RefLib, ref_available, build_oracle  # noqa: F401
