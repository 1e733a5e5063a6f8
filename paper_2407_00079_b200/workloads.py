"""Synthetic workloads for the configs in BASELINE.json (LLaMA2-70B KV shape).

Nothing here is timed; it builds block selections (which blocks move where)
exactly as the reference defines them:

* ``TransferWorkload`` -- Config 2: requests whose ``hash_ids`` follow
  ``generate_workload`` (proj/src/trace.cpp:163-222): the first
  floor(cache_ratio * blocks) ids come from one shared hot chain, the rest are
  fresh.  The prefill instance holds every unique block once (shared prefix
  deduplicated, as a prefix cache does); the prefill -> decode stream moves a
  request's WHOLE chain (proj/src/sim_engine.cpp:463-464), landing in slots
  the decode allocator hands out.
* ``MatchWorkload`` -- Config 4: Kimi-like trace, token streams of Zipf-chosen
  sessions; requests share a prefix of their session's stream.

Shapes: LLaMA2-70B has 80 layers and 8 KV heads x 128 dim, so one token of
one layer's K (or V) is 2,048 B in fp16 and 327,680 B over all layers, K+V
(kv_bytes_per_token, proj/src/config.cpp:216).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List

import numpy as np

LLAMA70B = dict(layers=80, heads=8, head_dim=128)


@dataclass
class TransferWorkload:
    n_req: int = 64
    tokens: int = 8192
    block_size: int = 16
    cache_ratio: float = 0.5
    wave: int = 16                 # requests resident on the decode side at once
    layers: int = 80
    heads: int = 8
    head_dim: int = 128
    dtype_bytes: int = 2
    decode_fragmentation: float = 0.2  # fraction of decode slots held by other requests
    seed: int = 1
    hash_ids: List[np.ndarray] = field(default_factory=list, repr=False)

    def __post_init__(self):
        self.blocks = -(-self.tokens // self.block_size)
        shared = int(np.floor(self.cache_ratio * self.blocks))
        # generate_workload id assignment (trace.cpp:188-218): hot chain ids
        # first (grown on demand), then globally fresh ids in request order.
        hot = np.arange(shared, dtype=np.int64)
        next_id = shared
        self.hash_ids = []
        for _ in range(self.n_req):
            fresh = np.arange(next_id, next_id + self.blocks - shared, dtype=np.int64)
            next_id += self.blocks - shared
            self.hash_ids.append(np.concatenate([hot, fresh]))
        self.src_slots = next_id  # one slot per unique block
        rng = np.random.default_rng(self.seed)
        slot_of = rng.permutation(self.src_slots).astype(np.int32)
        self.src_tables = [slot_of[h] for h in self.hash_ids]
        need = self.wave * self.blocks
        self.dst_slots = int(np.ceil(need / (1.0 - self.decode_fragmentation)))
        n_busy = self.dst_slots - need
        self.dst_preoccupied = np.sort(
            rng.choice(self.dst_slots, size=n_busy, replace=False)).astype(np.int32)

    @property
    def n_waves(self) -> int:
        return -(-self.n_req // self.wave)

    def wave_requests(self, w: int) -> range:
        return range(w * self.wave, min(self.n_req, (w + 1) * self.wave))

    @property
    def slab_bytes(self) -> int:
        return self.block_size * self.heads * self.head_dim * self.dtype_bytes

    @property
    def kv_bytes_per_token(self) -> int:
        return self.layers * 2 * self.heads * self.head_dim * self.dtype_bytes

    def payload_bytes(self) -> int:
        """Bytes one pass moves: every request's whole chain, all layers, K and V."""
        return self.n_req * self.blocks * self.layers * 2 * self.slab_bytes

    def wave_src_table(self, w: int) -> np.ndarray:
        return np.concatenate([self.src_tables[r] for r in self.wave_requests(w)])

    def decode_tables(self, allocator_factory) -> List[np.ndarray]:
        """Decode block tables per wave from the product allocator: every wave
        starts from the same fragmented pool (the previous wave's requests
        have finished decoding and released their slots)."""
        out = []
        for w in range(self.n_waves):
            alloc = allocator_factory(self.dst_slots)
            alloc.mark(self.dst_preoccupied)
            tabs = [np.array(alloc.take(self.blocks), copy=True) for _ in self.wave_requests(w)]
            out.append(np.concatenate(tabs))
        return out

    def describe(self) -> dict:
        return {"workload": "config2: 64 req x 8K tok, 50% shared prefix, LLaMA2-70B KV",
                "requests": self.n_req, "tokens_per_request": self.tokens,
                "block_size": self.block_size, "layers": self.layers,
                "kv_heads": self.heads, "head_dim": self.head_dim,
                "kv_dtype": {1: "fp8", 2: "fp16", 4: "fp32"}[self.dtype_bytes],
                "cache_ratio": self.cache_ratio, "decode_wave": self.wave,
                "unique_src_blocks": self.src_slots, "decode_slots": self.dst_slots,
                "payload_bytes_per_step": self.payload_bytes()}


@dataclass
class LongContextWorkload:
    """Config 3: one 128K-token request, streamed in 2,048-token chunks
    (prefill_chunk, proj/src/config.cpp:219) layer by layer; with P pairs each
    pair owns a contiguous layer range (a CPP stage = a layer range,
    proj/tests/oracles.hpp:120-137), so total work is fixed (strong scaling)."""
    tokens: int = 131072
    block_size: int = 16
    chunk_tokens: int = 2048
    layers: int = 80
    heads: int = 8
    head_dim: int = 128
    dtype_bytes: int = 2
    decode_fragmentation: float = 0.2
    seed: int = 3

    def __post_init__(self):
        self.blocks = -(-self.tokens // self.block_size)
        rng = np.random.default_rng(self.seed)
        self.src_slots = self.blocks
        self.src_table = rng.permutation(self.src_slots).astype(np.int32)
        self.dst_slots = int(np.ceil(self.blocks / (1.0 - self.decode_fragmentation)))
        self.dst_preoccupied = np.sort(rng.choice(
            self.dst_slots, size=self.dst_slots - self.blocks, replace=False)).astype(np.int32)
        self.chunk_blocks = self.chunk_tokens // self.block_size

    @property
    def slab_bytes(self) -> int:
        return self.block_size * self.heads * self.head_dim * self.dtype_bytes

    def layer_range(self, pair: int, pairs: int):
        return (pair * self.layers // pairs, (pair + 1) * self.layers // pairs)

    def payload_bytes(self, pair: int = 0, pairs: int = 1) -> int:
        lo, hi = self.layer_range(pair, pairs)
        return self.blocks * (hi - lo) * 2 * self.slab_bytes

    def decode_table(self, allocator_factory) -> np.ndarray:
        alloc = allocator_factory(self.dst_slots)
        alloc.mark(self.dst_preoccupied)
        return np.array(alloc.take(self.blocks), copy=True)

    def describe(self) -> dict:
        return {"workload": "config3: 1 x 128K-token request, 2048-token chunks, layer-wise, "
                            "layer-range shards per pair", "tokens": self.tokens,
                "block_size": self.block_size, "chunk_tokens": self.chunk_tokens,
                "layers": self.layers, "kv_heads": self.heads, "head_dim": self.head_dim,
                "kv_dtype": {1: "fp8", 2: "fp16", 4: "fp32"}[self.dtype_bytes],
                "payload_bytes_total": self.payload_bytes()}


@dataclass
class MatchWorkload:
    """Config 4: Kimi-like trace; N requests, lengths U[8K, 24K], Zipf(alpha)
    session choice over `sessions` sessions; each request reuses a prefix of
    its session's token stream (30-100% of its length) then fresh tokens.
    The instance index holds the blocks earlier turns of every drawn session
    left behind, topped up with unrelated keys to exactly `pool_keys`."""
    n_req: int = 4096
    min_tokens: int = 8192
    max_tokens: int = 24576
    block_size: int = 16
    sessions: int = 10000
    zipf_alpha: float = 1.0
    pool_keys: int = 1 << 20
    vocab: int = 32000
    seed: int = 4

    def build(self):
        rng = np.random.default_rng(self.seed)
        p = 1.0 / np.arange(1, self.sessions + 1) ** self.zipf_alpha
        p /= p.sum()
        sess = rng.choice(self.sessions, size=self.n_req, p=p)
        lens = rng.integers(self.min_tokens, self.max_tokens + 1, size=self.n_req)
        streams = {}
        for s in np.unique(sess):
            streams[int(s)] = np.random.default_rng(self.seed * 1000003 + int(s)).integers(
                0, self.vocab, size=self.max_tokens).astype(np.int32)
        toks = []
        for r in range(self.n_req):
            n = int(lens[r])
            share = int(n * rng.uniform(0.3, 1.0))
            fresh = rng.integers(0, self.vocab, size=n - share).astype(np.int32)
            toks.append(np.concatenate([streams[int(sess[r])][:share], fresh]))
        self.tok_off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        self.tokens = np.concatenate(toks).astype(np.int32)
        # earlier turns: each drawn session left a random-depth prefix behind
        self.session_ids = sorted(streams)
        depth = rng.integers(0, self.max_tokens // self.block_size + 1, size=len(streams))
        self.warm_tok_off = np.concatenate(
            [[0], np.cumsum(depth * self.block_size)]).astype(np.int64)
        self.warm_tokens = np.concatenate(
            [streams[s][: int(d) * self.block_size] for s, d in zip(self.session_ids, depth)]
            + [np.zeros(0, np.int32)]).astype(np.int32)
        self.filler_rng_seed = int(rng.integers(1 << 62))
        return self

    @property
    def n_blocks(self) -> int:
        lens = np.diff(self.tok_off)
        return int(((lens + self.block_size - 1) // self.block_size).sum())

    def filler_keys(self, n: int, salt: int = 0) -> np.ndarray:
        """Unrelated resident keys (never equal to a chain key with overwhelming
        probability: they are drawn uniformly from [2^62, 2^63 - 2^20));
        `salt` gives each prefill instance its own."""
        rng = np.random.default_rng(self.filler_rng_seed + salt)
        return rng.integers(1 << 62, (1 << 63) - (1 << 20), size=n, dtype=np.int64)

    def describe(self) -> dict:
        return {"workload": "config4: Kimi-like replay, Zipf prefix sharing, 1M-block pool",
                "requests": self.n_req, "tokens": f"U[{self.min_tokens},{self.max_tokens}]",
                "block_size": self.block_size, "sessions": self.sessions,
                "zipf_alpha": self.zipf_alpha, "pool_keys": self.pool_keys,
                "query_blocks": self.n_blocks}
