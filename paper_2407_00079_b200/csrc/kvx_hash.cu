// kvx_hash.cu -- K1: batched prefix block hashing (stage 1a).
//
// Reference: kvcsim::chain_hash (proj/src/kvcache.cpp:14-23) defines the key
// mixer; the paper's PrefixHash defines keys as prefix
// chained.  The per-block content hash is build-defined: a fold of
// chain_hash over the block's token ids starting from 0.
//
// Mapping: one warp per request.  Each lane folds one block's tokens (the
// content hash is a serial fold, so a block is the unit of parallelism); the
// prefix chain across blocks is then a serial fold too, done warp-uniformly
// over the 32 contents fetched with __shfl_sync, lane j keeping key j.  Token
// loads are 128-bit when the request's token range is 16-byte aligned and the
// block size is a multiple of 4; the per-lane stride is bs*4 bytes, so the
// 32 lanes walk 32 adjacent 64-byte spans and L1 serves the follow-up loads.
#include "kvx_common.cuh"

namespace kvx {
namespace {

__device__ __forceinline__ int64_t fold_tokens_scalar(const int32_t* __restrict__ t, int n) {
  int64_t h = 0;
  for (int i = 0; i < n; ++i)
    h = chain_hash(h, static_cast<uint64_t>(static_cast<uint32_t>(__ldg(t + i))));
  return h;
}

__device__ __forceinline__ int64_t fold_tokens_vec4(const int32_t* __restrict__ t, int n) {
  // n is a multiple of 4 and t is 16-byte aligned.
  const int4* v = reinterpret_cast<const int4*>(t);
  int64_t h = 0;
#pragma unroll 4
  for (int i = 0; i < n / 4; ++i) {
    const int4 q = __ldg(v + i);
    h = chain_hash(h, static_cast<uint64_t>(static_cast<uint32_t>(q.x)));
    h = chain_hash(h, static_cast<uint64_t>(static_cast<uint32_t>(q.y)));
    h = chain_hash(h, static_cast<uint64_t>(static_cast<uint32_t>(q.z)));
    h = chain_hash(h, static_cast<uint64_t>(static_cast<uint32_t>(q.w)));
  }
  return h;
}

__global__ void __launch_bounds__(256) block_hash_kernel(const int32_t* __restrict__ tokens,
                                                         const int64_t* __restrict__ tok_off,
                                                         int64_t n_req, int bs,
                                                         const int64_t* __restrict__ key_off,
                                                         int64_t* __restrict__ keys) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
       r < n_req; r += warps) {
    const int64_t lo = tok_off[r];
    const int64_t hi = tok_off[r + 1];
    const int64_t nblk = (hi - lo + bs - 1) / bs;
    int64_t* out = keys + key_off[r];
    const bool vec = ((bs & 3) == 0) &&
                     ((reinterpret_cast<uintptr_t>(tokens + lo) & 15) == 0);  // warp-uniform
    int64_t prev = 0;
    for (int64_t b0 = 0; b0 < nblk; b0 += 32) {
      const int64_t b = b0 + lane;
      uint64_t content = 0;
      if (b < nblk) {
        const int64_t t0 = lo + b * bs;
        const int n = static_cast<int>(min(static_cast<int64_t>(bs), hi - t0));
        content = static_cast<uint64_t>((vec && n == bs) ? fold_tokens_vec4(tokens + t0, n)
                                                          : fold_tokens_scalar(tokens + t0, n));
      }
      const int cnt = static_cast<int>(min(static_cast<int64_t>(32), nblk - b0));
      int64_t mine = 0;
      for (int j = 0; j < cnt; ++j) {
        const uint64_t c = __shfl_sync(0xffffffffu, content, j);
        prev = chain_hash(prev, c);
        if (lane == j) mine = prev;
      }
      if (b < nblk) out[b] = mine;
    }
  }
}

}  // namespace
}  // namespace kvx

using namespace kvx;

extern "C" int kvx_chain_hash_batch(const int32_t* d_tokens, const int64_t* d_tok_off,
                                    int64_t n_req, int64_t bs, const int64_t* d_key_off,
                                    int64_t* d_keys, void* stream) {
  KVX_REQUIRE(n_req >= 0, "kvx_chain_hash_batch: n_req must be >= 0");
  KVX_REQUIRE(bs >= 1 && bs <= (1 << 20), "kvx_chain_hash_batch: block size must be >= 1");
  if (n_req == 0) return KVX_OK;
  KVX_REQUIRE(d_tok_off && d_key_off && d_keys, "kvx_chain_hash_batch: NULL array");
  int dev = 0;
  KVX_CUDA(cudaGetDevice(&dev));
  const int threads = 256;
  const int64_t want = (n_req + (threads / 32) - 1) / (threads / 32);
  const int64_t cap = static_cast<int64_t>(sm_count(dev)) * 8;
  const int blocks = static_cast<int>(want < cap ? want : cap);
  block_hash_kernel<<<blocks, threads, 0, as_stream(stream)>>>(d_tokens, d_tok_off, n_req,
                                                               static_cast<int>(bs), d_key_off,
                                                               d_keys);
  KVX_LAUNCH_CHECK("block_hash_kernel");
  return KVX_OK;
}
