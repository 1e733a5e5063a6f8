// kvx_hash.cu -- K1: batched prefix block hashing (stage 1a).
//
// Reference: kvcsim::chain_hash (proj/src/kvcache.cpp:14-23) defines the key
// mixer; the paper's PrefixHash defines keys as prefix
// chained.  The per-block content hash is build-defined: a fold of
// chain_hash over the block's token ids starting from 0.
//
// chain_hash is not associative, so both folds are serial; the parallelism is
// blocks (content hashes are independent) and requests (key chains are
// independent).  Two phases, so no lane ever repeats another lane's work:
//   content_hash_kernel  flattened over all blocks of the batch (32 per warp,
//                        perfectly balanced); each lane folds one block's
//                        tokens and parks the content hash in keys[].  Token
//                        loads are 128-bit when the block is 16-byte aligned
//                        and bs % 4 == 0, scalar otherwise; lanes walk
//                        adjacent 4*bs-byte spans so L1 serves the follow-ups.
//   key_fold_kernel      one LANE per request: key_i = chain_hash(key_{i-1},
//                        content_i) in place, 8 contents prefetched per step.
//                        32-thread CTAs spread the (latency-bound) chains over
//                        every SM.
// Pure integer work: 64-bit multiplies are IMAD sequences (no native 64-bit
// multiplier), tensor cores do not apply.
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

// Flattened over the batch's blocks: warp w owns blocks [32w, 32w + 32) of the
// concatenated key array, so every warp does the same amount of hashing no
// matter how request lengths vary.  Lane 0 finds the owning request by binary
// search over key_off and broadcasts it; lanes past that request's end walk
// forward (a warp spans at most a few short requests).
__global__ void __launch_bounds__(256) content_hash_kernel(const int32_t* __restrict__ tokens,
                                                           const int64_t* __restrict__ tok_off,
                                                           int64_t n_req, int bs,
                                                           const int64_t* __restrict__ key_off,
                                                           int64_t* __restrict__ keys) {
  const int lane = threadIdx.x & 31;
  const int64_t total = key_off[n_req];
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t w = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
       32 * w < total; w += warps) {
    const int64_t g0 = 32 * w;
    int64_t r = 0;
    if (lane == 0) {  // last r with key_off[r] <= g0
      int64_t lo = 0, hi = n_req - 1;
      while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (__ldg(key_off + mid) <= g0) lo = mid;
        else hi = mid - 1;
      }
      r = lo;
    }
    r = __shfl_sync(0xffffffffu, r, 0);
    const int64_t g = g0 + lane;
    if (g < total) {
      while (__ldg(key_off + r + 1) <= g) ++r;
      const int64_t b = g - __ldg(key_off + r);
      const int64_t t0 = __ldg(tok_off + r) + b * bs;
      const int64_t t1 = __ldg(tok_off + r + 1);
      const int n = static_cast<int>(min(static_cast<int64_t>(bs), t1 - t0));
      const bool vec = n == bs && ((bs & 3) == 0) &&
                       ((reinterpret_cast<uintptr_t>(tokens + t0) & 15) == 0);
      keys[g] = vec ? fold_tokens_vec4(tokens + t0, n) : fold_tokens_scalar(tokens + t0, n);
    }
  }
}

// One lane per request; contents are prefetched one 8-block batch ahead so
// the serial chain never waits on memory.
__global__ void __launch_bounds__(32) key_fold_kernel(const int64_t* __restrict__ key_off,
                                                      int64_t n_req, int64_t* __restrict__ keys) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n_req) return;
  const int64_t k0 = key_off[r], k1 = key_off[r + 1];
  int64_t prev = 0;
  int64_t cur[8], nxt[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) cur[j] = (k0 + j < k1) ? keys[k0 + j] : 0;
  for (int64_t k = k0; k < k1; k += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) nxt[j] = (k + 8 + j < k1) ? keys[k + 8 + j] : 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (k + j < k1) {
        prev = chain_hash(prev, static_cast<uint64_t>(cur[j]));
        keys[k + j] = prev;
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) cur[j] = nxt[j];
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
  cudaStream_t s = as_stream(stream);
  const int threads = 256;
  const int blocks = sm_count(dev) * 8;  // 2048 threads per SM, grid-stride over blocks
  content_hash_kernel<<<blocks, threads, 0, s>>>(d_tokens, d_tok_off, n_req, static_cast<int>(bs),
                                                 d_key_off, d_keys);
  KVX_LAUNCH_CHECK("content_hash_kernel");
  key_fold_kernel<<<static_cast<int>((n_req + 31) / 32), 32, 0, s>>>(d_key_off, n_req, d_keys);
  KVX_LAUNCH_CHECK("key_fold_kernel");
  return KVX_OK;
}
