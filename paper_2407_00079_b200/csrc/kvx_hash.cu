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
//   content_hash_kernel  one warp per request; lane j folds block (32w + j)'s
//                        tokens and parks the content hash in keys[].  Token
//                        loads are 128-bit when the request's token range is
//                        16-byte aligned and bs % 4 == 0 (warp-uniform test),
//                        scalar otherwise; lanes walk adjacent 4*bs-byte spans
//                        so L1 serves the follow-up loads of each line.
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

__global__ void __launch_bounds__(256) content_hash_kernel(const int32_t* __restrict__ tokens,
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
    for (int64_t b = lane; b < nblk; b += 32) {
      const int64_t t0 = lo + b * bs;
      const int n = static_cast<int>(min(static_cast<int64_t>(bs), hi - t0));
      out[b] = (vec && n == bs) ? fold_tokens_vec4(tokens + t0, n)
                                : fold_tokens_scalar(tokens + t0, n);
    }
  }
}

__global__ void __launch_bounds__(32) key_fold_kernel(const int64_t* __restrict__ key_off,
                                                      int64_t n_req, int64_t* __restrict__ keys) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n_req) return;
  const int64_t k0 = key_off[r], k1 = key_off[r + 1];
  int64_t prev = 0;
  int64_t k = k0;
  for (; k + 8 <= k1; k += 8) {
    int64_t c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j] = keys[k + j];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      prev = chain_hash(prev, static_cast<uint64_t>(c[j]));
      c[j] = prev;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) keys[k + j] = c[j];
  }
  for (; k < k1; ++k) {
    prev = chain_hash(prev, static_cast<uint64_t>(keys[k]));
    keys[k] = prev;
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
  const int64_t want = (n_req + (threads / 32) - 1) / (threads / 32);
  const int64_t cap = static_cast<int64_t>(sm_count(dev)) * 8;
  const int blocks = static_cast<int>(want < cap ? want : cap);
  content_hash_kernel<<<blocks, threads, 0, s>>>(d_tokens, d_tok_off, n_req, static_cast<int>(bs),
                                                 d_key_off, d_keys);
  KVX_LAUNCH_CHECK("content_hash_kernel");
  key_fold_kernel<<<static_cast<int>((n_req + 31) / 32), 32, 0, s>>>(d_key_off, n_req, d_keys);
  KVX_LAUNCH_CHECK("key_fold_kernel");
  return KVX_OK;
}
