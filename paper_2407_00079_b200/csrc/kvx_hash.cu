// kvx_hash.cu -- K1: batched prefix block hashing (stage 1a).
//
// Reference: kvcsim::chain_hash (proj/src/kvcache.cpp:14-23) defines the key
// mixer; the paper's PrefixHash defines keys as prefix
// chained.  The per-block content hash is build-defined: a fold of
// chain_hash over the block's token ids starting from 0.
//
//   content_i = fold(chain_hash, tokens of block i, from 0)      (parallel over blocks)
//   key_i     = chain_hash(key_{i-1}, content_i), key_{-1} = 0     (serial per request)
//
// chain_hash is not associative, so the key chain of a request is a strictly
// serial fold (~100 cycles of dependent int64 arithmetic per block), while the
// content hashes are independent and ALU-throughput bound.  One persistent,
// cooperatively launched kernel overlaps the two:
//   * producer warps hash contents in WINDOW-MAJOR order -- window 0 (blocks
//     0..31) of every request, then window 1 of every request, ... -- one
//     (request, window) task per warp, lane = block, 128-bit token loads when
//     aligned.  Contents are parked in keys[] (chain_hash results are >= 0;
//     keys[] was pre-filled with -1 by block_hash_prep_kernel);
//   * folding lanes (lane = request, claimed from a counter) on SMs reserved
//     for them by %smid -- one folding warp per SM sub-partition, because a
//     lone chain runs at its ~97-cycle dependency latency while four per
//     sub-partition are issue bound (tests/perf/hash_micro.cu) -- walk their
//     request's keys[] 16 at a time: wait until the whole batch is produced
//     (re-polled with one round of parallel volatile loads and exponential
//     back-off -- tight polling measurably starves the producers of L2
//     bandwidth), prefetch the next batch, chain, overwrite in place.
//     Producers join the folding when the content tasks run out.
// Measured on the Config 4 batch (4,096 requests, 4.17 M blocks): content
// production alone 161 us; sequential produce-then-fold 373 us; this kernel
// 237 us (tests/perf/hash_phase.py, KVX_HASH_FOLD_SMS sweeps the reserve).
// Window-major production keeps every request's fold right behind its
// producer, so the batch costs ~max(content throughput, longest fold) instead
// of their sum.  Waiting happens only inside this single cooperative launch
// (all CTAs co-resident), never between separate launches.
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "kvx_common.cuh"

namespace kvx {
namespace {

constexpr int kHashThreads = 256;  // 8 warps: warp 0 folds (when assigned), 1..7 produce
constexpr int kFoldBatch = 16;
#ifndef KVX_HASH_MIN_CTAS
#define KVX_HASH_MIN_CTAS 3  // resident CTAs per SM (r01 sweep: 3 best; more spills or slows the fold)
#endif

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

// 16 tokens starting M tokens into a 16-byte aligned window: five aligned
// 128-bit loads cover them whatever the block's alignment, and the token
// selection is resolved at compile time (no per-token address arithmetic).
template <int M>
__device__ __forceinline__ int64_t fold16(const int32_t* __restrict__ aligned, int64_t h) {
  const int4* v = reinterpret_cast<const int4*>(aligned);
  uint32_t t[20];
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    const int4 q = __ldg(v + i);
    t[4 * i] = static_cast<uint32_t>(q.x);
    t[4 * i + 1] = static_cast<uint32_t>(q.y);
    t[4 * i + 2] = static_cast<uint32_t>(q.z);
    t[4 * i + 3] = static_cast<uint32_t>(q.w);
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) h = chain_hash(h, static_cast<uint64_t>(t[M + i]));
  return h;
}

// Content hash of a full block whose size is a multiple of 16 tokens; the
// caller guarantees the 16-byte window [t0 & ~3, t0 & ~3 + bs + 4) is inside
// the token array.
__device__ __forceinline__ int64_t fold_tokens_x16(const int32_t* __restrict__ tokens, int64_t t0,
                                                   int bs) {
  const int m = static_cast<int>(t0 & 3);
  const int32_t* a = tokens + (t0 - m);
  int64_t h = 0;
  for (int c = 0; c < bs; c += 16, a += 16) {
    switch (m) {
      case 0: h = fold16<0>(a, h); break;
      case 1: h = fold16<1>(a, h); break;
      case 2: h = fold16<2>(a, h); break;
      default: h = fold16<3>(a, h); break;
    }
  }
  return h;
}

__device__ __forceinline__ int64_t ld_volatile(const int64_t* p) {
  int64_t v;
  asm volatile("ld.volatile.global.s64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

// keys[0 .. total) = -1 ("content not ready"); ws[0] = max windows per request.
__global__ void __launch_bounds__(256) block_hash_prep_kernel(const int64_t* __restrict__ key_off,
                                                              int64_t n_req,
                                                              int64_t* __restrict__ keys,
                                                              unsigned long long* __restrict__ ws) {
  const int64_t total = key_off[n_req];
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = tid; i < total; i += stride) keys[i] = -1;
  unsigned long long wmax = 0;
  for (int64_t r = tid; r < n_req; r += stride) {
    const auto w = static_cast<unsigned long long>((key_off[r + 1] - key_off[r] + 31) / 32);
    wmax = w > wmax ? w : wmax;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long x = __shfl_down_sync(0xffffffffu, wmax, o);
    wmax = x > wmax ? x : wmax;
  }
  if ((threadIdx.x & 31) == 0 && wmax) atomicMax(ws, wmax);
}

__device__ __forceinline__ uint32_t sm_id() {
  uint32_t id;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
  return id;
}

// Fold whole requests, claimed one per lane from ws[1], until none are left.
// The next 16 contents are loaded while the current 16 are chained, so a
// request whose contents are all produced runs at the chain_hash dependency
// latency (~97 cycles per block measured, tests/perf/hash_micro.cu).
__device__ __forceinline__ void fold_requests(const int64_t* __restrict__ key_off, int64_t n_req,
                                              int64_t* keys, unsigned long long* ws) {
  while (true) {
    const int64_t r = static_cast<int64_t>(atomicAdd(ws + 1, 1ull));
    if (r >= n_req) return;
    const int64_t k0 = key_off[r], k1 = key_off[r + 1];
    int64_t prev = 0;
    int64_t c[kFoldBatch];
#pragma unroll
    for (int j = 0; j < kFoldBatch; ++j) c[j] = (k0 + j < k1) ? ld_volatile(keys + k0 + j) : 0;
    for (int64_t k = k0; k < k1; k += kFoldBatch) {
      const int m = static_cast<int>(min(static_cast<int64_t>(kFoldBatch), k1 - k));
      // Wait for the whole batch, re-polling every missing entry in ONE round
      // of parallel loads (polling them one by one would serialise an L2
      // round trip per block whenever the fold catches up with production).
      unsigned backoff = 512;  // ns; polling harder steals L2 bandwidth from the producers
      while (true) {
        bool ready = true;
#pragma unroll
        for (int j = 0; j < kFoldBatch; ++j) ready = ready && (j >= m || c[j] >= 0);
        if (ready) break;
        __nanosleep(backoff);
        backoff = backoff < 4096 ? backoff * 2 : backoff;
#pragma unroll
        for (int j = 0; j < kFoldBatch; ++j)
          if (j < m && c[j] < 0) c[j] = ld_volatile(keys + k + j);
      }
      int64_t nx[kFoldBatch];  // prefetch the next batch while this one is chained
#pragma unroll
      for (int j = 0; j < kFoldBatch; ++j)
        nx[j] = (k + kFoldBatch + j < k1) ? ld_volatile(keys + k + kFoldBatch + j) : 0;
#pragma unroll
      for (int j = 0; j < kFoldBatch; ++j) {
        if (j < m) {
          prev = chain_hash(prev, static_cast<uint64_t>(c[j]));
          keys[k + j] = prev;
        }
      }
#pragma unroll
      for (int j = 0; j < kFoldBatch; ++j) c[j] = nx[j];
    }
  }
}

// Roles by SM: the first CTA to arrive on each of the first `fold_sms` SMs
// runs kFoldWarps folding warps (one per SM sub-partition: a lone chain runs
// at its dependency latency, four per sub-partition would be issue bound);
// other CTAs on those SMs exit.  Every other warp produces contents, then
// joins the folding of whatever is still unclaimed.
#ifndef KVX_HASH_FOLD_WARPS
#define KVX_HASH_FOLD_WARPS 4
#endif
constexpr int kFoldWarps = KVX_HASH_FOLD_WARPS;

__global__ void __launch_bounds__(kHashThreads, KVX_HASH_MIN_CTAS) block_hash_fused_kernel(
    const int32_t* __restrict__ tokens, const int64_t* __restrict__ tok_off, int64_t n_req,
    int bs, const int64_t* __restrict__ key_off, int64_t* keys, unsigned long long* ws,
    int fold_sms) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int sm = static_cast<int>(sm_id());
  if (sm < fold_sms) {
    __shared__ unsigned long long ticket;
    if (threadIdx.x == 0) ticket = atomicAdd(ws + 3 + sm, 1ull);
    __syncthreads();
    if (ticket == 0 && warp < kFoldWarps) fold_requests(key_off, n_req, keys, ws);
    return;
  }
  const int64_t tasks = static_cast<int64_t>(ws[0]) * n_req;
  const int64_t total_tok = tok_off[n_req];
  const bool x16_ok = (bs & 15) == 0 && (reinterpret_cast<uintptr_t>(tokens) & 15) == 0;
  constexpr int64_t kClaim = 8;  // tasks per claim: keeps the shared counter cold
  while (true) {
    int64_t t0 = 0;
    if (lane == 0) t0 = static_cast<int64_t>(atomicAdd(ws + 2, static_cast<unsigned long long>(kClaim)));
    t0 = __shfl_sync(0xffffffffu, t0, 0);
    if (t0 >= tasks) break;
    const int64_t t_end = min(t0 + kClaim, tasks);
    // window-major: task t = (window w = t / n_req, request r = t % n_req), every
    // request's window w before any w+1; one division per claim, then step
    int64_t w = t0 / n_req;
    int64_t r = t0 - w * n_req - 1;
    for (int64_t t = t0; t < t_end; ++t) {
      if (++r == n_req) {
        r = 0;
        ++w;
      }
      const int64_t k0 = key_off[r];
      const int64_t nblk = key_off[r + 1] - k0;
      if (w * 32 >= nblk) continue;  // warp-uniform: request shorter than this window
      const int64_t b = w * 32 + lane;
      if (b < nblk) {
        const int64_t tb = tok_off[r] + b * bs;
        const int n = static_cast<int>(min(static_cast<int64_t>(bs), tok_off[r + 1] - tb));
        int64_t h;
        if (n == bs && x16_ok && tb + bs + 4 <= total_tok)
          h = fold_tokens_x16(tokens, tb, bs);  // any alignment: 5 aligned LDG.128 / 16 tokens
        else if (n == bs && ((bs & 3) == 0) && ((reinterpret_cast<uintptr_t>(tokens + tb) & 15) == 0))
          h = fold_tokens_vec4(tokens + tb, n);
        else
          h = fold_tokens_scalar(tokens + tb, n);
        keys[k0 + b] = h;
      }
    }
  }
  if (fold_sms >= 0) fold_requests(key_off, n_req, keys, ws);
}

struct Workspace {
  std::mutex mu;
  unsigned long long* ws[64] = {nullptr};
  int grid[64] = {0};
};

Workspace& workspace() {
  static Workspace w;
  return w;
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
  KVX_REQUIRE(dev < 64, "kvx_chain_hash_batch: device index too large");
  cudaStream_t s = as_stream(stream);
  Workspace& W = workspace();
  unsigned long long* ws;
  int grid;
  {
    std::lock_guard<std::mutex> lk(W.mu);
    if (!W.ws[dev]) {
      KVX_CUDA(cudaMalloc(reinterpret_cast<void**>(&W.ws[dev]),
                          (3 + sm_count(dev)) * sizeof(unsigned long long)));
      int per_sm = 0;
      KVX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, block_hash_fused_kernel,
                                                             kHashThreads, 0));
      W.grid[dev] = std::max(1, per_sm) * sm_count(dev);
    }
    ws = W.ws[dev];
    grid = W.grid[dev];
  }
  // ws: [0] max windows, [1] fold claims, [2] content claims, [3 + sm] per-SM CTA tickets
  KVX_CUDA(cudaMemsetAsync(ws, 0, (3 + sm_count(dev)) * sizeof(unsigned long long), s));
  block_hash_prep_kernel<<<sm_count(dev) * 4, 256, 0, s>>>(d_key_off, n_req, d_keys, ws);
  KVX_LAUNCH_CHECK("block_hash_prep_kernel");
  // SMs reserved for folding: kFoldWarps * 32 request lanes each, at most a
  // quarter of the chip (the rest of the requests are folded by producers
  // once the content tasks are exhausted).
  const int sms = sm_count(dev);
  const int64_t lanes_per_fold_sm = static_cast<int64_t>(kFoldWarps) * 32;
  int fold_sms = static_cast<int>(std::min<int64_t>(
      std::max<int64_t>(1, (n_req + lanes_per_fold_sm - 1) / lanes_per_fold_sm), sms / 4));
  if (const char* e = std::getenv("KVX_HASH_FOLD_SMS")) fold_sms = std::atoi(e);  // tuning/debug
  int bsi = static_cast<int>(bs);
  void* args[] = {const_cast<int32_t**>(&d_tokens), const_cast<int64_t**>(&d_tok_off), &n_req,
                  &bsi, const_cast<int64_t**>(&d_key_off), &d_keys, &ws, &fold_sms};
  KVX_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(block_hash_fused_kernel),
                                       dim3(grid), dim3(kHashThreads), args, 0, s));
  KVX_LAUNCH_CHECK("block_hash_fused_kernel");
  return KVX_OK;
}
