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
// content hashes are independent and ALU-throughput bound.  Two kernels:
//
// K1b halfwarp_hash_kernel (block sizes that are multiples of 16 -- every
//     configuration the bench and the reference's workloads use; described
//     at the kernel).  One CTA per SM; each half-warp owns one request at a
//     time: 15 lanes hash contents, lane 0 folds keys, contents pass through
//     shared memory, requests are claimed longest first.  Config 4 batch
//     (4,096 requests, 4.17 M blocks): 197 us.
//
// K1a block_hash_fused_kernel (any block size; KVX_HASH_KERNEL=fused forces
//     it).  One persistent, cooperatively launched kernel:
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
//   Config 4 batch: content production alone 161 us; sequential
//   produce-then-fold 373 us; this kernel 236 us.  Waiting happens only inside
//   this single cooperative launch (all CTAs co-resident).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>

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
  // key_off may be a slice of a larger batch (absolute positions)
  const int64_t first = key_off[0], total = key_off[n_req];
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = first + tid; i < total; i += stride) keys[i] = -1;
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

// ---- K1b: half-warp per request (block sizes that are multiples of 16) ------
//
// Each half-warp owns one request at a time: lane 0 folds the key chain, lanes
// 1..15 hash the contents of 15 consecutive blocks (a "round").  Every step
// all 16 lanes run ONE chain_hash in the same instruction stream -- content
// lanes on their next token, the folding lane on the next finished content --
// so the serial fold costs no extra issue slots and contents never leave the
// SM: content lanes park a finished round in shared memory, the folding lane
// consumes it during the next round (15 folds per 16-step round, which
// balances the 15 x 16 content steps).  Tokens arrive by cp.async 16-byte
// copies into a (kPrefetch + 1)-slot shared-memory ring, kPrefetch 16-step
// sub-rounds ahead (a block's 16 tokens plus up to 3 of misalignment: every
// block of a request has the same alignment because bs % 16 == 0).  The key
// chain of a 1,536-block request therefore runs at ~16/15 x one chain_hash
// latency per block with no L2 round trip in its dependency path, and the
// requests are claimed longest first (order kernel below) so the longest
// chains start at t = 0.  Compared with block_hash_fused_kernel (producer warps
// -> L2 -> polling fold lanes on reserved SMs) this removes the content
// staging traffic, the polling and the reserved SMs.
namespace hw {
#ifndef KVX_HASH_PREFETCH
#define KVX_HASH_PREFETCH 3
#endif
constexpr int kPrefetch = KVX_HASH_PREFETCH;  // sub-rounds of tokens in flight
constexpr int kSlots = kPrefetch + 1;
constexpr int kContentLanes = 15;
constexpr int kRowWords = 20;                   // 16 tokens + misalignment, 16-B rows
constexpr int kSlotWords = kContentLanes * kRowWords;
constexpr int kOrderBuckets = 2048;             // longest-first claim order, by block count
constexpr int64_t kOrderMaxReq = int64_t(1) << 22;  // larger batches claim in index order
#ifndef KVX_HASH_HW_WARPS
#define KVX_HASH_HW_WARPS 12  // warps in the one CTA per SM (3 per SM sub-partition)
#endif
constexpr int kMaxWarps = 20;  // 20 x 9.7 KB of staging fits the 227 KB opt-in
// The kernel is launched with exactly one CTA per SM: the dynamic shared
// memory request is padded past half of the SM's capacity, because with
// several small CTAs per SM the block scheduler placed them unevenly (ncu:
// 6 K .. 512 K active cycles per SM at 4 x 148 CTAs) and the SMs holding 5
// CTAs stretched the longest key chains.
constexpr size_t kMinCtaSmem = 120 * 1024;
constexpr size_t kMaxCtaSmem = 227 * 1024;

// chain_hash with the HIGH words of its four right shifts (x >> 2, >> 30,
// >> 27, >> 31) computed on the FMA pipe as mul.hi by 2^(32-k) -- one IMAD.HI
// for each SHF it replaces, so the instruction count is unchanged while the
// ALU pipe, the step's bound (23 ALU vs 8 FMA-pipe SASS per step), carries
// four fewer.  The multipliers arrive in registers (a kernel argument) so
// ptxas cannot fold them back into shifts.  Bit-identical to chain_hash.
struct HiShift {
  uint32_t m2, m30, m27, m31;  // 2^30, 2^2, 2^5, 2^1
};
__device__ __forceinline__ uint64_t shr64_fma(uint64_t x, int k, uint32_t m) {
  const uint32_t lo = static_cast<uint32_t>(x), hi = static_cast<uint32_t>(x >> 32);
  const uint32_t nlo = __funnelshift_r(lo, hi, k);
  const uint32_t nhi = __umulhi(hi, m);
  return (static_cast<uint64_t>(nhi) << 32) | nlo;
}
template <bool kFma>
__device__ __forceinline__ int64_t chain_hash_hw(int64_t prev, uint64_t content, const HiShift& k) {
  if (!kFma) return chain_hash(prev, content);
  uint64_t x = static_cast<uint64_t>(prev) + 0x9E3779B97F4A7C15ull;
  x ^= content + 0x9E3779B97F4A7C15ull + (x << 6) + shr64_fma(x, 2, k.m2);
  x ^= shr64_fma(x, 30, k.m30);
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= shr64_fma(x, 27, k.m27);
  x *= 0x94D049BB133111EBull;
  x ^= shr64_fma(x, 31, k.m31);
  return static_cast<int64_t>(x & 0x7FFFFFFFFFFFFFFFull);
}

// One 16-step sub-round of one round of one request, written by the
// prefetching side when it issues the tokens, read by the hashing side.
struct alignas(16) SubDesc {
  int32_t rem0;   // tokens from block 0's position in this sub-round to the request end
  int32_t nb;     // blocks in the round (0: no work)
  int32_t flags;  // 1: first sub-round of the block, 2: last (round done), 4: round 0 of the
                  // request, 8: last round of the request
  int32_t m;      // token misalignment of the request (all its blocks share it: bs % 16 == 0)
  int64_t kb;     // key index of block 0 of the round
  int64_t r;      // request index
};

// kvx_hash_match_batch runs the hash with `enabled` set: the keys were
// preset to -1 (no key is negative: chain_hash masks the sign bit), and a
// match kernel beside the hash reads each key once it is no longer -1.  No
// fence or extra store on the hash's side (a release per round would wait for
// the round's in-flight token prefetches).
struct Publish {
  int enabled;
};

// Staging of one request stream (one chain per lane) of one half-warp.
struct HalfSmem {
  uint32_t tok[kSlots][kSlotWords];  // [slot][block row][word]
  SubDesc desc[kSlots];
  uint32_t clo[16], chi[16];         // finished contents of the last round, split words
};

template <int V>
struct WarpSmem {
  HalfSmem h[V][2];   // [chain][half]
  uint32_t zero[16];  // the high word of a token
};

// Prefetching cursor of one half-warp.  Request fields are uniform over the
// half; `a` / `prem` are the lane's own block (lane j copies block j).
struct Cursor {
  const int32_t* a;  // 16-B aligned token pointer of this lane's block at sub-round u
  int32_t prem;      // tokens from a to the request end
  int32_t ntok, nblk, k, u, m;
  int64_t kb0;
  int64_t r;  // request index
  bool live;
};

// Claim requests (index into the longest-first order) until a non-empty one
// or the batch is exhausted.  Called by all 32 lanes; halves claim independently.
// `first` (uniform over the half): a pre-assigned first claim, or ~0 -- then
// the shared counter hands out indices from `base` on.
__device__ __forceinline__ void claim(Cursor& c, bool need, int hl, int j, int bs,
                                      const int32_t* __restrict__ tokens,
                                      const int64_t* __restrict__ tok_off,
                                      const int64_t* __restrict__ key_off, int64_t n_req,
                                      const int32_t* __restrict__ order,
                                      unsigned long long* ctr, unsigned long long& first,
                                      unsigned long long base) {
  while (__any_sync(0xffffffffu, need)) {
    unsigned long long idx = 0;
    if (need && first != ~0ull) {
      idx = first;
      first = ~0ull;
    } else {
      if (need && hl == 0) idx = base + atomicAdd(ctr, 1ull);
      idx = __shfl_sync(0xffffffffu, idx, 0, 16);
    }
    if (need) {
      if (idx >= static_cast<unsigned long long>(n_req)) {
        c.live = false;
        need = false;
      } else {
        const int64_t r = order ? static_cast<int64_t>(order[idx]) : static_cast<int64_t>(idx);
        const int64_t kb0 = key_off[r], tb0 = tok_off[r];
        c.nblk = static_cast<int32_t>(key_off[r + 1] - kb0);
        c.ntok = static_cast<int32_t>(tok_off[r + 1] - tb0);
        c.kb0 = kb0;
        c.r = r;
        c.m = static_cast<int32_t>(tb0 & 3);
        c.k = 0;
        c.u = 0;
        const int jj = j < 0 ? 0 : j;
        c.a = tokens + (tb0 - c.m) + static_cast<int64_t>(jj) * bs;
        c.prem = c.ntok + c.m - jj * bs;
        c.live = true;
        need = c.nblk <= 0;
      }
    }
  }
}

// Token copies carry an L2 evict-first hint: the token stream is read once
// and must not displace what stays hot in L2 (the instance indices the
// prefix match probes right after the hash).
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int bytes) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;" ::"r"(dst),
               "l"(src), "r"(bytes), "l"(pol));
}

// Issue the cursor's sub-round into `slot`: lane 0 of the half writes the
// descriptor, content lane j copies its block's 16 tokens (5 aligned 16-byte
// chunks; bytes past the request end are zero-filled, never read).
__device__ __forceinline__ void issue(const Cursor& c, HalfSmem& H, int slot, int hl, int j,
                                      int bs, int nsub, const int32_t* tokens) {
  const int nb = c.live ? min(kContentLanes, c.nblk - kContentLanes * c.k) : 0;
  if (hl == 0) {
    SubDesc d;
    d.rem0 = c.ntok - kContentLanes * c.k * bs - 16 * c.u;
    d.nb = nb;
    d.flags = (c.u == 0 ? 1 : 0) | (c.u == nsub - 1 ? 2 : 0) | (c.k == 0 ? 4 : 0) |
              (kContentLanes * (c.k + 1) >= c.nblk ? 8 : 0);
    d.m = c.m;
    d.kb = c.kb0 + static_cast<int64_t>(kContentLanes) * c.k;
    d.r = c.r;
    H.desc[slot] = d;
  }
  if (j >= 0 && j < nb) {
    const uint32_t dst =
        static_cast<uint32_t>(__cvta_generic_to_shared(&H.tok[slot][j * kRowWords]));
    if (c.prem >= 20) {
#pragma unroll
      for (int q = 0; q < 5; ++q) cp_async16(dst + 16 * q, c.a + 4 * q, 16);
    } else {
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        const int bytes = max(0, min(4, c.prem - 4 * q)) * 4;
        cp_async16(dst + 16 * q, bytes ? static_cast<const void*>(c.a + 4 * q)
                                       : static_cast<const void*>(tokens), bytes);
      }
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");  // uniform group count per lane
}

__device__ __forceinline__ bool step_cursor(Cursor& c, int bs, int nsub) {
  if (!c.live) return false;
  if (++c.u < nsub) {
    c.a += 16;
    c.prem -= 16;
    return false;
  }
  c.u = 0;
  ++c.k;
  c.a += 14 * bs + 16;
  c.prem -= 14 * bs + 16;
  return kContentLanes * c.k >= c.nblk;
}

__global__ void __launch_bounds__(1024) order_kernel(const int64_t* __restrict__ key_off,
                                                     int64_t n_req, int32_t* __restrict__ order,
                                                     unsigned long long* ctr) {
  __shared__ int hist[kOrderBuckets];
  __shared__ int part[1024];
  const int t = threadIdx.x;
  asm volatile("griddepcontrol.launch_dependents;");  // the hash grid may get resident now
  for (int b = t; b < kOrderBuckets; b += blockDim.x) hist[b] = 0;
  if (t == 0) *ctr = 0;
  __syncthreads();
  auto bucket = [&](int64_t r) {
    const int64_t n = key_off[r + 1] - key_off[r];
    return kOrderBuckets - 1 -
           static_cast<int>(min(max(n, int64_t(0)), static_cast<int64_t>(kOrderBuckets - 1)));
  };
  for (int64_t r = t; r < n_req; r += blockDim.x) atomicAdd(&hist[bucket(r)], 1);
  __syncthreads();
  // exclusive scan of hist (2 buckets per thread)
  const int per = kOrderBuckets / 1024;
  int s = 0;
  for (int i = 0; i < per; ++i) s += hist[t * per + i];
  part[t] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int v = t >= o ? part[t - o] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  int run = part[t] - s;
  for (int i = 0; i < per; ++i) {
    const int c = hist[t * per + i];
    hist[t * per + i] = run;
    run += c;
  }
  __syncthreads();
  for (int64_t r = t; r < n_req; r += blockDim.x)
    order[atomicAdd(&hist[bucket(r)], 1)] = static_cast<int32_t>(r);
}

// V independent request streams per half-warp (every lane advances V chains
// per step).  V = 1 is the shipped kernel: V = 2 was slower on the Config 4
// batch at every width, also with a compact (select-only, unroll 4) step loop
// (profiles/r01/hash_halfwarp.md).
template <int V, bool kFma = false>
__global__ void __launch_bounds__(kMaxWarps * 32, 1) halfwarp_hash_kernel(
    const int32_t* __restrict__ tokens, const int64_t* __restrict__ tok_off, int64_t n_req,
    int bs, const int64_t* __restrict__ key_off, int64_t* __restrict__ keys,
    const int32_t* __restrict__ order, unsigned long long* ctr, int prio, HiShift hs) {
  extern __shared__ __align__(16) unsigned char hw_smem_raw[];
  WarpSmem<V>& S = reinterpret_cast<WarpSmem<V>*>(hw_smem_raw)[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const int half = lane >> 4;
  const int hl = lane & 15;        // lane within the half-warp; 0 folds
  const int j = hl - 1;            // content block row (-1 on the folding lane)
  const bool folder = hl == 0;
  const int nsub = bs >> 4;
  if (lane < 16) S.zero[lane] = 0;
  // launched programmatically dependent on the order kernel (when there is
  // one): wait for its order / counter before reading anything
  asm volatile("griddepcontrol.wait;" ::: "memory");

  // First claims by warp priority: the warp scheduler issues the highest
  // ready warp id first, so the highest warp of every SM sub-partition takes
  // the longest requests (their key chains set the batch time and then run
  // at their dependency latency), the next warps the next longest; later
  // claims come from the shared counter, longest first.  prio == 0: every
  // claim from the counter (the r01 behaviour).
  const int nwarps = static_cast<int>(blockDim.x >> 5), warp = static_cast<int>(threadIdx.x >> 5);
  const unsigned long long halves = 2ull * V * nwarps * gridDim.x;
  unsigned long long first[V];
#pragma unroll
  for (int v = 0; v < V; ++v)
    first[v] = prio ? ((static_cast<unsigned long long>(nwarps - 1 - warp) * gridDim.x +
                        blockIdx.x) * 2 + half) * V + v
                    : ~0ull;
  const unsigned long long base = prio ? halves : 0ull;

  Cursor P[V];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    P[v].live = false;
    P[v].a = tokens;
    P[v].prem = P[v].ntok = P[v].nblk = P[v].k = P[v].u = P[v].m = 0;
    P[v].kb0 = 0;
    claim(P[v], true, hl, j, bs, tokens, tok_off, key_off, n_req, order, ctr, first[v], base);
  }
#pragma unroll 1
  for (int i = 0; i < kPrefetch; ++i) {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      issue(P[v], S.h[v][half], i, hl, j, bs, nsub, tokens);
      claim(P[v], step_cursor(P[v], bs, nsub), hl, j, bs, tokens, tok_off, key_off, n_req, order,
            ctr, first[v], base);
    }
  }

  int64_t h[V];
  int fn[V], freset[V];   // blocks to fold in this sub-round, chain restart
  int64_t fkb[V];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    h[v] = 0;
    fn[v] = freset[v] = 0;
    fkb[v] = 0;
  }
#pragma unroll 1
  for (uint32_t it = 0;; ++it) {
    // issue sub-round it + kPrefetch into the slot sub-round it - 1 used
#pragma unroll
    for (int v = 0; v < V; ++v) {
      issue(P[v], S.h[v][half], (it + kPrefetch) % kSlots, hl, j, bs, nsub, tokens);
      claim(P[v], step_cursor(P[v], bs, nsub), hl, j, bs, tokens, tok_off, key_off, n_req, order,
            ctr, first[v], base);
    }
    // V commit groups per sub-round: wait until only kPrefetch sub-rounds are pending
    asm volatile("cp.async.wait_group %0;" ::"n"(kPrefetch * V) : "memory");
    __syncwarp();
    const int slot = it % kSlots;
    SubDesc d[V];
    bool idle = true;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      d[v] = S.h[v][half].desc[slot];
      idle = idle && d[v].nb == 0 && fn[v] == 0;
    }
    if (__all_sync(0xffffffffu, idle)) break;

    const uint32_t* lo[V];
    const uint32_t* hi[V];
    int lim[V];
    bool fast = true;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      HalfSmem& H = S.h[v][half];
      if (folder) {
        lo[v] = H.clo;
        hi[v] = H.chi;
        lim[v] = fn[v];
        if (freset[v] && fn[v] > 0) h[v] = 0;
        fast = fast && (fn[v] == 0 || fn[v] == kContentLanes);
      } else {
        lo[v] = &H.tok[slot][j * kRowWords + d[v].m];
        hi[v] = S.zero;
        // rows past the round: don't care
        lim[v] = j < d[v].nb ? max(0, min(16, d[v].rem0 - j * bs)) : 16;
        if (d[v].flags & 1) h[v] = 0;
        fast = fast && lim[v] == 16;
      }
    }
    if (__all_sync(0xffffffffu, fast)) {
      // full sub-round: no per-step selects; the folding lane keeps the key
      // after its 15th fold (or its old chain value when it had nothing)
      int64_t h0[V], h14[V];
#pragma unroll
      for (int v = 0; v < V; ++v) h0[v] = h14[v] = h[v];
#pragma unroll
      for (int s = 0; s < 16; ++s) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const uint64_t in = (static_cast<uint64_t>(hi[v][s]) << 32) | lo[v][s];
          h[v] = chain_hash_hw<kFma>(h[v], in, hs);
          if (s == kContentLanes - 1) h14[v] = h[v];
          if (s < kContentLanes && folder && fn[v] > 0) keys[fkb[v] + s] = h[v];
        }
      }
      if (folder) {
#pragma unroll
        for (int v = 0; v < V; ++v) h[v] = fn[v] > 0 ? h14[v] : h0[v];
      }
    } else {
#pragma unroll
      for (int s = 0; s < 16; ++s) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const uint64_t in = (static_cast<uint64_t>(hi[v][s]) << 32) | lo[v][s];
          const int64_t hn = chain_hash_hw<kFma>(h[v], in, hs);
          const bool act = s < lim[v];
          h[v] = act ? hn : h[v];
          if (folder && fn[v] > 0 && act) keys[fkb[v] + s] = h[v];
        }
      }
    }
    __syncwarp();
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const bool round_done = d[v].nb > 0 && (d[v].flags & 2);
      if (round_done && !folder) {
        S.h[v][half].clo[j] = static_cast<uint32_t>(h[v]);
        S.h[v][half].chi[j] = static_cast<uint32_t>(static_cast<uint64_t>(h[v]) >> 32);
      }
      fn[v] = round_done ? d[v].nb : 0;
      fkb[v] = d[v].kb;
      freset[v] = d[v].flags & 4;
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}
// ---- K1b, software-pipelined control ---------------------------------------
// The same half-warp algorithm with the per-sub-round bookkeeping taken off
// the key chain's critical path.  In halfwarp_hash_kernel a lone warp runs a
// 1,536-block request at ~156 cycles per step against ~107 for the bare
// chain_hash chain: each 16-step sub-round first issues the next prefetch,
// waits, reads its descriptor, votes, branches -- in program order, before
// the first chain step.  Here iteration `it` runs the 16 chain steps of
// sub-round it with everything sub-round it+1 needs computed in the SAME
// branch-free basic block (predicated cp.async and descriptor stores,
// cursor advance by selects, the it+1 descriptor read and its two votes), so
// the instruction scheduler hides that work in the chain's idle issue slots;
// only the rare claim of a new request stays behind a branch.
__device__ __forceinline__ void cp_async16_pred(uint32_t dst, const void* src, int bytes, bool on) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " @p cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;\n}\n" ::"r"(dst),
      "l"(src), "r"(bytes), "l"(pol), "r"(static_cast<int>(on)));
}

// Issue of the cursor's sub-round into `slot` (see issue()): the descriptor
// and the rows of full blocks without branches (five 16-byte copies each);
// a row that reaches past its request's last token -- the last round of a
// request only -- takes the zero-filling copies behind one warp-uniform,
// rarely taken branch, so the common path carries no per-chunk size math.
__device__ __forceinline__ void issue_p(const Cursor& c, HalfSmem& H, int slot, int hl, int j,
                                        int bs, int nsub, const int32_t* tokens) {
  const int nb = c.live ? min(kContentLanes, c.nblk - kContentLanes * c.k) : 0;
  SubDesc d;
  d.rem0 = c.ntok - kContentLanes * c.k * bs - 16 * c.u;
  d.nb = nb;
  d.flags = (c.u == 0 ? 1 : 0) | (c.u == nsub - 1 ? 2 : 0) | (c.k == 0 ? 4 : 0) |
            (kContentLanes * (c.k + 1) >= c.nblk ? 8 : 0);
  d.m = c.m;
  d.kb = c.kb0 + static_cast<int64_t>(kContentLanes) * c.k;
  d.r = c.r;
  if (hl == 0) H.desc[slot] = d;  // predicated stores
  const bool copy = j >= 0 && j < nb;
  const bool full = c.prem >= 20;
  const int row = copy ? j : 0;
  const uint32_t dst =
      static_cast<uint32_t>(__cvta_generic_to_shared(&H.tok[slot][row * kRowWords]));
#pragma unroll
  for (int q = 0; q < 5; ++q) cp_async16_pred(dst + 16 * q, c.a + 4 * q, 16, copy && full);
  if (__any_sync(0xffffffffu, copy && !full)) {
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const int bytes = max(0, min(4, c.prem - 4 * q)) * 4;
      cp_async16_pred(dst + 16 * q, bytes ? static_cast<const void*>(c.a + 4 * q)
                                          : static_cast<const void*>(tokens),
                      bytes, copy && !full);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// The r02 first cut of issue_p (every chunk's size computed every sub-round);
// kept for the measurement knob KVX_HASH_ISSUE=0.
__device__ __forceinline__ void issue_p0(const Cursor& c, HalfSmem& H, int slot, int hl, int j,
                                         int bs, int nsub, const int32_t* tokens) {
  const int nb = c.live ? min(kContentLanes, c.nblk - kContentLanes * c.k) : 0;
  SubDesc d;
  d.rem0 = c.ntok - kContentLanes * c.k * bs - 16 * c.u;
  d.nb = nb;
  d.flags = (c.u == 0 ? 1 : 0) | (c.u == nsub - 1 ? 2 : 0) | (c.k == 0 ? 4 : 0) |
            (kContentLanes * (c.k + 1) >= c.nblk ? 8 : 0);
  d.m = c.m;
  d.kb = c.kb0 + static_cast<int64_t>(kContentLanes) * c.k;
  d.r = c.r;
  if (hl == 0) H.desc[slot] = d;  // predicated stores
  const bool copy = j >= 0 && j < nb;
  const int row = copy ? j : 0;
  const uint32_t dst =
      static_cast<uint32_t>(__cvta_generic_to_shared(&H.tok[slot][row * kRowWords]));
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    const int bytes = max(0, min(4, c.prem - 4 * q)) * 4;
    cp_async16_pred(dst + 16 * q, bytes ? static_cast<const void*>(c.a + 4 * q)
                                        : static_cast<const void*>(tokens),
                    bytes, copy);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// Branch-free cursor advance (see step_cursor); true when the request's
// last round was issued (a new request must be claimed).
__device__ __forceinline__ bool step_cursor_p(Cursor& c, int bs, int nsub) {
  const bool live = c.live;
  const int u1 = c.u + 1;
  const bool wrap = u1 >= nsub;
  const int adv = live ? (wrap ? 14 * bs + 16 : 16) : 0;
  c.u = live ? (wrap ? 0 : u1) : c.u;
  c.k += (live && wrap) ? 1 : 0;
  c.a += adv;
  c.prem -= adv;
  return live && wrap && kContentLanes * c.k >= c.nblk;
}

// What the lanes of a half need to run one sub-round.
struct Ctl {
  const uint32_t* lo;
  const uint32_t* hi;
  int lim;        // steps that count for this lane (16 on the fast path)
  int nb, flags;  // of the sub-round's descriptor
  int64_t kb, r;
  bool fast, idle;
};

__device__ __forceinline__ Ctl make_ctl(HalfSmem& H, const uint32_t* zero, int slot, bool folder,
                                        int j, int bs, int fn_next) {
  const SubDesc d = H.desc[slot];
  Ctl c;
  c.nb = d.nb;
  c.flags = d.flags;
  c.kb = d.kb;
  c.r = d.r;
  if (folder) {
    c.lo = H.clo;
    c.hi = H.chi;
    c.lim = fn_next;
  } else {
    c.lo = &H.tok[slot][j * kRowWords + d.m];
    c.hi = zero;
    c.lim = j < d.nb ? max(0, min(16, d.rem0 - j * bs)) : 16;
  }
  const bool fast = folder ? (fn_next == 0 || fn_next == kContentLanes) : c.lim == 16;
  c.fast = __all_sync(0xffffffffu, fast);
  c.idle = __all_sync(0xffffffffu, d.nb == 0 && fn_next == 0);
  return c;
}

template <bool kLazyIssue>
__global__ void __launch_bounds__(kMaxWarps * 32, 1) halfwarp_hash_kernel_p(
    const int32_t* __restrict__ tokens, const int64_t* __restrict__ tok_off, int64_t n_req,
    int bs, const int64_t* __restrict__ key_off, int64_t* __restrict__ keys,
    const int32_t* __restrict__ order, unsigned long long* ctr, int prio, Publish pubv) {
  (void)pubv;
  extern __shared__ __align__(16) unsigned char hw_smem_raw[];
  WarpSmem<1>& S = reinterpret_cast<WarpSmem<1>*>(hw_smem_raw)[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const int half = lane >> 4;
  const int hl = lane & 15;
  const int j = hl - 1;
  const bool folder = hl == 0;
  const int nsub = bs >> 4;
  HalfSmem& H = S.h[0][half];
  if (lane < 16) S.zero[lane] = 0;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // a consumer launched programmatically dependent on this kernel (the prefix
  // match of kvx_hash_match_batch) may become resident now: every CTA of this
  // grid already is, so the consumer's waits on the queue always progress
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  const int nwarps = static_cast<int>(blockDim.x >> 5), warp = static_cast<int>(threadIdx.x >> 5);
  const unsigned long long halves = 2ull * nwarps * gridDim.x;
  unsigned long long first =
      prio ? (static_cast<unsigned long long>(nwarps - 1 - warp) * gridDim.x + blockIdx.x) * 2 + half
           : ~0ull;
  const unsigned long long base = prio ? halves : 0ull;

  Cursor P;
  P.live = false;
  P.a = tokens;
  P.prem = P.ntok = P.nblk = P.k = P.u = P.m = 0;
  P.kb0 = 0;
  P.r = 0;
  claim(P, true, hl, j, bs, tokens, tok_off, key_off, n_req, order, ctr, first, base);
#pragma unroll 1
  for (int i = 0; i < kPrefetch; ++i) {
    if (kLazyIssue) issue_p(P, H, i, hl, j, bs, nsub, tokens);
    else issue_p0(P, H, i, hl, j, bs, nsub, tokens);
    const bool need = step_cursor_p(P, bs, nsub);
    if (__any_sync(0xffffffffu, need))
      claim(P, need, hl, j, bs, tokens, tok_off, key_off, n_req, order, ctr, first, base);
  }
  // sub-round 0's tokens and control
  asm volatile("cp.async.wait_group %0;" ::"n"(kPrefetch - 1) : "memory");
  __syncwarp();
  int fn = 0, freset = 0;  // folds of the current sub-round (the previous round's blocks)
  int64_t fkb = 0;
  Ctl c = make_ctl(H, S.zero, 0, folder, j, bs, 0);
  int64_t h = 0;
#pragma unroll 1
  for (uint32_t it = 0;; ++it) {
    if (c.idle) break;
    if (folder) {
      if (freset && fn > 0) h = 0;
    } else if (c.flags & 1) {
      h = 0;
    }
    // the folder's work in sub-round it+1: the blocks of the round finishing now
    const bool round_done = c.nb > 0 && (c.flags & 2);
    const int fn_next = round_done ? c.nb : 0;
    const int nslot = static_cast<int>((it + 1) % kSlots);
    Ctl cn;
    bool need;
    if (c.fast) {
      int64_t h0 = h, h14 = h;
#pragma unroll
      for (int s = 0; s < 16; ++s) {
        const uint64_t in = (static_cast<uint64_t>(c.hi[s]) << 32) | c.lo[s];
        h = chain_hash(h, in);
        if (s == kContentLanes - 1) h14 = h;
        if (s < kContentLanes && folder && fn > 0) keys[fkb + s] = h;
      }
      if (folder) h = fn > 0 ? h14 : h0;
      // next sub-round's work, scheduled into the chain's idle issue slots
      if (kLazyIssue) issue_p(P, H, static_cast<int>((it + kPrefetch) % kSlots), hl, j, bs, nsub, tokens);
      else issue_p0(P, H, static_cast<int>((it + kPrefetch) % kSlots), hl, j, bs, nsub, tokens);
      need = step_cursor_p(P, bs, nsub);
      asm volatile("cp.async.wait_group %0;" ::"n"(kPrefetch - 1) : "memory");
      cn = make_ctl(H, S.zero, nslot, folder, j, bs, fn_next);
    } else {
#pragma unroll
      for (int s = 0; s < 16; ++s) {
        const uint64_t in = (static_cast<uint64_t>(c.hi[s]) << 32) | c.lo[s];
        const int64_t hn = chain_hash(h, in);
        const bool act = s < c.lim;
        h = act ? hn : h;
        if (folder && fn > 0 && act) keys[fkb + s] = h;
      }
      if (kLazyIssue) issue_p(P, H, static_cast<int>((it + kPrefetch) % kSlots), hl, j, bs, nsub, tokens);
      else issue_p0(P, H, static_cast<int>((it + kPrefetch) % kSlots), hl, j, bs, nsub, tokens);
      need = step_cursor_p(P, bs, nsub);
      asm volatile("cp.async.wait_group %0;" ::"n"(kPrefetch - 1) : "memory");
      cn = make_ctl(H, S.zero, nslot, folder, j, bs, fn_next);
    }
    // hand the finished round's contents to the folder (read next sub-round)
    if (round_done && !folder) {
      H.clo[j] = static_cast<uint32_t>(h);
      H.chi[j] = static_cast<uint32_t>(static_cast<uint64_t>(h) >> 32);
    }

    fn = fn_next;
    fkb = c.kb;
    freset = c.flags & 4;
    __syncwarp();
    if (__any_sync(0xffffffffu, need))
      claim(P, need, hl, j, bs, tokens, tok_off, key_off, n_req, order, ctr, first, base);
    c = cn;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

}  // namespace hw

// Claim counters and the longest-first order are per (device, stream):
// batches on different streams of one device run concurrently without
// sharing them, batches on one stream are ordered by the stream.
struct Scratch {
  unsigned long long* ws = nullptr;  // 3 + SM count counters
  int32_t* order = nullptr;
  int64_t order_cap = 0;
};

struct Workspace {
  std::mutex mu;
  std::map<std::pair<int, void*>, Scratch> scratch;
  int grid[64] = {0};
  bool hw_attr[64] = {false};
};

Workspace& workspace() {
  static Workspace w;
  return w;
}

}  // namespace
}  // namespace kvx

namespace kvx {
namespace {
// key_off = exclusive scan of ceil((tok_off[r+1] - tok_off[r]) / bs): one CTA,
// 1024 threads x 8 requests per pass, warp-shuffle scans, a running carry
// (4,096 requests = one pass; the launch is latency, not bandwidth, bound).
constexpr int kScanThreads = 1024, kScanPer = 8;
__global__ void __launch_bounds__(kScanThreads) key_offsets_kernel(
    const int64_t* __restrict__ tok_off, int64_t n_req, int64_t bs, int64_t* __restrict__ key_off) {
  __shared__ int64_t warp_tot[kScanThreads / 32];
  __shared__ int64_t carry_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (int64_t base = 0; base < n_req; base += int64_t{kScanThreads} * kScanPer) {
    int64_t v[kScanPer];
    int64_t mine = 0;
    const int64_t r0 = base + static_cast<int64_t>(threadIdx.x) * kScanPer;
#pragma unroll
    for (int j = 0; j < kScanPer; ++j) {
      const int64_t r = r0 + j;
      v[j] = r < n_req ? (tok_off[r + 1] - tok_off[r] + bs - 1) / bs : 0;
      mine += v[j];
    }
    int64_t incl = mine;  // inclusive scan over the warp
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int64_t w = warp_tot[lane], wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t t = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += t;
      }
      warp_tot[lane] = wi - w;  // exclusive prefix of the warps
    }
    __syncthreads();
    int64_t run = carry_s + warp_tot[warp] + incl - mine;
#pragma unroll
    for (int j = 0; j < kScanPer; ++j) {
      const int64_t r = r0 + j;
      if (r < n_req) key_off[r] = run;
      run += v[j];
    }
    __syncthreads();
    if (threadIdx.x == kScanThreads - 1) carry_s = run;  // last thread holds the pass total
    __syncthreads();
  }
  if (threadIdx.x == 0) key_off[n_req] = carry_s;
}
}  // namespace
}  // namespace kvx

namespace kvx {
namespace {
// keys[key_off[0] .. key_off[n_req]) = -1 (the batch's key range, read on the device).
__global__ void __launch_bounds__(256) keys_unset_kernel(const int64_t* __restrict__ key_off,
                                                         int64_t n_req, int64_t* keys) {
  const int64_t first = key_off[0], last = key_off[n_req];
  for (int64_t i = first + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < last;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    keys[i] = -1;
}

}  // namespace

// Requests in decreasing block count (the hash's counting sort), for kernels
// that schedule long requests first (the prefix match); ws: one u64 of scratch.
int order_by_length(const int64_t* d_key_off, int64_t n_req, int32_t* d_order,
                    unsigned long long* d_ws, cudaStream_t s) {
  KVX_REQUIRE(n_req <= hw::kOrderMaxReq, "order_by_length: batch too large");
  hw::order_kernel<<<1, 1024, 0, s>>>(d_key_off, n_req, d_order, d_ws);
  KVX_LAUNCH_CHECK("order_kernel");
  return KVX_OK;
}
}  // namespace kvx

using namespace kvx;

extern "C" int kvx_key_offsets(const int64_t* d_tok_off, int64_t n_req, int64_t bs,
                               int64_t* d_key_off, void* stream) {
  KVX_REQUIRE(n_req >= 0 && bs >= 1, "kvx_key_offsets: bad n_req / block size");
  KVX_REQUIRE(d_tok_off && d_key_off, "kvx_key_offsets: NULL array");
  key_offsets_kernel<<<1, kScanThreads, 0, as_stream(stream)>>>(d_tok_off, n_req, bs, d_key_off);
  KVX_LAUNCH_CHECK("key_offsets_kernel");
  return KVX_OK;
}

namespace {
// The block hash; with pub.queue set (half-warp kernel only) every request is
// appended to the completion queue once its keys are stored.  *published
// reports whether the launched kernel publishes.
int hash_launch(const int32_t* d_tokens, const int64_t* d_tok_off, int64_t n_req, int64_t bs,
                const int64_t* d_key_off, int64_t* d_keys, void* stream, hw::Publish pub,
                bool* published, const int32_t** order_used = nullptr);
}  // namespace

extern "C" int kvx_chain_hash_batch(const int32_t* d_tokens, const int64_t* d_tok_off,
                                    int64_t n_req, int64_t bs, const int64_t* d_key_off,
                                    int64_t* d_keys, void* stream) {
  bool published = false;
  return hash_launch(d_tokens, d_tok_off, n_req, bs, d_key_off, d_keys, stream,
                     hw::Publish{0}, &published);
}

namespace {
int hash_launch(const int32_t* d_tokens, const int64_t* d_tok_off, int64_t n_req, int64_t bs,
                const int64_t* d_key_off, int64_t* d_keys, void* stream, hw::Publish pub,
                bool* published, const int32_t** order_used) {
  *published = false;
  if (order_used) *order_used = nullptr;
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
  std::lock_guard<std::mutex> lk(W.mu);  // host bookkeeping only; launches are async
  Scratch& X = W.scratch[{dev, stream}];
  if (!X.ws)
    KVX_CUDA(cudaMalloc(reinterpret_cast<void**>(&X.ws),
                        (3 + sm_count(dev)) * sizeof(unsigned long long)));
  if (!W.grid[dev]) {
    int per_sm = 0;
    KVX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, block_hash_fused_kernel,
                                                           kHashThreads, 0));
    W.grid[dev] = std::max(1, per_sm) * sm_count(dev);
  }
  ws = X.ws;
  grid = W.grid[dev];
  // Block sizes that are multiples of 16 (every configuration the bench and the
  // reference's workloads use): the half-warp kernel.  KVX_HASH_KERNEL=fused
  // selects the producer/fold kernel for comparison.
  const char* kern = std::getenv("KVX_HASH_KERNEL");
  const bool use_hw = (bs % 16) == 0 && (reinterpret_cast<uintptr_t>(d_tokens) & 15) == 0 &&
                      !(kern && std::strcmp(kern, "fused") == 0);
  if (use_hw) {
    int32_t* order = nullptr;
    int warps = KVX_HASH_HW_WARPS;
    if (const char* e = std::getenv("KVX_HASH_HW_WARPS")) warps = std::atoi(e);  // tuning
    warps = std::max(1, std::min(warps, hw::kMaxWarps));
    const size_t per_warp = sizeof(hw::WarpSmem<1>);
    warps = std::min<int>(warps, static_cast<int>(hw::kMaxCtaSmem / per_warp));
    const size_t smem = std::max(hw::kMinCtaSmem, warps * per_warp);
    int64_t order_max = hw::kOrderMaxReq;
    if (const char* e = std::getenv("KVX_HASH_ORDER_MAX")) order_max = std::atoll(e);  // tests
    if (n_req <= order_max && X.order_cap < n_req) {
      if (X.order) KVX_CUDA(cudaFree(X.order));  // cudaFree waits for the device
      X.order = nullptr;
      X.order_cap = 0;
      const int64_t cap = std::max<int64_t>(n_req, 4096);
      KVX_CUDA(cudaMalloc(reinterpret_cast<void**>(&X.order), cap * sizeof(int32_t)));
      X.order_cap = cap;
    }
    if (n_req <= order_max) order = X.order;
    if (!W.hw_attr[dev]) {
      KVX_CUDA(cudaFuncSetAttribute(hw::halfwarp_hash_kernel<1, false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(hw::kMaxCtaSmem)));
      KVX_CUDA(cudaFuncSetAttribute(hw::halfwarp_hash_kernel<1, true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(hw::kMaxCtaSmem)));
      KVX_CUDA(cudaFuncSetAttribute(hw::halfwarp_hash_kernel_p<true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(hw::kMaxCtaSmem)));
      KVX_CUDA(cudaFuncSetAttribute(hw::halfwarp_hash_kernel_p<false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(hw::kMaxCtaSmem)));
      W.hw_attr[dev] = true;
    }
    if (order) {
      hw::order_kernel<<<1, 1024, 0, s>>>(d_key_off, n_req, order, ws + 1);  // also zeroes ws[1]
      KVX_LAUNCH_CHECK("hash order_kernel");
    } else {
      KVX_CUDA(cudaMemsetAsync(ws + 1, 0, sizeof(unsigned long long), s));
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sm_count(dev));
    cfg.blockDim = dim3(warps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    static const bool pdl = [] {
      const char* e = std::getenv("KVX_HASH_PDL");
      return !(e && e[0] == '0');
    }();
    cfg.numAttrs = (order && pdl) ? 1 : 0;  // PDL only behind our own order kernel
    const int bsi = static_cast<int>(bs);
    unsigned long long* ctr = ws + 1;
    static const int prio = [] {
      const char* e = std::getenv("KVX_HASH_PRIO");  // measurement knob: 0 = counter-only claims
      return e ? std::atoi(e) : 1;
    }();
    static const bool fma_shifts = [] {
      const char* e = std::getenv("KVX_HASH_FMA");  // measurement knob: high-word shifts on FMA
      return e && e[0] == '1';
    }();
    const hw::HiShift hs{1u << 30, 1u << 2, 1u << 5, 1u << 1};
    static const int pipelined = [] {
      const char* e = std::getenv("KVX_HASH_PIPE");  // 0: the r01 loop (measurement knob)
      return e ? std::atoi(e) : 1;
    }();
    static const bool lazy_issue = [] {
      const char* e = std::getenv("KVX_HASH_ISSUE");  // 0: per-chunk sizes every sub-round
      return !(e && e[0] == '0');
    }();
    if (pipelined) {
      KVX_CUDA(cudaLaunchKernelEx(&cfg,
                                  lazy_issue ? hw::halfwarp_hash_kernel_p<true>
                                             : hw::halfwarp_hash_kernel_p<false>,
                                  d_tokens, d_tok_off, n_req, bsi, d_key_off, d_keys,
                                  static_cast<const int32_t*>(order), ctr, order ? prio : 0, pub));
      *published = pub.enabled != 0;
      if (order_used) *order_used = order;
    } else {
      KVX_CUDA(cudaLaunchKernelEx(&cfg,
                                  fma_shifts ? hw::halfwarp_hash_kernel<1, true>
                                             : hw::halfwarp_hash_kernel<1, false>,
                                  d_tokens, d_tok_off, n_req, bsi, d_key_off, d_keys,
                                  static_cast<const int32_t*>(order), ctr, order ? prio : 0, hs));
    }
    KVX_LAUNCH_CHECK("halfwarp_hash_kernel");
    return KVX_OK;
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

// The follower's claim counter per (device, stream).
struct QueueScratch {
  unsigned long long* ctr = nullptr;
};
std::mutex g_queue_mu;
std::map<std::pair<int, void*>, QueueScratch> g_queues;
}  // namespace

// Stage 1 in one stream-ordered call: the block hash, and the prefix match of
// each request following the hash's key production window by window (a
// match kernel resident beside the hash takes the requests in the hash's
// longest-first order and reads a window's keys once none is still the -1
// they were preset to).  A prefix match ends at the first miss, typically
// long before the request's last key exists, so the match of the batch hides
// under the hash instead of following it.  Results are those of kvx_chain_hash_batch followed by
// kvx_match_prefix_batch; block sizes the half-warp kernel does not take run
// exactly that sequence.
extern "C" int kvx_hash_match_batch(const int32_t* d_tokens, const int64_t* d_tok_off,
                                    int64_t n_req, int64_t bs, const int64_t* d_key_off,
                                    int64_t* d_keys, const kvx_index* const* idx,
                                    const int32_t* inst_ids, int64_t n_inst, int64_t* d_len_out,
                                    int64_t* d_best_len, int32_t* d_best_id, void* stream) {
  KVX_REQUIRE(n_inst >= 1, "find_best_prefix_match: empty prefill pool");
  KVX_REQUIRE(n_inst <= KVX_MAX_INSTANCES, "kvx_hash_match_batch: too many instances");
  KVX_REQUIRE(idx != nullptr && inst_ids != nullptr, "kvx_hash_match_batch: NULL instances");
  KVX_REQUIRE(n_req >= 0, "kvx_hash_match_batch: n_req must be >= 0");
  KVX_REQUIRE((d_best_len == nullptr) == (d_best_id == nullptr),
              "kvx_hash_match_batch: best_len and best_id go together");
  if (n_req == 0) return KVX_OK;
  KVX_REQUIRE(d_tok_off && d_key_off && d_keys, "kvx_hash_match_batch: NULL array");
  int dev = 0;
  KVX_CUDA(cudaGetDevice(&dev));
  cudaStream_t s = as_stream(stream);
  QueueScratch* q = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_queue_mu);
    q = &g_queues[{dev, stream}];
    if (!q->ctr) KVX_CUDA(cudaMalloc(reinterpret_cast<void**>(&q->ctr), 64));
  }
  KVX_CUDA(cudaMemsetAsync(q->ctr, 0, sizeof(unsigned long long), s));
  // every key -1 until the hash stores it (the follower's readiness test)
  keys_unset_kernel<<<sm_count(dev) * 4, 256, 0, s>>>(d_key_off, n_req, d_keys);
  KVX_LAUNCH_CHECK("keys_unset_kernel");
  if (d_best_len && n_inst > 1)  // the packed atomicMax words start at 0
    KVX_CUDA(cudaMemsetAsync(d_best_len, 0, sizeof(int64_t) * n_req, s));
  bool published = false;
  const int32_t* order = nullptr;
  int rc = hash_launch(d_tokens, d_tok_off, n_req, bs, d_key_off, d_keys, stream,
                       hw::Publish{1}, &published, &order);
  if (rc) return rc;
  if (!published)  // the producer / fold kernel (bs % 16 != 0): hash, then match
    return kvx_match_prefix_batch(idx, inst_ids, n_inst, d_keys, d_key_off, n_req, d_len_out,
                                  d_best_len, d_best_id, stream);
  rc = match_follow_launch(idx, inst_ids, n_inst, d_keys, d_key_off, n_req, d_len_out,
                           d_best_len, d_best_id, order, q->ctr, stream);
  if (rc) return rc;
  if (d_best_len && n_inst > 1)
    return kvx_best_unpack(reinterpret_cast<const uint64_t*>(d_best_len), n_req, d_best_len,
                           d_best_id, stream);
  return KVX_OK;
}

namespace kvx {
// The hash of kvx_hash_match_batch (keys preset to -1 by the caller; a match
// kernel may follow them) for other callers: request-sharded stage 1
// (kvx_xmatch_hash_match).  *published: the half-warp kernel ran (bs % 16 ==
// 0, 16-byte aligned tokens); otherwise a kernel that cannot be followed ran.
int hash_publish_launch(const int32_t* d_tokens, const int64_t* d_tok_off, int64_t n_req,
                        int64_t bs, const int64_t* d_key_off, int64_t* d_keys, void* stream,
                        bool* published) {
  return ::hash_launch(d_tokens, d_tok_off, n_req, bs, d_key_off, d_keys, stream, hw::Publish{1},
                       published);
}
}  // namespace kvx
