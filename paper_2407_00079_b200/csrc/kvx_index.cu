// kvx_index.cu -- the block index (residency side of the block manager) and
// K2, the batched prefix-match query (stage 1b).
//
// Reference semantics:
//   residency      CachePool::contains / resident_ map  (proj/include/kvcsim/kvcache.hpp:74,98)
//   match_prefix   largest k with blocks[0..k) resident, stops at the FIRST
//                  miss even if later blocks are resident (proj/src/kvcache.cpp:150-154)
//   best match     max over instances; ties -> lowest instance id; first
//                  instance seeds (proj/src/conductor.cpp:57-73)
//
// Table: open addressing, linear probing, power-of-two slots, structure of
// arrays (keys[] and values[] separate) so a match probe touches only the
// 8-byte key array -- 4 keys per 32-byte sector.  Slot = mix64(key) & mask.
// Erase writes a tombstone; tombstones are dropped by a rebuild that the host
// triggers from an upper bound on occupied slots (no per-call sync).
//
// Match mapping: one warp per (request, instance) task.  Each lane probes two
// query keys per iteration (64 keys per warp step, two independent probe
// chains per lane in flight); __ballot_sync over "miss" and __ffs give the
// first miss, so the warp exits at the first window containing a miss.  The
// per-request argmax over instances is one atomicMax per task on a packed
// (len << 32 | ~id) word, which reproduces the lowest-id tie-break.
#include <algorithm>
#include <cstring>

#include "kvx_common.cuh"

namespace kvx {
namespace {

constexpr double kMaxLoad = 0.70;     // occupied (live + tombstones) / slots
constexpr double kTargetLoad = 0.40;  // after a rebuild

struct Counters {
  unsigned long long live;
  unsigned long long used;      // live + tombstones
  unsigned long long rejected;  // reserved sentinel keys seen by insert
};

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

__global__ void fill_i64(int64_t* __restrict__ p, int64_t n, int64_t v) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = v;
}

__device__ __forceinline__ void insert_one(int64_t* __restrict__ tkeys,
                                           int64_t* __restrict__ tvals, uint64_t mask,
                                           int64_t key, int64_t val, unsigned long long& added) {
  uint64_t s = mix64(static_cast<uint64_t>(key)) & mask;
  while (true) {
    int64_t cur = tkeys[s];
    if (cur == key) {
      tvals[s] = val;
      return;
    }
    if (cur == kKeyEmpty) {
      const int64_t prev = static_cast<int64_t>(atomicCAS(
          reinterpret_cast<unsigned long long*>(tkeys + s),
          static_cast<unsigned long long>(kKeyEmpty), static_cast<unsigned long long>(key)));
      if (prev == kKeyEmpty) {
        tvals[s] = val;
        ++added;
        return;
      }
      if (prev == key) {
        tvals[s] = val;
        return;
      }
    }
    s = (s + 1) & mask;
  }
}

__global__ void __launch_bounds__(256) insert_kernel(int64_t* __restrict__ tkeys,
                                                     int64_t* __restrict__ tvals, uint64_t mask,
                                                     const int64_t* __restrict__ keys,
                                                     const int64_t* __restrict__ vals, int64_t n,
                                                     Counters* __restrict__ ctr) {
  unsigned long long added = 0, rejected = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t key = keys[i];
    if (is_reserved(key)) {
      ++rejected;
      continue;
    }
    insert_one(tkeys, tvals, mask, key, vals ? vals[i] : i, added);
  }
  added = warp_sum(added);
  rejected = warp_sum(rejected);
  if ((threadIdx.x & 31) == 0) {
    if (added) {
      atomicAdd(&ctr->live, added);
      atomicAdd(&ctr->used, added);
    }
    if (rejected) atomicAdd(&ctr->rejected, rejected);
  }
}

__global__ void __launch_bounds__(256) erase_kernel(int64_t* __restrict__ tkeys, uint64_t mask,
                                                    const int64_t* __restrict__ keys, int64_t n,
                                                    Counters* __restrict__ ctr) {
  unsigned long long removed = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t key = keys[i];
    if (is_reserved(key)) continue;
    uint64_t s = mix64(static_cast<uint64_t>(key)) & mask;
    while (true) {
      const int64_t cur = tkeys[s];
      if (cur == kKeyEmpty) break;
      if (cur == key) {
        const int64_t prev = static_cast<int64_t>(
            atomicCAS(reinterpret_cast<unsigned long long*>(tkeys + s),
                      static_cast<unsigned long long>(key),
                      static_cast<unsigned long long>(kKeyTomb)));
        if (prev == key) ++removed;
        break;
      }
      s = (s + 1) & mask;
    }
  }
  removed = warp_sum(removed);
  if ((threadIdx.x & 31) == 0 && removed)
    atomicAdd(&ctr->live, static_cast<unsigned long long>(-static_cast<long long>(removed)));
}

// Erase keys [0, ne) and insert keys [ne, ne + ni) in ONE launch (the drop-in
// block manager's put: evicted ids out, new ids in).  Safe to run together:
// inserts claim only EMPTY slots (never tombstones) and stop at their own key,
// an erase only turns its own key into a tombstone, and the two sets are
// disjoint (a block being admitted is never its own victim).
__global__ void __launch_bounds__(256) update_kernel(int64_t* __restrict__ tkeys,
                                                     int64_t* __restrict__ tvals, uint64_t mask,
                                                     const int64_t* __restrict__ erase, int64_t ne,
                                                     const int64_t* __restrict__ ins,
                                                     const int64_t* __restrict__ vals, int64_t ni,
                                                     Counters* __restrict__ ctr) {
  unsigned long long added = 0, removed = 0, rejected = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < ne + ni;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (i < ne) {
      const int64_t key = erase[i];
      if (is_reserved(key)) continue;
      uint64_t s = mix64(static_cast<uint64_t>(key)) & mask;
      while (true) {
        const int64_t cur = tkeys[s];
        if (cur == kKeyEmpty) break;
        if (cur == key) {
          const int64_t prev = static_cast<int64_t>(
              atomicCAS(reinterpret_cast<unsigned long long*>(tkeys + s),
                        static_cast<unsigned long long>(key),
                        static_cast<unsigned long long>(kKeyTomb)));
          if (prev == key) ++removed;
          break;
        }
        s = (s + 1) & mask;
      }
    } else {
      const int64_t j = i - ne;
      const int64_t key = ins[j];
      if (is_reserved(key)) {
        ++rejected;
        continue;
      }
      insert_one(tkeys, tvals, mask, key, vals ? vals[j] : j, added);
    }
  }
  added = warp_sum(added);
  removed = warp_sum(removed);
  rejected = warp_sum(rejected);
  if ((threadIdx.x & 31) == 0) {
    if (added != removed)
      atomicAdd(&ctr->live, static_cast<unsigned long long>(static_cast<long long>(added) -
                                                            static_cast<long long>(removed)));
    if (added) atomicAdd(&ctr->used, added);
    if (rejected) atomicAdd(&ctr->rejected, rejected);
  }
}

__device__ __forceinline__ int64_t find_slot(const int64_t* __restrict__ tkeys, uint64_t mask,
                                             int64_t key) {
  if (is_reserved(key)) return -1;
  uint64_t s = mix64(static_cast<uint64_t>(key)) & mask;
  while (true) {
    const int64_t cur = __ldg(tkeys + s);
    if (cur == key) return static_cast<int64_t>(s);
    if (cur == kKeyEmpty) return -1;
    s = (s + 1) & mask;
  }
}

__global__ void __launch_bounds__(256) lookup_kernel(const int64_t* __restrict__ tkeys,
                                                     const int64_t* __restrict__ tvals,
                                                     uint64_t mask,
                                                     const int64_t* __restrict__ keys, int64_t n,
                                                     int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = find_slot(tkeys, mask, keys[i]);
    out[i] = s < 0 ? -1 : tvals[s];
  }
}

__global__ void __launch_bounds__(256) rehash_kernel(const int64_t* __restrict__ okeys,
                                                     const int64_t* __restrict__ ovals,
                                                     int64_t oslots, int64_t* __restrict__ nkeys,
                                                     int64_t* __restrict__ nvals, uint64_t nmask,
                                                     Counters* __restrict__ ctr) {
  unsigned long long added = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < oslots;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t key = okeys[i];
    if (is_reserved(key)) continue;
    insert_one(nkeys, nvals, nmask, key, ovals[i], added);
  }
  added = warp_sum(added);
  if ((threadIdx.x & 31) == 0 && added) {
    atomicAdd(&ctr->live, added);
    atomicAdd(&ctr->used, added);
  }
}

// ---- K2: batched prefix match ------------------------------------------

struct MatchParams {
  const int64_t* keys[KVX_MAX_INSTANCES];
  uint64_t mask[KVX_MAX_INSTANCES];
  int32_t ids[KVX_MAX_INSTANCES];
  int32_t n_inst;
  int32_t packed_only;  // leave the packed (len<<32 | ~id) word for a cross-GPU MAX
  // cross-GPU exchange inside the kernel: atomicMax of the packed word into
  // every rank's result buffer (peer mappings; NVLink remote atomics)
  unsigned long long* dests[KVX_MAX_PEERS];
  int32_t n_dests;
  // request-sharded batches (follower only): the keys of requests
  // [owner_end[j-1], owner_end[j]) live in owner_keys[j] (a peer GPU's buffer)
  const int64_t* owner_keys[KVX_MAX_PEERS];
  int64_t owner_end[KVX_MAX_PEERS];
  int32_t n_owner;
};

// U independent probe chains per lane: every chain's next slot load is issued
// before any is resolved, so each lane keeps U random L2/HBM reads in flight.
template <int U>
__device__ __forceinline__ void probe_multi(const int64_t* __restrict__ tk, uint64_t mask,
                                            const int64_t (&k)[U], const bool (&v)[U],
                                            bool (&hit)[U]) {
  bool done[U];
  uint64_t s[U];
  bool all = true;
#pragma unroll
  for (int j = 0; j < U; ++j) {
    done[j] = !v[j] || is_reserved(k[j]);
    hit[j] = false;
    s[j] = mix64(static_cast<uint64_t>(k[j])) & mask;
    all = all && done[j];
  }
  while (!all) {
    int64_t c[U];
#pragma unroll
    for (int j = 0; j < U; ++j) c[j] = done[j] ? kKeyEmpty : __ldg(tk + s[j]);
    all = true;
#pragma unroll
    for (int j = 0; j < U; ++j) {
      if (!done[j]) {
        if (c[j] == k[j]) {
          hit[j] = true;
          done[j] = true;
        } else if (c[j] == kKeyEmpty) {
          done[j] = true;
        } else {
          s[j] = (s[j] + 1) & mask;
        }
      }
      all = all && done[j];
    }
  }
}

// Sector probing: each round loads the whole 32-byte sector (4 slots) that
// holds a chain's next slot with one 256-bit load and scans it, so a
// linear-probe chain resolves in one round unless it runs past its sector
// (rare at the index's <= 0.40 load) -- against one round per slot when
// probing slot by slot.  The prefix match is latency bound (a warp step waits
// for the slowest of its probes), so rounds, not bytes, set its time.
__device__ __forceinline__ void ld_sector(const int64_t* p, int64_t (&w)[4]) {
  asm volatile("ld.global.nc.v4.b64 {%0,%1,%2,%3}, [%4];"
               : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3])
               : "l"(p));
}

template <int U>
__device__ __forceinline__ void probe_sector(const int64_t* __restrict__ tk, uint64_t mask,
                                             const int64_t (&k)[U], const bool (&v)[U],
                                             bool (&hit)[U]) {
  bool done[U];
  uint64_t base[U];
  int off[U];
  bool all = true;
#pragma unroll
  for (int j = 0; j < U; ++j) {
    done[j] = !v[j] || is_reserved(k[j]);
    hit[j] = false;
    const uint64_t s = mix64(static_cast<uint64_t>(k[j])) & mask;
    base[j] = s & ~uint64_t{3};  // tables have >= 1024 slots: sectors never wrap
    off[j] = static_cast<int>(s & 3);
    all = all && done[j];
  }
  while (!all) {
    int64_t w[U][4];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      if (!done[j]) ld_sector(tk + base[j], w[j]);
    }
    all = true;
#pragma unroll
    for (int j = 0; j < U; ++j) {
      if (!done[j]) {
        bool found = false, empty = false;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const bool act = q >= off[j] && !found && !empty;
          found = found || (act && w[j][q] == k[j]);
          empty = empty || (act && w[j][q] == kKeyEmpty);
        }
        if (found || empty) {
          hit[j] = found;
          done[j] = true;
        } else {
          base[j] = (base[j] + 4) & mask;
          off[j] = 0;
        }
      }
      all = all && done[j];
    }
  }
}

#ifndef KVX_PROBE_CHAINS
#define KVX_PROBE_CHAINS 4
#endif
constexpr int kProbeChains = KVX_PROBE_CHAINS;  // per lane -> 32 x this query keys per warp step

__device__ __forceinline__ unsigned long long pack_best(int64_t len, int32_t id) {
  // Larger len wins; on equal len the LOWER id must win, so store ~ordered(id).
  const uint32_t ordered = static_cast<uint32_t>(id) ^ 0x80000000u;
  return (static_cast<unsigned long long>(len) << 32) | static_cast<unsigned long long>(~ordered);
}

// The per-task epilogue shared by both match kernels (lane 0 of the warp /
// thread 0 of the CTA that owns the task).
__device__ __forceinline__ void match_result(const MatchParams& p, int64_t t, int64_t r, int i,
                                             int64_t len, int64_t* __restrict__ len_out,
                                             int64_t* __restrict__ best_len,
                                             int32_t* __restrict__ best_id) {
  if (len_out) len_out[t] = len;
  if (p.n_dests > 0) {
    const unsigned long long v = pack_best(len, p.ids[i]);
    for (int j = 0; j < p.n_dests; ++j) atomicMax(p.dests[j] + r, v);
  } else if (best_len) {
    if (p.n_inst == 1 && !p.packed_only) {
      best_len[r] = len;
      best_id[r] = p.ids[0];
    } else {
      atomicMax(reinterpret_cast<unsigned long long*>(best_len + r), pack_best(len, p.ids[i]));
    }
  }
}

__global__ void __launch_bounds__(256) match_kernel(const __grid_constant__ MatchParams p,
                                                    const int64_t* __restrict__ keys,
                                                    const int64_t* __restrict__ key_off,
                                                    int64_t n_req,
                                                    int64_t* __restrict__ len_out,
                                                    int64_t* __restrict__ best_len,
                                                    int32_t* __restrict__ best_id) {
  const int lane = threadIdx.x & 31;
  const int64_t tasks = n_req * p.n_inst;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
       t < tasks; t += warps) {
    // 32-bit division when it suffices (a 64-bit one is a long subroutine)
    const int64_t r = tasks <= 0xFFFFFFFFll
                          ? static_cast<int64_t>(static_cast<uint32_t>(t) / static_cast<uint32_t>(p.n_inst))
                          : t / p.n_inst;
    const int i = static_cast<int>(t - r * p.n_inst);
    const int64_t* __restrict__ tk = p.keys[i];
    const uint64_t mask = p.mask[i];
    const int64_t base = key_off[r];
    const int64_t n = key_off[r + 1] - base;
    const int64_t* __restrict__ q = keys + base;
    int64_t len = 0;
    for (int64_t k0 = 0;; k0 += 32 * kProbeChains) {
      int64_t qk[kProbeChains];
      bool qv[kProbeChains], hit[kProbeChains];
#pragma unroll
      for (int j = 0; j < kProbeChains; ++j) {
        const int64_t idx = k0 + 32 * j + lane;
        qv[j] = idx < n;
        qk[j] = qv[j] ? __ldg(q + idx) : 0;
      }
      probe_multi<kProbeChains>(tk, mask, qk, qv, hit);
      bool stop = false;
#pragma unroll
      for (int j = 0; j < kProbeChains; ++j) {
        const unsigned miss = __ballot_sync(0xffffffffu, !hit[j]);  // out-of-range = miss
        if (!stop && miss) {
          len = k0 + 32 * j + __ffs(miss) - 1;
          stop = true;
        }
      }
      if (stop) break;
    }
    if (lane == 0) match_result(p, t, r, i, len, len_out, best_len, best_id);
  }
}

// K2 with G warps per (request, instance) task: the request's 128-key
// windows go to the warps in waves (window = wave * G + warp), so a long
// matched prefix costs ceil(windows / G) dependent probe rounds instead of
// one per window; each warp's first miss is folded into a shared atomicMin,
// and the task ends after the first wave whose windows all lie past it (all
// windows before the minimum were fully probed: it IS the first miss).  The
// extra probes are the speculative windows of the wave that holds the miss.
// One (request r, instance i) task of K2 on a CTA of G warps (first_miss:
// the CTA's shared word).  Ends with the CTA synchronised.
template <int G, int C, bool kSector>
__device__ __forceinline__ void match_task(const MatchParams& p, const int64_t* __restrict__ keys,
                                           const int64_t* __restrict__ key_off, int64_t r, int i,
                                           int64_t* __restrict__ len_out,
                                           int64_t* __restrict__ best_len,
                                           int32_t* __restrict__ best_id, long long& first_miss) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int64_t kWin = 32 * C;
  const int64_t t = r * p.n_inst + i;
  const int64_t* __restrict__ tk = p.keys[i];
  const uint64_t mask = p.mask[i];
  const int64_t base = key_off[r];
  const int64_t n = key_off[r + 1] - base;
  const int64_t* __restrict__ q = keys + base;
  if (threadIdx.x == 0) first_miss = n;  // no miss: the whole chain matches
  __syncthreads();
  // this warp's query keys of the first wave; each wave then loads the next
  // wave's keys before probing, so their L2 round trip overlaps the probes
  int64_t nq[C];
#pragma unroll
  for (int j = 0; j < C; ++j) {
    const int64_t idx = warp * kWin + 32 * j + lane;
    nq[j] = idx < n ? __ldg(q + idx) : 0;
  }
  for (int64_t wave = 0;; ++wave) {
    const int64_t k0 = (wave * G + warp) * kWin;
    int64_t qk[C];
#pragma unroll
    for (int j = 0; j < C; ++j) qk[j] = nq[j];
    if (k0 + G * kWin < n) {
#pragma unroll
      for (int j = 0; j < C; ++j) {
        const int64_t idx = k0 + G * kWin + 32 * j + lane;
        nq[j] = idx < n ? __ldg(q + idx) : 0;
      }
    }
    if (k0 < n && k0 < static_cast<int64_t>(*reinterpret_cast<volatile long long*>(&first_miss))) {
      bool qv[C], hit[C];
#pragma unroll
      for (int j = 0; j < C; ++j) qv[j] = k0 + 32 * j + lane < n;
      if (kSector) probe_sector<C>(tk, mask, qk, qv, hit);
      else probe_multi<C>(tk, mask, qk, qv, hit);
#pragma unroll
      for (int j = 0; j < C; ++j) {
        const unsigned miss = __ballot_sync(0xffffffffu, !hit[j] && qv[j]);
        if (miss) {  // the window's first miss (out-of-range lanes are not misses here)
          if (lane == 0) atomicMin(&first_miss, static_cast<long long>(k0 + 32 * j + __ffs(miss) - 1));
          break;
        }
      }
    }
    __syncthreads();
    const int64_t fm = static_cast<int64_t>(first_miss);
    const int64_t covered = (wave + 1) * G * kWin;
    if (fm < covered || covered >= n) break;  // uniform over the CTA
  }
  if (threadIdx.x == 0) {
    const int64_t len = static_cast<int64_t>(first_miss);
    match_result(p, t, r, i, len, len_out, best_len, best_id);
  }
  __syncthreads();  // first_miss is re-initialised for the next task
}

template <int G, int C, int MINB = 1, bool kSector = false>
__global__ void __launch_bounds__(G * 32, MINB) match_group_kernel(
    const __grid_constant__ MatchParams p, const int64_t* __restrict__ keys,
    const int64_t* __restrict__ key_off, int64_t n_req, int64_t* __restrict__ len_out,
    int64_t* __restrict__ best_len, int32_t* __restrict__ best_id,
    const int32_t* __restrict__ order) {
  __shared__ long long first_miss;
  const int64_t tasks = n_req * p.n_inst;
  for (int64_t tt = blockIdx.x; tt < tasks; tt += gridDim.x) {
    const int64_t ro = tasks <= 0xFFFFFFFFll
                           ? static_cast<int64_t>(static_cast<uint32_t>(tt) / static_cast<uint32_t>(p.n_inst))
                           : tt / p.n_inst;
    const int i = static_cast<int>(tt - ro * p.n_inst);
    // longest requests first when an order is given (they set the batch time)
    const int64_t r = order ? static_cast<int64_t>(__ldg(order + ro)) : ro;
    match_task<G, C, kSector>(p, keys, key_off, r, i, len_out, best_len, best_id, first_miss);
  }
}

// Set when a follower gave up waiting for a request's keys (kvx_hash_match_check).
__device__ unsigned long long g_queue_timeouts = 0;

// K2 following the block hash running beside it (kvx_hash_match_batch).  A
// CTA takes requests in the hash's own longest-first claim order; each warp
// loads its window's keys from L2 and re-polls (back-off, 5 s limit) the ones
// that are still -1, the value the keys were preset to -- no key is negative,
// and each 8-byte key is stored whole -- so a window is probed as soon as the
// hash has produced it.  The match stops at the first miss, usually long
// before the request's hash ends.  Launched programmatically dependent on the
// hash, which triggers only once all of its CTAs are resident, so every
// awaited key is eventually stored.
template <int G, int C, bool kSector>
__global__ void __launch_bounds__(G * 32) match_follow_kernel(
    const __grid_constant__ MatchParams p, const int64_t* __restrict__ keys,
    const int64_t* __restrict__ key_off, int64_t n_req, int64_t* __restrict__ len_out,
    int64_t* __restrict__ best_len, int32_t* __restrict__ best_id,
    const int32_t* __restrict__ order, unsigned long long* claim) {
  __shared__ long long first_miss;
  __shared__ long long req;
  __shared__ int stop;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int64_t kWin = 32 * C;
  while (true) {
    if (threadIdx.x == 0) {
      const unsigned long long pos = atomicAdd(claim, 1ull);
      req = pos < static_cast<unsigned long long>(n_req)
                ? (order ? static_cast<long long>(order[pos]) : static_cast<long long>(pos))
                : -1;
      stop = 0;
    }
    __syncthreads();
    const int64_t r = static_cast<int64_t>(req);
    if (r < 0) return;
    const int64_t base = key_off[r];
    const int64_t n = key_off[r + 1] - base;
    const int64_t* kb = keys;
    if (p.n_owner > 0) {  // read the keys where their shard's GPU stores them (NVLink loads)
      int j = 0;
      while (j + 1 < p.n_owner && r >= p.owner_end[j]) ++j;
      kb = p.owner_keys[j];
    }
    const int64_t* q = kb + base;
    for (int i = 0; i < p.n_inst; ++i) {
      const int64_t t = r * p.n_inst + i;
      const int64_t* __restrict__ tk = p.keys[i];
      const uint64_t mask = p.mask[i];
      if (threadIdx.x == 0) first_miss = n;
      __syncthreads();
      for (int64_t wave = 0;; ++wave) {
        const int64_t k0 = (wave * G + warp) * kWin;
        if (k0 < n && k0 < static_cast<int64_t>(*reinterpret_cast<volatile long long*>(&first_miss))) {
          int64_t qk[C];
          bool qv[C], hit[C];
          // L2 only (ld.global.cg): the keys are stored during this kernel by
          // other SMs, and a line read earlier may sit stale in this SM's L1
#pragma unroll
          for (int j = 0; j < C; ++j) {
            const int64_t idx = k0 + 32 * j + lane;
            qv[j] = idx < n;
            qk[j] = qv[j] ? __ldcg(q + idx) : 0;
          }
          bool pending = false;
#pragma unroll
          for (int j = 0; j < C; ++j) pending = pending || qk[j] < 0;
          if (__any_sync(0xffffffffu, pending)) {
            unsigned ns = 64;
            unsigned long long t0, tn;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            while (__any_sync(0xffffffffu, pending)) {
              __nanosleep(ns);
              ns = ns < 1024 ? 2 * ns : ns;
              pending = false;
#pragma unroll
              for (int j = 0; j < C; ++j) {
                if (qk[j] < 0) qk[j] = __ldcg(q + k0 + 32 * j + lane);
                pending = pending || qk[j] < 0;
              }
              asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
              if (tn - t0 > 5000000000ull) {  // never stored: report, don't hang
                if (lane == 0) {
                  g_queue_timeouts = 1;
                  stop = 1;
                }
                break;
              }
            }
          }
          if (kSector) probe_sector<C>(tk, mask, qk, qv, hit);
          else probe_multi<C>(tk, mask, qk, qv, hit);
#pragma unroll
          for (int j = 0; j < C; ++j) {
            const unsigned miss = __ballot_sync(0xffffffffu, !hit[j] && qv[j]);
            if (miss) {
              if (lane == 0) atomicMin(&first_miss, static_cast<long long>(k0 + 32 * j + __ffs(miss) - 1));
              break;
            }
          }
        }
        __syncthreads();
        const int64_t fm = static_cast<int64_t>(first_miss);
        const int64_t covered = (wave + 1) * G * kWin;
        if (stop || fm < covered || covered >= n) break;  // uniform over the CTA
      }
      if (threadIdx.x == 0 && !stop) {
        const int64_t len = static_cast<int64_t>(first_miss);
        match_result(p, t, r, i, len, len_out, best_len, best_id);
      }
      __syncthreads();
      if (stop) break;
    }
  }
}

// packed may alias best_len (in-place unpack).
__global__ void unpack_best_kernel(const unsigned long long* packed, int64_t* best_len,
                                   int32_t* __restrict__ best_id, int64_t n_req) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n_req;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const unsigned long long v = packed[r];
    best_len[r] = static_cast<int64_t>(v >> 32);
    best_id[r] = static_cast<int32_t>(~static_cast<uint32_t>(v & 0xffffffffu) ^ 0x80000000u);
  }
}

int grid_for(int64_t n, int threads, int dev, int per_sm = 8) {
  const int64_t want = (n + threads - 1) / threads;
  const int64_t cap = static_cast<int64_t>(sm_count(dev)) * per_sm;
  return static_cast<int>(std::max<int64_t>(1, std::min(want, cap)));
}

int64_t next_pow2(int64_t v) {
  int64_t p = 1024;
  while (p < v) p <<= 1;
  return p;
}

}  // namespace
}  // namespace kvx

using namespace kvx;

struct kvx_index {
  int device = 0;
  int64_t* keys = nullptr;
  int64_t* vals = nullptr;
  int64_t slots = 0;
  Counters* ctr = nullptr;   // device counters
  int64_t used_ub = 0;       // host upper bound on occupied slots
};

namespace {

int alloc_table(kvx_index* x, int64_t slots, cudaStream_t s, int64_t** keys, int64_t** vals) {
  KVX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(keys), sizeof(int64_t) * slots, s));
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(vals), sizeof(int64_t) * slots, s);
  if (e != cudaSuccess) {
    cudaFreeAsync(*keys, s);
    return cuda_error(e, "kvx_index: cudaMallocAsync(values)");
  }
  fill_i64<<<grid_for(slots, 256, x->device), 256, 0, s>>>(*keys, slots, kKeyEmpty);
  KVX_LAUNCH_CHECK("fill_i64");
  return KVX_OK;
}

int read_counters(kvx_index* x, cudaStream_t s, Counters* h) {
  KVX_CUDA(cudaMemcpyAsync(h, x->ctr, sizeof(Counters), cudaMemcpyDeviceToHost, s));
  KVX_CUDA(cudaStreamSynchronize(s));
  return KVX_OK;
}

int rebuild(kvx_index* x, int64_t new_slots, cudaStream_t s) {
  int64_t *nk = nullptr, *nv = nullptr;
  int st = alloc_table(x, new_slots, s, &nk, &nv);
  if (st) return st;
  KVX_CUDA(cudaMemsetAsync(x->ctr, 0, 2 * sizeof(unsigned long long), s));  // live, used
  if (x->keys) {
    rehash_kernel<<<grid_for(x->slots, 256, x->device), 256, 0, s>>>(
        x->keys, x->vals, x->slots, nk, nv, static_cast<uint64_t>(new_slots - 1), x->ctr);
    KVX_LAUNCH_CHECK("rehash_kernel");
    KVX_CUDA(cudaFreeAsync(x->keys, s));
    KVX_CUDA(cudaFreeAsync(x->vals, s));
  }
  x->keys = nk;
  x->vals = nv;
  x->slots = new_slots;
  return KVX_OK;
}

// Ensure n more keys fit under kMaxLoad.  Only syncs when the cheap upper
// bound says the table might be too full.
int ensure_room(kvx_index* x, int64_t n, cudaStream_t s) {
  if (static_cast<double>(x->used_ub + n) <= kMaxLoad * static_cast<double>(x->slots))
    return KVX_OK;
  Counters h;
  int st = read_counters(x, s, &h);
  if (st) return st;
  const int64_t live = static_cast<int64_t>(h.live), used = static_cast<int64_t>(h.used);
  x->used_ub = used;
  if (static_cast<double>(used + n) <= kMaxLoad * static_cast<double>(x->slots)) return KVX_OK;
  int64_t want = x->slots;
  while (static_cast<double>(live + n) > kTargetLoad * static_cast<double>(want)) want <<= 1;
  st = rebuild(x, want, s);
  if (st) return st;
  x->used_ub = live;
  return KVX_OK;
}

int match_impl(const kvx_index* const* idx, const int32_t* inst_ids, int64_t n_inst,
               const int64_t* d_keys, const int64_t* d_key_off, int64_t n_req,
               int64_t* d_len_out, int64_t* d_best_len, int32_t* d_best_id, bool packed_only,
               void* stream, uint64_t* const* dests = nullptr, int n_dests = 0);

}  // namespace

extern "C" {

int kvx_index_create(int device, int64_t capacity_hint, kvx_index** out) {
  KVX_REQUIRE(out != nullptr, "kvx_index_create: out is NULL");
  KVX_REQUIRE(capacity_hint >= 0, "kvx_index_create: capacity_hint must be >= 0");
  int ndev = 0;
  KVX_CUDA(cudaGetDeviceCount(&ndev));
  KVX_REQUIRE(device >= 0 && device < ndev, "kvx_index_create: bad device");
  DeviceGuard g(device);
  auto* x = new kvx_index();
  x->device = device;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&x->ctr), sizeof(Counters));
  if (e != cudaSuccess) {
    delete x;
    return cuda_error(e, "kvx_index_create: cudaMalloc(counters)");
  }
  e = cudaMemsetAsync(x->ctr, 0, sizeof(Counters), nullptr);
  if (e != cudaSuccess) {
    kvx_index_destroy(x);
    return cuda_error(e, "kvx_index_create: cudaMemset(counters)");
  }
  int64_t slots = next_pow2(static_cast<int64_t>(static_cast<double>(capacity_hint) / kTargetLoad) + 1);
  int st = rebuild(x, slots, nullptr);
  if (st == KVX_OK) {
    e = cudaStreamSynchronize(nullptr);
    if (e != cudaSuccess) st = cuda_error(e, "kvx_index_create");
  }
  if (st) {
    kvx_index_destroy(x);
    return st;
  }
  *out = x;
  return KVX_OK;
}

int kvx_index_destroy(kvx_index* x) {
  if (!x) return KVX_OK;
  DeviceGuard g(x->device);
  cudaDeviceSynchronize();
  if (x->keys) cudaFreeAsync(x->keys, nullptr);
  if (x->vals) cudaFreeAsync(x->vals, nullptr);
  if (x->ctr) cudaFree(x->ctr);
  cudaStreamSynchronize(nullptr);
  delete x;
  return KVX_OK;
}

int kvx_index_device(const kvx_index* x) { return x ? x->device : -1; }

int kvx_index_insert(kvx_index* x, const int64_t* d_keys, const int64_t* d_values, int64_t n,
                     void* stream) {
  KVX_REQUIRE(x != nullptr, "kvx_index_insert: NULL index");
  KVX_REQUIRE(n >= 0, "kvx_index_insert: n must be >= 0");
  if (n == 0) return KVX_OK;
  KVX_REQUIRE(d_keys != nullptr, "kvx_index_insert: NULL keys");
  DeviceGuard g(x->device);
  cudaStream_t s = as_stream(stream);
  int st = ensure_room(x, n, s);
  if (st) return st;
  insert_kernel<<<grid_for(n, 256, x->device), 256, 0, s>>>(
      x->keys, x->vals, static_cast<uint64_t>(x->slots - 1), d_keys, d_values, n, x->ctr);
  KVX_LAUNCH_CHECK("insert_kernel");
  x->used_ub += n;
  return KVX_OK;
}

int kvx_index_erase(kvx_index* x, const int64_t* d_keys, int64_t n, void* stream) {
  KVX_REQUIRE(x != nullptr, "kvx_index_erase: NULL index");
  KVX_REQUIRE(n >= 0, "kvx_index_erase: n must be >= 0");
  if (n == 0) return KVX_OK;
  KVX_REQUIRE(d_keys != nullptr, "kvx_index_erase: NULL keys");
  DeviceGuard g(x->device);
  erase_kernel<<<grid_for(n, 256, x->device), 256, 0, as_stream(stream)>>>(
      x->keys, static_cast<uint64_t>(x->slots - 1), d_keys, n, x->ctr);
  KVX_LAUNCH_CHECK("erase_kernel");
  return KVX_OK;
}

int kvx_index_update(kvx_index* x, const int64_t* d_erase, int64_t ne, const int64_t* d_insert,
                     const int64_t* d_values, int64_t ni, void* stream) {
  KVX_REQUIRE(x != nullptr, "kvx_index_update: NULL index");
  KVX_REQUIRE(ne >= 0 && ni >= 0, "kvx_index_update: counts must be >= 0");
  if (ne + ni == 0) return KVX_OK;
  KVX_REQUIRE((ne == 0 || d_erase) && (ni == 0 || d_insert), "kvx_index_update: NULL keys");
  DeviceGuard g(x->device);
  cudaStream_t s = as_stream(stream);
  if (ni) {
    int st = ensure_room(x, ni, s);
    if (st) return st;
  }
  update_kernel<<<grid_for(ne + ni, 256, x->device), 256, 0, s>>>(
      x->keys, x->vals, static_cast<uint64_t>(x->slots - 1), d_erase, ne, d_insert, d_values, ni,
      x->ctr);
  KVX_LAUNCH_CHECK("update_kernel");
  x->used_ub += ni;
  return KVX_OK;
}

int kvx_index_l2_pin(const kvx_index* x, void* stream, int on) {
  KVX_REQUIRE(x != nullptr && stream != nullptr, "kvx_index_l2_pin: NULL index or stream");
  DeviceGuard g(x->device);
  cudaStreamAttrValue attr = {};
  if (on) {
    int max_persist = 0, max_window = 0;
    KVX_CUDA(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, x->device));
    KVX_CUDA(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, x->device));
    KVX_REQUIRE(max_persist > 0 && max_window > 0, "kvx_index_l2_pin: no persisting L2 on this device");
    const size_t bytes = static_cast<size_t>(x->slots) * sizeof(int64_t);
    const size_t window = std::min(bytes, static_cast<size_t>(max_window));
    const size_t carve = std::min(window, static_cast<size_t>(max_persist));
    size_t cur = 0;
    KVX_CUDA(cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize));
    if (cur < carve) KVX_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve));
    attr.accessPolicyWindow.base_ptr = x->keys;
    attr.accessPolicyWindow.num_bytes = window;
    attr.accessPolicyWindow.hitRatio = static_cast<float>(std::min(1.0, double(carve) / double(window)));
    attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  }
  KVX_CUDA(cudaStreamSetAttribute(as_stream(stream), cudaStreamAttributeAccessPolicyWindow, &attr));
  return KVX_OK;
}

int kvx_index_lookup(const kvx_index* x, const int64_t* d_keys, int64_t n, int64_t* d_out,
                     void* stream) {
  KVX_REQUIRE(x != nullptr, "kvx_index_lookup: NULL index");
  KVX_REQUIRE(n >= 0, "kvx_index_lookup: n must be >= 0");
  if (n == 0) return KVX_OK;
  KVX_REQUIRE(d_keys && d_out, "kvx_index_lookup: NULL array");
  DeviceGuard g(x->device);
  lookup_kernel<<<grid_for(n, 256, x->device), 256, 0, as_stream(stream)>>>(
      x->keys, x->vals, static_cast<uint64_t>(x->slots - 1), d_keys, n, d_out);
  KVX_LAUNCH_CHECK("lookup_kernel");
  return KVX_OK;
}

int kvx_index_clear(kvx_index* x, void* stream) {
  KVX_REQUIRE(x != nullptr, "kvx_index_clear: NULL index");
  DeviceGuard g(x->device);
  cudaStream_t s = as_stream(stream);
  fill_i64<<<grid_for(x->slots, 256, x->device), 256, 0, s>>>(x->keys, x->slots, kKeyEmpty);
  KVX_LAUNCH_CHECK("fill_i64");
  KVX_CUDA(cudaMemsetAsync(x->ctr, 0, 2 * sizeof(unsigned long long), s));
  x->used_ub = 0;
  return KVX_OK;
}

int kvx_index_reserve(kvx_index* x, int64_t min_keys, void* stream) {
  KVX_REQUIRE(x != nullptr, "kvx_index_reserve: NULL index");
  KVX_REQUIRE(min_keys >= 0, "kvx_index_reserve: min_keys must be >= 0");
  DeviceGuard g(x->device);
  cudaStream_t s = as_stream(stream);
  Counters h;
  int st = read_counters(x, s, &h);
  if (st) return st;
  const int64_t live = static_cast<int64_t>(h.live);
  const int64_t want = next_pow2(static_cast<int64_t>(
      static_cast<double>(std::max(min_keys, live)) / kTargetLoad) + 1);
  st = rebuild(x, want, s);
  if (st) return st;
  x->used_ub = live;
  return KVX_OK;
}

int kvx_index_stats(kvx_index* x, int64_t* live, int64_t* tombstones, int64_t* slots,
                    int64_t* rejected, void* stream) {
  KVX_REQUIRE(x != nullptr, "kvx_index_stats: NULL index");
  DeviceGuard g(x->device);
  Counters h;
  int st = read_counters(x, as_stream(stream), &h);
  if (st) return st;
  if (live) *live = static_cast<int64_t>(h.live);
  if (tombstones) *tombstones = static_cast<int64_t>(h.used - h.live);
  if (slots) *slots = x->slots;
  if (rejected) *rejected = static_cast<int64_t>(h.rejected);
  return KVX_OK;
}

int kvx_match_prefix_batch(const kvx_index* const* idx, const int32_t* inst_ids, int64_t n_inst,
                           const int64_t* d_keys, const int64_t* d_key_off, int64_t n_req,
                           int64_t* d_len_out, int64_t* d_best_len, int32_t* d_best_id,
                           void* stream) {
  KVX_REQUIRE(n_inst >= 1, "find_best_prefix_match: empty prefill pool");
  KVX_REQUIRE(n_inst <= KVX_MAX_INSTANCES, "kvx_match_prefix_batch: too many instances");
  KVX_REQUIRE(idx != nullptr && inst_ids != nullptr, "kvx_match_prefix_batch: NULL instances");
  KVX_REQUIRE(n_req >= 0, "kvx_match_prefix_batch: n_req must be >= 0");
  KVX_REQUIRE((d_best_len == nullptr) == (d_best_id == nullptr),
              "kvx_match_prefix_batch: best_len and best_id go together");
  if (n_req == 0) return KVX_OK;
  // d_keys may be NULL when every chain is empty (the kernel reads keys only
  // inside a request's [key_off[r], key_off[r+1]) range)
  KVX_REQUIRE(d_key_off, "kvx_match_prefix_batch: NULL key offsets");
  return match_impl(idx, inst_ids, n_inst, d_keys, d_key_off, n_req, d_len_out, d_best_len,
                    d_best_id, false, stream);
}

int kvx_match_prefix_packed(const kvx_index* const* idx, const int32_t* inst_ids, int64_t n_inst,
                            const int64_t* d_keys, const int64_t* d_key_off, int64_t n_req,
                            uint64_t* d_packed, void* stream) {
  KVX_REQUIRE(n_inst >= 1, "find_best_prefix_match: empty prefill pool");
  KVX_REQUIRE(n_inst <= KVX_MAX_INSTANCES, "kvx_match_prefix_packed: too many instances");
  KVX_REQUIRE(idx != nullptr && inst_ids != nullptr, "kvx_match_prefix_packed: NULL instances");
  KVX_REQUIRE(n_req >= 0, "kvx_match_prefix_packed: n_req must be >= 0");
  if (n_req == 0) return KVX_OK;
  KVX_REQUIRE(d_key_off && d_packed, "kvx_match_prefix_packed: NULL array");
  return match_impl(idx, inst_ids, n_inst, d_keys, d_key_off, n_req, nullptr,
                    reinterpret_cast<int64_t*>(d_packed), nullptr, true, stream);
}

int kvx_best_unpack(const uint64_t* d_packed, int64_t n_req, int64_t* d_best_len,
                    int32_t* d_best_id, void* stream) {
  KVX_REQUIRE(n_req >= 0, "kvx_best_unpack: n_req must be >= 0");
  if (n_req == 0) return KVX_OK;
  KVX_REQUIRE(d_packed && d_best_len && d_best_id, "kvx_best_unpack: NULL array");
  int dev = 0;
  KVX_CUDA(cudaGetDevice(&dev));
  unpack_best_kernel<<<grid_for(n_req, 256, dev), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const unsigned long long*>(d_packed), d_best_len, d_best_id, n_req);
  KVX_LAUNCH_CHECK("unpack_best_kernel");
  return KVX_OK;
}

}  // extern "C"

namespace {
int match_impl(const kvx_index* const* idx, const int32_t* inst_ids, int64_t n_inst,
               const int64_t* d_keys, const int64_t* d_key_off, int64_t n_req,
               int64_t* d_len_out, int64_t* d_best_len, int32_t* d_best_id, bool packed_only,
               void* stream, uint64_t* const* dests, int n_dests) {
  MatchParams p{};
  p.n_inst = static_cast<int32_t>(n_inst);
  p.packed_only = packed_only ? 1 : 0;
  p.n_dests = n_dests;
  for (int j = 0; j < n_dests; ++j) p.dests[j] = reinterpret_cast<unsigned long long*>(dests[j]);
  const int dev = idx[0] ? idx[0]->device : -1;
  for (int64_t i = 0; i < n_inst; ++i) {
    KVX_REQUIRE(idx[i] != nullptr, "kvx_match_prefix_batch: NULL index");
    KVX_REQUIRE(idx[i]->device == dev, "kvx_match_prefix_batch: indices on different devices");
    p.keys[i] = idx[i]->keys;
    p.mask[i] = static_cast<uint64_t>(idx[i]->slots - 1);
    p.ids[i] = inst_ids[i];
  }
  DeviceGuard g(dev);
  cudaStream_t s = as_stream(stream);
  if (d_best_len && (n_inst > 1 || packed_only) && n_dests == 0)
    KVX_CUDA(cudaMemsetAsync(d_best_len, 0, sizeof(int64_t) * n_req, s));
  const int64_t tasks = n_req * n_inst;
  // warps per task x probe chains per lane (measured, profiles/r02/match.md)
  static const int group = [] {
    const char* e = std::getenv("KVX_MATCH_GROUP");  // 1 = the warp-per-task kernel
    const int v = e ? std::atoi(e) : 2;
    return v == 1 || v == 2 || v == 4 || v == 8 ? v : 2;
  }();
  static const int chains = [] {
    const char* e = std::getenv("KVX_MATCH_CHAINS");
    const int v = e ? std::atoi(e) : 2;
    return v == 1 || v == 2 || v == 4 ? v : 2;
  }();
  if (group > 1) {
    const int64_t cap = static_cast<int64_t>(sm_count(dev)) * (64 / group);  // 2048 threads / SM
    const int blocks = static_cast<int>(std::max<int64_t>(1, std::min(tasks, cap)));
    const int threads = 32 * group;
    static const bool ordered = [] {
      const char* e = std::getenv("KVX_MATCH_ORDER");  // longest requests first (measurement)
      return e && e[0] == '1';
    }();
    int32_t* order = nullptr;
    unsigned long long* ows = nullptr;
    if (ordered && n_req <= (int64_t{1} << 22)) {
      KVX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&order), n_req * sizeof(int32_t) + 16, s));
      ows = reinterpret_cast<unsigned long long*>(order + ((n_req + 1) & ~int64_t{1}));
      int rc = order_by_length(d_key_off, n_req, order, ows, s);
      if (rc) return rc;
    }
#define KVX_MATCH_G(G, C)                                                                  \
  match_group_kernel<G, C><<<blocks, threads, 0, s>>>(p, d_keys, d_key_off, n_req, d_len_out, \
                                                      d_best_len, d_best_id, order)
    // Sector probing shortens each probe chain to ~one dependent round, which
    // is what a small batch waits for (148 requests: 18.9 vs 24.3 us); a full
    // Config 4 batch is set by the burst of its first wave through L2, where
    // the 256-bit loads cost more than they save (34.8 vs 32.7 us):
    // profiles/r02/match.md.  KVX_MATCH_SECTOR=0/1 forces either.
    static const int sector_knob = [] {
      const char* e = std::getenv("KVX_MATCH_SECTOR");
      return e ? std::atoi(e) : -1;
    }();
    const bool sector = sector_knob >= 0 ? sector_knob == 1 : tasks <= 1024;
    static const bool full_occ = [] {
      const char* e = std::getenv("KVX_MATCH_OCC");  // measurement knob
      return e && e[0] == '1';
    }();
    switch (sector ? 1000 + group * 10 + chains
                   : (full_occ && group == 2 && chains == 2 ? 220 : group * 10 + chains)) {
#define KVX_MATCH_GS(G, C)                                                                    \
  match_group_kernel<G, C, 1, true><<<blocks, threads, 0, s>>>(p, d_keys, d_key_off, n_req,     \
                                                               d_len_out, d_best_len, d_best_id, \
                                                               order)
      case 1021: KVX_MATCH_GS(2, 1); break;
      case 1022: KVX_MATCH_GS(2, 2); break;
      case 1024: KVX_MATCH_GS(2, 4); break;
      case 1041: KVX_MATCH_GS(4, 1); break;
      case 1042: KVX_MATCH_GS(4, 2); break;
      case 1081: KVX_MATCH_GS(8, 1); break;
#undef KVX_MATCH_GS
      case 21: KVX_MATCH_G(2, 1); break;
      case 41: KVX_MATCH_G(4, 1); break;
      case 42: KVX_MATCH_G(4, 2); break;
      case 44: KVX_MATCH_G(4, 4); break;
      case 81: KVX_MATCH_G(8, 1); break;
      case 82: KVX_MATCH_G(8, 2); break;
      case 84: KVX_MATCH_G(8, 4); break;
      case 24: KVX_MATCH_G(2, 4); break;
      case 220:  // 2 x 2 at full residency: 32 CTAs of 64 threads per SM (<= 32 registers)
        match_group_kernel<2, 2, 32><<<static_cast<int>(std::max<int64_t>(
                                          1, std::min<int64_t>(tasks, sm_count(dev) * 32))),
                                      threads, 0, s>>>(p, d_keys, d_key_off, n_req, d_len_out,
                                                       d_best_len, d_best_id, order);
        break;
      default: KVX_MATCH_G(2, 2);
    }
#undef KVX_MATCH_G
    KVX_LAUNCH_CHECK("match_group_kernel");
    if (order) KVX_CUDA(cudaFreeAsync(order, s));
  } else {
  const int threads = 256;
  const int64_t want = (tasks + (threads / 32) - 1) / (threads / 32);
  const int64_t cap = static_cast<int64_t>(sm_count(dev)) * 16;
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min(want, cap)));
  match_kernel<<<blocks, threads, 0, s>>>(p, d_keys, d_key_off, n_req, d_len_out, d_best_len,
                                          d_best_id);
  KVX_LAUNCH_CHECK("match_kernel");
  }
  if (d_best_len && n_inst > 1 && !packed_only) {
    unpack_best_kernel<<<grid_for(n_req, 256, dev), 256, 0, s>>>(
        reinterpret_cast<const unsigned long long*>(d_best_len), d_best_len, d_best_id, n_req);
    KVX_LAUNCH_CHECK("unpack_best_kernel");
  }
  return KVX_OK;
}
}  // namespace

namespace kvx {
// K2 following the hash's key progress (kvx_hash_match_batch): params as
// kvx_match_prefix_batch; launched programmatically dependent on the hash.
int match_follow_launch(const kvx_index* const* idx, const int32_t* inst_ids, int64_t n_inst,
                        const int64_t* d_keys, const int64_t* d_key_off, int64_t n_req,
                        int64_t* d_len_out, int64_t* d_best_len, int32_t* d_best_id,
                        const int32_t* d_order, unsigned long long* d_claim, void* stream,
                        uint64_t* const* dests, int n_dests, const int64_t* const* owner_keys,
                        const int64_t* owner_end, int n_owner) {
  MatchParams p{};
  p.n_owner = n_owner;
  for (int j = 0; j < n_owner; ++j) {
    p.owner_keys[j] = owner_keys[j];
    p.owner_end[j] = owner_end[j];
  }
  p.n_inst = static_cast<int32_t>(n_inst);
  p.n_dests = n_dests;  // cross-GPU: packed atomicMax into every rank's result buffer
  for (int j = 0; j < n_dests; ++j) p.dests[j] = reinterpret_cast<unsigned long long*>(dests[j]);
  const int dev = idx[0]->device;
  for (int64_t i = 0; i < n_inst; ++i) {
    KVX_REQUIRE(idx[i] != nullptr && idx[i]->device == dev,
                "kvx_hash_match_batch: NULL index or indices on different devices");
    p.keys[i] = idx[i]->keys;
    p.mask[i] = static_cast<uint64_t>(idx[i]->slots - 1);
    p.ids[i] = inst_ids[i];
  }
  DeviceGuard g(dev);
  // resident beside the hash (one 384-thread CTA per SM): a few 64-thread CTAs per SM
  const int blocks = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>(n_req, static_cast<int64_t>(sm_count(dev)) * 6)));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(64);
  cfg.stream = as_stream(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (n_req * n_inst <= 1024)
    KVX_CUDA(cudaLaunchKernelEx(&cfg, match_follow_kernel<2, 2, true>, p, d_keys, d_key_off,
                                n_req, d_len_out, d_best_len, d_best_id, d_order, d_claim));
  else
    KVX_CUDA(cudaLaunchKernelEx(&cfg, match_follow_kernel<2, 2, false>, p, d_keys, d_key_off,
                                n_req, d_len_out, d_best_len, d_best_id, d_order, d_claim));
  KVX_LAUNCH_CHECK("match_follow_kernel");
  return KVX_OK;
}
}  // namespace kvx

extern "C" int kvx_hash_match_check(void* stream) {
  int dev = -1;
  if (stream) {
    KVX_CUDA(cudaStreamGetDevice(as_stream(stream), &dev));
  } else {
    KVX_CUDA(cudaGetDevice(&dev));
  }
  DeviceGuard g(dev);
  KVX_CUDA(cudaStreamSynchronize(as_stream(stream)));
  unsigned long long t = 0, zero = 0;
  KVX_CUDA(cudaMemcpyFromSymbol(&t, g_queue_timeouts, sizeof(t)));
  if (!t) return KVX_OK;
  KVX_CUDA(cudaMemcpyToSymbol(g_queue_timeouts, &zero, sizeof(zero)));
  return set_error(KVX_ECUDA, "kvx_hash_match_check: a match task waited 5 s for keys the "
                              "hash never published; its results are missing");
}

// ---- cross-GPU best match without a collective --------------------------
// SURVEY 8(e) case ii: one prefill instance (or several) per GPU.  The match
// kernel of every rank atomically MAXes each request's packed word straight
// into EVERY rank's result buffer through CUDA IPC mappings (NVLink remote
// atomics), so the exchange is part of the kernel; 64-bit flags written with
// stream memory operations then tell each rank that all ranks' atomics have
// landed (no kernel spins on another's flag).  Result buffers are double
// buffered by step parity: a rank zeroes the buffer for step e+1 before it
// announces step e, and every rank starts step e+1 only after all step-e
// announcements, so no atomic can hit a buffer before it was zeroed.
//
// Request-sharded hashing (kvx_xmatch_key_buffer / kvx_xmatch_share_keys):
// every rank hashes only its shard of the batch into its copy of a shared key
// buffer, then copy-engine pushes that shard into every peer's copy (CUDA IPC)
// and raises a per-rank "keys of step e landed" flag there; each rank's
// stream waits for all peers' flags before its match.  A rank's pushes of
// step e+1 are queued after its xmatch_run of step e, which waited for every
// rank's step-e announcement (written after that rank's match kernel), so no
// push can overwrite keys a peer is still matching.
struct kvx_xmatch {
  int device = 0, rank = 0, world = 1;
  int64_t max_req = 0;
  // [buf0 | buf1 | flags | keyflags | readyflags | doneflags], KVX_MAX_PEERS words per flag set
  uint8_t* mem = nullptr;
  uint64_t* peer_buf[KVX_MAX_PEERS][2] = {};
  uint64_t* peer_flags[KVX_MAX_PEERS] = {};
  void* peer_mem[KVX_MAX_PEERS] = {};
  uint64_t epoch = 0;
  // shared key buffer (optional): two halves, by the parity of the fused step
  int64_t max_keys = 0;
  int64_t* keys = nullptr;
  uint64_t fused_epoch = 0;
  bool peer_same_gpu = false;  // some peer shares this physical GPU: no fused stage 1
  int32_t* order = nullptr;    // fused stage 1: whole-batch longest-first order + claim counter
  unsigned long long* claim = nullptr;
  uint8_t uuid[16] = {};
  int64_t* peer_keys[KVX_MAX_PEERS] = {};
  uint64_t key_epoch = 0;
  cudaStream_t copy_stream = nullptr;  // share_keys pushes; fused stage 1's side work
  cudaEvent_t copy_dep = nullptr;
  cudaEvent_t side_done = nullptr;  // fused stage 1: the side stream's order + preset
  uint64_t* buf(int b) const { return reinterpret_cast<uint64_t*>(mem) + b * max_req; }
  uint64_t* flags() const { return reinterpret_cast<uint64_t*>(mem) + 2 * max_req; }
  uint64_t* keyflags() const { return flags() + KVX_MAX_PEERS; }
  uint64_t* readyflags() const { return flags() + 2 * KVX_MAX_PEERS; }
  uint64_t* doneflags() const { return flags() + 3 * KVX_MAX_PEERS; }
  size_t bytes() const {
    return (2 * static_cast<size_t>(max_req) + 4 * KVX_MAX_PEERS) * sizeof(uint64_t);
  }
};

extern "C" {
static int xmatch_finish(kvx_xmatch* x, uint64_t e, int64_t n_req, int64_t* d_best_len,
                         int32_t* d_best_id, cudaStream_t s);
}

namespace {
struct XmatchBlob {
  int32_t magic, rank, world, pad;
  int64_t max_req;
  uint8_t handle[KVX_IPC_HANDLE_BYTES];
  int64_t max_keys;  // 0: no shared key buffer
  uint8_t key_handle[KVX_IPC_HANDLE_BYTES];
  uint8_t uuid[16];  // physical GPU
};
constexpr int32_t kXmatchMagic = 0x6b76786d;  // "kvxm"
}  // namespace

extern "C" {

int kvx_xmatch_create(int device, int rank, int world, int64_t max_req, kvx_xmatch** out) {
  KVX_REQUIRE(out != nullptr, "kvx_xmatch_create: NULL out");
  KVX_REQUIRE(world >= 1 && world <= KVX_MAX_PEERS && rank >= 0 && rank < world,
              "kvx_xmatch_create: bad rank / world");
  KVX_REQUIRE(max_req >= 1, "kvx_xmatch_create: max_req must be >= 1");
  DeviceGuard g(device);
  auto* x = new kvx_xmatch();
  x->device = device;
  x->rank = rank;
  x->world = world;
  x->max_req = max_req;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&x->mem), x->bytes());
  if (e == cudaSuccess) e = cudaMemset(x->mem, 0, x->bytes());
  if (e == cudaSuccess) e = cudaDeviceSynchronize();  // zeroed before any peer maps it
  if (e != cudaSuccess) {
    kvx_xmatch_destroy(x);
    return cuda_error(e, "kvx_xmatch_create");
  }
  x->peer_buf[rank][0] = x->buf(0);
  x->peer_buf[rank][1] = x->buf(1);
  x->peer_flags[rank] = x->flags();
  cudaDeviceProp prop{};
  if (cudaGetDeviceProperties(&prop, device) == cudaSuccess)
    std::memcpy(x->uuid, &prop.uuid, sizeof(x->uuid));
  *out = x;
  return KVX_OK;
}

int kvx_xmatch_destroy(kvx_xmatch* x) {
  if (!x) return KVX_OK;
  DeviceGuard g(x->device);
  cudaDeviceSynchronize();
  for (int j = 0; j < KVX_MAX_PEERS; ++j) {
    if (x->peer_mem[j]) kvx_ipc_close(x->peer_mem[j]);
    if (x->peer_keys[j] && j != x->rank) kvx_ipc_close(x->peer_keys[j]);
  }
  if (x->copy_stream) cudaStreamDestroy(x->copy_stream);
  if (x->copy_dep) cudaEventDestroy(x->copy_dep);
  if (x->side_done) cudaEventDestroy(x->side_done);
  if (x->keys) cudaFree(x->keys);
  if (x->order) cudaFree(x->order);
  if (x->claim) cudaFree(x->claim);
  if (x->mem) cudaFree(x->mem);
  delete x;
  return KVX_OK;
}

int kvx_xmatch_export(kvx_xmatch* x, uint8_t* blob, int64_t cap, int64_t* len) {
  KVX_REQUIRE(x && len, "kvx_xmatch_export: NULL argument");
  *len = static_cast<int64_t>(sizeof(XmatchBlob));
  if (!blob) return KVX_OK;
  KVX_REQUIRE(cap >= *len, "kvx_xmatch_export: blob too small");
  XmatchBlob b{};
  b.magic = kXmatchMagic;
  b.rank = x->rank;
  b.world = x->world;
  b.max_req = x->max_req;
  int rc = kvx_ipc_export(x->mem, b.handle);
  if (rc) return rc;
  b.max_keys = x->max_keys;
  std::memcpy(b.uuid, x->uuid, sizeof(b.uuid));
  if (x->keys) {
    rc = kvx_ipc_export(x->keys, b.key_handle);
    if (rc) return rc;
  }
  std::memcpy(blob, &b, sizeof(b));
  return KVX_OK;
}

int kvx_xmatch_connect(kvx_xmatch* x, const uint8_t* blob, int64_t len) {
  KVX_REQUIRE(x && blob && len >= static_cast<int64_t>(sizeof(XmatchBlob)),
              "kvx_xmatch_connect: bad blob");
  XmatchBlob b;
  std::memcpy(&b, blob, sizeof(b));
  KVX_REQUIRE(b.magic == kXmatchMagic && b.world == x->world && b.max_req == x->max_req &&
                  b.rank >= 0 && b.rank < x->world && b.max_keys == x->max_keys,
              "kvx_xmatch_connect: peer does not match (rank / world / max_req / key buffer)");
  if (b.rank == x->rank) return KVX_OK;  // self
  KVX_REQUIRE(x->peer_mem[b.rank] == nullptr, "kvx_xmatch_connect: peer already connected");
  if (std::memcmp(b.uuid, x->uuid, sizeof(b.uuid)) == 0) x->peer_same_gpu = true;
  void* p = nullptr;
  int rc = kvx_ipc_open(b.handle, x->device, &p);
  if (rc) return rc;
  x->peer_mem[b.rank] = p;
  auto* words = static_cast<uint64_t*>(p);
  x->peer_buf[b.rank][0] = words;
  x->peer_buf[b.rank][1] = words + x->max_req;
  x->peer_flags[b.rank] = words + 2 * x->max_req;
  if (x->max_keys) {
    rc = kvx_ipc_open(b.key_handle, x->device, &p);
    if (rc) return rc;
    x->peer_keys[b.rank] = static_cast<int64_t*>(p);
  }
  return KVX_OK;
}

int kvx_xmatch_key_buffer(kvx_xmatch* x, int64_t max_keys, int64_t** d_keys) {
  KVX_REQUIRE(x && d_keys && max_keys >= 1, "kvx_xmatch_key_buffer: bad arguments");
  if (x->keys) {
    KVX_REQUIRE(max_keys <= x->max_keys, "kvx_xmatch_key_buffer: already sized smaller");
    *d_keys = x->keys;
    return KVX_OK;
  }
  for (int j = 0; j < x->world; ++j)
    KVX_REQUIRE(j == x->rank || x->peer_mem[j] == nullptr,
                "kvx_xmatch_key_buffer: call before exporting / connecting");
  DeviceGuard g(x->device);
  KVX_CUDA(cudaMalloc(reinterpret_cast<void**>(&x->keys), 2 * sizeof(int64_t) * max_keys));
  KVX_CUDA(cudaStreamCreateWithFlags(&x->copy_stream, cudaStreamNonBlocking));
  KVX_CUDA(cudaEventCreateWithFlags(&x->copy_dep, cudaEventDisableTiming));
  KVX_CUDA(cudaEventCreateWithFlags(&x->side_done, cudaEventDisableTiming));
  x->max_keys = max_keys;
  x->peer_keys[x->rank] = x->keys;
  *d_keys = x->keys;
  return KVX_OK;
}

int kvx_xmatch_share_keys(kvx_xmatch* x, int64_t key_lo, int64_t key_hi, void* stream) {
  KVX_REQUIRE(x && x->keys, "kvx_xmatch_share_keys: no key buffer");
  KVX_REQUIRE(0 <= key_lo && key_lo <= key_hi && key_hi <= x->max_keys,
              "kvx_xmatch_share_keys: key range out of the buffer");
  for (int j = 0; j < x->world; ++j)
    KVX_REQUIRE(x->peer_keys[j] != nullptr, "kvx_xmatch_share_keys: not connected to every rank");
  DeviceGuard g(x->device);
  const uint64_t e = ++x->key_epoch;
  // the pushes follow this rank's hash of its shard (queued on `stream`)
  KVX_CUDA(cudaEventRecord(x->copy_dep, as_stream(stream)));
  KVX_CUDA(cudaStreamWaitEvent(x->copy_stream, x->copy_dep, 0));
  const size_t bytes = sizeof(int64_t) * static_cast<size_t>(key_hi - key_lo);
  for (int k = 1; k < x->world; ++k) {  // start with the next rank: spread the pushes
    const int j = (x->rank + k) % x->world;
    if (bytes)
      KVX_CUDA(cudaMemcpyAsync(x->peer_keys[j] + key_lo, x->keys + key_lo, bytes,
                               cudaMemcpyDefault, x->copy_stream));
  }
  for (int k = 1; k < x->world; ++k) {  // "my shard of step e landed" (after the copies)
    const int j = (x->rank + k) % x->world;
    int rc = kvx_signal_write(x->copy_stream, x->peer_flags[j] + KVX_MAX_PEERS + x->rank, e);
    if (rc) return rc;
  }
  for (int j = 0; j < x->world; ++j) {  // every peer's shard is here before the match
    if (j == x->rank) continue;
    int rc = kvx_signal_wait(stream, x->keyflags() + j, e);
    if (rc) return rc;
  }
  return KVX_OK;
}

int kvx_xmatch_run(kvx_xmatch* x, const kvx_index* const* idx, const int32_t* inst_ids,
                   int64_t n_inst, const int64_t* d_keys, const int64_t* d_key_off, int64_t n_req,
                   int64_t* d_best_len, int32_t* d_best_id, void* stream) {
  KVX_REQUIRE(x != nullptr, "kvx_xmatch_run: NULL exchange");
  KVX_REQUIRE(n_inst >= 1, "find_best_prefix_match: empty prefill pool");
  KVX_REQUIRE(n_inst <= KVX_MAX_INSTANCES, "kvx_xmatch_run: too many instances");
  KVX_REQUIRE(idx != nullptr && inst_ids != nullptr, "kvx_xmatch_run: NULL instances");
  KVX_REQUIRE(n_req >= 0 && n_req <= x->max_req, "kvx_xmatch_run: n_req out of range");
  KVX_REQUIRE(d_key_off && d_best_len && d_best_id, "kvx_xmatch_run: NULL array");
  for (int j = 0; j < x->world; ++j)
    KVX_REQUIRE(x->peer_buf[j][0] != nullptr, "kvx_xmatch_run: not connected to every rank");
  DeviceGuard g(x->device);
  cudaStream_t s = as_stream(stream);
  const uint64_t e = ++x->epoch;
  const int b = static_cast<int>(e & 1);
  uint64_t* dests[KVX_MAX_PEERS];
  for (int j = 0; j < x->world; ++j) dests[j] = x->peer_buf[j][b];
  if (n_req > 0) {
    int rc = match_impl(idx, inst_ids, n_inst, d_keys, d_key_off, n_req, nullptr, nullptr, nullptr,
                        true, stream, dests, x->world);
    if (rc) return rc;
  }
  return xmatch_finish(x, e, n_req, d_best_len, d_best_id, s);
}

// After every rank's match atomics for step e: announce, wait for all, unpack.
static int xmatch_finish(kvx_xmatch* x, uint64_t e, int64_t n_req, int64_t* d_best_len,
                         int32_t* d_best_id, cudaStream_t s) {
  const int b = static_cast<int>(e & 1);
  void* stream = s;
  // the other parity's buffer was unpacked last step: zero it before announcing
  KVX_CUDA(cudaMemsetAsync(x->buf(b ^ 1), 0, sizeof(uint64_t) * x->max_req, s));
  for (int j = 0; j < x->world; ++j) {  // "my atomics for step e have landed" -> every rank
    int rc = kvx_signal_write(stream, x->peer_flags[j] + x->rank, e);
    if (rc) return rc;
  }
  for (int j = 0; j < x->world; ++j) {  // wait for every rank's announcement
    int rc = kvx_signal_wait(stream, x->flags() + j, e);
    if (rc) return rc;
  }
  if (n_req > 0) {
    unpack_best_kernel<<<grid_for(n_req, 256, x->device), 256, 0, s>>>(
        reinterpret_cast<const unsigned long long*>(x->buf(b)), d_best_len, d_best_id, n_req);
    KVX_LAUNCH_CHECK("unpack_best_kernel");
  }
  return KVX_OK;
}


// Request-sharded stage 1 with the key exchange inside the match kernel (see
// kvx.h).  Per step e (parity par = e & 1 selects the key-buffer half):
//   wait ready(e) from every peer   (its half `par` is preset to -1)
//   hash this rank's shard into the local half `par`
//   follow: match the WHOLE batch against the local instances beside the
//           hash, reading each request's keys where its shard's GPU stores
//           them (local, or NVLink loads of the peer's half) as they appear;
//           packed atomicMax into every rank's result buffer
//   signal done(e) to every peer    (my reads of their half `par` ended)
//   announce / wait / unpack the results (xmatch_finish)
//   wait done(e - 1) from every peer, preset my half par ^ 1, signal ready(e + 1)
// Every wait is a stream memop; nothing blocks the host.  (Pushing each key
// into the peers' buffers from the hash kernel instead measured 407 us per
// Config 4 step on 2 GPUs: the remote stores stall the key-folding lane.)
int kvx_xmatch_hash_match(kvx_xmatch* x, const int32_t* d_tokens, const int64_t* d_tok_off,
                          const int64_t* shard_bounds, int64_t bs, const int64_t* d_key_off,
                          int64_t n_req, const kvx_index* const* idx, const int32_t* inst_ids,
                          int64_t n_inst, int64_t* d_best_len, int32_t* d_best_id,
                          int64_t** d_keys_out, void* stream) {
  KVX_REQUIRE(x && x->keys, "kvx_xmatch_hash_match: no key buffer");
  KVX_REQUIRE(n_inst >= 1, "find_best_prefix_match: empty prefill pool");
  KVX_REQUIRE(n_inst <= KVX_MAX_INSTANCES, "kvx_xmatch_hash_match: too many instances");
  KVX_REQUIRE(idx != nullptr && inst_ids != nullptr, "kvx_xmatch_hash_match: NULL instances");
  KVX_REQUIRE(n_req >= 1 && n_req <= x->max_req, "kvx_xmatch_hash_match: n_req out of range");
  KVX_REQUIRE(shard_bounds != nullptr && shard_bounds[0] == 0 && shard_bounds[x->world] == n_req,
              "kvx_xmatch_hash_match: shard bounds must run from 0 to n_req");
  for (int j = 0; j < x->world; ++j)
    KVX_REQUIRE(shard_bounds[j] <= shard_bounds[j + 1], "kvx_xmatch_hash_match: bad shard bounds");
  KVX_REQUIRE(d_tokens && d_tok_off && d_key_off && d_best_len && d_best_id,
              "kvx_xmatch_hash_match: NULL array");
  KVX_REQUIRE(bs >= 16 && bs % 16 == 0 && (reinterpret_cast<uintptr_t>(d_tokens) & 15) == 0,
              "kvx_xmatch_hash_match: needs bs % 16 == 0 and 16-byte aligned tokens");
  KVX_REQUIRE(!x->peer_same_gpu,
              "kvx_xmatch_hash_match: a peer shares this GPU (its kernels would wait on ours); "
              "use kvx_xmatch_share_keys + kvx_xmatch_run");
  for (int j = 0; j < x->world; ++j)
    KVX_REQUIRE(x->peer_keys[j] != nullptr && x->peer_buf[j][0] != nullptr,
                "kvx_xmatch_hash_match: not connected to every rank");
  DeviceGuard g(x->device);
  cudaStream_t s = as_stream(stream);
  if (!x->order) {
    KVX_CUDA(cudaMalloc(reinterpret_cast<void**>(&x->order), sizeof(int32_t) * x->max_req));
    KVX_CUDA(cudaMalloc(reinterpret_cast<void**>(&x->claim), 64));
  }
  const uint64_t e = ++x->fused_epoch;
  const int par = static_cast<int>(e & 1);
  int64_t* mine = x->keys + par * x->max_keys;
  // a half is preset whole (all bytes 0xff: every key -1), so the next step
  // may be a batch of any size
  const size_t half_bytes = sizeof(int64_t) * static_cast<size_t>(x->max_keys);
  int rc = KVX_OK;
  if (e == 1) {  // the first step's half: preset and announce
    KVX_CUDA(cudaMemsetAsync(mine, 0xff, half_bytes, s));
    for (int j = 0; j < x->world; ++j) {
      if (j == x->rank) continue;
      rc = kvx_signal_write(stream, x->peer_flags[j] + 2 * KVX_MAX_PEERS + x->rank, e);
      if (rc) return rc;
    }
  } else {  // this step's half was preset by the previous step's side work
    KVX_CUDA(cudaStreamWaitEvent(s, x->side_done, 0));
  }
  // Side stream, beside this step's hash: the whole-batch order for the
  // follower, then the NEXT step's half -- once every peer has finished
  // reading it (step e - 1) -- preset and announced.
  KVX_CUDA(cudaEventRecord(x->copy_dep, s));
  KVX_CUDA(cudaStreamWaitEvent(x->copy_stream, x->copy_dep, 0));
  // whole-batch longest-first order for the follower (also zeroes its claim counter)
  rc = order_by_length(d_key_off, n_req, x->order, x->claim, x->copy_stream);
  if (rc) return rc;
  KVX_CUDA(cudaEventRecord(x->copy_dep, x->copy_stream));
  for (int j = 0; j < x->world; ++j) {
    if (j == x->rank) continue;
    rc = kvx_signal_wait(x->copy_stream, x->doneflags() + j, e - 1);
    if (rc) return rc;
  }
  KVX_CUDA(cudaMemsetAsync(x->keys + (par ^ 1) * x->max_keys, 0xff, half_bytes, x->copy_stream));
  for (int j = 0; j < x->world; ++j) {
    if (j == x->rank) continue;
    rc = kvx_signal_write(x->copy_stream, x->peer_flags[j] + 2 * KVX_MAX_PEERS + x->rank, e + 1);
    if (rc) return rc;
  }
  KVX_CUDA(cudaEventRecord(x->side_done, x->copy_stream));
  for (int j = 0; j < x->world; ++j) {  // every peer's half `par` is preset
    if (j == x->rank) continue;
    rc = kvx_signal_wait(stream, x->readyflags() + j, e);
    if (rc) return rc;
  }
  KVX_CUDA(cudaStreamWaitEvent(s, x->copy_dep, 0));  // the order
  const int64_t r0 = shard_bounds[x->rank], r1 = shard_bounds[x->rank + 1];
  if (r1 > r0) {
    bool published = false;
    rc = hash_publish_launch(d_tokens, d_tok_off + r0, r1 - r0, bs, d_key_off + r0, mine, stream,
                             &published);
    if (rc) return rc;
    KVX_REQUIRE(published, "kvx_xmatch_hash_match: the publishing hash kernel did not run");
  }
  const uint64_t me = ++x->epoch;  // the result exchange's own step counter
  const int b = static_cast<int>(me & 1);
  uint64_t* dests[KVX_MAX_PEERS];
  const int64_t* owners[KVX_MAX_PEERS];
  int64_t owner_end[KVX_MAX_PEERS];
  for (int j = 0; j < x->world; ++j) {
    dests[j] = x->peer_buf[j][b];
    owners[j] = x->peer_keys[j] + par * x->max_keys;  // peer_keys[rank] is the local buffer
    owner_end[j] = shard_bounds[j + 1];
  }
  rc = match_follow_launch(idx, inst_ids, n_inst, mine, d_key_off, n_req, nullptr, nullptr,
                           nullptr, x->order, x->claim, stream, dests, x->world, owners,
                           owner_end, x->world);
  if (rc) return rc;
  for (int j = 0; j < x->world; ++j) {  // my reads of every peer's half `par` are done
    if (j == x->rank) continue;
    rc = kvx_signal_write(stream, x->peer_flags[j] + 3 * KVX_MAX_PEERS + x->rank, e);
    if (rc) return rc;
  }
  rc = xmatch_finish(x, me, n_req, d_best_len, d_best_id, s);
  if (rc) return rc;
  if (d_keys_out) *d_keys_out = mine;
  return KVX_OK;
}

}  // extern "C"
