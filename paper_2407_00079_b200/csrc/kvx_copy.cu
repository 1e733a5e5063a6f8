// kvx_copy.cu -- paged KV pools and the byte stages: K3 gather (stage 2),
// K5 scatter (stage 4) and the fused paged -> paged copy (stages 2+3+4, whose
// destination may be a peer GPU's pool mapped over NVLink).
//
// There is no byte-level reference.  What moves is defined
// by the reference's block selection: the whole hash_ids chain of a request
// for the prefill -> decode stream (proj/src/sim_engine.cpp:463-464), a chain
// range [local_prefix, used_prefix) for a migration
// (proj/src/sim_engine.cpp:405-416), landing positions per insert_replicated
// (proj/src/kvcache.cpp:133-148).  Sizes follow kv_bytes_per_token
// (proj/src/config.cpp:216).
//
// Every stage is one generic slab copy: unit u = (plane, b) with plane =
// (layer - lo)*2 + kv; the source / destination address of a unit is either
// a paged slot (table[b]) or a contiguous buffer position (b).  Two
// implementations, both HBM-bound (no tensor-core work exists here):
//   LSU  -- 512-thread CTAs, each CTA streams work items of up to 32 KiB:
//           128-bit loads (ld.global.nc.L1::no_allocate) of the next item are
//           issued before the current item's evict-first (.cs) stores, 8 per
//           thread in flight.
//   TMA  -- one elected thread per CTA drives cp.async.bulk global->shared
//           (mbarrier complete_tx) and shared->global bulk stores through a
//           shared-memory ring (default 6 x 16 KiB stages, 4 loads in
//           flight, 2 CTAs per SM = 128 KiB per SM) with no register staging.
// Measured (Config 2, N=1): LSU 0.966 of HBM, TMA 0.91 -- LSU is the default.
#include <algorithm>
#include <cstdlib>

#include "kvx_common.cuh"

namespace kvx {
namespace {

int g_copy_impl = 0;

// CTAs of a copy that crosses PCIe (a host pool on either side).  16 CTAs x
// 512 threads x 8 x 16 B in flight = 1 MiB outstanding, well above the
// PCIe bandwidth-delay product; KVX_HOST_COPY_CTAS overrides (measurement).
int host_copy_ctas() {
  static const int v = [] {
    const char* e = std::getenv("KVX_HOST_COPY_CTAS");
    const int x = e ? std::atoi(e) : 16;
    return x >= 1 ? x : 16;
  }();
  return v;
}

struct SlabCopy {
  const uint8_t* src;
  uint8_t* dst;
  int64_t src_plane;  // bytes between (layer, kv) planes on the source side
  int64_t dst_plane;
  const int32_t* src_table;  // NULL: contiguous side
  const int32_t* dst_table;
  int64_t n;       // blocks per plane
  int64_t planes;  // (hi - lo) * 2
  int64_t slab;    // bytes per unit, multiple of 16
  uint32_t src_slots;  // valid table entries: [0, slots) (paged sides; < 2^31)
  uint32_t dst_slots;
};

// Set when a table entry outside [0, slots) was met (that block is skipped,
// not copied), per device; kvx_copy_check() reports and clears it.
__device__ unsigned long long g_bad_table_entries = 0;
// Set when a pull copy gave up waiting for its readiness flag (kvx_copy_check).
__device__ unsigned long long g_wait_timeouts = 0;

__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Coherent 16-B load (the pull copy reads a peer pool that another GPU
// writes while the kernel may already be running: the read-only .nc path is
// not ordered by the flag acquire).
__device__ __forceinline__ int4 ld_coherent(const int4* p) {
  int4 r;
  asm volatile("ld.global.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p)
               : "memory");
  return r;
}

// Addresses of unit u; false (and flagged) when a table entry is out of range.
template <class Idx = int64_t>
__device__ __forceinline__ bool unit_addrs(const SlabCopy& c, Idx u, const uint8_t*& s,
                                           uint8_t*& d, bool count = false) {
  const Idx n = static_cast<Idx>(c.n);
  const Idx plane = u / n;
  const Idx b = u - plane * n;
  // one unsigned 32-bit compare per side also rejects negative entries
  const uint32_t sb = c.src_table ? static_cast<uint32_t>(__ldg(c.src_table + b))
                                  : static_cast<uint32_t>(b);
  const uint32_t db = c.dst_table ? static_cast<uint32_t>(__ldg(c.dst_table + b))
                                  : static_cast<uint32_t>(b);
  const bool ok = sb < c.src_slots && db < c.dst_slots;
  s = c.src + static_cast<int64_t>(plane) * c.src_plane + static_cast<int64_t>(sb) * c.slab;
  d = c.dst + static_cast<int64_t>(plane) * c.dst_plane + static_cast<int64_t>(db) * c.slab;
  if (!ok && count) g_bad_table_entries = 1;  // a plain idempotent store: no atomics in the copy loop
  return ok;
}

constexpr int kLsuThreads = 512;
constexpr int kLsuUnroll = 4;
constexpr int64_t kLsuItem = 16LL * kLsuThreads * kLsuUnroll;  // 32 KiB

// Plain form (one work item in flight per thread; write-back stores).  Kept as
// the KVX_LSU_VARIANT=1 measurement baseline.
__global__ void __launch_bounds__(kLsuThreads) copy_lsu_plain_kernel(const SlabCopy c) {
  const int64_t parts = (c.slab + kLsuItem - 1) / kLsuItem;
  const int64_t items = c.planes * c.n * parts;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int64_t u = it / parts;
    const int64_t off = (it - u * parts) * kLsuItem;
    const uint8_t* s;
    uint8_t* d;
    const bool ok = unit_addrs(c, u, s, d, off == 0);
    const int64_t bytes = ok ? min(kLsuItem, c.slab - off) : 0;
    const int4* sv = reinterpret_cast<const int4*>(s + off);
    int4* dv = reinterpret_cast<int4*>(d + off);
    const int nv = static_cast<int>(bytes >> 4);
    int4 r[kLsuUnroll];
#pragma unroll
    for (int j = 0; j < kLsuUnroll; ++j) {
      const int v = threadIdx.x + j * kLsuThreads;
      if (v < nv) r[j] = ld_stream(sv + v);
    }
#pragma unroll
    for (int j = 0; j < kLsuUnroll; ++j) {
      const int v = threadIdx.x + j * kLsuThreads;
      if (v < nv) dv[v] = r[j];
    }
  }
}

__device__ __forceinline__ void st_stream(int4* p, const int4& v) {
  asm volatile("st.global.cs.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// The LSU copy kernel: evict-first (.cs) stores -- the copied KV is not read
// again soon, so it should not displace L2 lines -- and the next work item's
// loads issued before the current item's stores (8 x 16 B in flight per
// thread).  r01: 0.966 of the measured HBM copy peak vs 0.951 for the plain
// form.
// Idx: uint32_t when the launch has < 2^32 work items (the host checks), so
// the per-item index arithmetic is 32-bit (64-bit division is a long
// subroutine that also cost the kernel register spills).
template <bool kCsStores, bool kPipelined, class Idx, bool kCoherent = false>
__device__ __forceinline__ void lsu_copy(const SlabCopy& c) {
  const Idx parts = static_cast<Idx>((c.slab + kLsuItem - 1) / kLsuItem);
  const Idx items = static_cast<Idx>(c.planes * c.n * parts);
  int4 r[kLsuUnroll];
  int nv = 0;
  int4* dv = nullptr;
  auto load = [&](Idx it, int4 (&buf)[kLsuUnroll], int& n, int4*& dst) {
    const Idx u = it / parts;
    const int64_t off = static_cast<int64_t>(it - u * parts) * kLsuItem;
    const uint8_t* s;
    uint8_t* d;
    const bool ok = unit_addrs<Idx>(c, u, s, d, off == 0);
    n = ok ? static_cast<int>(min(kLsuItem, c.slab - off) >> 4) : 0;
    const int4* sv = reinterpret_cast<const int4*>(s + off);
    dst = reinterpret_cast<int4*>(d + off);
#pragma unroll
    for (int j = 0; j < kLsuUnroll; ++j) {
      const int v = threadIdx.x + j * kLsuThreads;
      if (v < n) buf[j] = kCoherent ? ld_coherent(sv + v) : ld_stream(sv + v);
    }
  };
  auto store = [&](const int4 (&buf)[kLsuUnroll], int n, int4* dst) {
#pragma unroll
    for (int j = 0; j < kLsuUnroll; ++j) {
      const int v = threadIdx.x + j * kLsuThreads;
      if (v < n) {
        if (kCsStores) st_stream(dst + v, buf[j]);
        else dst[v] = buf[j];
      }
    }
  };
  Idx it = blockIdx.x;
  if (it >= items) return;
  load(it, r, nv, dv);
  for (; it < items; it += gridDim.x) {
    if (kPipelined && it + gridDim.x < items) {
      int4 r2[kLsuUnroll];
      int nv2;
      int4* dv2;
      load(it + gridDim.x, r2, nv2, dv2);
      store(r, nv, dv);
#pragma unroll
      for (int j = 0; j < kLsuUnroll; ++j) r[j] = r2[j];
      nv = nv2;
      dv = dv2;
    } else {
      store(r, nv, dv);
      if (it + gridDim.x < items) load(it + gridDim.x, r, nv, dv);
    }
  }
}

template <class Idx>
__global__ void __launch_bounds__(kLsuThreads, 2) copy_lsu_kernel(const SlabCopy c) {
  // A launch made with programmatic stream serialization (the streamer's
  // independent layer-wise units) lets the next unit's CTAs start now; with
  // no programmatic dependent this is a no-op.
  asm volatile("griddepcontrol.launch_dependents;");
  lsu_copy<true, true, Idx>(c);
}

// PEER_PULL receiver, one layer-wise unit = a one-warp gate kernel + the pull
// copy launched programmatically dependent on it.  The gate waits for the
// sender's readiness flag (system-scope acquire; the sender's stream write
// fences the unit's KV first) and only then releases the copy, so while the
// decode GPU waits for a slow prefill exactly ONE warp is resident -- the
// copy's CTAs are not scheduled ahead of their data (they would otherwise
// occupy every SM and starve decode kernels).  The gate itself is launched
// programmatically dependent on the previous unit's copy, so in steady state
// it has already passed when that copy drains and unit k+1 ramps up while unit
// k finishes.  Gives up after 20 s: *status (the streamer's failure word) and
// g_wait_timeouts are set, the copies skip, kvx_streamer_check /
// kvx_copy_check report it instead of the GPU hanging.
__global__ void __launch_bounds__(32) pull_gate_kernel(const unsigned long long* __restrict__ flag,
                                                       unsigned long long value,
                                                       unsigned long long* __restrict__ status) {
  if (threadIdx.x == 0) {
    unsigned long long t0, t, v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    unsigned ns = 32;
    while (true) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
      if (v >= value) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 20000000000ull) {
        *status = 1;
        g_wait_timeouts = 1;
        break;
      }
      __nanosleep(ns);
      ns = ns < 1024 ? 2 * ns : ns;
    }
  }
  __syncwarp();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// The pull copy: coherent loads of the peer pool (another GPU wrote it while
// this grid may already have been launched), evict-first local stores.  It
// is launched (programmatically dependent on its gate) only once the gate saw
// the unit's flag, so thread 0's own system-scope acquire of the flag passes
// at once and orders the CTA's loads after the sender's writes (the CTA
// barrier carries it); it does NOT wait for the gate grid to complete, which
// would serialise it behind the previous unit's copy.  A gate that timed out
// raised *status: the copy then skips.  Then the next unit's gate may be
// scheduled.
template <class Idx>
__global__ void __launch_bounds__(kLsuThreads, 2) copy_pull_kernel(
    const SlabCopy c, const unsigned long long* __restrict__ flag, unsigned long long value,
    const unsigned long long* __restrict__ status) {
  __shared__ int go;
  if (threadIdx.x == 0) {
    int ok = 1;
    while (true) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
      if (v >= value) break;
      if (*reinterpret_cast<const volatile unsigned long long*>(status)) {
        ok = 0;
        break;
      }
      __nanosleep(64);
    }
    go = ok;
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (go) lsu_copy<true, true, Idx, true>(c);
}

// Receiver -> sender "source blocks consumed" word of a PEER_PULL step: the
// consumed unit count, with bit 62 set when a unit of the step timed out (the
// sender's GEQ wait passes either way; the receiver's host sees the failure
// through kvx_streamer_check).
__global__ void pull_done_kernel(const unsigned long long* __restrict__ status,
                                 unsigned long long* __restrict__ peer_flag,
                                 unsigned long long value) {
  const unsigned long long v = *status ? (value | (1ull << 62)) : value;
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(peer_flag), "l"(v) : "memory");
}

// ---- TMA bulk-copy pipeline ----------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_load(void* smem, const void* gsrc, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(smem)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_store(void* gdst, const void* smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(smem)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int STAGES, int AHEAD, int STAGE_BYTES>
__global__ void __launch_bounds__(32) copy_tma_kernel(const SlabCopy c) {
  static_assert(AHEAD < STAGES, "need a free stage beyond the loads in flight");
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[STAGES];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");

  constexpr int64_t kStage = STAGE_BYTES;
  const int64_t parts = (c.slab + kStage - 1) / kStage;
  const int64_t items = c.planes * c.n * parts;
  // this CTA's items: blockIdx.x, blockIdx.x + gridDim.x, ...
  const int64_t mine = items > blockIdx.x ? (items - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  auto item_addr = [&](int64_t k, const uint8_t*& s, uint8_t*& d, uint32_t& bytes, bool count) {
    const int64_t it = blockIdx.x + k * gridDim.x;
    const int64_t u = it / parts;
    const int64_t off = (it - u * parts) * kStage;
    const bool ok = unit_addrs(c, u, s, d);
    s += off;
    d += off;
    bytes = ok ? static_cast<uint32_t>(min(kStage, c.slab - off)) : 0u;
    if (!ok && count) g_bad_table_entries = 1;
  };

  for (int64_t k = 0; k < mine + AHEAD; ++k) {
    // consume item k - AHEAD: its load has landed -> bulk store it out
    const int64_t kc = k - AHEAD;
    if (kc >= 0) {
      const int st = static_cast<int>(kc % STAGES);
      mbar_wait(&bars[st], static_cast<uint32_t>((kc / STAGES) & 1));
      const uint8_t* s;
      uint8_t* d;
      uint32_t bytes;
      item_addr(kc, s, d, bytes, false);
      if (bytes) bulk_store(d, smem + st * kStage, bytes);
      else asm volatile("cp.async.bulk.commit_group;" ::: "memory");  // keep the group count
    }
    // produce item k into its stage once the store that last used it (item
    // k - STAGES; stores committed so far: items <= kc) has read shared memory
    if (k < mine) {
      if (k >= STAGES) bulk_wait_read<STAGES - AHEAD>();
      const int st = static_cast<int>(k % STAGES);
      const uint8_t* s;
      uint8_t* d;
      uint32_t bytes;
      item_addr(k, s, d, bytes, true);
      mbar_expect_tx(&bars[st], bytes);  // 0 bytes: the arrive alone completes the phase
      if (bytes) bulk_load(smem + st * kStage, s, bytes, &bars[st]);
    }
  }
  bulk_wait_all();
}

// TMA pipeline shapes: {stages, loads in flight, stage bytes, CTAs per SM}.
// Bytes in flight per SM = loads in flight x stage bytes x CTAs per SM.
template <int STAGES, int AHEAD, int STAGE_BYTES>
int launch_tma(const SlabCopy& c, int dev, int ctas_per_sm, cudaStream_t s) {
  constexpr int kSmem = STAGES * STAGE_BYTES;
  static bool attr_set[64] = {false};
  if (dev >= 0 && dev < 64 && !attr_set[dev]) {
    KVX_CUDA(cudaFuncSetAttribute(copy_tma_kernel<STAGES, AHEAD, STAGE_BYTES>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    attr_set[dev] = true;
  }
  const int64_t items = c.planes * c.n * ((c.slab + STAGE_BYTES - 1) / STAGE_BYTES);
  const int blocks = static_cast<int>(
      std::min<int64_t>(items, static_cast<int64_t>(sm_count(dev)) * ctas_per_sm));
  copy_tma_kernel<STAGES, AHEAD, STAGE_BYTES><<<blocks, 32, kSmem, s>>>(c);
  KVX_LAUNCH_CHECK("copy_tma_kernel");
  return KVX_OK;
}

// overlap_prev: launch with programmatic stream serialization (the copy may
// start while the previous kernel on the stream runs; caller guarantees the
// two touch disjoint bytes).  LSU copy only.
// max_ctas > 0 caps the grid (copies that cross PCIe: a few CTAs keep the link
// busy and leave the other SMs to compute).
int launch_copy(const SlabCopy& c, int dev, cudaStream_t s, bool overlap_prev = false,
                int max_ctas = 0) {
  const int64_t units = c.planes * c.n;
  if (units == 0 || c.slab == 0) return KVX_OK;
  const int sms = sm_count(dev);
  if (g_copy_impl == 1 && max_ctas == 0) {
    static const int cfg = [] {
      const char* e = std::getenv("KVX_TMA_CFG");  // tuning knob
      return e ? std::atoi(e) : 0;
    }();
    // One issuing thread per CTA is the limiter with a single CTA per SM
    // (r01 sweep: 12x16K/8 ahead, 1 CTA/SM = 0.55 of HBM; 6x16K/4 ahead,
    // 2 CTAs/SM = 0.92), so the default runs several CTAs per SM.
    switch (cfg) {
      case 1: return launch_tma<8, 4, 16384>(c, dev, 1, s);    //  64 KB in flight / SM
      case 3: return launch_tma<6, 4, 32768>(c, dev, 1, s);    // 128 KB
      case 4: return launch_tma<4, 2, 16384>(c, dev, 4, s);    // 128 KB
      case 5: return launch_tma<6, 4, 16384>(c, dev, 3, s);    // 192 KB
      case 6: return launch_tma<12, 8, 16384>(c, dev, 1, s);   // 128 KB, one CTA per SM
      default: return launch_tma<6, 4, 16384>(c, dev, 2, s);   // 128 KB
    }
  } else {
    static const int ctas_per_sm = [] {
      const char* e = std::getenv("KVX_LSU_CTAS");  // tuning knob (default 4 = 2048 threads/SM)
      const int v = e ? std::atoi(e) : 4;
      return v >= 1 && v <= 4 ? v : 4;
    }();
    const int64_t items = units * ((c.slab + kLsuItem - 1) / kLsuItem);
    int64_t cap = static_cast<int64_t>(sms) * ctas_per_sm;
    if (max_ctas > 0) cap = std::min<int64_t>(cap, max_ctas);
    const int blocks = static_cast<int>(std::min<int64_t>(items, cap));
    static const int variant = [] {
      const char* e = std::getenv("KVX_LSU_VARIANT");  // measurement knob
      return e ? std::atoi(e) : 0;
    }();
    if (variant == 1) {
      copy_lsu_plain_kernel<<<blocks, kLsuThreads, 0, s>>>(c);
    } else if (overlap_prev) {
      // programmatic dependent launch: this copy may start while the previous
      // kernel on the stream is still running (caller guarantees independence)
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(blocks);
      cfg.blockDim = dim3(kLsuThreads);
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      if (items + blocks < (int64_t{1} << 32))
        KVX_CUDA(cudaLaunchKernelEx(&cfg, copy_lsu_kernel<uint32_t>, c));
      else
        KVX_CUDA(cudaLaunchKernelEx(&cfg, copy_lsu_kernel<int64_t>, c));
    } else if (items + blocks < (int64_t{1} << 32)) {
      copy_lsu_kernel<uint32_t><<<blocks, kLsuThreads, 0, s>>>(c);
    } else {
      copy_lsu_kernel<int64_t><<<blocks, kLsuThreads, 0, s>>>(c);
    }
    KVX_LAUNCH_CHECK("copy_lsu_kernel");
  }
  return KVX_OK;
}

// ---- synthetic content ------------------------------------------------------

__global__ void __launch_bounds__(256) fill_kernel(uint8_t* __restrict__ base, uint32_t pool_id,
                                                   int64_t slots, int64_t units, int64_t slab) {
  const int64_t words = slab >> 3;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int64_t lk = u / slots;
    const int64_t slot = u - lk * slots;
    const uint64_t seed = slab_seed(pool_id, static_cast<uint32_t>(lk >> 1),
                                    static_cast<uint32_t>(lk & 1), static_cast<uint32_t>(slot));
    ulonglong2* p = reinterpret_cast<ulonglong2*>(base + u * slab);
    for (int64_t v = threadIdx.x; v < (words >> 1); v += blockDim.x) {
      ulonglong2 w;
      w.x = mix64(seed + 2 * v);
      w.y = mix64(seed + 2 * v + 1);
      p[v] = w;
    }
  }
}

__global__ void __launch_bounds__(256) verify_kernel(const uint8_t* __restrict__ base,
                                                     int64_t slots, int64_t slab,
                                                     const int32_t* __restrict__ dst_table,
                                                     uint32_t src_pool_id,
                                                     const int32_t* __restrict__ src_table,
                                                     int64_t n, int32_t layer_lo, int64_t planes,
                                                     unsigned long long* __restrict__ mismatch) {
  const int64_t words = slab >> 3;
  unsigned long long bad = 0;
  for (int64_t u = blockIdx.x; u < planes * n; u += gridDim.x) {
    const int64_t plane = u / n;
    const int64_t b = u - plane * n;
    const int64_t layer = layer_lo + (plane >> 1);
    const int kv = static_cast<int>(plane & 1);
    if (dst_table[b] < 0 || dst_table[b] >= slots || src_table[b] < 0) {  // out of range: all words bad
      if (threadIdx.x == 0) bad += static_cast<unsigned long long>(words);
      continue;
    }
    const uint64_t seed = slab_seed(src_pool_id, static_cast<uint32_t>(layer),
                                    static_cast<uint32_t>(kv),
                                    static_cast<uint32_t>(src_table[b]));
    const ulonglong2* p = reinterpret_cast<const ulonglong2*>(
        base + ((layer * 2 + kv) * slots + dst_table[b]) * slab);
    for (int64_t v = threadIdx.x; v < (words >> 1); v += blockDim.x) {
      const ulonglong2 w = p[v];
      bad += (w.x != mix64(seed + 2 * v)) + (w.y != mix64(seed + 2 * v + 1));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) bad += __shfl_down_sync(0xffffffffu, bad, o);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(mismatch, bad);
}

}  // namespace
}  // namespace kvx

using namespace kvx;

struct kvx_pool {
  kvx_pool_desc d;
  int64_t slab = 0;
  int64_t bytes = 0;
  uint8_t* base = nullptr;
  bool owned = false;
  bool host = false;  // pinned, device-mapped CPU DRAM (the KVCache DRAM tier)
};

namespace {

int check_desc(const kvx_pool_desc* d) {
  KVX_REQUIRE(d != nullptr, "kvx_pool: NULL descriptor");
  KVX_REQUIRE(d->layers >= 1 && d->layers <= 32767, "kvx_pool: layers must be in [1, 32767]");
  KVX_REQUIRE(d->block_size >= 1 && d->heads >= 1 && d->head_dim >= 1,
              "kvx_pool: block_size, heads, head_dim must be >= 1");
  KVX_REQUIRE(d->dtype_bytes == 1 || d->dtype_bytes == 2 || d->dtype_bytes == 4,
              "kvx_pool: dtype_bytes must be 1, 2 or 4");
  KVX_REQUIRE(d->slots >= 1 && d->slots <= 0x7FFFFFFF, "kvx_pool: slots must be in [1, 2^31)");
  const int64_t slab = static_cast<int64_t>(d->block_size) * d->heads * d->head_dim * d->dtype_bytes;
  KVX_REQUIRE(slab % 16 == 0, "kvx_pool: slab bytes must be a multiple of 16");
  return KVX_OK;
}

int check_range(const kvx_pool* p, int64_t n, int32_t lo, int32_t hi) {
  KVX_REQUIRE(p != nullptr, "NULL pool");
  KVX_REQUIRE(n >= 0, "block count must be >= 0");
  KVX_REQUIRE(lo >= 0 && lo <= hi && hi <= p->d.layers, "bad layer range");
  return KVX_OK;
}

}  // namespace

namespace kvx {
namespace {
// Checks and the SlabCopy of a paged -> paged copy of blocks [0, n), layers [lo, hi).
int paged_copy_args(const kvx_pool* src, const int32_t* d_src_table, const kvx_pool* dst,
                    const int32_t* d_dst_table, int64_t n, int32_t lo, int32_t hi, SlabCopy* c,
                    bool* empty) {
  int st = check_range(src, n, lo, hi);
  if (st) return st;
  st = check_range(dst, n, lo, hi);
  if (st) return st;
  KVX_REQUIRE(src->slab == dst->slab, "kvx_copy_paged: slab sizes differ");
  *empty = n == 0 || lo == hi;
  if (*empty) return KVX_OK;
  KVX_REQUIRE(d_src_table && d_dst_table, "kvx_copy_paged: NULL table");
  c->src = src->base + static_cast<int64_t>(lo) * 2 * src->d.slots * src->slab;
  c->src_plane = src->d.slots * src->slab;
  c->src_table = d_src_table;
  c->dst = dst->base + static_cast<int64_t>(lo) * 2 * dst->d.slots * dst->slab;
  c->dst_plane = dst->d.slots * dst->slab;
  c->dst_table = d_dst_table;
  c->n = n;
  c->src_slots = static_cast<uint32_t>(src->d.slots);
  c->dst_slots = static_cast<uint32_t>(dst->d.slots);
  c->planes = static_cast<int64_t>(hi - lo) * 2;
  c->slab = src->slab;
  return KVX_OK;
}
}  // namespace
}  // namespace kvx

extern "C" {

int kvx_pool_create(const kvx_pool_desc* desc, kvx_pool** out) {
  int st = check_desc(desc);
  if (st) return st;
  KVX_REQUIRE(out != nullptr, "kvx_pool_create: out is NULL");
  DeviceGuard g(desc->device);
  auto* p = new kvx_pool();
  p->d = *desc;
  p->slab = static_cast<int64_t>(desc->block_size) * desc->heads * desc->head_dim * desc->dtype_bytes;
  p->bytes = static_cast<int64_t>(desc->layers) * 2 * desc->slots * p->slab;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&p->base), static_cast<size_t>(p->bytes));
  if (e != cudaSuccess) {
    delete p;
    return cuda_error(e, "kvx_pool_create: cudaMalloc");
  }
  p->owned = true;
  *out = p;
  return KVX_OK;
}

int kvx_pool_create_view(const kvx_pool_desc* desc, void* d_base, kvx_pool** out) {
  int st = check_desc(desc);
  if (st) return st;
  KVX_REQUIRE(out != nullptr && d_base != nullptr, "kvx_pool_create_view: NULL");
  KVX_REQUIRE((reinterpret_cast<uintptr_t>(d_base) & 15) == 0,
              "kvx_pool_create_view: base must be 16-byte aligned");
  auto* p = new kvx_pool();
  p->d = *desc;
  p->slab = static_cast<int64_t>(desc->block_size) * desc->heads * desc->head_dim * desc->dtype_bytes;
  p->bytes = static_cast<int64_t>(desc->layers) * 2 * desc->slots * p->slab;
  p->base = static_cast<uint8_t*>(d_base);
  p->owned = false;
  *out = p;
  return KVX_OK;
}

int kvx_pool_create_host(const kvx_pool_desc* desc, kvx_pool** out) {
  int st = check_desc(desc);
  if (st) return st;
  KVX_REQUIRE(out != nullptr, "kvx_pool_create_host: out is NULL");
  DeviceGuard g(desc->device);
  auto* p = new kvx_pool();
  p->d = *desc;
  p->slab = static_cast<int64_t>(desc->block_size) * desc->heads * desc->head_dim * desc->dtype_bytes;
  p->bytes = static_cast<int64_t>(desc->layers) * 2 * desc->slots * p->slab;
  // pinned + mapped: kernels on any GPU address it directly (UVA: the host
  // pointer is the device pointer), reads and writes cross PCIe
  cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&p->base), static_cast<size_t>(p->bytes),
                                cudaHostAllocPortable | cudaHostAllocMapped);
  if (e != cudaSuccess) {
    delete p;
    return cuda_error(e, "kvx_pool_create_host: cudaHostAlloc");
  }
  p->owned = true;
  p->host = true;
  *out = p;
  return KVX_OK;
}

int kvx_pool_is_host(const kvx_pool* p) { return p && p->host ? 1 : 0; }

int kvx_pool_destroy(kvx_pool* p) {
  if (!p) return KVX_OK;
  if (p->owned && p->base && p->host) {
    cudaFreeHost(p->base);
  } else if (p->owned && p->base) {
    DeviceGuard g(p->d.device);
    cudaFree(p->base);
  }
  delete p;
  return KVX_OK;
}

void* kvx_pool_base(const kvx_pool* p) { return p ? p->base : nullptr; }
int64_t kvx_pool_slab_bytes(const kvx_pool* p) { return p ? p->slab : 0; }
int64_t kvx_pool_bytes(const kvx_pool* p) { return p ? p->bytes : 0; }
int kvx_pool_device(const kvx_pool* p) { return p ? p->d.device : -1; }
int32_t kvx_pool_layers(const kvx_pool* p) { return p ? p->d.layers : 0; }

int kvx_set_copy_impl(int impl) {
  KVX_REQUIRE(impl == 0 || impl == 1, "kvx_set_copy_impl: impl must be 0 (LSU) or 1 (TMA)");
  g_copy_impl = impl;
  return KVX_OK;
}

int kvx_pool_fill_synthetic(kvx_pool* p, uint32_t pool_id, void* stream) {
  KVX_REQUIRE(p != nullptr, "kvx_pool_fill_synthetic: NULL pool");
  DeviceGuard g(p->d.device);
  const int64_t units = static_cast<int64_t>(p->d.layers) * 2 * p->d.slots;
  const int blocks = static_cast<int>(std::min<int64_t>(units, sm_count(p->d.device) * 8));
  fill_kernel<<<blocks, 256, 0, as_stream(stream)>>>(p->base, pool_id, p->d.slots, units, p->slab);
  KVX_LAUNCH_CHECK("fill_kernel");
  return KVX_OK;
}

int kvx_pool_verify(const kvx_pool* dst, const int32_t* d_dst_table, uint32_t src_pool_id,
                    const int32_t* d_src_table, int64_t n, int32_t layer_lo, int32_t layer_hi,
                    uint64_t* d_mismatch, void* stream) {
  int st = check_range(dst, n, layer_lo, layer_hi);
  if (st) return st;
  KVX_REQUIRE(d_mismatch != nullptr, "kvx_pool_verify: NULL counter");
  if (n == 0 || layer_hi == layer_lo) return KVX_OK;
  KVX_REQUIRE(d_dst_table && d_src_table, "kvx_pool_verify: NULL table");
  DeviceGuard g(dst->d.device);
  const int64_t planes = static_cast<int64_t>(layer_hi - layer_lo) * 2;
  const int blocks =
      static_cast<int>(std::min<int64_t>(planes * n, sm_count(dst->d.device) * 8));
  verify_kernel<<<blocks, 256, 0, as_stream(stream)>>>(
      dst->base, dst->d.slots, dst->slab, d_dst_table, src_pool_id, d_src_table, n, layer_lo,
      planes, reinterpret_cast<unsigned long long*>(d_mismatch));
  KVX_LAUNCH_CHECK("verify_kernel");
  return KVX_OK;
}

int kvx_gather(const kvx_pool* p, const int32_t* d_src_table, int64_t n, int32_t lo, int32_t hi,
               void* d_buf, void* stream) {
  int st = check_range(p, n, lo, hi);
  if (st) return st;
  if (n == 0 || lo == hi) return KVX_OK;
  KVX_REQUIRE(d_src_table && d_buf, "kvx_gather: NULL table or buffer");
  KVX_REQUIRE((reinterpret_cast<uintptr_t>(d_buf) & 15) == 0, "kvx_gather: buffer not 16B aligned");
  SlabCopy c;
  c.src = p->base + static_cast<int64_t>(lo) * 2 * p->d.slots * p->slab;
  c.src_plane = p->d.slots * p->slab;
  c.src_table = d_src_table;
  c.dst = static_cast<uint8_t*>(d_buf);
  c.dst_plane = n * p->slab;
  c.dst_table = nullptr;
  c.n = n;
  c.src_slots = static_cast<uint32_t>(p->d.slots);
  c.dst_slots = static_cast<uint32_t>(n);
  c.planes = static_cast<int64_t>(hi - lo) * 2;
  c.slab = p->slab;
  DeviceGuard g(p->d.device);
  return launch_copy(c, p->d.device, as_stream(stream), false, p->host ? host_copy_ctas() : 0);
}

int kvx_scatter(kvx_pool* p, const int32_t* d_dst_table, int64_t n, int32_t lo, int32_t hi,
                const void* d_buf, void* stream) {
  int st = check_range(p, n, lo, hi);
  if (st) return st;
  if (n == 0 || lo == hi) return KVX_OK;
  KVX_REQUIRE(d_dst_table && d_buf, "kvx_scatter: NULL table or buffer");
  KVX_REQUIRE((reinterpret_cast<uintptr_t>(d_buf) & 15) == 0,
              "kvx_scatter: buffer not 16B aligned");
  SlabCopy c;
  c.src = static_cast<const uint8_t*>(d_buf);
  c.src_plane = n * p->slab;
  c.src_table = nullptr;
  c.dst = p->base + static_cast<int64_t>(lo) * 2 * p->d.slots * p->slab;
  c.dst_plane = p->d.slots * p->slab;
  c.dst_table = d_dst_table;
  c.n = n;
  c.src_slots = static_cast<uint32_t>(n);
  c.dst_slots = static_cast<uint32_t>(p->d.slots);
  c.planes = static_cast<int64_t>(hi - lo) * 2;
  c.slab = p->slab;
  DeviceGuard g(p->d.device);
  return launch_copy(c, p->d.device, as_stream(stream), false, p->host ? host_copy_ctas() : 0);
}

int kvx_copy_paged(const kvx_pool* src, const int32_t* d_src_table, kvx_pool* dst,
                   const int32_t* d_dst_table, int64_t n, int32_t lo, int32_t hi, void* stream) {
  SlabCopy c;
  bool empty = false;
  const int st = kvx::paged_copy_args(src, d_src_table, dst, d_dst_table, n, lo, hi, &c, &empty);
  if (st || empty) return st;
  // the kernel runs on the device of the stream's pools: a host (DRAM-tier)
  // pool is accessed by the GPU of the other side
  const int dev = src->host ? dst->d.device : src->d.device;
  DeviceGuard g(dev);
  return launch_copy(c, dev, as_stream(stream), false,
                     (src->host || dst->host) ? host_copy_ctas() : 0);
}

}  // extern "C"

namespace kvx {
namespace {
cudaLaunchAttribute pdl_attr() {
  cudaLaunchAttribute a;
  a.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a.val.programmaticStreamSerializationAllowed = 1;
  return a;
}
}  // namespace

int pull_gate(const uint64_t* d_flag, uint64_t value, uint64_t* d_status, void* stream,
              bool overlap_prev) {
  KVX_REQUIRE(d_flag && d_status, "pull_gate: NULL flag or status");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(32);
  cfg.stream = as_stream(stream);
  cudaLaunchAttribute attr[1] = {pdl_attr()};
  cfg.attrs = overlap_prev ? attr : nullptr;
  cfg.numAttrs = overlap_prev ? 1 : 0;
  KVX_CUDA(cudaLaunchKernelEx(&cfg, pull_gate_kernel,
                              reinterpret_cast<const unsigned long long*>(d_flag),
                              static_cast<unsigned long long>(value),
                              reinterpret_cast<unsigned long long*>(d_status)));
  KVX_LAUNCH_CHECK("pull_gate_kernel");
  return KVX_OK;
}

int pull_done(const uint64_t* d_status, uint64_t* d_peer_flag, uint64_t value, void* stream) {
  KVX_REQUIRE(d_status && d_peer_flag, "pull_done: NULL status or flag");
  pull_done_kernel<<<1, 1, 0, as_stream(stream)>>>(
      reinterpret_cast<const unsigned long long*>(d_status),
      reinterpret_cast<unsigned long long*>(d_peer_flag), static_cast<unsigned long long>(value));
  KVX_LAUNCH_CHECK("pull_done_kernel");
  return KVX_OK;
}

int copy_paged_pull(const kvx_pool* src, const int32_t* d_src_table, kvx_pool* dst,
                    const int32_t* d_dst_table, int64_t n, int32_t lo, int32_t hi, void* stream,
                    const uint64_t* d_flag, uint64_t value, const uint64_t* d_status,
                    bool after_gate) {
  SlabCopy c;
  bool empty = false;
  const int st = paged_copy_args(src, d_src_table, dst, d_dst_table, n, lo, hi, &c, &empty);
  if (st || empty) return st;
  const int dev = dst->d.device;  // the pulling GPU
  DeviceGuard g(dev);
  const int64_t items = c.planes * c.n * ((c.slab + kLsuItem - 1) / kLsuItem);
  const int blocks = static_cast<int>(std::min<int64_t>(items, static_cast<int64_t>(sm_count(dev)) * 4));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(kLsuThreads);
  cfg.stream = as_stream(stream);
  cudaLaunchAttribute attr[1] = {pdl_attr()};
  cfg.attrs = after_gate ? attr : nullptr;
  cfg.numAttrs = after_gate ? 1 : 0;
  KVX_REQUIRE(d_flag && d_status, "copy_paged_pull: NULL flag or status");
  const auto* fl = reinterpret_cast<const unsigned long long*>(d_flag);
  const auto* stw = reinterpret_cast<const unsigned long long*>(d_status);
  const unsigned long long v = value;
  if (items + blocks < (int64_t{1} << 32))
    KVX_CUDA(cudaLaunchKernelEx(&cfg, copy_pull_kernel<uint32_t>, c, fl, v, stw));
  else
    KVX_CUDA(cudaLaunchKernelEx(&cfg, copy_pull_kernel<int64_t>, c, fl, v, stw));
  KVX_LAUNCH_CHECK("copy_pull_kernel");
  return KVX_OK;
}

int copy_paged_overlapped(const kvx_pool* src, const int32_t* d_src_table, kvx_pool* dst,
                          const int32_t* d_dst_table, int64_t n, int32_t lo, int32_t hi,
                          void* stream) {
  SlabCopy c;
  bool empty = false;
  const int st = paged_copy_args(src, d_src_table, dst, d_dst_table, n, lo, hi, &c, &empty);
  if (st || empty) return st;
  DeviceGuard g(src->d.device);
  return launch_copy(c, src->d.device, as_stream(stream), true);
}
}  // namespace kvx

extern "C" {

int kvx_copy_check(void* stream) {
  // the flags are per device: read the ones of the device that owns `stream`
  int dev = -1;
  if (stream) {
    KVX_CUDA(cudaStreamGetDevice(as_stream(stream), &dev));
  } else {
    KVX_CUDA(cudaGetDevice(&dev));
  }
  DeviceGuard g(dev);
  KVX_CUDA(cudaStreamSynchronize(as_stream(stream)));
  unsigned long long timeouts = 0, bad = 0, zero = 0;
  KVX_CUDA(cudaMemcpyFromSymbol(&timeouts, g_wait_timeouts, sizeof(timeouts)));
  if (timeouts) {
    KVX_CUDA(cudaMemcpyToSymbol(g_wait_timeouts, &zero, sizeof(zero)));
    return set_error(KVX_ECUDA, "kvx_copy_check: a pull copy timed out waiting for its unit");
  }
  KVX_CUDA(cudaMemcpyFromSymbol(&bad, g_bad_table_entries, sizeof(bad)));
  if (bad == 0) return KVX_OK;
  KVX_CUDA(cudaMemcpyToSymbol(g_bad_table_entries, &zero, sizeof(zero)));
  return set_error(KVX_EINVAL,
                   "block table entries out of [0, slots): those blocks were skipped, not copied");
}

}  // extern "C"
