// kvx_stream.cpp -- the layer-wise prefill -> decode KV stream (stages 2->3->4)
// as a host C++ engine over libkvx's kernels and copy engines.
//
// Reference behaviour it makes real:
//   * the stream of a finished prefill: whole request chain, layer-wise,
//     overlapping the prefill (proj/src/sim_engine.cpp:455-470; the paper's
//     launch/wait per layer);
//   * chunked pipeline prefill produces KV chunk by chunk (prefill_chunk =
//     2048 tokens, proj/src/config.cpp:219; perf_model.cpp:87-110), so a long
//     request streams (token chunk, layer range) units in chunk-major order;
//   * one in-order transfer queue per sender (sender_busy_until_ms,
//     proj/src/sim_engine.cpp:409-411).
// A unit = (block range of the request, layer range).  Modes:
//   LOCAL_FUSED   one GPU: paged->paged copy kernel per unit
//   LOCAL_STAGED  one GPU: gather -> ring slot -> scatter (two streams)
//   PEER_FUSED    sender kernel stores straight into the receiver's pool (IPC view)
//   PEER_PULL     receiver kernel loads the sender's pool (IPC view) over NVLink
//                 and stores into its own pool; per-unit readiness flags from the
//                 sender, each unit released by a one-warp gate kernel; the
//                 prefill GPU's SMs stay free
//   PEER_CE       sender gathers into a ring slot, the copy engine moves it into
//                 the receiver's ring (IPC), the receiver scatters; 64-bit flags
//                 written with stream memory operations order the three queues
//                 across processes (no kernel ever spins on another's flag).
//   PEER_NCCL     comparison: gather -> ncclSend / ncclRecv (a 2-rank NCCL
//                 communicator of the pair, libnccl loaded at run time) ->
//                 scatter; sends / receives on a second queue, ring slots
//                 ordered by events.
// Sequence numbers only grow, so flags never need resetting (no ABA).
// The two ends may also be two processes on ONE GPU (same device UUID in the
// handshake): then no kernel ever waits for the other process -- every wait is
// a stream memory operation -- because nothing guarantees that kernels of two
// processes sharing a GPU run at the same time.
#include <cuda_runtime.h>

#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <cstring>
#include <string>
#include <vector>

#include "kvx.h"
#include "kvx_common.cuh"

using kvx::as_stream;
using kvx::set_error;

struct kvx_streamer {
  kvx_streamer_desc d{};
  kvx_pool* src = nullptr;
  kvx_pool* dst = nullptr;
  int device = 0;
  cudaStream_t s_main = nullptr;     // gather / fused copy (sender, local) or scatter (receiver)
  cudaStream_t s_second = nullptr;   // LOCAL_STAGED scatter stream
  kvx_xfer* xfer = nullptr;          // PEER_CE copy queue
  std::vector<void*> ring;           // local staging slots (cudaMalloc, IPC-exportable)
  std::vector<void*> peer_ring;      // receiver's slots as mapped on the sender
  std::vector<uint64_t> slot_ticket; // PEER_CE: copy that last read each gather slot
  std::vector<cudaEvent_t> slot_ev;  // LOCAL_STAGED: scatter that last read each slot
  std::vector<cudaEvent_t> gather_ev;
  uint64_t* flag = nullptr;          // local 64-bit flag word (peer writes it)
  uint64_t* pull_status = nullptr;   // PEER_PULL receiver: nonzero once a unit's gate timed out
  bool same_gpu = false;             // the peer process runs on this very GPU
  int pull_wait = 0;                 // PEER_PULL receiver: kPullGate / kPullInline / kPullStream
  void* nccl_comm = nullptr;         // PEER_NCCL: the pair's 2-rank communicator
  uint8_t nccl_id[128] = {};         // PEER_NCCL: the sender's ncclUniqueId
  uint64_t* peer_flag = nullptr;     // the peer's flag word, mapped here
  kvx_pool* peer_view = nullptr;     // PEER_FUSED: receiver's pool as seen by the sender
  uint64_t seq = 0;                  // units issued (sender) / consumed (receiver)
  // optional per-launch timing of the dominant kernel
  bool timing = false;
  uint64_t timing_stride = 1;  // time every stride-th dominant launch (event records cost host time)
  uint64_t timing_count = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timed;
  std::vector<double> timed_bytes;
  size_t timed_used = 0;
  // CUDA-graph record / replay of one step (LOCAL_FUSED): the units of the
  // sends between record_begin and record_end become kernel nodes of one graph
  bool recording = false;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  uint64_t graph_launches = 0, graph_units = 0, rec_launch0 = 0, rec_seq0 = 0;
  size_t graph_timed = 0;  // timed pairs [0, graph_timed) are graph nodes (re-recorded per replay)
};

namespace {

int ev_pair(kvx_streamer* s, cudaEvent_t* a, cudaEvent_t* b) {
  if (s->timed_used == s->timed.size()) {
    cudaEvent_t x, y;
    KVX_CUDA(cudaEventCreate(&x));
    KVX_CUDA(cudaEventCreate(&y));
    s->timed.push_back({x, y});
    s->timed_bytes.push_back(0);
  }
  *a = s->timed[s->timed_used].first;
  *b = s->timed[s->timed_used].second;
  return KVX_OK;
}

// Whether the next dominant launch will be bracketed by timing events.
bool will_sample(const kvx_streamer* s) {
  return s->timing && (s->timing_count % s->timing_stride == 0);
}

// Wrap one dominant launch with timing events when enabled.
template <class F>
int timed_launch(kvx_streamer* s, cudaStream_t st, double bytes, F&& launch) {
  cudaEvent_t a = nullptr, b = nullptr;
  const bool on = s->timing && (s->timing_count++ % s->timing_stride == 0);
  // while recording a graph the pair becomes two event-record nodes that
  // re-record on every replay
  const unsigned flags = s->recording ? cudaEventRecordExternal : cudaEventRecordDefault;
  if (on) {
    int rc = ev_pair(s, &a, &b);
    if (rc) return rc;
    KVX_CUDA(cudaEventRecordWithFlags(a, st, flags));
  }
  int rc = launch();
  if (rc) return rc;
  if (on) {
    KVX_CUDA(cudaEventRecordWithFlags(b, st, flags));
    s->timed_bytes[s->timed_used] = bytes;
    ++s->timed_used;
  }
  return KVX_OK;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("KVX_STREAM_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

int device_uuid(int dev, uint8_t out[16]) {
  cudaDeviceProp p;
  KVX_CUDA(cudaGetDeviceProperties(&p, dev));
  std::memcpy(out, &p.uuid, 16);
  return KVX_OK;
}

// How a PEER_PULL receiver waits for the sender's unit flag:
//   kPullGate   (default) a one-warp gate kernel waits; the copy launches
//               programmatically dependent on it (only the gate is resident
//               while the data is not there)
//   kPullInline the copy itself waits (thread 0 of every CTA), launched
//               programmatically dependent on the previous unit's copy: the
//               r01 design -- the next unit's whole grid sits resident while
//               the sender has not produced it
//   kPullStream the stream front end waits (cuStreamWaitValue64); the copy is
//               a plain launch
// KVX_PULL_GATE=gate|inline|stream selects it (measurement knob); two
// processes sharing one GPU always use kPullStream.
enum { kPullGate = 0, kPullInline = 1, kPullStream = 2 };
int pull_wait_mode() {
  static const int m = [] {
    const char* e = std::getenv("KVX_PULL_GATE");
    if (e && std::strcmp(e, "stream") == 0) return static_cast<int>(kPullStream);
    if (e && std::strcmp(e, "inline") == 0) return static_cast<int>(kPullInline);
    return static_cast<int>(kPullGate);
  }();
  return m;
}

bool is_peer(const kvx_streamer* s) {
  return s->d.mode == KVX_STREAM_PEER_FUSED || s->d.mode == KVX_STREAM_PEER_CE ||
         s->d.mode == KVX_STREAM_PEER_PULL || s->d.mode == KVX_STREAM_PEER_NCCL;
}

// ---- NCCL, loaded at run time (PEER_NCCL only): libkvx has no link-time
// NCCL dependency; in a process that already loaded libnccl.so.2 (e.g. with
// torch) dlopen returns that same library.
struct Nccl {
  int (*get_unique_id)(void*) = nullptr;
  int (*comm_destroy)(void*) = nullptr;
  int (*send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  const char* (*error_string)(int) = nullptr;
  void* init_rank = nullptr;  // ncclCommInitRank(ncclComm_t*, int, ncclUniqueId, int)
  bool ok = false;
};
struct Id128 {  // ncclUniqueId (passed by value to ncclCommInitRank)
  char b[128];
};
Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    n.get_unique_id = reinterpret_cast<int (*)(void*)>(dlsym(h, "ncclGetUniqueId"));
    n.comm_destroy = reinterpret_cast<int (*)(void*)>(dlsym(h, "ncclCommDestroy"));
    n.send = reinterpret_cast<int (*)(const void*, size_t, int, int, void*, cudaStream_t)>(
        dlsym(h, "ncclSend"));
    n.recv = reinterpret_cast<int (*)(void*, size_t, int, int, void*, cudaStream_t)>(
        dlsym(h, "ncclRecv"));
    n.error_string = reinterpret_cast<const char* (*)(int)>(dlsym(h, "ncclGetErrorString"));
    n.init_rank = dlsym(h, "ncclCommInitRank");
    n.ok = n.get_unique_id && n.comm_destroy && n.send && n.recv && n.init_rank;
  });
  return n;
}
constexpr int kNcclUint8 = 0;  // ncclUint8 in nccl.h's ncclDataType_t

int nccl_error(int rc, const char* where) {
  const char* msg = nccl().error_string ? nccl().error_string(rc) : "?";
  return set_error(KVX_ECUDA, std::string(where) + ": NCCL error " + std::to_string(rc) + " (" +
                                  msg + ")");
}

struct ExportBlob {
  int32_t magic;
  int32_t mode;
  int32_t ring;
  int32_t has_pool;
  int64_t slot_bytes;
  uint8_t flag[KVX_IPC_HANDLE_BYTES];
  uint8_t pool[KVX_IPC_HANDLE_BYTES];
  uint8_t uuid[16];  // the exporting GPU (two processes may share one GPU)
  uint8_t nccl_id[128];  // PEER_NCCL: the sender's ncclUniqueId
  // followed by ring * KVX_IPC_HANDLE_BYTES slot handles
};
constexpr int32_t kMagic = 0x6b767873;  // "kvxs"

}  // namespace

extern "C" {

int kvx_streamer_create(const kvx_streamer_desc* desc, kvx_pool* src, kvx_pool* dst,
                        kvx_streamer** out) {
  KVX_REQUIRE(desc && out, "kvx_streamer_create: NULL argument");
  const int mode = desc->mode, role = desc->role;
  KVX_REQUIRE(mode >= KVX_STREAM_LOCAL_FUSED && mode <= KVX_STREAM_PEER_NCCL,
              "kvx_streamer_create: bad mode");
  const bool local = mode == KVX_STREAM_LOCAL_FUSED || mode == KVX_STREAM_LOCAL_STAGED;
  KVX_REQUIRE(local == (role == KVX_ROLE_LOCAL), "kvx_streamer_create: mode/role mismatch");
  KVX_REQUIRE(role != KVX_ROLE_LOCAL || (src && dst), "local streamer needs src and dst pools");
  KVX_REQUIRE(role != KVX_ROLE_SENDER || src, "sender needs a src pool");
  KVX_REQUIRE(role != KVX_ROLE_RECEIVER || dst, "receiver needs a dst pool");
  const bool staged = mode == KVX_STREAM_LOCAL_STAGED || mode == KVX_STREAM_PEER_CE ||
                      mode == KVX_STREAM_PEER_NCCL;
  KVX_REQUIRE(!staged || (desc->ring >= 1 && desc->slot_bytes > 0),
              "staged modes need ring >= 1 and slot_bytes > 0");
  auto* s = new kvx_streamer();
  s->d = *desc;
  s->src = src;
  s->dst = dst;
  s->device = src ? kvx_pool_device(src) : kvx_pool_device(dst);
  s->timing = desc->time_launches != 0;
  kvx::DeviceGuard g(s->device);
  auto fail = [&](int rc) {
    kvx_streamer_destroy(s);
    return rc;
  };
  cudaError_t e = cudaStreamCreateWithFlags(&s->s_main, cudaStreamNonBlocking);
  if (e != cudaSuccess) return fail(kvx::cuda_error(e, "kvx_streamer_create: stream"));
  if (mode == KVX_STREAM_LOCAL_STAGED || mode == KVX_STREAM_PEER_NCCL) {
    e = cudaStreamCreateWithFlags(&s->s_second, cudaStreamNonBlocking);
    if (e != cudaSuccess) return fail(kvx::cuda_error(e, "kvx_streamer_create: stream"));
  }
  if (staged) {
    for (int i = 0; i < desc->ring; ++i) {
      void* p = nullptr;
      e = cudaMalloc(&p, static_cast<size_t>(desc->slot_bytes));
      if (e != cudaSuccess) return fail(kvx::cuda_error(e, "kvx_streamer_create: ring"));
      s->ring.push_back(p);
      cudaEvent_t ev1 = nullptr, ev2 = nullptr;
      e = cudaEventCreateWithFlags(&ev1, cudaEventDisableTiming);
      if (e == cudaSuccess) s->slot_ev.push_back(ev1);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev2, cudaEventDisableTiming);
      if (e == cudaSuccess) s->gather_ev.push_back(ev2);
      if (e != cudaSuccess) return fail(kvx::cuda_error(e, "kvx_streamer_create: event"));
    }
    s->slot_ticket.assign(desc->ring, 0);
  }
  if (is_peer(s)) {
    e = cudaMalloc(reinterpret_cast<void**>(&s->flag), 256);
    if (e != cudaSuccess) return fail(kvx::cuda_error(e, "kvx_streamer_create: flag"));
    s->pull_status = s->flag + 8;  // same allocation, not written by the peer
    e = cudaMemsetAsync(s->flag, 0, 256, s->s_main);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->s_main);  // zero before the peer maps it
    if (e != cudaSuccess) return fail(kvx::cuda_error(e, "kvx_streamer_create: flag"));
  }
  if (mode == KVX_STREAM_PEER_CE && role == KVX_ROLE_SENDER) {
    int rc = kvx_xfer_create(s->device, &s->xfer);
    if (rc) return fail(rc);
  }
  if (mode == KVX_STREAM_PEER_NCCL) {
    if (!nccl().ok) return fail(set_error(KVX_ECUDA, "kvx_streamer_create: libnccl.so.2 not loadable"));
    if (role == KVX_ROLE_SENDER) {
      const int rc = nccl().get_unique_id(s->nccl_id);
      if (rc) return fail(nccl_error(rc, "ncclGetUniqueId"));
    }
  }
  *out = s;
  return KVX_OK;
}

int kvx_streamer_destroy(kvx_streamer* s) {
  if (!s) return KVX_OK;
  kvx::DeviceGuard g(s->device);
  if (s->recording) {
    cudaGraph_t dropped = nullptr;
    cudaStreamEndCapture(s->s_main, &dropped);
    if (dropped) cudaGraphDestroy(dropped);
  }
  if (s->graph_exec) cudaGraphExecDestroy(s->graph_exec);
  if (s->graph) cudaGraphDestroy(s->graph);
  if (s->s_main) cudaStreamSynchronize(s->s_main);
  if (s->s_second) cudaStreamSynchronize(s->s_second);
  if (s->nccl_comm) nccl().comm_destroy(s->nccl_comm);
  if (s->xfer) kvx_xfer_destroy(s->xfer);
  for (void* p : s->peer_ring) kvx_ipc_close(p);
  if (s->peer_flag) kvx_ipc_close(s->peer_flag);
  if (s->peer_view) {
    void* base = kvx_pool_base(s->peer_view);
    kvx_pool_destroy(s->peer_view);
    kvx_ipc_close(base);
  }
  for (void* p : s->ring) cudaFree(p);
  for (auto ev : s->slot_ev) cudaEventDestroy(ev);
  for (auto ev : s->gather_ev) cudaEventDestroy(ev);
  for (auto& pr : s->timed) {
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  if (s->flag) cudaFree(s->flag);
  if (s->s_main) cudaStreamDestroy(s->s_main);
  if (s->s_second) cudaStreamDestroy(s->s_second);
  delete s;
  return KVX_OK;
}

int kvx_streamer_export(kvx_streamer* s, uint8_t* blob, int64_t cap, int64_t* len) {
  KVX_REQUIRE(s && len, "kvx_streamer_export: NULL argument");
  KVX_REQUIRE(is_peer(s), "kvx_streamer_export: only peer streamers export");
  const int64_t need = static_cast<int64_t>(sizeof(ExportBlob)) +
                       static_cast<int64_t>(s->ring.size()) * KVX_IPC_HANDLE_BYTES;
  *len = need;
  if (!blob) return KVX_OK;
  KVX_REQUIRE(cap >= need, "kvx_streamer_export: blob too small");
  ExportBlob b{};
  b.magic = kMagic;
  b.mode = s->d.mode;
  b.ring = static_cast<int32_t>(s->ring.size());
  b.slot_bytes = s->d.slot_bytes;
  int rc = device_uuid(s->device, b.uuid);
  if (rc) return rc;
  std::memcpy(b.nccl_id, s->nccl_id, sizeof(b.nccl_id));
  rc = kvx_ipc_export(s->flag, b.flag);
  if (rc) return rc;
  if (s->d.role == KVX_ROLE_RECEIVER && s->d.mode == KVX_STREAM_PEER_FUSED) {
    rc = kvx_ipc_export(kvx_pool_base(s->dst), b.pool);
    if (rc) return rc;
    b.has_pool = 1;
  }
  if (s->d.role == KVX_ROLE_SENDER && s->d.mode == KVX_STREAM_PEER_PULL) {
    rc = kvx_ipc_export(kvx_pool_base(s->src), b.pool);
    if (rc) return rc;
    b.has_pool = 1;
  }
  std::memcpy(blob, &b, sizeof(b));
  for (size_t i = 0; i < s->ring.size(); ++i) {
    rc = kvx_ipc_export(s->ring[i], blob + sizeof(b) + i * KVX_IPC_HANDLE_BYTES);
    if (rc) return rc;
  }
  return KVX_OK;
}

int kvx_streamer_connect(kvx_streamer* s, const uint8_t* blob, int64_t len,
                         const kvx_pool_desc* peer_pool) {
  KVX_REQUIRE(s && blob && len >= static_cast<int64_t>(sizeof(ExportBlob)),
              "kvx_streamer_connect: bad blob");
  ExportBlob b;
  std::memcpy(&b, blob, sizeof(b));
  KVX_REQUIRE(b.magic == kMagic && b.mode == s->d.mode, "kvx_streamer_connect: peer mismatch");
  kvx::DeviceGuard g(s->device);
  uint8_t mine[16];
  int rc = device_uuid(s->device, mine);
  if (rc) return rc;
  s->same_gpu = std::memcmp(mine, b.uuid, 16) == 0;
  s->pull_wait = s->same_gpu ? kPullStream : pull_wait_mode();
  void* p = nullptr;
  rc = kvx_ipc_open(b.flag, s->device, &p);
  if (rc) return rc;
  s->peer_flag = static_cast<uint64_t*>(p);
  const bool maps_pool = (s->d.role == KVX_ROLE_SENDER && s->d.mode == KVX_STREAM_PEER_FUSED) ||
                         (s->d.role == KVX_ROLE_RECEIVER && s->d.mode == KVX_STREAM_PEER_PULL);
  if (maps_pool) {
    KVX_REQUIRE(b.has_pool && peer_pool, "kvx_streamer_connect: peer pool missing");
    rc = kvx_ipc_open(b.pool, s->device, &p);
    if (rc) return rc;
    kvx_pool_desc d = *peer_pool;
    d.device = s->device;
    rc = kvx_pool_create_view(&d, p, &s->peer_view);
    if (rc) return rc;
  }
  if (s->d.mode == KVX_STREAM_PEER_NCCL) {
    // the pair's communicator: sender rank 0 (its id), receiver rank 1;
    // collective -- both ends connect at about the same time
    KVX_REQUIRE(b.ring == static_cast<int32_t>(s->ring.size()) && b.slot_bytes == s->d.slot_bytes,
                "kvx_streamer_connect: ring shapes differ");
    KVX_REQUIRE(!s->same_gpu, "kvx_streamer_connect: NCCL needs the two ends on different GPUs");
    Id128 id;
    std::memcpy(id.b, s->d.role == KVX_ROLE_SENDER ? s->nccl_id : b.nccl_id, sizeof(id.b));
    typedef int (*InitRank)(void**, int, Id128, int);
    const int rc2 = reinterpret_cast<InitRank>(nccl().init_rank)(
        &s->nccl_comm, 2, id, s->d.role == KVX_ROLE_SENDER ? 0 : 1);
    if (rc2) return nccl_error(rc2, "ncclCommInitRank");
  }
  if (s->d.role == KVX_ROLE_SENDER && s->d.mode == KVX_STREAM_PEER_CE) {
    KVX_REQUIRE(b.ring == static_cast<int32_t>(s->ring.size()) && b.slot_bytes == s->d.slot_bytes,
                "kvx_streamer_connect: ring shapes differ");
    KVX_REQUIRE(len >= static_cast<int64_t>(sizeof(b)) + b.ring * KVX_IPC_HANDLE_BYTES,
                "kvx_streamer_connect: truncated blob");
    for (int i = 0; i < b.ring; ++i) {
      rc = kvx_ipc_open(blob + sizeof(b) + i * KVX_IPC_HANDLE_BYTES, s->device, &p);
      if (rc) return rc;
      s->peer_ring.push_back(p);
    }
  }
  return KVX_OK;
}

void* kvx_streamer_stream(kvx_streamer* s) { return s ? reinterpret_cast<void*>(s->s_main) : nullptr; }

// Enqueue the units of one block range: chunk-major over [0, n) in
// chunk_blocks, layer ranges of layers_per_chunk inside [layer_lo, layer_hi).
int kvx_streamer_send(kvx_streamer* s, const int32_t* d_src_table, const int32_t* d_dst_table,
                      int64_t n, int64_t chunk_blocks, int32_t layer_lo, int32_t layer_hi,
                      int32_t layers_per_chunk) {
  KVX_REQUIRE(s && s->d.role != KVX_ROLE_RECEIVER, "kvx_streamer_send: not a sender");
  KVX_REQUIRE(n >= 0 && chunk_blocks >= 1 && layers_per_chunk >= 1 && layer_lo <= layer_hi,
              "kvx_streamer_send: bad ranges");
  const bool needs_dst = s->d.mode != KVX_STREAM_PEER_CE && s->d.mode != KVX_STREAM_PEER_PULL &&
                         s->d.mode != KVX_STREAM_PEER_NCCL;
  KVX_REQUIRE(d_src_table && (!needs_dst || d_dst_table), "kvx_streamer_send: NULL table");
  kvx::DeviceGuard g(s->device);
  const int64_t slab = kvx_pool_slab_bytes(s->src);
  const int R = static_cast<int>(s->ring.size());
  bool first_unit = true;
  for (int64_t b0 = 0; b0 < n; b0 += chunk_blocks) {
    const int64_t nb = std::min(chunk_blocks, n - b0);
    for (int32_t l0 = layer_lo; l0 < layer_hi; l0 += layers_per_chunk) {
      const int32_t l1 = std::min(layer_hi, l0 + layers_per_chunk);
      const int64_t payload = static_cast<int64_t>(l1 - l0) * 2 * nb * slab;
      const uint64_t c = s->seq++;
      int rc = KVX_OK;
      switch (s->d.mode) {
        case KVX_STREAM_LOCAL_FUSED: {
          // The units of ONE send touch disjoint (chunk, layer) slabs, so each
          // unit after the first may overlap its predecessor (programmatic
          // dependent launch; KVX_STREAM_PDL=0: off).  The first unit of a
          // call waits for everything before it (an earlier send may have
          // written the same decode slots), and a launch sampled for timing
          // runs isolated so its duration is its own.
          // (a pool copied into itself keeps its units strictly ordered)
          const bool overlap =
              pdl_enabled() && !first_unit && !will_sample(s) && s->src != s->dst;
          rc = timed_launch(s, s->s_main, 2.0 * payload, [&] {
            return overlap ? kvx::copy_paged_overlapped(s->src, d_src_table + b0, s->dst,
                                                        d_dst_table + b0, nb, l0, l1, s->s_main)
                           : kvx_copy_paged(s->src, d_src_table + b0, s->dst, d_dst_table + b0,
                                            nb, l0, l1, s->s_main);
          });
          break;
        }
        case KVX_STREAM_PEER_PULL:
          // the KV of unit c is in the pool once the work queued so far on the
          // sender's queue (the prefill of that layer, in a serving engine) is done
          KVX_REQUIRE(s->peer_flag, "kvx_streamer_send: not connected");
          rc = kvx_signal_write(s->s_main, s->peer_flag, c + 1);
          break;
        case KVX_STREAM_PEER_FUSED: {
          KVX_REQUIRE(s->peer_view, "kvx_streamer_send: not connected");
          // disjoint (chunk, layer) slabs of the receiver's pool: as LOCAL_FUSED
          const bool overlap = pdl_enabled() && !first_unit && !will_sample(s);
          rc = timed_launch(s, s->s_main, 1.0 * payload, [&] {
            return overlap ? kvx::copy_paged_overlapped(s->src, d_src_table + b0, s->peer_view,
                                                        d_dst_table + b0, nb, l0, l1, s->s_main)
                           : kvx_copy_paged(s->src, d_src_table + b0, s->peer_view,
                                            d_dst_table + b0, nb, l0, l1, s->s_main);
          });
          break;
        }
        case KVX_STREAM_LOCAL_STAGED: {
          KVX_REQUIRE(payload <= s->d.slot_bytes, "kvx_streamer_send: unit larger than a slot");
          const int slot = static_cast<int>(c % R);
          if (c >= static_cast<uint64_t>(R)) KVX_CUDA(cudaStreamWaitEvent(s->s_main, s->slot_ev[slot], 0));
          rc = timed_launch(s, s->s_main, 2.0 * payload, [&] {
            return kvx_gather(s->src, d_src_table + b0, nb, l0, l1, s->ring[slot], s->s_main);
          });
          if (rc) return rc;
          KVX_CUDA(cudaEventRecord(s->gather_ev[slot], s->s_main));
          KVX_CUDA(cudaStreamWaitEvent(s->s_second, s->gather_ev[slot], 0));
          rc = kvx_scatter(s->dst, d_dst_table + b0, nb, l0, l1, s->ring[slot], s->s_second);
          if (rc) return rc;
          KVX_CUDA(cudaEventRecord(s->slot_ev[slot], s->s_second));
          break;
        }
        case KVX_STREAM_PEER_CE: {
          KVX_REQUIRE(!s->peer_ring.empty(), "kvx_streamer_send: not connected");
          KVX_REQUIRE(payload <= s->d.slot_bytes, "kvx_streamer_send: unit larger than a slot");
          const int slot = static_cast<int>(c % R);
          if (s->slot_ticket[slot]) {  // the copy that last read this gather slot
            rc = kvx_transfer_wait_stream(s->xfer, s->slot_ticket[slot], s->s_main);
            if (rc) return rc;
          }
          rc = timed_launch(s, s->s_main, 2.0 * payload, [&] {
            return kvx_gather(s->src, d_src_table + b0, nb, l0, l1, s->ring[slot], s->s_main);
          });
          if (rc) return rc;
          if (c >= static_cast<uint64_t>(R)) {  // receiver drained its slot (unit c - R)
            rc = kvx_signal_wait(kvx_xfer_stream(s->xfer), s->flag, c - R + 1);
            if (rc) return rc;
          }
          rc = kvx_transfer_submit(s->xfer, s->peer_ring[slot], s->ring[slot], payload, s->s_main,
                                   &s->slot_ticket[slot]);
          if (rc) return rc;
          rc = kvx_transfer_signal(s->xfer, s->peer_flag, c + 1);  // unit c landed
          break;
        }
        case KVX_STREAM_PEER_NCCL: {
          KVX_REQUIRE(s->nccl_comm, "kvx_streamer_send: not connected");
          KVX_REQUIRE(payload <= s->d.slot_bytes, "kvx_streamer_send: unit larger than a slot");
          const int slot = static_cast<int>(c % R);
          // the send that last read this slot is done before the gather rewrites it
          if (c >= static_cast<uint64_t>(R)) KVX_CUDA(cudaStreamWaitEvent(s->s_main, s->slot_ev[slot], 0));
          rc = timed_launch(s, s->s_main, 2.0 * payload, [&] {
            return kvx_gather(s->src, d_src_table + b0, nb, l0, l1, s->ring[slot], s->s_main);
          });
          if (rc) return rc;
          KVX_CUDA(cudaEventRecord(s->gather_ev[slot], s->s_main));
          KVX_CUDA(cudaStreamWaitEvent(s->s_second, s->gather_ev[slot], 0));
          const int nrc = nccl().send(s->ring[slot], static_cast<size_t>(payload), kNcclUint8, 1,
                                      s->nccl_comm, s->s_second);
          if (nrc) return nccl_error(nrc, "ncclSend");
          KVX_CUDA(cudaEventRecord(s->slot_ev[slot], s->s_second));
          break;
        }
        default:
          return set_error(KVX_EINVAL, "kvx_streamer_send: bad mode");
      }
      if (rc) return rc;
      first_unit = false;
    }
  }
  return KVX_OK;
}

int kvx_streamer_recv(kvx_streamer* s, const int32_t* d_src_table, const int32_t* d_dst_table,
                      int64_t n, int64_t chunk_blocks, int32_t layer_lo, int32_t layer_hi,
                      int32_t layers_per_chunk) {
  KVX_REQUIRE(s && s->d.role == KVX_ROLE_RECEIVER, "kvx_streamer_recv: not a receiver");
  KVX_REQUIRE(n >= 0 && chunk_blocks >= 1 && layers_per_chunk >= 1 && layer_lo <= layer_hi,
              "kvx_streamer_recv: bad ranges");
  kvx::DeviceGuard g(s->device);
  const int64_t slab = kvx_pool_slab_bytes(s->dst);
  const int R = static_cast<int>(s->ring.size());
  bool first_unit = true;
  for (int64_t b0 = 0; b0 < n; b0 += chunk_blocks) {
    const int64_t nb = std::min(chunk_blocks, n - b0);
    for (int32_t l0 = layer_lo; l0 < layer_hi; l0 += layers_per_chunk) {
      const int32_t l1 = std::min(layer_hi, l0 + layers_per_chunk);
      const int64_t payload = static_cast<int64_t>(l1 - l0) * 2 * nb * slab;
      const uint64_t c = s->seq++;
      if (s->d.mode == KVX_STREAM_PEER_FUSED) continue;  // bytes land without us
      KVX_REQUIRE(d_dst_table, "kvx_streamer_recv: NULL table");
      if (s->d.mode == KVX_STREAM_PEER_PULL) {
        KVX_REQUIRE(d_src_table && s->peer_view, "kvx_streamer_recv: pull needs the src table");
        // Unit c is released by the sender's flag reaching c + 1.  Across two
        // GPUs a one-warp gate kernel waits for it and the copy launches
        // programmatically dependent on the gate; the gate of a unit after
        // the first of a call is itself dependent on the previous unit's copy,
        // so unit c+1 ramps up while unit c drains, yet only the gate is
        // resident while the data is not there.  On a shared GPU (or with
        // KVX_PULL_GATE=stream) the stream front end waits instead.  A launch
        // sampled for timing runs isolated.
        const bool sampled = will_sample(s);
        const bool pdl = pdl_enabled();
        int rc = KVX_OK;
        bool after_gate = false;  // launch the copy programmatically dependent
        if (s->pull_wait == kPullGate) {
          rc = kvx::pull_gate(s->flag, c + 1, s->pull_status, s->s_main,
                              pdl && !first_unit && !sampled);
          after_gate = pdl && !sampled;
        } else if (s->pull_wait == kPullInline) {
          after_gate = pdl && !first_unit && !sampled;  // on the previous unit's copy
          if (first_unit || sampled) rc = kvx_signal_wait(s->s_main, s->flag, c + 1);
        } else {
          rc = kvx_signal_wait(s->s_main, s->flag, c + 1);
        }
        first_unit = false;
        if (rc) return rc;
        rc = timed_launch(s, s->s_main, 1.0 * payload, [&] {
          return kvx::copy_paged_pull(s->peer_view, d_src_table + b0, s->dst, d_dst_table + b0, nb,
                                      l0, l1, s->s_main, s->flag, c + 1, s->pull_status,
                                      after_gate);
        });
        if (rc) return rc;
        continue;
      }
      if (s->d.mode == KVX_STREAM_PEER_NCCL) {
        KVX_REQUIRE(s->nccl_comm, "kvx_streamer_recv: not connected");
        KVX_REQUIRE(payload <= s->d.slot_bytes, "kvx_streamer_recv: unit larger than a slot");
        const int slot = static_cast<int>(c % R);
        // the scatter that last read this slot is done before the next receive lands in it
        if (c >= static_cast<uint64_t>(R)) KVX_CUDA(cudaStreamWaitEvent(s->s_second, s->slot_ev[slot], 0));
        const int nrc = nccl().recv(s->ring[slot], static_cast<size_t>(payload), kNcclUint8, 0,
                                    s->nccl_comm, s->s_second);
        if (nrc) return nccl_error(nrc, "ncclRecv");
        KVX_CUDA(cudaEventRecord(s->gather_ev[slot], s->s_second));
        KVX_CUDA(cudaStreamWaitEvent(s->s_main, s->gather_ev[slot], 0));
        int rc = timed_launch(s, s->s_main, 2.0 * payload, [&] {
          return kvx_scatter(s->dst, d_dst_table + b0, nb, l0, l1, s->ring[slot], s->s_main);
        });
        if (rc) return rc;
        KVX_CUDA(cudaEventRecord(s->slot_ev[slot], s->s_main));
        continue;
      }
      const int slot = static_cast<int>(c % R);
      int rc = kvx_signal_wait(s->s_main, s->flag, c + 1);
      if (rc) return rc;
      rc = timed_launch(s, s->s_main, 2.0 * payload, [&] {
        return kvx_scatter(s->dst, d_dst_table + b0, nb, l0, l1, s->ring[slot], s->s_main);
      });
      if (rc) return rc;
      rc = kvx_signal_write(s->s_main, s->peer_flag, c + 1);  // slot drained
      if (rc) return rc;
    }
  }
  return KVX_OK;
}

// Close a step: PEER_FUSED sender publishes its unit count; the receiver's
// stream waits for it.  Then `stream` (if given) waits for all queued work.
int kvx_streamer_finish(kvx_streamer* s, void* stream) {
  KVX_REQUIRE(s != nullptr, "kvx_streamer_finish: NULL");
  kvx::DeviceGuard g(s->device);
  if (s->d.mode == KVX_STREAM_PEER_FUSED) {
    int rc = s->d.role == KVX_ROLE_SENDER ? kvx_signal_write(s->s_main, s->peer_flag, s->seq)
                                          : kvx_signal_wait(s->s_main, s->flag, s->seq);
    if (rc) return rc;
  }
  if (s->d.mode == KVX_STREAM_PEER_PULL) {
    // receiver -> sender: source blocks consumed (bit 62 set if a unit timed
    // out; the receiver's host learns it from kvx_streamer_check)
    int rc = s->d.role == KVX_ROLE_RECEIVER
                 ? kvx::pull_done(s->pull_status, s->peer_flag, s->seq, s->s_main)
                 : kvx_signal_wait(s->s_main, s->flag, s->seq);
    if (rc) return rc;
  }
  if (stream) {
    cudaEvent_t ev;
    KVX_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    std::vector<cudaStream_t> qs = {s->s_main};
    if (s->s_second) qs.push_back(s->s_second);
    if (s->xfer) qs.push_back(as_stream(kvx_xfer_stream(s->xfer)));
    for (cudaStream_t q : qs) {
      KVX_CUDA(cudaEventRecord(ev, q));
      KVX_CUDA(cudaStreamWaitEvent(as_stream(stream), ev, 0));
    }
    KVX_CUDA(cudaEventDestroy(ev));
  }
  return KVX_OK;
}

// Make the streamer's queues wait for work already queued on `stream`.
int kvx_streamer_after(kvx_streamer* s, void* stream) {
  KVX_REQUIRE(s != nullptr, "kvx_streamer_after: NULL");
  kvx::DeviceGuard g(s->device);
  cudaEvent_t ev;
  KVX_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  KVX_CUDA(cudaEventRecord(ev, as_stream(stream)));
  KVX_CUDA(cudaStreamWaitEvent(s->s_main, ev, 0));
  if (s->s_second) KVX_CUDA(cudaStreamWaitEvent(s->s_second, ev, 0));
  if (s->xfer) KVX_CUDA(cudaStreamWaitEvent(as_stream(kvx_xfer_stream(s->xfer)), ev, 0));
  KVX_CUDA(cudaEventDestroy(ev));
  return KVX_OK;
}

// Host-blocking: average duration and algorithmic bytes of the timed launches
// since the last reset.
int kvx_streamer_launch_stats(kvx_streamer* s, int64_t* launches, double* avg_ms,
                              double* avg_bytes, int reset) {
  KVX_REQUIRE(s && launches && avg_ms && avg_bytes, "kvx_streamer_launch_stats: NULL");
  kvx::DeviceGuard g(s->device);
  double ms_sum = 0, bytes_sum = 0;
  for (size_t i = 0; i < s->timed_used; ++i) {
    KVX_CUDA(cudaEventSynchronize(s->timed[i].second));
    float ms = 0;
    KVX_CUDA(cudaEventElapsedTime(&ms, s->timed[i].first, s->timed[i].second));
    ms_sum += ms;
    bytes_sum += s->timed_bytes[i];
  }
  *launches = static_cast<int64_t>(s->timed_used);
  *avg_ms = s->timed_used ? ms_sum / s->timed_used : 0.0;
  *avg_bytes = s->timed_used ? bytes_sum / s->timed_used : 0.0;
  if (reset) s->timed_used = s->graph_timed;  // a recorded graph keeps its pairs
  return KVX_OK;
}

// ---- CUDA-graph record / replay (LOCAL_FUSED) ------------------------------
// A step of fine-grained layer-wise units (Config 3 at one 2,048-token chunk
// x one layer = 8 MiB per unit: 5,120 launches) is bound by host launch cost.
// Record the step's sends once as a graph, then replay it: one
// cudaGraphLaunch per step.  The tables are read at replay time, so their
// contents may change between replays (same device pointers and ranges).
int kvx_streamer_record_begin(kvx_streamer* s) {
  KVX_REQUIRE(s && s->d.mode == KVX_STREAM_LOCAL_FUSED,
              "kvx_streamer_record_begin: graph record/replay is for the local fused mode");
  KVX_REQUIRE(!s->recording, "kvx_streamer_record_begin: already recording");
  kvx::DeviceGuard g(s->device);
  if (s->graph_exec) KVX_CUDA(cudaGraphExecDestroy(s->graph_exec));
  if (s->graph) KVX_CUDA(cudaGraphDestroy(s->graph));
  s->graph_exec = nullptr;
  s->graph = nullptr;
  s->graph_timed = 0;
  s->timed_used = 0;
  s->rec_launch0 = kvx_launch_count();
  s->rec_seq0 = s->seq;
  KVX_CUDA(cudaStreamBeginCapture(s->s_main, cudaStreamCaptureModeRelaxed));
  s->recording = true;
  return KVX_OK;
}

int kvx_streamer_record_end(kvx_streamer* s) {
  KVX_REQUIRE(s && s->recording, "kvx_streamer_record_end: not recording");
  kvx::DeviceGuard g(s->device);
  s->recording = false;
  cudaGraph_t graph = nullptr;
  KVX_CUDA(cudaStreamEndCapture(s->s_main, &graph));
  cudaError_t e = cudaGraphInstantiate(&s->graph_exec, graph, 0);
  if (e != cudaSuccess) {
    cudaGraphDestroy(graph);
    s->graph_exec = nullptr;
    return kvx::cuda_error(e, "kvx_streamer_record_end: cudaGraphInstantiate");
  }
  s->graph = graph;
  // the recorded units have not run: launches and units count on replay
  s->graph_launches = kvx_launch_count() - s->rec_launch0;
  kvx::uncount_launches(s->graph_launches);
  s->graph_units = s->seq - s->rec_seq0;
  s->seq = s->rec_seq0;
  s->graph_timed = s->timed_used;
  return KVX_OK;
}

int kvx_streamer_replay(kvx_streamer* s) {
  KVX_REQUIRE(s && s->graph_exec && !s->recording, "kvx_streamer_replay: nothing recorded");
  kvx::DeviceGuard g(s->device);
  KVX_CUDA(cudaGraphLaunch(s->graph_exec, s->s_main));
  kvx::count_launch(s->graph_launches);
  s->seq += s->graph_units;
  return KVX_OK;
}

int kvx_streamer_set_timing(kvx_streamer* s, int on, int stride) {
  KVX_REQUIRE(s != nullptr && stride >= 1, "kvx_streamer_set_timing: bad arguments");
  s->timing = on != 0;
  s->timing_stride = static_cast<uint64_t>(stride);
  s->timing_count = 0;
  return KVX_OK;
}

uint64_t kvx_streamer_units(const kvx_streamer* s) { return s ? s->seq : 0; }

int kvx_streamer_check(kvx_streamer* s) {
  KVX_REQUIRE(s != nullptr, "kvx_streamer_check: NULL");
  kvx::DeviceGuard g(s->device);
  KVX_CUDA(cudaStreamSynchronize(s->s_main));
  if (s->s_second) KVX_CUDA(cudaStreamSynchronize(s->s_second));
  if (s->xfer) KVX_CUDA(cudaStreamSynchronize(as_stream(kvx_xfer_stream(s->xfer))));
  if (s->pull_status && s->d.role == KVX_ROLE_RECEIVER) {
    uint64_t st = 0;
    KVX_CUDA(cudaMemcpy(&st, s->pull_status, sizeof(st), cudaMemcpyDeviceToHost));
    if (st) {
      KVX_CUDA(cudaMemset(s->pull_status, 0, sizeof(st)));
      kvx_copy_check(s->s_main);  // clears the device-wide timeout flag too
      return set_error(KVX_ECUDA,
                       "kvx_streamer_check: a pulled unit timed out waiting for the sender "
                       "(20 s); its decode slots were not written");
    }
  }
  return kvx_copy_check(s->s_main);
}

int kvx_streamer_same_gpu(const kvx_streamer* s) { return s && s->same_gpu ? 1 : 0; }

int kvx_streamer_set_pull_wait(kvx_streamer* s, int mode) {
  KVX_REQUIRE(s && mode >= KVX_PULL_WAIT_GATE && mode <= KVX_PULL_WAIT_STREAM,
              "kvx_streamer_set_pull_wait: bad arguments");
  KVX_REQUIRE(s->d.mode == KVX_STREAM_PEER_PULL && s->d.role == KVX_ROLE_RECEIVER,
              "kvx_streamer_set_pull_wait: only PEER_PULL receivers wait for units");
  s->pull_wait = s->same_gpu ? kPullStream : mode;  // one GPU: never a waiting kernel
  return KVX_OK;
}

}  // extern "C"
