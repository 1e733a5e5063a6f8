// kvx_runtime.cu -- error plumbing, launch accounting, transfer engine, IPC
// and stream-ordered signals for libkvx.
//
// The transfer engine replaces the reference's analytic Messenger model
// (estimate_transfer_time, proj/src/perf_model.cpp:51-59) and its per-sender
// FIFO (sender_busy_until_ms, proj/src/sim_engine.cpp:409-411): every source
// GPU owns one in-order copy-engine queue, so transfers from one sender
// serialise exactly like the reference's FIFO while different senders run
// concurrently over NVSwitch.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <mutex>
#include <vector>

#include "kvx_common.cuh"

namespace kvx {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
}  // namespace

int set_error(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}

int cuda_error(cudaError_t e, const char* where) {
  const int st = (e == cudaErrorMemoryAllocation) ? KVX_ENOMEM : KVX_ECUDA;
  return set_error(st, std::string(where) + ": " + cudaGetErrorName(e) + " (" +
                           cudaGetErrorString(e) + ")");
}

void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
void uncount_launches(uint64_t n) { g_launches.fetch_sub(n, std::memory_order_relaxed); }

int sm_count(int dev) {
  static std::mutex mu;
  static std::vector<int> cache;
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 0) return 148;
  if (static_cast<int>(cache.size()) <= dev) cache.resize(dev + 1, 0);
  if (cache[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}

// ---- driver entry points for stream memory operations -------------------
// Resolved at run time through the runtime so libkvx.so has no link-time
// dependency on libcuda (the CPU build container has none).
namespace {
typedef CUresult (*PFN_writeValue64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
typedef CUresult (*PFN_waitValue64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
PFN_writeValue64 p_write64 = nullptr;
PFN_waitValue64 p_wait64 = nullptr;
std::once_flag g_memops_once;
int g_memops_status = KVX_ECUDA;

void load_memops() {
  cudaDriverEntryPointQueryResult q1, q2;
  void* w = nullptr;
  void* v = nullptr;
  if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &w, cudaEnableDefault, &q1) ==
          cudaSuccess &&
      cudaGetDriverEntryPoint("cuStreamWaitValue64", &v, cudaEnableDefault, &q2) ==
          cudaSuccess &&
      q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess && w && v) {
    p_write64 = reinterpret_cast<PFN_writeValue64>(w);
    p_wait64 = reinterpret_cast<PFN_waitValue64>(v);
    g_memops_status = KVX_OK;
  }
}

int memops_ready() {
  std::call_once(g_memops_once, load_memops);
  if (g_memops_status != KVX_OK)
    return set_error(KVX_ECUDA, "cuStreamWriteValue64/cuStreamWaitValue64 unavailable");
  return KVX_OK;
}
}  // namespace

}  // namespace kvx

using namespace kvx;

// ---- transfer engine -------------------------------------------------------
struct kvx_xfer {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::vector<cudaEvent_t> ring;  // ticket -> ring[ticket % size]
  cudaEvent_t dep = nullptr;      // producer-stream dependency of the next submit
  uint64_t next_ticket = 1;
};

namespace {
constexpr size_t kTicketRing = 1024;
}

extern "C" {

int kvx_abi_version(void) { return KVX_ABI_VERSION; }
const char* kvx_last_error(void) { return g_last_error.c_str(); }
uint64_t kvx_launch_count(void) { return g_launches.load(); }

int kvx_sync(void* stream) {
  KVX_CUDA(cudaStreamSynchronize(as_stream(stream)));
  return KVX_OK;
}

int64_t kvx_chain_hash(int64_t prev_key, uint64_t content_hash) {
  return kvx::chain_hash(prev_key, content_hash);
}

int kvx_xfer_create(int device, kvx_xfer** out) {
  KVX_REQUIRE(out != nullptr, "kvx_xfer_create: out is NULL");
  DeviceGuard g(device);
  auto* x = new kvx_xfer();
  x->device = device;
  cudaError_t e = cudaStreamCreateWithFlags(&x->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete x;
    return cuda_error(e, "kvx_xfer_create: cudaStreamCreate");
  }
  x->ring.resize(kTicketRing, nullptr);
  e = cudaEventCreateWithFlags(&x->dep, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    kvx_xfer_destroy(x);
    return cuda_error(e, "kvx_xfer_create: cudaEventCreate");
  }
  for (auto& ev : x->ring) {
    e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e != cudaSuccess) {
      kvx_xfer_destroy(x);
      return cuda_error(e, "kvx_xfer_create: cudaEventCreate");
    }
  }
  *out = x;
  return KVX_OK;
}

int kvx_xfer_destroy(kvx_xfer* x) {
  if (!x) return KVX_OK;
  DeviceGuard g(x->device);
  if (x->stream) cudaStreamSynchronize(x->stream);
  for (auto ev : x->ring)
    if (ev) cudaEventDestroy(ev);
  if (x->dep) cudaEventDestroy(x->dep);
  if (x->stream) cudaStreamDestroy(x->stream);
  delete x;
  return KVX_OK;
}

void* kvx_xfer_stream(kvx_xfer* x) { return x ? reinterpret_cast<void*>(x->stream) : nullptr; }

int kvx_transfer_submit(kvx_xfer* x, void* dst, const void* src, int64_t bytes,
                        void* after_stream, uint64_t* ticket) {
  KVX_REQUIRE(x != nullptr, "kvx_transfer_submit: NULL engine");
  KVX_REQUIRE(bytes >= 0, "kvx_transfer_submit: bytes must be >= 0");
  KVX_REQUIRE(bytes == 0 || (dst && src), "kvx_transfer_submit: NULL buffer");
  DeviceGuard g(x->device);
  if (after_stream) {
    // Order after the producer (e.g. the gather of this layer) without a
    // host round trip: record on the producer stream, wait on the queue (the
    // wait captures the event's state, so the event is reusable at once).
    KVX_CUDA(cudaEventRecord(x->dep, as_stream(after_stream)));
    KVX_CUDA(cudaStreamWaitEvent(x->stream, x->dep, 0));
  }
  if (bytes > 0)
    KVX_CUDA(cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyDefault, x->stream));
  const uint64_t t = x->next_ticket++;
  KVX_CUDA(cudaEventRecord(x->ring[t % kTicketRing], x->stream));
  if (ticket) *ticket = t;
  return KVX_OK;
}

static int ticket_event(kvx_xfer* x, uint64_t ticket, cudaEvent_t* ev) {
  KVX_REQUIRE(x != nullptr, "transfer: NULL engine");
  KVX_REQUIRE(ticket >= 1 && ticket < x->next_ticket, "transfer: unknown ticket");
  // A ticket older than the ring was re-recorded by a later copy on the same
  // in-order queue; waiting on it then over-waits, which is still correct.
  *ev = x->ring[ticket % kTicketRing];
  return KVX_OK;
}

int kvx_transfer_wait(kvx_xfer* x, uint64_t ticket) {
  cudaEvent_t ev = nullptr;
  int st = ticket_event(x, ticket, &ev);
  if (st) return st;
  DeviceGuard g(x->device);
  KVX_CUDA(cudaEventSynchronize(ev));
  return KVX_OK;
}

int kvx_transfer_wait_stream(kvx_xfer* x, uint64_t ticket, void* stream) {
  cudaEvent_t ev = nullptr;
  int st = ticket_event(x, ticket, &ev);
  if (st) return st;
  KVX_CUDA(cudaStreamWaitEvent(as_stream(stream), ev, 0));
  return KVX_OK;
}

int kvx_transfer_query(kvx_xfer* x, uint64_t ticket) {
  cudaEvent_t ev = nullptr;
  int st = ticket_event(x, ticket, &ev);
  if (st) return st;
  cudaError_t e = cudaEventQuery(ev);
  if (e == cudaErrorNotReady) return KVX_EAGAIN;
  KVX_CUDA(e);
  return KVX_OK;
}

int kvx_transfer_signal(kvx_xfer* x, void* d_flag, uint64_t value) {
  KVX_REQUIRE(x != nullptr, "kvx_transfer_signal: NULL engine");
  DeviceGuard g(x->device);
  return kvx_signal_write(x->stream, d_flag, value);
}

// ---- IPC / peers / signals -------------------------------------------------

int kvx_ipc_export(void* d_ptr, uint8_t handle[KVX_IPC_HANDLE_BYTES]) {
  static_assert(sizeof(cudaIpcMemHandle_t) == KVX_IPC_HANDLE_BYTES, "ipc handle size");
  KVX_REQUIRE(d_ptr && handle, "kvx_ipc_export: NULL");
  cudaIpcMemHandle_t h;
  KVX_CUDA(cudaIpcGetMemHandle(&h, d_ptr));
  std::memcpy(handle, &h, sizeof(h));
  return KVX_OK;
}

int kvx_ipc_open(const uint8_t handle[KVX_IPC_HANDLE_BYTES], int device, void** d_ptr) {
  KVX_REQUIRE(handle && d_ptr, "kvx_ipc_open: NULL");
  DeviceGuard g(device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  KVX_CUDA(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return KVX_OK;
}

int kvx_ipc_close(void* d_ptr) {
  KVX_CUDA(cudaIpcCloseMemHandle(d_ptr));
  return KVX_OK;
}

int kvx_enable_peer(int device, int peer_device) {
  if (device == peer_device) return KVX_OK;
  DeviceGuard g(device);
  int can = 0;
  KVX_CUDA(cudaDeviceCanAccessPeer(&can, device, peer_device));
  KVX_REQUIRE(can, "kvx_enable_peer: devices cannot access each other");
  cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return KVX_OK;
  }
  KVX_CUDA(e);
  return KVX_OK;
}

// ---- small host-side plumbing for C / C++ hosts (no CUDA runtime of their own) --

int kvx_stream_create(int device, void** out) {
  KVX_REQUIRE(out != nullptr, "kvx_stream_create: NULL out");
  DeviceGuard g(device);
  cudaStream_t s = nullptr;
  KVX_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  *out = s;
  return KVX_OK;
}

int kvx_stream_destroy(void* stream) {
  if (!stream) return KVX_OK;
  KVX_CUDA(cudaStreamSynchronize(as_stream(stream)));
  KVX_CUDA(cudaStreamDestroy(as_stream(stream)));
  return KVX_OK;
}

int kvx_host_alloc(int64_t bytes, void** out) {
  KVX_REQUIRE(out && bytes > 0, "kvx_host_alloc: bad arguments");
  KVX_CUDA(cudaHostAlloc(out, static_cast<size_t>(bytes),
                         cudaHostAllocPortable | cudaHostAllocMapped));
  return KVX_OK;
}

int kvx_host_free(void* p) {
  if (p) KVX_CUDA(cudaFreeHost(p));
  return KVX_OK;
}

int kvx_memcpy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  KVX_REQUIRE(bytes >= 0 && (bytes == 0 || (dst && src)), "kvx_memcpy_async: bad arguments");
  if (bytes) KVX_CUDA(cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyDefault,
                                      as_stream(stream)));
  return KVX_OK;
}

int kvx_wait_host_word(const volatile int64_t* word, int64_t target, void* stream) {
  KVX_REQUIRE(word != nullptr, "kvx_wait_host_word: NULL word");
  // Spin on the pinned word the GPU writes (a kernel result or a stream-
  // ordered flag) until it reaches `target`: no synchronise call on the fast
  // path.  Every 4096 polls the stream is asked whether it failed, or went
  // idle without writing.
  for (uint64_t i = 1;; ++i) {
    if (*word >= target) return KVX_OK;
    if ((i & 4095) == 0) {
      cudaError_t e = cudaStreamQuery(as_stream(stream));
      if (e == cudaSuccess) {
        if (*word >= target) return KVX_OK;
        return set_error(KVX_ECUDA, "kvx_wait_host_word: stream idle, word never written");
      }
      if (e != cudaErrorNotReady) return cuda_error(e, "kvx_wait_host_word");
    }
  }
}

int kvx_signal_write(void* stream, void* d_flag, uint64_t value) {
  KVX_REQUIRE(d_flag != nullptr, "kvx_signal_write: NULL flag");
  int st = memops_ready();
  if (st) return st;
  // Default flags: the store is ordered after (fenced behind) prior work.
  CUresult r = p_write64(reinterpret_cast<CUstream>(stream),
                         reinterpret_cast<CUdeviceptr>(d_flag), value, 0);
  if (r != CUDA_SUCCESS)
    return set_error(KVX_ECUDA, "cuStreamWriteValue64 failed: " + std::to_string(r));
  return KVX_OK;
}

int kvx_signal_wait(void* stream, const void* d_flag, uint64_t value) {
  KVX_REQUIRE(d_flag != nullptr, "kvx_signal_wait: NULL flag");
  int st = memops_ready();
  if (st) return st;
  CUresult r = p_wait64(reinterpret_cast<CUstream>(stream),
                        reinterpret_cast<CUdeviceptr>(const_cast<void*>(d_flag)), value,
                        CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS)
    return set_error(KVX_ECUDA, "cuStreamWaitValue64 failed: " + std::to_string(r));
  return KVX_OK;
}

}  // extern "C"
