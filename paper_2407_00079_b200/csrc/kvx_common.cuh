// kvx_common.cuh -- shared device helpers and host error plumbing for libkvx.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include "kvx.h"

namespace kvx {

// ---- hashing (bit-identical to kvcsim::chain_hash, proj/src/kvcache.cpp:14-23)
__host__ __device__ __forceinline__ int64_t chain_hash(int64_t prev_key, uint64_t content) {
  uint64_t x = static_cast<uint64_t>(prev_key) + 0x9E3779B97F4A7C15ull;
  x ^= content + 0x9E3779B97F4A7C15ull + (x << 6) + (x >> 2);
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return static_cast<int64_t>(x & 0x7FFFFFFFFFFFFFFFull);
}

// splitmix64 finalizer: slot hash of the index and the synthetic KV generator.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t slab_seed(uint32_t pool_id, uint32_t layer,
                                                       uint32_t kv, uint32_t slot) {
  const uint64_t hi = (static_cast<uint64_t>(pool_id & 0xFFFFu) << 16) |
                      (static_cast<uint64_t>(layer & 0x7FFFu) << 1) |
                      static_cast<uint64_t>(kv & 1u);
  return mix64((hi << 32) | static_cast<uint64_t>(slot));
}

constexpr int64_t kKeyEmpty = KVX_KEY_EMPTY;
constexpr int64_t kKeyTomb = KVX_KEY_TOMBSTONE;
__host__ __device__ __forceinline__ bool is_reserved(int64_t k) { return k <= kKeyTomb; }

// ---- host side -----------------------------------------------------------
int set_error(int status, const std::string& msg);
int cuda_error(cudaError_t e, const char* where);
void count_launch(uint64_t n = 1);
void uncount_launches(uint64_t n);  // launches recorded into a graph, not run

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Guard that switches to `dev` for the scope (restores the caller's device).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

int sm_count(int dev);

// kvx_copy_paged whose launch may overlap the previous kernel on the stream
// (programmatic dependent launch): only for copies independent of it, e.g.
// the streamer's layer-wise units, which touch disjoint (chunk, layer) slabs.
int copy_paged_overlapped(const kvx_pool* src, const int32_t* d_src_table, kvx_pool* dst,
                          const int32_t* d_dst_table, int64_t n, int32_t lo, int32_t hi,
                          void* stream);
// PEER_PULL receiver pieces (kvx_copy.cu): a one-warp gate that waits for the
// sender's flag (d_flag >= value, system-scope acquire; 20 s timeout sets
// *d_status), the pull copy (after_gate: programmatically dependent on the
// gate; re-acquires the flag, skips when *d_status != 0), and the end-of-step
// "consumed" word.
int pull_gate(const uint64_t* d_flag, uint64_t value, uint64_t* d_status, void* stream,
              bool overlap_prev);
int copy_paged_pull(const kvx_pool* src, const int32_t* d_src_table, kvx_pool* dst,
                    const int32_t* d_dst_table, int64_t n, int32_t lo, int32_t hi, void* stream,
                    const uint64_t* d_flag, uint64_t value, const uint64_t* d_status,
                    bool after_gate);
int pull_done(const uint64_t* d_status, uint64_t* d_peer_flag, uint64_t value, void* stream);
// K2 following the hash's key production (kvx_index.cu; kvx_hash_match_batch:
// keys preset to -1); d_order: the hash's claim order (NULL: index order).
int match_follow_launch(const kvx_index* const* idx, const int32_t* inst_ids, int64_t n_inst,
                        const int64_t* d_keys, const int64_t* d_key_off, int64_t n_req,
                        int64_t* d_len_out, int64_t* d_best_len, int32_t* d_best_id,
                        const int32_t* d_order, unsigned long long* d_claim, void* stream,
                        uint64_t* const* dests = nullptr, int n_dests = 0,
                        const int64_t* const* owner_keys = nullptr,
                        const int64_t* owner_end = nullptr, int n_owner = 0);
// Requests of a batch in decreasing block count (kvx_hash.cu).
int order_by_length(const int64_t* d_key_off, int64_t n_req, int32_t* d_order,
                    unsigned long long* d_ws, cudaStream_t s);
int hash_publish_launch(const int32_t* d_tokens, const int64_t* d_tok_off, int64_t n_req,
                        int64_t bs, const int64_t* d_key_off, int64_t* d_keys, void* stream,
                        bool* published);

}  // namespace kvx

#define KVX_CUDA(expr)                                         \
  do {                                                         \
    cudaError_t _e = (expr);                                   \
    if (_e != cudaSuccess) return ::kvx::cuda_error(_e, #expr); \
  } while (0)

#define KVX_LAUNCH_CHECK(where)                                  \
  do {                                                           \
    cudaError_t _e = cudaGetLastError();                         \
    if (_e != cudaSuccess) return ::kvx::cuda_error(_e, where);  \
    ::kvx::count_launch();                                       \
  } while (0)

#define KVX_REQUIRE(cond, msg)                                     \
  do {                                                             \
    if (!(cond)) return ::kvx::set_error(KVX_EINVAL, (msg));       \
  } while (0)
