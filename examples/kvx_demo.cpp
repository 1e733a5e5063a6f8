// kvx_demo.cpp -- the hot path driven from C++ through the C ABI only
// (include/kvx.h), the way a serving engine's host code would use it:
//   1. hash two requests that share a prefix (stage 1a),
//   2. index request A's blocks on a "prefill instance" and prefix-match B (1b),
//   3. stream B's KV layer-wise from a prefill pool into a decode pool whose
//      block table comes from the decode allocator (stages 2-4, one GPU),
//   4. verify every landed word on the device.
// Prints "kvx_demo OK" and exits 0 on success.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kvx.h"

#define CHECK(x)                                                                      \
  do {                                                                                \
    int rc_ = (x);                                                                    \
    if (rc_ != KVX_OK) {                                                              \
      std::fprintf(stderr, "%s failed: %d %s\n", #x, rc_, kvx_last_error());          \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)

template <class T>
T* to_device(const std::vector<T>& h) {
  T* d = nullptr;
  cudaMalloc(&d, h.size() * sizeof(T) + 16);
  cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
  return d;
}

int main() {
  const int64_t bs = 16;
  // request A: 40 blocks; request B shares A's first 25 blocks, then diverges
  std::vector<int32_t> tokens;
  for (int i = 0; i < 40 * bs; ++i) tokens.push_back((i * 7919 + 13) % 32000);
  for (int i = 0; i < 32 * bs; ++i) tokens.push_back(i < 25 * bs ? tokens[i] : 31000 - i);
  std::vector<int64_t> tok_off = {0, 40 * bs, 72 * bs}, key_off = {0, 40, 72};
  int32_t* d_tok = to_device(tokens);
  int64_t* d_tok_off = to_device(tok_off);
  int64_t* d_key_off = to_device(key_off);
  int64_t* d_keys = nullptr;
  cudaMalloc(&d_keys, 72 * sizeof(int64_t));
  CHECK(kvx_chain_hash_batch(d_tok, d_tok_off, 2, bs, d_key_off, d_keys, nullptr));

  kvx_index* inst = nullptr;
  CHECK(kvx_index_create(0, 64, &inst));
  CHECK(kvx_index_insert(inst, d_keys, nullptr, 40, nullptr));  // A is cached on the instance
  const kvx_index* insts[1] = {inst};
  const int32_t ids[1] = {3};
  int64_t* d_best = nullptr;
  int32_t* d_best_id = nullptr;
  cudaMalloc(&d_best, sizeof(int64_t));
  cudaMalloc(&d_best_id, sizeof(int32_t));
  std::vector<int64_t> b_off = {0, 32};
  int64_t* d_b_off = to_device(b_off);
  CHECK(kvx_match_prefix_batch(insts, ids, 1, d_keys + 40, d_b_off, 1, nullptr, d_best, d_best_id,
                               nullptr));
  int64_t best = -1;
  cudaMemcpy(&best, d_best, sizeof(best), cudaMemcpyDeviceToHost);
  if (best != 25) {
    std::fprintf(stderr, "prefix match: got %lld, want 25\n", static_cast<long long>(best));
    return 1;
  }

  // stages 2-4: B's 32 blocks, 6 layers of an 8-head x 128 fp16 KV shape
  kvx_pool_desc pd{6, static_cast<int32_t>(bs), 8, 128, 2, 64, 0};
  kvx_pool *src = nullptr, *dst = nullptr;
  CHECK(kvx_pool_create(&pd, &src));
  pd.slots = 48;
  CHECK(kvx_pool_create(&pd, &dst));
  CHECK(kvx_pool_fill_synthetic(src, 5, nullptr));
  std::vector<int32_t> src_table(32), dst_table(32);
  for (int i = 0; i < 32; ++i) src_table[i] = (i * 37) % 64;
  kvx_slot_alloc* alloc = nullptr;
  CHECK(kvx_slot_alloc_create(48, &alloc));
  const int32_t busy[3] = {0, 1, 7};  // slots held by requests already decoding
  CHECK(kvx_slot_alloc_mark(alloc, busy, 3));
  CHECK(kvx_slot_alloc_take(alloc, 32, dst_table.data()));
  int32_t* d_st = to_device(src_table);
  int32_t* d_dt = to_device(dst_table);
  kvx_streamer_desc sd{KVX_STREAM_LOCAL_FUSED, KVX_ROLE_LOCAL, 0, 0, 0};
  kvx_streamer* st = nullptr;
  CHECK(kvx_streamer_create(&sd, src, dst, &st));
  // 2048-token chunks = 128 blocks: here 8-block chunks, one layer per unit
  CHECK(kvx_streamer_send(st, d_st, d_dt, 32, 8, 0, 6, 1));
  CHECK(kvx_streamer_finish(st, nullptr));
  CHECK(kvx_sync(kvx_streamer_stream(st)));
  uint64_t* d_bad = nullptr;
  cudaMalloc(&d_bad, sizeof(uint64_t));
  cudaMemset(d_bad, 0, sizeof(uint64_t));
  CHECK(kvx_pool_verify(dst, d_dt, 5, d_st, 32, 0, 6, d_bad, nullptr));
  uint64_t bad = 1;
  cudaMemcpy(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost);
  if (bad != 0 || kvx_streamer_units(st) != 4 * 6) {
    std::fprintf(stderr, "stream: %llu mismatched words\n", static_cast<unsigned long long>(bad));
    return 1;
  }
  kvx_streamer_destroy(st);
  kvx_slot_alloc_destroy(alloc);
  kvx_pool_destroy(src);
  kvx_pool_destroy(dst);
  kvx_index_destroy(inst);
  std::printf("kvx_demo OK: prefix match 25 blocks, %llu units streamed bit-exact, %llu kernels\n",
              static_cast<unsigned long long>(4 * 6),
              static_cast<unsigned long long>(kvx_launch_count()));
  return 0;
}
