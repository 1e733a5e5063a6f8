// kvx_host.cpp -- host-side pieces of the data plane: the decode instance's
// slot allocator (the paged block table the scatter lands in) and raw device
// allocations that can be exported over CUDA IPC.
//
// The reference has no decode block table -- decode instances only count KV
// tokens (proj/src/sim_engine.cpp:161-175) -- so the allocator is
// build-defined: deterministic lowest-free-slot allocation, so
// that the same request sequence always yields the same decode block tables
// and the oracle (oracle/kvx_oracle.c: kvo_alloc_lowest_free) can restate it.
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "kvx_common.cuh"

struct kvx_slot_alloc {
  int64_t slots = 0;
  int64_t free = 0;
  std::vector<uint64_t> used;  // bit set: 1 = slot taken
};

using namespace kvx;

extern "C" {

int kvx_device_alloc(int device, int64_t bytes, void** d_ptr) {
  KVX_REQUIRE(d_ptr != nullptr && bytes > 0, "kvx_device_alloc: bad arguments");
  DeviceGuard g(device);
  KVX_CUDA(cudaMalloc(d_ptr, static_cast<size_t>(bytes)));
  return KVX_OK;
}

int kvx_device_free(int device, void* d_ptr) {
  if (!d_ptr) return KVX_OK;
  DeviceGuard g(device);
  KVX_CUDA(cudaFree(d_ptr));
  return KVX_OK;
}

int kvx_slot_alloc_create(int64_t slots, kvx_slot_alloc** out) {
  KVX_REQUIRE(out != nullptr, "kvx_slot_alloc_create: out is NULL");
  KVX_REQUIRE(slots >= 0 && slots <= 0x7FFFFFFF, "kvx_slot_alloc_create: bad slot count");
  auto* a = new kvx_slot_alloc();
  a->slots = slots;
  a->free = slots;
  a->used.assign(static_cast<size_t>((slots + 63) / 64), 0);
  if (slots % 64) a->used.back() = ~0ull << (slots % 64);  // bits past the end: taken
  *out = a;
  return KVX_OK;
}

int kvx_slot_alloc_destroy(kvx_slot_alloc* a) {
  delete a;
  return KVX_OK;
}

int64_t kvx_slot_alloc_free_count(const kvx_slot_alloc* a) { return a ? a->free : 0; }

int kvx_slot_alloc_take(kvx_slot_alloc* a, int64_t n, int32_t* table_out) {
  KVX_REQUIRE(a != nullptr, "kvx_slot_alloc_take: NULL allocator");
  KVX_REQUIRE(n >= 0 && (n == 0 || table_out), "kvx_slot_alloc_take: bad arguments");
  if (n > a->free) return set_error(KVX_ENOMEM, "kvx_slot_alloc_take: decode pool exhausted");
  int64_t got = 0;
  for (size_t w = 0; w < a->used.size() && got < n; ++w) {
    uint64_t freebits = ~a->used[w];
    while (freebits && got < n) {
      const int bit = __builtin_ctzll(freebits);
      freebits &= freebits - 1;
      a->used[w] |= 1ull << bit;
      table_out[got++] = static_cast<int32_t>(w * 64 + bit);
    }
  }
  a->free -= got;
  return KVX_OK;
}

int kvx_slot_alloc_mark(kvx_slot_alloc* a, const int32_t* slots, int64_t n) {
  KVX_REQUIRE(a != nullptr && (n == 0 || slots), "kvx_slot_alloc_mark: bad arguments");
  for (int64_t i = 0; i < n; ++i) {
    const int64_t s = slots[i];
    KVX_REQUIRE(s >= 0 && s < a->slots, "kvx_slot_alloc_mark: slot out of range");
    uint64_t& w = a->used[static_cast<size_t>(s / 64)];
    const uint64_t bit = 1ull << (s % 64);
    if (!(w & bit)) {
      w |= bit;
      --a->free;
    }
  }
  return KVX_OK;
}

int kvx_slot_alloc_release(kvx_slot_alloc* a, const int32_t* slots, int64_t n) {
  KVX_REQUIRE(a != nullptr && (n == 0 || slots), "kvx_slot_alloc_release: bad arguments");
  for (int64_t i = 0; i < n; ++i) {
    const int64_t s = slots[i];
    KVX_REQUIRE(s >= 0 && s < a->slots, "kvx_slot_alloc_release: slot out of range");
    uint64_t& w = a->used[static_cast<size_t>(s / 64)];
    const uint64_t bit = 1ull << (s % 64);
    if (w & bit) {
      w &= ~bit;
      ++a->free;
    }
  }
  return KVX_OK;
}

}  // extern "C"
