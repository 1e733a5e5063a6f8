// kvx_store.cpp -- one instance's KVCache store: paged pool + block index
// (key -> slot) + slot allocator, and the migration data path between two
// stores (hot-spot replication).
//
// Reference semantics (kvcsim):
//   * the Conductor's migration plan replicates the best holder's chain range
//     [local_prefix, used_prefix) onto the chosen instance
//     (proj/src/conductor.cpp:254-260; engine issue proj/src/sim_engine.cpp:399-419);
//   * at migration begin the engine aborts if the source evicted ANY block of
//     the range (proj/src/sim_engine.cpp:605-639) -- here: KVX_EABORTED, and
//     nothing is changed on either side;
//   * landing = insert_replicated (proj/src/kvcache.cpp:133-148): blocks
//     already resident at the destination are skipped.
// The bytes move with the same paged -> paged copy kernel as the stream
// (kvx_copy_paged); when the two stores live on different GPUs the kernel
// writes through a peer mapping of the destination pool (NVLink).
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <cstdint>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "kvx.h"
#include "kvx_common.cuh"

struct kvx_store {
  int device = 0;
  kvx_pool_desc desc{};
  std::map<int, kvx_pool*> views;  // this pool as seen from other GPUs (migration pulls)
  kvx_pool* pool = nullptr;
  kvx_index* index = nullptr;
  kvx_slot_alloc* alloc = nullptr;
  cudaStream_t stream = nullptr;
  int64_t* d_scratch = nullptr;  // keys / values staging
  int64_t scratch_words = 0;
};

namespace {

int ensure_scratch(kvx_store* s, int64_t words) {
  if (words <= s->scratch_words) return KVX_OK;
  int64_t cap = std::max<int64_t>(1024, s->scratch_words);
  while (cap < words) cap *= 2;
  kvx::DeviceGuard g(s->device);
  if (s->d_scratch) cudaFree(s->d_scratch);
  s->d_scratch = nullptr;
  s->scratch_words = 0;
  KVX_CUDA(cudaMalloc(reinterpret_cast<void**>(&s->d_scratch), cap * sizeof(int64_t)));
  s->scratch_words = cap;
  return KVX_OK;
}

// Host-blocking lookup of keys in a store: slot per key, -1 when absent.
int lookup_host(kvx_store* s, const int64_t* h_keys, int64_t n, std::vector<int64_t>& out) {
  out.assign(static_cast<size_t>(n), -1);
  if (n == 0) return KVX_OK;
  int rc = ensure_scratch(s, 2 * n);
  if (rc) return rc;
  kvx::DeviceGuard g(s->device);
  KVX_CUDA(cudaMemcpyAsync(s->d_scratch, h_keys, n * sizeof(int64_t), cudaMemcpyHostToDevice,
                           s->stream));
  rc = kvx_index_lookup(s->index, s->d_scratch, n, s->d_scratch + n, s->stream);
  if (rc) return rc;
  KVX_CUDA(cudaMemcpyAsync(out.data(), s->d_scratch + n, n * sizeof(int64_t),
                           cudaMemcpyDeviceToHost, s->stream));
  KVX_CUDA(cudaStreamSynchronize(s->stream));
  return KVX_OK;
}

int insert_host(kvx_store* s, const int64_t* keys, const int64_t* slots, int64_t n) {
  if (n == 0) return KVX_OK;
  int rc = ensure_scratch(s, 2 * n);
  if (rc) return rc;
  kvx::DeviceGuard g(s->device);
  KVX_CUDA(cudaMemcpyAsync(s->d_scratch, keys, n * sizeof(int64_t), cudaMemcpyHostToDevice,
                           s->stream));
  KVX_CUDA(cudaMemcpyAsync(s->d_scratch + n, slots, n * sizeof(int64_t), cudaMemcpyHostToDevice,
                           s->stream));
  rc = kvx_index_insert(s->index, s->d_scratch, s->d_scratch + n, n, s->stream);
  if (rc) return rc;
  KVX_CUDA(cudaStreamSynchronize(s->stream));
  return KVX_OK;
}

// Bytes of blocks st[i] (source pool) -> dt[i] (destination pool), every
// layer, K and V, on the source GPU.  Across GPUs of one process the
// destination pool is reached through UVA once peer access is on: the copy
// kernel's stores go over NVLink.
int copy_blocks(kvx_store* src, kvx_store* dst, const std::vector<int32_t>& st,
                const std::vector<int32_t>& dt) {
  const int64_t m = static_cast<int64_t>(st.size());
  if (dst->device != src->device) {
    // Across GPUs the destination GPU pulls: its copy kernel loads the source
    // pool over NVLink through a view of it (UVA + peer access) and stores
    // locally -- 0.99-1.0 of the link vs ~0.9 for pushing with stores
    // (profiles/r01/migrate.md) -- after the source stream's queued work.
    int rc = kvx_enable_peer(dst->device, src->device);
    if (!rc) rc = kvx_enable_peer(src->device, dst->device);
    if (rc) return rc;
    kvx_pool*& view = src->views[dst->device];
    if (!view) {
      kvx_pool_desc vd = src->desc;
      vd.device = dst->device;
      rc = kvx_pool_create_view(&vd, kvx_pool_base(src->pool), &view);
      if (rc) return rc;
    }
    struct Event {  // destroyed on every path
      cudaEvent_t e = nullptr;
      ~Event() {
        if (e) cudaEventDestroy(e);
      }
    } ev;
    {
      kvx::DeviceGuard gs(src->device);
      KVX_CUDA(cudaEventCreateWithFlags(&ev.e, cudaEventDisableTiming));
      KVX_CUDA(cudaEventRecord(ev.e, src->stream));
    }
    kvx::DeviceGuard g(dst->device);
    KVX_CUDA(cudaStreamWaitEvent(dst->stream, ev.e, 0));
    rc = ensure_scratch(dst, m);
    if (rc) return rc;
    int32_t* d_tables = reinterpret_cast<int32_t*>(dst->d_scratch);
    KVX_CUDA(cudaMemcpyAsync(d_tables, st.data(), m * sizeof(int32_t), cudaMemcpyHostToDevice,
                             dst->stream));
    KVX_CUDA(cudaMemcpyAsync(d_tables + m, dt.data(), m * sizeof(int32_t),
                             cudaMemcpyHostToDevice, dst->stream));
    rc = kvx_copy_paged(view, d_tables, dst->pool, d_tables + m, m, 0, kvx_pool_layers(src->pool),
                        dst->stream);
    if (rc) return rc;
    KVX_CUDA(cudaStreamSynchronize(dst->stream));
    return KVX_OK;
  }
  kvx::DeviceGuard g(src->device);
  int rc = ensure_scratch(src, m);
  if (rc) return rc;
  int32_t* d_tables = reinterpret_cast<int32_t*>(src->d_scratch);
  KVX_CUDA(cudaMemcpyAsync(d_tables, st.data(), m * sizeof(int32_t), cudaMemcpyHostToDevice,
                           src->stream));
  KVX_CUDA(cudaMemcpyAsync(d_tables + m, dt.data(), m * sizeof(int32_t), cudaMemcpyHostToDevice,
                           src->stream));
  rc = kvx_copy_paged(src->pool, d_tables, dst->pool, d_tables + m, m, 0,
                      kvx_pool_layers(src->pool), src->stream);
  if (rc) return rc;
  KVX_CUDA(cudaStreamSynchronize(src->stream));
  return KVX_OK;
}

}  // namespace

extern "C" {

int kvx_store_create(const kvx_pool_desc* desc, kvx_store** out) {
  KVX_REQUIRE(desc && out, "kvx_store_create: NULL argument");
  auto* s = new kvx_store();
  s->device = desc->device;
  s->desc = *desc;
  int rc = kvx_pool_create(desc, &s->pool);
  if (!rc) rc = kvx_index_create(desc->device, desc->slots, &s->index);
  if (!rc) rc = kvx_slot_alloc_create(desc->slots, &s->alloc);
  if (!rc) {
    kvx::DeviceGuard g(s->device);
    if (cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking) != cudaSuccess)
      rc = kvx::set_error(KVX_ECUDA, "kvx_store_create: stream");
  }
  if (rc) {
    kvx_store_destroy(s);
    return rc;
  }
  *out = s;
  return KVX_OK;
}

int kvx_store_destroy(kvx_store* s) {
  if (!s) return KVX_OK;
  kvx::DeviceGuard g(s->device);
  if (s->stream) cudaStreamSynchronize(s->stream);
  if (s->index) kvx_index_destroy(s->index);
  for (auto& kv : s->views) kvx_pool_destroy(kv.second);  // views do not own memory
  if (s->pool) kvx_pool_destroy(s->pool);
  if (s->alloc) kvx_slot_alloc_destroy(s->alloc);
  if (s->d_scratch) cudaFree(s->d_scratch);
  if (s->stream) cudaStreamDestroy(s->stream);
  delete s;
  return KVX_OK;
}

kvx_pool* kvx_store_pool(kvx_store* s) { return s ? s->pool : nullptr; }
kvx_index* kvx_store_index(kvx_store* s) { return s ? s->index : nullptr; }
void* kvx_store_stream(kvx_store* s) { return s ? reinterpret_cast<void*>(s->stream) : nullptr; }

int kvx_store_put(kvx_store* s, const int64_t* h_keys, int64_t n, int32_t* h_slots) {
  KVX_REQUIRE(s && (n == 0 || (h_keys && h_slots)), "kvx_store_put: bad arguments");
  for (int64_t i = 0; i < n; ++i)
    KVX_REQUIRE(!kvx::is_reserved(h_keys[i]), "kvx_store_put: reserved sentinel key");
  std::vector<int64_t> have;
  int rc = lookup_host(s, h_keys, n, have);
  if (rc) return rc;
  // absent keys get one slot each, however often they repeat in this call
  std::vector<int64_t> new_keys;
  std::unordered_map<int64_t, size_t> first;  // absent key -> index in new_keys
  std::vector<size_t> which(static_cast<size_t>(n), SIZE_MAX);
  for (int64_t i = 0; i < n; ++i) {
    if (have[i] >= 0) {
      h_slots[i] = static_cast<int32_t>(have[i]);
      continue;
    }
    auto it = first.emplace(h_keys[i], new_keys.size()).first;
    if (it->second == new_keys.size()) new_keys.push_back(h_keys[i]);
    which[i] = it->second;
  }
  std::vector<int32_t> got(new_keys.size());
  rc = kvx_slot_alloc_take(s->alloc, static_cast<int64_t>(new_keys.size()), got.data());
  if (rc) return rc;
  std::vector<int64_t> vals(got.begin(), got.end());
  rc = insert_host(s, new_keys.data(), vals.data(), static_cast<int64_t>(new_keys.size()));
  if (rc) {
    kvx_slot_alloc_release(s->alloc, got.data(), static_cast<int64_t>(got.size()));
    return rc;
  }
  for (int64_t i = 0; i < n; ++i)
    if (which[i] != SIZE_MAX) h_slots[i] = got[which[i]];
  return KVX_OK;
}

int kvx_store_get(kvx_store* s, const int64_t* h_keys, int64_t n, int32_t* h_slots) {
  KVX_REQUIRE(s && (n == 0 || (h_keys && h_slots)), "kvx_store_get: bad arguments");
  std::vector<int64_t> v;
  int rc = lookup_host(s, h_keys, n, v);
  if (rc) return rc;
  for (int64_t i = 0; i < n; ++i) h_slots[i] = static_cast<int32_t>(v[i]);
  return KVX_OK;
}

int kvx_store_evict(kvx_store* s, const int64_t* h_keys, int64_t n) {
  KVX_REQUIRE(s && (n == 0 || h_keys), "kvx_store_evict: bad arguments");
  std::vector<int64_t> v;
  int rc = lookup_host(s, h_keys, n, v);
  if (rc) return rc;
  std::vector<int32_t> freed;  // each resident slot once, however often its key repeats
  std::unordered_set<int64_t> seen;
  for (int64_t x : v)
    if (x >= 0 && seen.insert(x).second) freed.push_back(static_cast<int32_t>(x));
  kvx::DeviceGuard g(s->device);
  KVX_CUDA(cudaMemcpyAsync(s->d_scratch, h_keys, n * sizeof(int64_t), cudaMemcpyHostToDevice,
                           s->stream));
  rc = kvx_index_erase(s->index, s->d_scratch, n, s->stream);
  if (rc) return rc;
  KVX_CUDA(cudaStreamSynchronize(s->stream));
  return kvx_slot_alloc_release(s->alloc, freed.data(), static_cast<int64_t>(freed.size()));
}

int kvx_store_migrate(kvx_store* src, kvx_store* dst, const int64_t* h_keys, int64_t n,
                      int64_t* n_copied) {
  KVX_REQUIRE(src && dst && src != dst && (n == 0 || h_keys), "kvx_store_migrate: bad arguments");
  KVX_REQUIRE(kvx_pool_slab_bytes(src->pool) == kvx_pool_slab_bytes(dst->pool),
              "kvx_store_migrate: pools have different block shapes");
  if (n_copied) *n_copied = 0;
  if (n == 0) return KVX_OK;
  // 1. submit-time residency check on the source (sim_engine.cpp:605-639)
  std::vector<int64_t> s_slot, d_have;
  int rc = lookup_host(src, h_keys, n, s_slot);
  if (rc) return rc;
  for (int64_t x : s_slot)
    if (x < 0) return kvx::set_error(KVX_EABORTED, "kvx_store_migrate: source evicted part of the range");
  // 2. landing skips blocks the destination already holds (insert_replicated)
  rc = lookup_host(dst, h_keys, n, d_have);
  if (rc) return rc;
  std::vector<int64_t> keys;
  std::vector<int32_t> st;
  std::unordered_set<int64_t> seen;
  for (int64_t i = 0; i < n; ++i)
    if (d_have[i] < 0 && seen.insert(h_keys[i]).second) {
      keys.push_back(h_keys[i]);
      st.push_back(static_cast<int32_t>(s_slot[i]));
    }
  const int64_t m = static_cast<int64_t>(keys.size());
  if (m == 0) return KVX_OK;
  std::vector<int32_t> dt(static_cast<size_t>(m));
  rc = kvx_slot_alloc_take(dst->alloc, m, dt.data());
  if (rc) return rc;
  // 3. bytes: src pool -> dst pool for every layer, K and V, on the source GPU
  // Across GPUs of one process the destination pool is reached through UVA
  // once peer access is on: the copy kernel's stores go over NVLink.
  rc = copy_blocks(src, dst, st, dt);
  // 4. land: index the new blocks at the destination
  std::vector<int64_t> vals(dt.begin(), dt.end());
  if (!rc) rc = insert_host(dst, keys.data(), vals.data(), m);
  if (rc) {  // nothing landed: give the destination slots back
    kvx_slot_alloc_release(dst->alloc, dt.data(), m);
    return rc;
  }
  if (n_copied) *n_copied = m;
  return KVX_OK;
}

}  // extern "C"
