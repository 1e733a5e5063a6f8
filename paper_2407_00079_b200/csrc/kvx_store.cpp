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
// (kvx_copy_paged); when the two stores live on different GPUs the
// destination GPU pulls through a peer mapping of the source pool (NVLink).
//
// Asynchronous migration (kvx_store_migrate_submit / _query / _wait): every
// source store owns ONE in-order migration FIFO -- the reference's per-sender
// link (begin = max(now, sender_busy_until_ms), sim_engine.cpp:409-411).  A
// migration BEGINS when it reaches the head of its sender's FIFO and the
// previous one finished: only then is the source checked (any block evicted
// -> aborted, KVX_EABORTED, nothing lands; sim_engine.cpp:605-639), the
// destination slots reserved and the copy launched.  Its source slots stay
// pinned until the copy is done, so an eviction meanwhile removes the key but
// the slot is not reused until then.  It lands (index insert at the
// destination, skipping blocks that became resident meanwhile) when it is
// DONE (sim_engine.cpp:641-650).  Progress is made by every submit / query /
// wait / progress call on the source store (no host threads).
#include <cuda_runtime.h>

#include <algorithm>
#include <deque>
#include <map>
#include <memory>
#include <cstdint>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "kvx.h"
#include "kvx_common.cuh"

namespace {
struct Migration {
  enum State { kQueued, kRunning, kDone, kAborted, kFailed } state = kQueued;
  uint64_t ticket = 0;
  kvx_store* dst = nullptr;
  std::vector<int64_t> keys;        // requested range (host copy)
  std::vector<int64_t> land_keys;   // keys copied (absent at the destination at begin)
  std::vector<int32_t> st, dt;      // source / destination slots of land_keys
  cudaEvent_t after = nullptr;      // submit-time dependency (after_stream)
  cudaEvent_t done = nullptr;       // recorded after the copy
  cudaStream_t q = nullptr;         // the stream the copy ran on
  int32_t* d_tables = nullptr;      // st | dt on the copying device
  int status = KVX_OK;
  int64_t copied = 0;
};
}  // namespace

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
  // migration FIFO of this store as a SENDER
  cudaStream_t mig_q = nullptr;  // copies that run on this GPU (same-GPU or pulled into it)
  std::deque<std::unique_ptr<Migration>> fifo;
  std::unordered_map<uint64_t, std::unique_ptr<Migration>> finished;
  uint64_t next_ticket = 1;
  std::unordered_map<int32_t, int> pinned;  // source slot -> in-flight copies reading it
  std::vector<int32_t> deferred_free;       // evicted while pinned
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
    if (cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&s->mig_q, cudaStreamNonBlocking) != cudaSuccess)
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
  for (auto& m : s->fifo) {  // in-flight copies finish; queued ones are dropped
    if (m->done) cudaEventSynchronize(m->done);
    if (m->done) cudaEventDestroy(m->done);
    if (m->after) cudaEventDestroy(m->after);
    if (m->d_tables) cudaFree(m->d_tables);
  }
  s->fifo.clear();
  for (auto& kv : s->finished) {
    if (kv.second->done) cudaEventDestroy(kv.second->done);
    if (kv.second->after) cudaEventDestroy(kv.second->after);
  }
  s->finished.clear();
  if (s->mig_q) {
    cudaStreamSynchronize(s->mig_q);
    cudaStreamDestroy(s->mig_q);
  }
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
  // a slot an in-flight migration still reads is released when that copy is done
  std::vector<int32_t> now;
  for (int32_t x : freed) {
    if (s->pinned.count(x)) s->deferred_free.push_back(x);
    else now.push_back(x);
  }
  return kvx_slot_alloc_release(s->alloc, now.data(), static_cast<int64_t>(now.size()));
}

}  // extern "C"

namespace {

int mig_launch(kvx_store* src, Migration* m);

// Begin the head migration of src's FIFO: residency check, destination slot
// reservation, copy launch.  The migration ends kRunning, kDone (nothing to
// copy), kAborted or kFailed.
int mig_begin(kvx_store* src, Migration* m) {
  kvx_store* dst = m->dst;
  const int64_t n = static_cast<int64_t>(m->keys.size());
  std::vector<int64_t> s_slot, d_have;
  int rc = lookup_host(src, m->keys.data(), n, s_slot);
  if (rc) return rc;
  for (int64_t x : s_slot)
    if (x < 0) {  // the source evicted part of the range before the link freed up
      m->state = Migration::kAborted;
      m->status = KVX_EABORTED;
      return KVX_OK;
    }
  rc = lookup_host(dst, m->keys.data(), n, d_have);
  if (rc) return rc;
  std::unordered_set<int64_t> seen;
  for (int64_t i = 0; i < n; ++i)
    if (d_have[i] < 0 && seen.insert(m->keys[i]).second) {
      m->land_keys.push_back(m->keys[i]);
      m->st.push_back(static_cast<int32_t>(s_slot[i]));
    }
  const int64_t k = static_cast<int64_t>(m->land_keys.size());
  if (k == 0) {
    m->state = Migration::kDone;
    return KVX_OK;
  }
  m->dt.resize(static_cast<size_t>(k));
  rc = kvx_slot_alloc_take(dst->alloc, k, m->dt.data());
  if (rc) {
    m->dt.clear();
    return rc;
  }
  rc = mig_launch(src, m);
  if (rc) {  // nothing launched: give the destination slots back
    kvx_slot_alloc_release(dst->alloc, m->dt.data(), k);
    m->dt.clear();
  }
  return rc;
}

// Launch the copy of a begun migration (slots reserved on both sides).
int mig_launch(kvx_store* src, Migration* m) {
  kvx_store* dst = m->dst;
  const int64_t k = static_cast<int64_t>(m->land_keys.size());
  int rc = KVX_OK;
  // the copy: same GPU on the source's FIFO queue; across GPUs the destination
  // GPU pulls through a view of the source pool (0.99-1.0 of the link,
  // profiles/r01/migrate.md), on the destination's queue
  const bool cross = dst->device != src->device;
  const int dev = cross ? dst->device : src->device;
  kvx_pool* from = src->pool;
  if (cross) {
    rc = kvx_enable_peer(dst->device, src->device);
    if (!rc) rc = kvx_enable_peer(src->device, dst->device);
    if (rc) return rc;
    kvx_pool*& view = src->views[dst->device];
    if (!view) {
      kvx_pool_desc vd = src->desc;
      vd.device = dst->device;
      rc = kvx_pool_create_view(&vd, kvx_pool_base(src->pool), &view);
      if (rc) return rc;
    }
    from = view;
  }
  m->q = cross ? dst->mig_q : src->mig_q;
  cudaEvent_t src_ready = nullptr;
  {
    kvx::DeviceGuard gs(src->device);  // after the KV queued on the source's stream
    KVX_CUDA(cudaEventCreateWithFlags(&src_ready, cudaEventDisableTiming));
    KVX_CUDA(cudaEventRecord(src_ready, src->stream));
  }
  kvx::DeviceGuard g(dev);
  cudaError_t e = cudaStreamWaitEvent(m->q, src_ready, 0);
  cudaEventDestroy(src_ready);
  KVX_CUDA(e);
  if (m->after) KVX_CUDA(cudaStreamWaitEvent(m->q, m->after, 0));
  KVX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&m->d_tables), 2 * k * sizeof(int32_t), m->q));
  KVX_CUDA(cudaMemcpyAsync(m->d_tables, m->st.data(), k * sizeof(int32_t),
                           cudaMemcpyHostToDevice, m->q));
  KVX_CUDA(cudaMemcpyAsync(m->d_tables + k, m->dt.data(), k * sizeof(int32_t),
                           cudaMemcpyHostToDevice, m->q));
  rc = kvx_copy_paged(from, m->d_tables, dst->pool, m->d_tables + k, k, 0,
                      kvx_pool_layers(src->pool), m->q);
  if (rc) return rc;
  KVX_CUDA(cudaFreeAsync(m->d_tables, m->q));
  m->d_tables = nullptr;
  KVX_CUDA(cudaEventCreateWithFlags(&m->done, cudaEventDisableTiming));
  KVX_CUDA(cudaEventRecord(m->done, m->q));
  for (int32_t x : m->st) ++src->pinned[x];
  m->state = Migration::kRunning;
  return KVX_OK;
}

// The head copy finished: unpin, land at the destination (skipping blocks it
// gained meanwhile), release deferred evictions.
int mig_finish(kvx_store* src, Migration* m) {
  for (int32_t x : m->st) {
    auto it = src->pinned.find(x);
    if (it != src->pinned.end() && --it->second == 0) src->pinned.erase(it);
  }
  std::vector<int32_t> release;
  for (size_t i = 0; i < src->deferred_free.size();) {
    const int32_t x = src->deferred_free[i];
    if (!src->pinned.count(x)) {
      release.push_back(x);
      src->deferred_free[i] = src->deferred_free.back();
      src->deferred_free.pop_back();
    } else {
      ++i;
    }
  }
  int rc = kvx_slot_alloc_release(src->alloc, release.data(), static_cast<int64_t>(release.size()));
  if (rc) return rc;
  kvx_store* dst = m->dst;
  const int64_t k = static_cast<int64_t>(m->land_keys.size());
  std::vector<int64_t> now;
  rc = lookup_host(dst, m->land_keys.data(), k, now);
  if (rc) return rc;
  std::vector<int64_t> keys, vals;
  std::vector<int32_t> unused;
  for (int64_t i = 0; i < k; ++i) {
    if (now[i] >= 0) unused.push_back(m->dt[i]);  // became resident meanwhile: keep that one
    else {
      keys.push_back(m->land_keys[i]);
      vals.push_back(m->dt[i]);
    }
  }
  rc = insert_host(dst, keys.data(), vals.data(), static_cast<int64_t>(keys.size()));
  if (rc) return rc;
  rc = kvx_slot_alloc_release(dst->alloc, unused.data(), static_cast<int64_t>(unused.size()));
  if (rc) return rc;
  m->copied = static_cast<int64_t>(keys.size());
  m->state = Migration::kDone;
  return KVX_OK;
}

// Advance src's FIFO as far as possible without blocking (block: wait for
// the running head's copy first).
int mig_progress(kvx_store* src, bool block) {
  while (!src->fifo.empty()) {
    Migration* m = src->fifo.front().get();
    if (m->state == Migration::kQueued) {
      int rc = mig_begin(src, m);
      if (rc) {  // a CUDA / allocation failure: report on this ticket, move on
        m->state = Migration::kFailed;
        m->status = rc;
      }
    }
    if (m->state == Migration::kRunning) {
      kvx::DeviceGuard g(m->dst->device == src->device ? src->device : m->dst->device);
      cudaError_t e = block ? cudaEventSynchronize(m->done) : cudaEventQuery(m->done);
      if (e == cudaErrorNotReady) return KVX_OK;
      if (e != cudaSuccess) {
        m->state = Migration::kFailed;
        m->status = kvx::cuda_error(e, "migration copy");
      } else {
        int rc = mig_finish(src, m);
        if (rc) {
          m->state = Migration::kFailed;
          m->status = rc;
        }
      }
    }
    std::unique_ptr<Migration> done = std::move(src->fifo.front());
    src->fifo.pop_front();
    src->finished[done->ticket] = std::move(done);
  }
  return KVX_OK;
}

}  // namespace

extern "C" {

int kvx_store_migrate_submit(kvx_store* src, kvx_store* dst, const int64_t* h_keys, int64_t n,
                             void* after_stream, uint64_t* ticket) {
  KVX_REQUIRE(src && dst && src != dst && (n == 0 || h_keys) && ticket,
              "kvx_store_migrate_submit: bad arguments");
  KVX_REQUIRE(kvx_pool_slab_bytes(src->pool) == kvx_pool_slab_bytes(dst->pool) &&
                  kvx_pool_layers(src->pool) == kvx_pool_layers(dst->pool),
              "kvx_store_migrate_submit: pools have different block shapes");
  auto m = std::make_unique<Migration>();
  m->ticket = src->next_ticket++;
  m->dst = dst;
  m->keys.assign(h_keys, h_keys + n);
  if (after_stream) {
    int dev = 0;
    KVX_CUDA(cudaStreamGetDevice(kvx::as_stream(after_stream), &dev));
    kvx::DeviceGuard g(dev);
    KVX_CUDA(cudaEventCreateWithFlags(&m->after, cudaEventDisableTiming));
    KVX_CUDA(cudaEventRecord(m->after, kvx::as_stream(after_stream)));
  }
  *ticket = m->ticket;
  src->fifo.push_back(std::move(m));
  return mig_progress(src, false);
}

int kvx_store_migrate_progress(kvx_store* src) {
  KVX_REQUIRE(src != nullptr, "kvx_store_migrate_progress: NULL");
  return mig_progress(src, false);
}

namespace {
int mig_result(kvx_store* src, uint64_t ticket, int64_t* n_copied, bool erase) {
  auto it = src->finished.find(ticket);
  Migration* m = it->second.get();
  if (n_copied) *n_copied = m->copied;
  const int st = m->status;
  if (erase) {
    if (m->done) cudaEventDestroy(m->done);
    if (m->after) cudaEventDestroy(m->after);
    src->finished.erase(it);
  }
  if (st == KVX_EABORTED)
    return kvx::set_error(KVX_EABORTED, "migration aborted: the source evicted part of the range "
                                        "before the transfer began");
  if (st) return st;
  return KVX_OK;
}
}  // namespace

int kvx_store_migrate_query(kvx_store* src, uint64_t ticket) {
  KVX_REQUIRE(src && ticket >= 1 && ticket < src->next_ticket, "kvx_store_migrate_query: bad ticket");
  int rc = mig_progress(src, false);
  if (rc) return rc;
  if (!src->finished.count(ticket)) {
    for (auto& m : src->fifo)
      if (m->ticket == ticket) return KVX_EAGAIN;
    return kvx::set_error(KVX_EINVAL, "kvx_store_migrate_query: ticket already collected");
  }
  return mig_result(src, ticket, nullptr, false);
}

int kvx_store_migrate_wait(kvx_store* src, uint64_t ticket, int64_t* n_copied) {
  KVX_REQUIRE(src && ticket >= 1 && ticket < src->next_ticket, "kvx_store_migrate_wait: bad ticket");
  if (n_copied) *n_copied = 0;
  while (!src->finished.count(ticket)) {
    bool queued = false;
    for (auto& m : src->fifo) queued = queued || m->ticket == ticket;
    if (!queued) return kvx::set_error(KVX_EINVAL, "kvx_store_migrate_wait: ticket already collected");
    int rc = mig_progress(src, true);
    if (rc) return rc;
  }
  return mig_result(src, ticket, n_copied, true);
}

int kvx_store_migrate(kvx_store* src, kvx_store* dst, const int64_t* h_keys, int64_t n,
                      int64_t* n_copied) {
  if (n_copied) *n_copied = 0;
  uint64_t t = 0;
  int rc = kvx_store_migrate_submit(src, dst, h_keys, n, nullptr, &t);
  if (rc) return rc;
  return kvx_store_migrate_wait(src, t, n_copied);
}

}  // extern "C"
