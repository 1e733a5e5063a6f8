// kvcsim_cachepool.cpp -- the GPU-backed kvcsim::CachePool (drop-in block
// manager; public API in include/kvcsim/kvcache.hpp).
//
// Semantics follow the reference block manager exactly
// (/root/reference/proj/src/kvcache.cpp):
//   * victim order: LRU by last use; LFU by (use count, last use);
//     LengthAware by (deepest position first, use count, last use); BlockId
//     breaks remaining ties (kvcache.cpp:48-63);
//   * a touch or an insert advances the logical clock (kvcache.cpp:65-70,90-96);
//   * the chain being admitted is never a victim, including its skip range
//     (kvcache.cpp:106-111); when every resident block is protected the miss
//     is counted but nothing is inserted (kvcache.cpp:84,89);
//   * admit: positions >= capacity are truncated misses (kvcache.cpp:124-127);
//     insert_replicated: resident blocks are skipped, a position >= capacity
//     stops the landing (kvcache.cpp:140-146).
// The structures are this file's own: protection is an epoch stamp on the
// entry (no per-call map of the chain), victims come from an ordered set of
// (rank, id) keys.  Residency queries (match_prefix, contains) are kernels on
// the B200 block index (libkvx: kvx_match_prefix_batch / kvx_index_lookup);
// every put mirrors its inserted and evicted ids into that index.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>

#include "kvcsim/kvcache.hpp"
#include "kvcsim/kvx_batch.hpp"
#include "kvx.h"

#if __has_include("kvcsim/errors.hpp")
#include "kvcsim/errors.hpp"
#else
namespace kvcsim {
class ValidationError : public std::runtime_error {
 public:
  explicit ValidationError(const std::string& what) : std::runtime_error(what) {}
};
}  // namespace kvcsim
#endif

#if __has_include("kvcsim/trace.hpp")
#include "kvcsim/trace.hpp"
#define KVCSIM_HAVE_TRACE 1
#endif

namespace kvcsim {

BlockId chain_hash(BlockId prev_key, std::uint64_t content_hash) {
  return kvx_chain_hash(prev_key, content_hash);
}

const char* to_string(CachePolicy policy) {
  switch (policy) {
    case CachePolicy::kLru: return "lru";
    case CachePolicy::kLfu: return "lfu";
    case CachePolicy::kLengthAware: return "length_aware";
  }
  return "?";
}

std::optional<CachePolicy> cache_policy_from_string(const std::string& name) {
  static const std::map<std::string, CachePolicy> kNames = {
      {"lru", CachePolicy::kLru}, {"lfu", CachePolicy::kLfu},
      {"length_aware", CachePolicy::kLengthAware}};
  const auto it = kNames.find(name);
  if (it == kNames.end()) return std::nullopt;
  return it->second;
}

// ---------------------------------------------------------------------------
// GPU plumbing.  This library has no CUDA runtime of its own: every device
// operation goes through libkvx's C ABI (one runtime per process, the one
// inside libkvx.so).  Per-call latency matters here -- the engine asks a
// pool one question at a time (conductor.cpp:65,198 issue 2P match_prefix
// calls per arrival) -- so a query never copies: its keys are staged in
// pinned, device-mapped host memory that the kernel reads directly, the
// kernel writes its answer into pinned memory, and the host polls that word
// (kvx_wait_host_word) instead of a device-to-host copy plus a stream
// synchronise.  Updates (a put's victims out, new blocks in) are one fused
// kernel (kvx_index_update) and do not wait at all.
namespace gpu {

[[noreturn]] void fail(int st, const char* what) {
  throw std::runtime_error(std::string("kvcsim gpu: ") + what + ": " + kvx_last_error() +
                           " (status " + std::to_string(st) + ")");
}

inline void ok(int st, const char* what) {
  if (st != KVX_OK) fail(st, what);
}

int selected_device() {
  static const int dev = [] {
    const char* env = std::getenv("KVCSIM_CUDA_DEVICE");
    return env ? std::atoi(env) : 0;
  }();
  return dev;
}

// One non-blocking stream per process for all pools (pools are single-owner
// and the engine is single-threaded, so one in-order queue suffices).
void* shared_stream() {
  static std::once_flag once;
  static void* s = nullptr;
  std::call_once(once, [] { ok(kvx_stream_create(selected_device(), &s), "kvx_stream_create"); });
  return s;
}

// Per-process call statistics (KVCSIM_GPU_STATS=1 prints them at exit).
struct Stats {
  uint64_t queries = 0, cached = 0, updates = 0, pools = 0, recycled = 0;
  double query_s = 0, update_s = 0, pool_s = 0;
  ~Stats() {
    if (std::getenv("KVCSIM_GPU_STATS"))
      std::fprintf(stderr,
                   "kvcsim gpu: %llu queries (%llu from the per-version cache) %.1f us avg, "
                   "%llu index updates %.1f us avg, %llu pools (%llu recycled) %.1f us avg\n",
                   static_cast<unsigned long long>(queries), static_cast<unsigned long long>(cached),
                   queries ? 1e6 * query_s / queries : 0.0, static_cast<unsigned long long>(updates),
                   updates ? 1e6 * update_s / updates : 0.0, static_cast<unsigned long long>(pools),
                   static_cast<unsigned long long>(recycled), pools ? 1e6 * pool_s / pools : 0.0);
  }
};
Stats& stats() {
  static Stats st;
  return st;
}

struct Timer {
  double& acc;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  explicit Timer(double& a) : acc(a) {}
  ~Timer() {
    acc += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
};

// Device resources of destroyed pools, reused by new ones: creating a GPU
// index and a pinned arena costs allocations and a device synchronise, and
// engines (and the reference's tests) create many short-lived pools.  Never
// freed at exit (process teardown releases them).
struct Recycled {
  kvx_index* idx;
  int64_t* arena;
  std::size_t half;
  uint64_t next_op;
};
std::vector<Recycled>& recycle_bin() {
  static auto* bin = new std::vector<Recycled>();
  return *bin;
}

class DeviceIndex {
 public:
  DeviceIndex() : dev_(selected_device()), stream_(shared_stream()) {
    Timer t(stats().pool_s);
    ++stats().pools;
    auto& bin = recycle_bin();
    if (!bin.empty()) {  // an emptied index and its arena from a destroyed pool
      const Recycled r = bin.back();
      bin.pop_back();
      idx_ = r.idx;
      arena_ = r.arena;
      half_ = r.half;
      next_op_ = r.next_op;
      ++stats().recycled;
      return;
    }
    ok(kvx_index_create(dev_, 0, &idx_), "kvx_index_create");
    grow(256);
  }
  ~DeviceIndex() {
    if (!idx_) return;
    // emptied on the shared stream (ordered before any later use of it);
    // the arena's ops counter travels with it
    if (kvx_index_clear(idx_, stream_) == KVX_OK) {
      recycle_bin().push_back({idx_, arena_, half_, next_op_});
      return;
    }
    kvx_sync(stream_);
    kvx_index_destroy(idx_);
    if (arena_) kvx_host_free(arena_);
  }
  DeviceIndex(const DeviceIndex&) = delete;
  DeviceIndex& operator=(const DeviceIndex&) = delete;

  const kvx_index* handle() const { return idx_; }

  void apply(const std::vector<BlockId>& erase, const std::vector<BlockId>& insert) {
    if (erase.empty() && insert.empty()) return;
    Timer t(stats().update_s);
    const std::size_t ne = erase.size(), ni = insert.size();
    int64_t* buf = stage(ne + ni);
    std::memcpy(buf, erase.data(), ne * sizeof(int64_t));
    std::memcpy(buf + ne, insert.data(), ni * sizeof(int64_t));
    ok(kvx_index_update(idx_, buf, static_cast<int64_t>(ne), buf + ne, nullptr,
                        static_cast<int64_t>(ni), stream_), "kvx_index_update");
    retire();
    ++version_;
    ++stats().updates;
  }

  std::size_t match(std::span<const BlockId> blocks) const {
    if (blocks.empty()) return 0;
    Timer t(stats().query_s);
    const std::size_t n = blocks.size();
    ++stats().queries;
    // the reference's conductor asks each pool the same chain twice per
    // arrival (conductor.cpp:65 then :198): answer a repeat from this pool's
    // last answer while the pool is unchanged (same version, same keys)
    if (cache_version_ == version_ && cache_keys_.size() == n &&
        std::memcmp(cache_keys_.data(), blocks.data(), n * sizeof(BlockId)) == 0) {
      ++stats().cached;
      return cache_len_;
    }
    int64_t* buf = stage(n + 2);
    buf[0] = 0;
    buf[1] = static_cast<int64_t>(n);
    std::memcpy(buf + 2, blocks.data(), n * sizeof(int64_t));
    volatile int64_t* res = result_word();
    *res = -1;
    const int32_t id = 0;
    const kvx_index* one[1] = {idx_};
    ok(kvx_match_prefix_batch(one, &id, 1, buf + 2, buf, 1, const_cast<int64_t*>(res), nullptr,
                              nullptr, stream_), "match_prefix");
    retire();
    ok(kvx_wait_host_word(res, 0, stream_), "match_prefix wait");
    cache_keys_.assign(blocks.begin(), blocks.end());
    cache_version_ = version_;
    cache_len_ = static_cast<std::size_t>(*res);
    return cache_len_;
  }

  bool contains(BlockId id) const {
    Timer t(stats().query_s);
    ++stats().queries;
    int64_t* buf = stage(1);
    buf[0] = id;
    volatile int64_t* res = result_word();
    *res = std::numeric_limits<int64_t>::min();
    ok(kvx_index_lookup(idx_, buf, 1, const_cast<int64_t*>(res), stream_), "lookup");
    retire();
    ok(kvx_wait_host_word(res, -1, stream_), "contains wait");  // -1 absent, >= 0 present
    return *res >= 0;
  }

 private:
  // Arena (pinned, mapped): [done][result][half 0 | half 1].  Operation k
  // stages its keys in half k % 2; before half h is overwritten the
  // operation that last read it (k - 2) must be done: each operation is
  // followed by a stream-ordered write of k into `done`.
  volatile int64_t* done_word() const { return arena_; }
  volatile int64_t* result_word() const { return arena_ + 1; }

  int64_t* stage(std::size_t words) const {
    if (words > half_) grow(words);
    const uint64_t k = next_op_;
    if (k >= 2) ok(kvx_wait_host_word(done_word(), static_cast<int64_t>(k - 2), stream_),
                   "staging reuse wait");
    return arena_ + 2 + (k & 1) * half_;
  }

  void retire() const {
    ok(kvx_signal_write(stream_, const_cast<int64_t*>(done_word()), next_op_), "signal");
    ++next_op_;
  }

  void grow(std::size_t words) const {
    std::size_t cap = std::max<std::size_t>(256, half_);
    while (cap < words) cap *= 2;
    if (arena_) {
      ok(kvx_sync(stream_), "arena drain");  // nothing in flight reads the old arena
      kvx_host_free(arena_);
      arena_ = nullptr;
    }
    void* p = nullptr;
    ok(kvx_host_alloc(static_cast<int64_t>((2 + 2 * cap) * sizeof(int64_t)), &p), "kvx_host_alloc");
    arena_ = static_cast<int64_t*>(p);
    half_ = cap;
    arena_[0] = static_cast<int64_t>(next_op_) - 1;  // every earlier op is done
  }

  int dev_;
  void* stream_;
  kvx_index* idx_ = nullptr;
  mutable int64_t* arena_ = nullptr;
  mutable std::size_t half_ = 0;
  mutable uint64_t next_op_ = 0;
  uint64_t version_ = 0;  // bumped by every update (answers cached per version)
  mutable uint64_t cache_version_ = ~0ull;
  mutable std::vector<BlockId> cache_keys_;
  mutable std::size_t cache_len_ = 0;
};

}  // namespace gpu

// ---------------------------------------------------------------------------

CachePool::CachePool(std::optional<std::size_t> capacity_blocks, CachePolicy policy)
    : capacity_(capacity_blocks), policy_(policy) {
  if (capacity_ && *capacity_ == 0)
    throw ValidationError("cache capacity must be >= 1 block (or unbounded)");
  dev_ = std::make_unique<gpu::DeviceIndex>();
}

CachePool::~CachePool() = default;
CachePool::CachePool(CachePool&&) noexcept = default;
CachePool& CachePool::operator=(CachePool&&) noexcept = default;

const void* CachePool::device_index() const { return dev_->handle(); }

CachePool::OrderKey CachePool::order_key(BlockId id, const Entry& e) const {
  const auto lu = static_cast<std::int64_t>(e.last_use);
  const auto uc = static_cast<std::int64_t>(e.use_count);
  switch (policy_) {
    case CachePolicy::kLru: return {lu, 0, 0, id};
    case CachePolicy::kLfu: return {uc, lu, 0, id};
    case CachePolicy::kLengthAware: return {-static_cast<std::int64_t>(e.position), uc, lu, id};
  }
  return {0, 0, 0, id};
}

void CachePool::reference(BlockId id, Entry& e) {
  order_.erase(order_key(id, e));
  e.last_use = ++clock_;
  ++e.use_count;
  order_.insert(order_key(id, e));
}

// Insert `id` at `position`, evicting unguarded victims while the pool is
// full.  Returns false when no room could be made.
bool CachePool::place(BlockId id, std::uint32_t position, std::vector<BlockId>& evicted,
                      std::vector<BlockId>& inserted) {
  if (capacity_) {
    while (meta_.size() >= *capacity_) {
      auto v = order_.begin();
      while (v != order_.end() && meta_.find(v->id)->second.guard == guard_epoch_) ++v;
      if (v == order_.end()) return false;  // everything resident is guarded
      const BlockId victim = v->id;
      order_.erase(v);
      meta_.erase(victim);
      evicted.push_back(victim);
    }
  }
  Entry e;
  e.last_use = ++clock_;
  e.use_count = 1;
  e.position = position;
  e.guard = guard_epoch_;
  order_.insert(order_key(id, e));
  meta_.emplace(id, e);
  inserted.push_back(id);
  return true;
}

void CachePool::sync_device(const std::vector<BlockId>& inserted,
                            const std::vector<BlockId>& evicted) {
  dev_->apply(evicted, inserted);
}

CachePool::AdmitResult CachePool::admit_and_touch(std::span<const BlockId> blocks) {
  return admit_and_touch(blocks, 0, 0);
}

namespace {
// INT64_MIN / INT64_MIN+1 are the device index's empty / tombstone markers
// (include/kvx.h); the only keys this block manager cannot hold.
void reject_sentinels(std::span<const BlockId> blocks) {
  for (BlockId id : blocks)
    if (id <= KVX_KEY_TOMBSTONE)
      throw ValidationError("block id " + std::to_string(id) +
                            " is reserved by the GPU block index (INT64_MIN, INT64_MIN+1)");
}
}  // namespace

CachePool::AdmitResult CachePool::admit_and_touch(std::span<const BlockId> blocks,
                                                  std::size_t skip_begin, std::size_t skip_end) {
  reject_sentinels(blocks);
  AdmitResult r;
  ++guard_epoch_;
  for (BlockId id : blocks) {  // the whole chain is protected, skip range included
    auto it = meta_.find(id);
    if (it != meta_.end()) it->second.guard = guard_epoch_;
  }
  std::vector<BlockId> inserted;
  for (std::size_t i = 0; i < blocks.size(); ++i) {
    if (i >= skip_begin && i < skip_end) continue;
    const BlockId id = blocks[i];
    auto it = meta_.find(id);
    if (it != meta_.end()) {
      ++r.hits;
      ++stats_.hits;
      reference(id, it->second);
      continue;
    }
    ++r.misses;
    ++stats_.misses;
    if (capacity_ && i >= *capacity_) {
      r.truncated = true;
      continue;
    }
    place(id, static_cast<std::uint32_t>(i), r.evicted, inserted);
  }
  sync_device(inserted, r.evicted);
  return r;
}

std::vector<BlockId> CachePool::insert_replicated(std::span<const BlockId> blocks,
                                                  std::size_t chain_offset) {
  reject_sentinels(blocks);
  std::vector<BlockId> evicted, inserted;
  ++guard_epoch_;
  for (BlockId id : blocks) {
    auto it = meta_.find(id);
    if (it != meta_.end()) it->second.guard = guard_epoch_;
  }
  for (std::size_t i = 0; i < blocks.size(); ++i) {
    const std::size_t position = chain_offset + i;
    if (meta_.count(blocks[i])) continue;
    if (capacity_ && position >= *capacity_) break;
    place(blocks[i], static_cast<std::uint32_t>(position), evicted, inserted);
  }
  sync_device(inserted, evicted);
  return evicted;
}

std::size_t CachePool::match_prefix(std::span<const BlockId> blocks) const {
  return dev_->match(blocks);
}

bool CachePool::contains(BlockId id) const { return dev_->contains(id); }

std::size_t match_prefix(const CachePool& index, std::span<const BlockId> request_blocks) {
  return index.match_prefix(request_blocks);
}

#ifdef KVCSIM_HAVE_TRACE
std::vector<PolicySweepPoint> policy_sweep(const std::vector<RequestRecord>& trace,
                                           CachePolicy policy,
                                           std::span<const std::optional<std::size_t>> capacities) {
  if (capacities.empty()) throw ValidationError("policy_sweep needs at least one capacity");
  std::vector<PolicySweepPoint> out;
  for (const auto& cap : capacities) {
    CachePool pool(cap, policy);
    for (const auto& rec : trace) pool.admit_and_touch(rec.hash_ids);
    out.push_back({cap, pool.stats().hit_ratio()});
  }
  return out;
}

std::vector<PopularityPoint> popularity_cdf(const std::vector<RequestRecord>& trace) {
  std::unordered_map<BlockId, std::uint64_t> refs;
  for (const auto& rec : trace)
    for (BlockId id : rec.hash_ids) ++refs[id];
  if (refs.empty()) return {};
  std::map<std::uint64_t, std::size_t> by_count;  // hits beyond first insert -> blocks
  for (const auto& kv : refs) ++by_count[kv.second - 1];
  std::vector<PopularityPoint> cdf;
  std::size_t acc = 0;
  for (const auto& [hits, n] : by_count) {
    acc += n;
    cdf.push_back({hits, static_cast<double>(acc) / static_cast<double>(refs.size())});
  }
  return cdf;
}
#endif

// ---------------------------------------------------------------------------
// Batched queries (kvcsim/kvx_batch.hpp)

std::vector<BestPrefixMatchBatch> find_best_prefix_match_batch(
    std::span<const CachePool* const> instances, std::span<const int> instance_ids,
    std::span<const BlockId> keys, std::span<const std::int64_t> key_offsets,
    std::vector<std::size_t>* per_instance) {
  if (instances.empty()) throw ValidationError("find_best_prefix_match: empty prefill pool");
  if (instances.size() != instance_ids.size())
    throw ValidationError("find_best_prefix_match_batch: ids and instances differ in length");
  if (key_offsets.empty()) return {};
  const std::size_t n_req = key_offsets.size() - 1;
  const std::size_t n_inst = instances.size();
  if (n_inst > KVX_MAX_INSTANCES) throw ValidationError("too many instances");
  std::vector<const kvx_index*> idx(n_inst);
  std::vector<int32_t> ids(n_inst);
  for (std::size_t i = 0; i < n_inst; ++i) {
    idx[i] = static_cast<const kvx_index*>(instances[i]->device_index());
    ids[i] = instance_ids[i];
  }
  void* s = gpu::shared_stream();
  const std::size_t nk = keys.size();
  // device layout: [key_off n_req+1][keys nk][len n_req*n_inst][best_len n_req][best_id n_req]
  const std::size_t words = (n_req + 1) + nk + n_req * n_inst + n_req + (n_req + 1) / 2 + 1;
  void* dv = nullptr;
  const int dev = gpu::selected_device();
  gpu::ok(kvx_device_alloc(dev, static_cast<int64_t>(words * sizeof(int64_t)), &dv),
          "kvx_device_alloc");
  struct Free {
    int dev;
    void* p;
    ~Free() { kvx_device_free(dev, p); }
  } guard{dev, dv};
  auto* d = static_cast<int64_t*>(dv);
  int64_t* d_off = d;
  int64_t* d_keys = d_off + (n_req + 1);
  int64_t* d_len = d_keys + nk;
  int64_t* d_best = d_len + n_req * n_inst;
  auto* d_bid = reinterpret_cast<int32_t*>(d_best + n_req);
  gpu::ok(kvx_memcpy_async(d_off, key_offsets.data(),
                           static_cast<int64_t>((n_req + 1) * sizeof(int64_t)), s), "H2D offsets");
  gpu::ok(kvx_memcpy_async(d_keys, keys.data(), static_cast<int64_t>(nk * sizeof(int64_t)), s),
          "H2D keys");
  gpu::ok(kvx_match_prefix_batch(idx.data(), ids.data(), static_cast<int64_t>(n_inst),
                                 d_keys, d_off, static_cast<int64_t>(n_req),
                                 per_instance ? d_len : nullptr, d_best, d_bid, s),
          "kvx_match_prefix_batch");
  std::vector<int64_t> best(n_req);
  std::vector<int32_t> bid(n_req);
  std::vector<int64_t> lens(per_instance ? n_req * n_inst : 0);
  gpu::ok(kvx_memcpy_async(best.data(), d_best, static_cast<int64_t>(n_req * sizeof(int64_t)), s),
          "D2H best");
  gpu::ok(kvx_memcpy_async(bid.data(), d_bid, static_cast<int64_t>(n_req * sizeof(int32_t)), s),
          "D2H ids");
  if (per_instance)
    gpu::ok(kvx_memcpy_async(lens.data(), d_len, static_cast<int64_t>(lens.size() * sizeof(int64_t)),
                             s), "D2H lens");
  gpu::ok(kvx_sync(s), "sync");  // before the allocation is freed and results are read
  std::vector<BestPrefixMatchBatch> out(n_req);
  for (std::size_t r = 0; r < n_req; ++r) out[r] = {static_cast<std::size_t>(best[r]), bid[r]};
  if (per_instance) per_instance->assign(lens.begin(), lens.end());
  return out;
}

}  // namespace kvcsim
