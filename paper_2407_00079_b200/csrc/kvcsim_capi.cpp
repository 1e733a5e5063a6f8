// kvcsim_capi.cpp -- C ABI (include/kvcsim_c.h) over the GPU-backed
// kvcsim::CachePool, translating C++ exceptions into kvx_status codes.
#include <stdexcept>
#include <string>
#include <vector>

#include "kvcsim/kvcache.hpp"
#include "kvcsim/kvx_batch.hpp"
#include "kvcsim_c.h"
#include "kvx.h"

#if __has_include("kvcsim/errors.hpp")
#include "kvcsim/errors.hpp"
#define KVCSIM_HAVE_ERRORS 1
#endif

struct kvcsim_pool {
  kvcsim::CachePool pool;
};

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return KVX_OK;
#ifdef KVCSIM_HAVE_ERRORS
  } catch (const kvcsim::ValidationError& e) {
    g_err = e.what();
    return KVX_EINVAL;
#endif
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    // ValidationError is a runtime_error too when errors.hpp was unavailable
    return std::string(e.what()).find("kvcsim gpu") == 0 ? KVX_ECUDA : KVX_EINVAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return KVX_ECUDA;
  }
}

kvcsim::CachePolicy policy_of(int p) {
  return p == 1 ? kvcsim::CachePolicy::kLfu
                : p == 2 ? kvcsim::CachePolicy::kLengthAware : kvcsim::CachePolicy::kLru;
}

std::span<const kvcsim::BlockId> span_of(const int64_t* k, int64_t n) {
  return {reinterpret_cast<const kvcsim::BlockId*>(k), static_cast<std::size_t>(n)};
}

void copy_out(const std::vector<kvcsim::BlockId>& v, int64_t* out, int64_t cap, int64_t* n) {
  for (std::size_t i = 0; i < v.size() && static_cast<int64_t>(i) < cap; ++i) out[i] = v[i];
  if (n) *n = static_cast<int64_t>(v.size());
}
}  // namespace

extern "C" {

const char* kvcsim_last_error(void) { return g_err.c_str(); }

int kvcsim_pool_create(int64_t capacity, int policy, kvcsim_pool** out) {
  if (!out) return KVX_EINVAL;
  return guarded([&] {
    std::optional<std::size_t> cap;
    if (capacity >= 0) cap = static_cast<std::size_t>(capacity);
    *out = new kvcsim_pool{kvcsim::CachePool(cap, policy_of(policy))};
  });
}

void kvcsim_pool_destroy(kvcsim_pool* p) { delete p; }

int kvcsim_pool_admit(kvcsim_pool* p, const int64_t* keys, int64_t n, int64_t skip_begin,
                      int64_t skip_end, int64_t* evicted, int64_t cap, int64_t* n_evicted,
                      int64_t* hits, int64_t* misses, int32_t* truncated) {
  return guarded([&] {
    const auto r = p->pool.admit_and_touch(span_of(keys, n), static_cast<std::size_t>(skip_begin),
                                           static_cast<std::size_t>(skip_end));
    copy_out(r.evicted, evicted, cap, n_evicted);
    if (hits) *hits = static_cast<int64_t>(r.hits);
    if (misses) *misses = static_cast<int64_t>(r.misses);
    if (truncated) *truncated = r.truncated ? 1 : 0;
  });
}

int kvcsim_pool_insert_replicated(kvcsim_pool* p, const int64_t* keys, int64_t n,
                                  int64_t chain_offset, int64_t* evicted, int64_t cap,
                                  int64_t* n_evicted) {
  return guarded([&] {
    copy_out(p->pool.insert_replicated(span_of(keys, n), static_cast<std::size_t>(chain_offset)),
             evicted, cap, n_evicted);
  });
}

int kvcsim_pool_match_prefix(const kvcsim_pool* p, const int64_t* keys, int64_t n,
                             int64_t* len) {
  return guarded([&] { *len = static_cast<int64_t>(p->pool.match_prefix(span_of(keys, n))); });
}

int kvcsim_pool_contains(const kvcsim_pool* p, int64_t key, int32_t* out) {
  return guarded([&] { *out = p->pool.contains(key) ? 1 : 0; });
}

int64_t kvcsim_pool_size(const kvcsim_pool* p) { return static_cast<int64_t>(p->pool.size()); }

void kvcsim_pool_stats(const kvcsim_pool* p, uint64_t* hits, uint64_t* misses) {
  *hits = p->pool.stats().hits;
  *misses = p->pool.stats().misses;
}

int kvcsim_find_best_prefix_match_batch(kvcsim_pool* const* pools, const int32_t* ids,
                                        int64_t n_inst, const int64_t* keys,
                                        const int64_t* key_off, int64_t n_req, int64_t* len_out,
                                        int64_t* best_len, int32_t* best_id) {
  return guarded([&] {
    std::vector<const kvcsim::CachePool*> inst(static_cast<std::size_t>(n_inst));
    std::vector<int> iid(static_cast<std::size_t>(n_inst));
    for (int64_t i = 0; i < n_inst; ++i) {
      inst[i] = &pools[i]->pool;
      iid[i] = ids[i];
    }
    const int64_t nk = n_req > 0 ? key_off[n_req] : 0;
    std::vector<std::size_t> per;
    const auto best = kvcsim::find_best_prefix_match_batch(
        inst, iid, span_of(keys, nk), {key_off, static_cast<std::size_t>(n_req + 1)},
        len_out ? &per : nullptr);
    for (int64_t r = 0; r < n_req; ++r) {
      best_len[r] = static_cast<int64_t>(best[r].prefix_blocks);
      best_id[r] = best[r].instance_id;
    }
    if (len_out)
      for (std::size_t i = 0; i < per.size(); ++i) len_out[i] = static_cast<int64_t>(per[i]);
  });
}

}  // extern "C"
