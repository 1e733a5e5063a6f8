/*
 * ref_shim.cpp -- extern "C" view of the UNMODIFIED reference implementation
 * (TEST INFRASTRUCTURE ONLY).
 *
 * oracle/Makefile compiles this file together with the reference's own
 * proj/src/{kvcache,conductor,perf_model}.cpp, in place under
 * /root/reference, with -Dkvcsim=kvref so the reference symbols live in
 * namespace kvref.  The result, oracle/_ref/libkvref.so, is what tests use to
 * pin the C restatement (kvx_oracle.c) and what bench.py times as the
 * "reference" CPU arm for prefix matching.  No reference source is copied
 * into this repository.
 *
 * Functions wrapped (reference file:line):
 *   chain_hash                 proj/src/kvcache.cpp:14-23
 *   CachePool ctor             proj/src/kvcache.cpp:41-46
 *   admit_and_touch            proj/src/kvcache.cpp:103-131
 *   insert_replicated          proj/src/kvcache.cpp:133-148
 *   match_prefix               proj/src/kvcache.cpp:150-158
 *   find_best_prefix_match     proj/src/conductor.cpp:57-73
 *   estimate_transfer_time     proj/src/perf_model.cpp:51-59
 */
#include <algorithm>
#include <array>
#include <cstdint>
#include <exception>
#include <optional>
#include <span>
#include <thread>
#include <vector>

#include "kvcsim/conductor.hpp"
#include "kvcsim/errors.hpp"
#include "kvcsim/kvcache.hpp"
#include "kvcsim/perf_model.hpp"

namespace {
kvref::CachePolicy policy_of(int p) {
  switch (p) {
    case 1: return kvref::CachePolicy::kLfu;
    case 2: return kvref::CachePolicy::kLengthAware;
    default: return kvref::CachePolicy::kLru;
  }
}
std::span<const kvref::BlockId> span_of(const int64_t* keys, int64_t n) {
  return {reinterpret_cast<const kvref::BlockId*>(keys), static_cast<std::size_t>(n)};
}
}  // namespace

extern "C" {

int64_t kvref_chain_hash(int64_t prev, uint64_t content) {
  return kvref::chain_hash(prev, content);
}

/* capacity < 0 means unbounded.  Returns NULL on ValidationError. */
void* kvref_pool_create(int64_t capacity, int policy) {
  try {
    std::optional<std::size_t> cap;
    if (capacity >= 0) cap = static_cast<std::size_t>(capacity);
    return new kvref::CachePool(cap, policy_of(policy));
  } catch (const std::exception&) {
    return nullptr;
  }
}

void kvref_pool_destroy(void* pool) { delete static_cast<kvref::CachePool*>(pool); }

/* Returns the number of evicted ids (all written when <= evicted_cap). */
int64_t kvref_pool_admit(void* pool, const int64_t* keys, int64_t n, int64_t skip_begin,
                         int64_t skip_end, int64_t* evicted, int64_t evicted_cap,
                         int64_t* hits, int64_t* misses, int32_t* truncated) {
  auto* p = static_cast<kvref::CachePool*>(pool);
  const auto r = p->admit_and_touch(span_of(keys, n), static_cast<std::size_t>(skip_begin),
                                    static_cast<std::size_t>(skip_end));
  for (std::size_t i = 0; i < r.evicted.size() && static_cast<int64_t>(i) < evicted_cap; ++i)
    evicted[i] = r.evicted[i];
  if (hits) *hits = static_cast<int64_t>(r.hits);
  if (misses) *misses = static_cast<int64_t>(r.misses);
  if (truncated) *truncated = r.truncated ? 1 : 0;
  return static_cast<int64_t>(r.evicted.size());
}

int64_t kvref_pool_insert_replicated(void* pool, const int64_t* keys, int64_t n,
                                     int64_t chain_offset, int64_t* evicted,
                                     int64_t evicted_cap) {
  auto* p = static_cast<kvref::CachePool*>(pool);
  const auto ev = p->insert_replicated(span_of(keys, n), static_cast<std::size_t>(chain_offset));
  for (std::size_t i = 0; i < ev.size() && static_cast<int64_t>(i) < evicted_cap; ++i)
    evicted[i] = ev[i];
  return static_cast<int64_t>(ev.size());
}

int64_t kvref_pool_match_prefix(const void* pool, const int64_t* keys, int64_t n) {
  return static_cast<int64_t>(
      static_cast<const kvref::CachePool*>(pool)->match_prefix(span_of(keys, n)));
}

int kvref_pool_contains(const void* pool, int64_t key) {
  return static_cast<const kvref::CachePool*>(pool)->contains(key) ? 1 : 0;
}

int64_t kvref_pool_size(const void* pool) {
  return static_cast<int64_t>(static_cast<const kvref::CachePool*>(pool)->size());
}

void kvref_pool_stats(const void* pool, uint64_t* hits, uint64_t* misses) {
  const auto& s = static_cast<const kvref::CachePool*>(pool)->stats();
  *hits = s.hits;
  *misses = s.misses;
}

/* Returns 0, or -1 when the reference throws ValidationError (empty pool). */
int kvref_find_best_prefix_match(void* const* pools, const int32_t* ids, int64_t n_inst,
                                 const int64_t* keys, int64_t n, int64_t* best_len,
                                 int32_t* best_id) {
  std::vector<kvref::PrefillSnapshot> snaps;
  for (int64_t i = 0; i < n_inst; ++i)
    snaps.push_back({ids[i], static_cast<const kvref::CachePool*>(pools[i]), 0.0, 0.0, 0.0});
  try {
    const auto b = kvref::find_best_prefix_match(snaps, span_of(keys, n));
    *best_len = static_cast<int64_t>(b.prefix_blocks);
    *best_id = b.instance_id;
    return 0;
  } catch (const kvref::ValidationError&) {
    return -1;
  }
}

/* CPU baseline: find_best_prefix_match for n_req requests, disjoint request
 * slices on nthreads std::threads (match_prefix is const, so concurrent
 * readers are safe -- kvcache.hpp:42-43). */
void kvref_match_batch_mt(void* const* pools, const int32_t* ids, int64_t n_inst,
                          const int64_t* keys, const int64_t* key_off, int64_t n_req,
                          int64_t* best_len, int32_t* best_id, int nthreads) {
  std::vector<kvref::PrefillSnapshot> snaps;
  for (int64_t i = 0; i < n_inst; ++i)
    snaps.push_back({ids[i], static_cast<const kvref::CachePool*>(pools[i]), 0.0, 0.0, 0.0});
  auto work = [&](int64_t lo, int64_t hi) {
    for (int64_t r = lo; r < hi; ++r) {
      const auto b = kvref::find_best_prefix_match(
          snaps, span_of(keys + key_off[r], key_off[r + 1] - key_off[r]));
      best_len[r] = static_cast<int64_t>(b.prefix_blocks);
      best_id[r] = b.instance_id;
    }
  };
  if (nthreads <= 1) {
    work(0, n_req);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nthreads; ++t)
    th.emplace_back(work, n_req * t / nthreads, n_req * (t + 1) / nthreads);
  for (auto& x : th) x.join();
}

/* CPU baseline for stage 1a: prefix block keys folded with the reference's
 * own chain_hash (the content hash -- a fold over the block's token ids -- is
 * build-defined), request slices on nthreads std::threads. */
void kvref_block_hash_mt(const int32_t* tokens, const int64_t* tok_off, int64_t n_req, int64_t bs,
                         const int64_t* key_off, int64_t* keys, int nthreads) {
  auto work = [&](int64_t lo, int64_t hi) {
    for (int64_t r = lo; r < hi; ++r) {
      int64_t key = 0;
      int64_t k = key_off[r];
      for (int64_t t = tok_off[r]; t < tok_off[r + 1]; t += bs) {
        const int64_t end = std::min(t + bs, tok_off[r + 1]);
        kvref::BlockId c = 0;
        for (int64_t i = t; i < end; ++i)
          c = kvref::chain_hash(c, static_cast<uint64_t>(static_cast<uint32_t>(tokens[i])));
        key = kvref::chain_hash(key, static_cast<uint64_t>(c));
        keys[k++] = key;
      }
    }
  };
  if (nthreads <= 1) {
    work(0, n_req);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nthreads; ++t)
    th.emplace_back(work, n_req * t / nthreads, n_req * (t + 1) / nthreads);
  for (auto& x : th) x.join();
}

/* kvref::schedule(..., kKvcacheCentric) for one request (conductor.cpp:126-262).
 * perf8 = alpha, beta, gamma, delta, epsilon, kv_bytes_per_token, link_bw, load_bw.
 * out_i = accepted, reject_reason(0/1/2), prefill_id, decode_id, local_prefix,
 *         used_prefix, migrate, migrate_source, migrate_prefix_blocks
 * out_d = queue_ms, transfer_ms, exec_ms, ttft_ms, tbt_ms.  Returns -1 on
 * ValidationError. */
int kvref_schedule(const double* perf8, int64_t chunk, int64_t stages, double l_ttft,
                   double l_tbt, double threshold, int64_t block_size, double now,
                   void* const* pools, const int32_t* ids, const double* busy,
                   const double* sender, const double* queued, int64_t n_pre,
                   const int32_t* dids, const int64_t* dbatch, const int64_t* dkv, int64_t n_dec,
                   int64_t input, const int64_t* keys, int64_t n_keys, int64_t* out_i,
                   double* out_d) {
  kvref::PerfModelParams p;
  p.alpha_mlp = perf8[0];
  p.beta_attn = perf8[1];
  p.gamma_decode = perf8[2];
  p.delta_decode = perf8[3];
  p.epsilon_decode = perf8[4];
  p.kv_bytes_per_token = perf8[5];
  p.link_bandwidth = perf8[6];
  p.load_bandwidth = perf8[7];
  p.prefill_chunk = chunk;
  p.cpp_group_size = stages;
  std::vector<kvref::PrefillSnapshot> pre;
  for (int64_t i = 0; i < n_pre; ++i)
    pre.push_back({ids[i], static_cast<const kvref::CachePool*>(pools[i]), busy[i], sender[i],
                   queued[i]});
  std::vector<kvref::DecodeSnapshot> dec;
  for (int64_t i = 0; i < n_dec; ++i) dec.push_back({dids[i], dbatch[i], dkv[i], std::nullopt});
  kvref::SLOConfig slo;
  slo.l_ttft_ms = l_ttft;
  slo.l_tbt_ms = l_tbt;
  kvref::ConductorConfig cc;
  cc.kvcache_balancing_threshold = threshold;
  cc.block_size = block_size;
  kvref::RequestRecord rec;
  rec.input_length = input;
  rec.output_length = 1;
  rec.hash_ids.assign(keys, keys + n_keys);
  const kvref::ScheduleContext ctx{pre, dec, slo, cc, p, now};
  try {
    const auto d = kvref::schedule(rec, ctx, kvref::SchedulerChoice::kKvcacheCentric);
    out_i[0] = d.accepted;
    out_i[1] = d.reject_reason == kvref::RejectReason::kTtftSlo   ? 1
               : d.reject_reason == kvref::RejectReason::kTbtSlo ? 2
                                                                  : 0;
    out_i[2] = d.prefill_id;
    out_i[3] = d.decode_id;
    out_i[4] = static_cast<int64_t>(d.local_prefix_blocks);
    out_i[5] = static_cast<int64_t>(d.used_prefix_blocks);
    out_i[6] = d.migration.has_value();
    out_i[7] = d.migration ? d.migration->source_id : 0;
    out_i[8] = d.migration ? static_cast<int64_t>(d.migration->prefix_blocks) : 0;
    out_d[0] = d.queue_ms;
    out_d[1] = d.transfer_ms;
    out_d[2] = d.exec_ms;
    out_d[3] = d.estimated_ttft_ms;
    out_d[4] = d.estimated_tbt_ms;
    return 0;
  } catch (const kvref::ValidationError&) {
    return -1;
  }
}

/* Bulk-load a reference pool (setup for the CPU baseline; not timed). */
void kvref_pool_insert_many(void* pool, const int64_t* keys, int64_t n) {
  auto* p = static_cast<kvref::CachePool*>(pool);
  const int64_t step = 4096;
  for (int64_t i = 0; i < n; i += step)
    p->insert_replicated(span_of(keys + i, std::min(step, n - i)), 0);
}

double kvref_estimate_transfer_time(int64_t tokens, double kv_bytes_per_token,
                                    double link_bandwidth, double sender_busy_until,
                                    double now) {
  kvref::PerfModelParams p;
  p.kv_bytes_per_token = kv_bytes_per_token;
  p.link_bandwidth = link_bandwidth;
  return kvref::estimate_transfer_time(tokens, p, sender_busy_until, now);
}

}  // extern "C"
