// replay_main.cpp -- drop-in proof driver.
//
// Built twice by oracle/dropin.mk from the SAME source:
//   ref_replay    : linked with the reference's own proj/src/kvcache.cpp
//   dropin_replay : compiled against include/kvcsim/kvcache.hpp (this repo)
//                   and linked with libkvcsim_gpu.so (GPU block index)
// Every other translation unit (sim_engine, conductor, overload, trace,
// perf_model, metrics, config) is the reference's, unmodified.  Each run
// prints one SimReport::to_json_string() per scenario; the two builds must
// print byte-identical output (tests/test_gpu_dropin_engine.py compares the
// GPU run with tests/golden/replay_reports.txt produced by ref_replay).
#include <algorithm>
#include <cstdio>
#include <string>
#include <vector>

#include "kvcsim/conductor.hpp"
#include "kvcsim/kvcache.hpp"
#include "kvcsim/sim_engine.hpp"
#include "kvcsim/trace.hpp"

using namespace kvcsim;

namespace {

// Several independent hot chains (one generate_workload per tenant, ids
// shifted into disjoint ranges), merged by arrival time.
std::vector<RequestRecord> tenants(int n_tenants, std::int64_t per_tenant, double rps,
                                   std::int64_t lo, std::int64_t hi, double cache_ratio,
                                   std::uint64_t seed) {
  std::vector<RequestRecord> all;
  for (int t = 0; t < n_tenants; ++t) {
    WorkloadSpec w;
    w.rate_rps = rps;
    w.request_count = per_tenant;
    w.input_length = LengthSpec{lo, hi};
    w.output_length = LengthSpec{16, 128};
    w.cache_ratio = cache_ratio;
    w.seed = seed * 7919 + static_cast<std::uint64_t>(t);
    auto part = generate_workload(w);
    for (auto& r : part) {
      for (auto& id : r.hash_ids) id += static_cast<std::int64_t>(t + 1) << 36;
      all.push_back(std::move(r));
    }
  }
  std::stable_sort(all.begin(), all.end(),
                   [](const RequestRecord& a, const RequestRecord& b) {
                     return a.timestamp_ms < b.timestamp_ms;
                   });
  for (std::size_t i = 0; i < all.size(); ++i) all[i].request_id = static_cast<std::int64_t>(i);
  return all;
}

struct Scenario {
  const char* name;
  int prefill, decode;
  std::optional<std::size_t> capacity;
  CachePolicy policy;
  SchedulerChoice scheduler;
  double threshold;
  int n_tenants;
  std::int64_t per_tenant;
  double rps;
  std::uint64_t seed;
  double link_bandwidth = 1.0e8;  // bytes/ms; slow links make sources evict mid-migration
};

}  // namespace

int main() {
  const Scenario scenarios[] = {
      {"4P4D_lru_cap96_centric", 4, 4, 96, CachePolicy::kLru, SchedulerChoice::kKvcacheCentric,
       2.0, 4, 60, 0.4, 1},
      {"2P2D_lfu_cap40_centric", 2, 2, 40, CachePolicy::kLfu, SchedulerChoice::kKvcacheCentric,
       1.5, 3, 50, 0.3, 2},
      {"3P1D_la_unbounded_centric", 3, 1, std::nullopt, CachePolicy::kLengthAware,
       SchedulerChoice::kKvcacheCentric, 4.0, 5, 40, 0.5, 3},
      {"4P2D_lru_cap24_cacheaware", 4, 2, 24, CachePolicy::kLru, SchedulerChoice::kCacheAware,
       4.0, 4, 40, 0.5, 4},
      {"8P4D_lfu_cap64_centric", 8, 4, 64, CachePolicy::kLfu, SchedulerChoice::kKvcacheCentric,
       1.2, 8, 40, 0.8, 5},
      {"4P2D_lru_cap20_centric_pressure", 4, 2, 20, CachePolicy::kLru,
       SchedulerChoice::kKvcacheCentric, 1.05, 6, 40, 3.0, 6, 2.0e6},
  };
  for (const auto& s : scenarios) {
    SimConfig cfg;
    cfg.cluster.prefill_instances = s.prefill;
    cfg.cluster.decode_instances = s.decode;
    cfg.cluster.cache_capacity_blocks = s.capacity;
    cfg.cluster.cache_policy = s.policy;
    cfg.scheduler = s.scheduler;
    cfg.conductor.kvcache_balancing_threshold = s.threshold;
    cfg.perf.cpp_group_size = 2;
    cfg.perf.link_bandwidth = s.link_bandwidth;
    cfg.seed = s.seed;
    const auto trace = tenants(s.n_tenants, s.per_tenant, s.rps, 2048, 24576, 0.6, s.seed);
    const SimReport rep = run(trace, cfg);
    std::printf("%s %s\n", s.name, rep.to_json_string(false).c_str());
  }
  return 0;
}
