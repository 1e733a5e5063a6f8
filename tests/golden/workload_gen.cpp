// workload_gen.cpp -- golden generator (TEST INFRASTRUCTURE): prints the
// reference's own kvcsim::generate_workload (proj/src/trace.cpp:163-222)
// hash_ids for the Config 2 / Config 1 specs, one request per line
// ("<input_length> <id> <id> ..."), so tests/test_workloads.py can pin
// paper_2407_00079_b200.workloads.TransferWorkload against it.
// Built and run by tests/golden/make_workload_golden.sh.
#include <cstdio>
#include <cstdlib>

#include "kvcsim/trace.hpp"

int main(int argc, char** argv) {
  kvcsim::WorkloadSpec w;
  w.rate_rps = 10.0;
  w.request_count = argc > 1 ? std::atoll(argv[1]) : 64;
  w.input_length = kvcsim::LengthSpec::fixed(argc > 2 ? std::atoll(argv[2]) : 8192);
  w.output_length = kvcsim::LengthSpec::fixed(1);
  w.cache_ratio = argc > 3 ? std::atof(argv[3]) : 0.5;
  w.block_size = argc > 4 ? std::atoll(argv[4]) : 16;
  w.seed = 1;
  for (const auto& r : kvcsim::generate_workload(w)) {
    std::printf("%lld", static_cast<long long>(r.input_length));
    for (auto id : r.hash_ids) std::printf(" %lld", static_cast<long long>(id));
    std::printf("\n");
  }
  return 0;
}
