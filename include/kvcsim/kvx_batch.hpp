/*
 * kvcsim/kvx_batch.hpp -- batched form of the Conductor's prefix-match query.
 *
 * The reference answers find_best_prefix_match one request at a time, P
 * match_prefix calls each (proj/src/conductor.cpp:57-73; schedule() repeats
 * the P calls at :198).  This extension answers a whole batch of requests
 * against P instance pools in one B200 kernel launch (kvx_match_prefix_batch),
 * with the reference's result convention: the longest prefix wins, ties go to
 * the lowest instance id, an empty instance list throws ValidationError.
 */
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "kvcsim/kvcache.hpp"

namespace kvcsim {

struct BestPrefixMatchBatch {
  std::size_t prefix_blocks = 0;
  int instance_id = 0;
};

// keys: the requests' block-key chains back to back; key_offsets: n_req + 1
// prefix offsets into keys.  per_instance (optional) receives the n_req x P
// match_prefix matrix, row-major.
std::vector<BestPrefixMatchBatch> find_best_prefix_match_batch(
    std::span<const CachePool* const> instances, std::span<const int> instance_ids,
    std::span<const BlockId> keys, std::span<const std::int64_t> key_offsets,
    std::vector<std::size_t>* per_instance = nullptr);

}  // namespace kvcsim
