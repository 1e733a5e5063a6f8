/*
 * kvcsim_c.h -- C ABI over the GPU-backed drop-in block manager
 * (kvcsim::CachePool in include/kvcsim/kvcache.hpp, libkvcsim_gpu.so).
 *
 * For hosts that cannot bind C++ (ctypes, cgo, JNI).  Each entry point is the
 * C face of one reference member function:
 *   kvcsim_pool_create            CachePool::CachePool      proj/include/kvcsim/kvcache.hpp:47
 *   kvcsim_pool_admit             CachePool::admit_and_touch  kvcache.hpp:61-64
 *   kvcsim_pool_insert_replicated CachePool::insert_replicated kvcache.hpp:68-69
 *   kvcsim_pool_match_prefix      CachePool::match_prefix    kvcache.hpp:72
 *   kvcsim_pool_contains          CachePool::contains        kvcache.hpp:74
 *   kvcsim_pool_size / _stats     size() / stats()           kvcache.hpp:75-78
 *   kvcsim_find_best_prefix_match_batch
 *                                 find_best_prefix_match, batched
 *                                                            proj/include/kvcsim/conductor.hpp:63-64
 * Status codes are kvx_status (include/kvx.h): KVX_EINVAL where the reference
 * throws ValidationError, KVX_ECUDA without a usable GPU.
 */
#ifndef KVCSIM_C_H_
#define KVCSIM_C_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct kvcsim_pool kvcsim_pool;

/* capacity < 0: unbounded.  policy: 0 LRU, 1 LFU, 2 LengthAware. */
int kvcsim_pool_create(int64_t capacity, int policy, kvcsim_pool** out);
void kvcsim_pool_destroy(kvcsim_pool* pool);
/* Writes up to evicted_cap evicted ids; *n_evicted is the full count. */
int kvcsim_pool_admit(kvcsim_pool* pool, const int64_t* keys, int64_t n, int64_t skip_begin,
                      int64_t skip_end, int64_t* evicted, int64_t evicted_cap,
                      int64_t* n_evicted, int64_t* hits, int64_t* misses, int32_t* truncated);
int kvcsim_pool_insert_replicated(kvcsim_pool* pool, const int64_t* keys, int64_t n,
                                  int64_t chain_offset, int64_t* evicted, int64_t evicted_cap,
                                  int64_t* n_evicted);
int kvcsim_pool_match_prefix(const kvcsim_pool* pool, const int64_t* keys, int64_t n,
                             int64_t* len);
int kvcsim_pool_contains(const kvcsim_pool* pool, int64_t key, int32_t* out);
int64_t kvcsim_pool_size(const kvcsim_pool* pool);
void kvcsim_pool_stats(const kvcsim_pool* pool, uint64_t* hits, uint64_t* misses);
/* HOST arrays; len_out (n_req x n_inst, optional), best_len / best_id (n_req). */
int kvcsim_find_best_prefix_match_batch(kvcsim_pool* const* pools, const int32_t* ids,
                                        int64_t n_inst, const int64_t* keys,
                                        const int64_t* key_off, int64_t n_req, int64_t* len_out,
                                        int64_t* best_len, int32_t* best_id);
const char* kvcsim_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* KVCSIM_C_H_ */
