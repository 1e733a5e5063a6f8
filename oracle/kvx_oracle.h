/*
 * kvx_oracle.h -- CPU restatement of the Mooncake/kvcsim KVCache hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * CUDA path in paper_2407_00079_b200/csrc.  Only tests/, the smoke() entry
 * of __graft_entry__.py and bench.py's cpu_baseline / --impl reference leg
 * may load it.  The product path never links or calls it.
 *
 * Parity anchors (reference = /root/reference, kvcsim):
 *   - kvo_chain_hash            proj/src/kvcache.cpp:14-23 (bit-exact port)
 *   - kvo_match_prefix          proj/src/kvcache.cpp:150-158 (first-miss rule)
 *   - kvo_best_prefix_match     proj/src/conductor.cpp:57-73 (argmax, lowest
 *                               id wins ties, first instance seeds)
 *   - block selection of the prefill->decode stream: the whole hash_ids chain
 *     of the request (proj/src/sim_engine.cpp:463-464); migration ranges
 *     [local_prefix, used_prefix) (proj/src/sim_engine.cpp:405-416).
 *   - gather/scatter bytes, the content hash over token ids, the synthetic KV
 *     generator and the decode allocator are NOT defined by the reference
 *     (SPEC.md:183 makes byte-level KV a non-goal).  They are defined here
 *     (and in DESIGN.md) and pinned by this repo's own known-answer tests.
 */
#ifndef KVX_ORACLE_H_
#define KVX_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- stage 1a: hashing ------------------------------------------------ */

/* Bit-exact restatement of kvcsim::chain_hash (proj/src/kvcache.cpp:14-23). */
int64_t kvo_chain_hash(int64_t prev_key, uint64_t content_hash);

/* Build-defined content hash of one block: fold chain_hash over the token
 * ids, starting from 0.  Token ids are widened as uint32 -> uint64. */
uint64_t kvo_content_hash(const int32_t* tokens, int64_t n_tokens);

/* Prefix-chained block keys for n_req requests.  Request r owns tokens
 * [tok_off[r], tok_off[r+1]); its ceil(len/bs) keys are written at
 * keys_out[key_off[r] ...] where key_off is the exclusive scan of the block
 * counts.  key_i = chain_hash(key_{i-1}, content_i), key_{-1} = 0; the last
 * block may be partial and hashes only the tokens it has. */
void kvo_block_hash_batch(const int32_t* tokens, const int64_t* tok_off, int64_t n_req,
                          int64_t bs, const int64_t* key_off, int64_t* keys_out);

/* ---- stage 1b: prefix match -------------------------------------------- */

/* A resident-key set: a sorted copy of the keys (binary search). */
typedef struct kvo_set kvo_set;
kvo_set* kvo_set_create(const int64_t* keys, int64_t n);
void kvo_set_destroy(kvo_set* s);
int kvo_set_contains(const kvo_set* s, int64_t key);

/* Largest k with keys[0..k) all resident (kvcache.cpp:150-154). */
int64_t kvo_match_prefix(const kvo_set* s, const int64_t* keys, int64_t n);

/* Batched: for each request r and instance i, len_out[r*n_inst+i]; best_len
 * and best_id follow find_best_prefix_match (conductor.cpp:57-73). */
void kvo_match_prefix_batch(const kvo_set* const* sets, const int32_t* inst_ids,
                            int64_t n_inst, const int64_t* keys, const int64_t* key_off,
                            int64_t n_req, int64_t* len_out, int64_t* best_len,
                            int32_t* best_id);

/* ---- stages 2-4: paged KV bytes ---------------------------------------- */

/* Paged pool layout (build-defined): base[((layer*2 + kv)*slots + slot)*slab]
 * with slab = bs*heads*dim*dtype_bytes bytes.  Transfer buffer layout for a
 * layer range [lo,hi): buf[(((l-lo)*2 + kv)*n + b)*slab]. */
void kvo_gather(const uint8_t* pool, int64_t slots, int64_t slab, const int32_t* src_table,
                int64_t n, int64_t layer_lo, int64_t layer_hi, uint8_t* buf, int nthreads);
void kvo_scatter(uint8_t* pool, int64_t slots, int64_t slab, const int32_t* dst_table,
                 int64_t n, int64_t layer_lo, int64_t layer_hi, const uint8_t* buf,
                 int nthreads);
/* Direct paged -> paged copy (the fused stage 2+3+4). */
void kvo_copy_paged(const uint8_t* src_pool, int64_t src_slots, const int32_t* src_table,
                    uint8_t* dst_pool, int64_t dst_slots, const int32_t* dst_table,
                    int64_t slab, int64_t n, int64_t layer_lo, int64_t layer_hi,
                    int nthreads);

/* Synthetic KV content (build-defined, counter based, every slab distinct):
 * word w of slab (pool_id, layer, kv, slot) = kvo_kv_word(...).  */
uint64_t kvo_mix64(uint64_t z);
uint64_t kvo_slab_seed(uint32_t pool_id, uint32_t layer, uint32_t kv, uint32_t slot);
uint64_t kvo_kv_word(uint64_t slab_seed, uint64_t word);
void kvo_fill_pool(uint8_t* pool, uint32_t pool_id, int64_t layers, int64_t slots,
                   int64_t slab, int nthreads);

/* Deterministic decode allocator: the n lowest free slots, ascending, are
 * marked used and written to table_out.  Returns the number allocated (< n
 * when the pool is exhausted; nothing is allocated in that case). */
int64_t kvo_alloc_lowest_free(uint8_t* used, int64_t slots, int64_t n, int32_t* table_out);

#ifdef __cplusplus
}
#endif
#endif
