/*
 * kvx.h -- C ABI of the B200-native KVCache hot path (libkvx.so).
 *
 * Four stages of Mooncake's KVCache path (arXiv 2407.00079), each a
 * hand-written sm_100a kernel or a copy-engine transfer:
 *   1a  batched prefix block hash        kvx_chain_hash_batch
 *   1b  batched prefix-match query       kvx_index_*, kvx_match_prefix_batch
 *   2   gather paged -> contiguous       kvx_gather
 *   3   layer-wise transfer              kvx_xfer_*, kvx_transfer_submit / _wait
 *   4   scatter contiguous -> paged      kvx_scatter
 *   2+3+4 fused paged -> paged           kvx_copy_paged (dst may be a peer view)
 *
 * Which reference interface each entry point replaces (reference =
 * /root/reference, kvcsim; see INTEGRATION.md for the bindings):
 *   kvx_chain_hash_batch   kvcsim::chain_hash            proj/include/kvcsim/kvcache.hpp:25
 *                                                         (proj/src/kvcache.cpp:14-23)
 *   kvx_index_insert       CachePool::admit_and_touch /  proj/include/kvcsim/kvcache.hpp:61-64
 *                          insert_replicated (residency  proj/include/kvcsim/kvcache.hpp:68-69
 *                          side of the block manager put)
 *   kvx_index_erase        eviction in insert_block      proj/src/kvcache.cpp:72-97
 *   kvx_index_lookup       CachePool::contains           proj/include/kvcsim/kvcache.hpp:74
 *   kvx_match_prefix_batch CachePool::match_prefix,      proj/include/kvcsim/kvcache.hpp:72,105
 *                          find_best_prefix_match        proj/include/kvcsim/conductor.hpp:63-64
 *   kvx_gather / kvx_scatter / kvx_copy_paged / kvx_transfer_*:
 *                          the analytic transfer model   proj/src/perf_model.cpp:51-59,
 *                          and migration/stream events   proj/src/sim_engine.cpp:399-419,455-476,605-650
 *                          (no byte-level reference exists)
 *
 * Conventions
 *   - Every function returns kvx_status; on failure kvx_last_error() holds a
 *     thread-local message.  KVX_EINVAL corresponds to kvcsim::ValidationError
 *     (proj/include/kvcsim/errors.hpp:18-21).
 *   - Pointers named d_* are device pointers on the device of the handle they
 *     are used with; `stream` is a cudaStream_t passed as void* (NULL = the
 *     legacy default stream).  Work is asynchronous and ordered on `stream`;
 *     only *_wait, kvx_index_stats and kvx_sync are host-blocking.
 *   - Calls on one handle must be externally serialised (the reference's
 *     CachePool is single-owner, proj/include/kvcsim/kvcache.hpp:42-43).
 *   - Block keys are int64.  Two values are reserved as table sentinels and
 *     are never resident: KVX_KEY_EMPTY and KVX_KEY_TOMBSTONE.
 *   - There is no CPU fallback: without a usable CUDA device every compute
 *     entry point returns KVX_ECUDA.
 */
#ifndef KVX_H_
#define KVX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVX_ABI_VERSION 1

typedef enum {
  KVX_OK = 0,
  KVX_EINVAL = 1,    /* precondition violated (kvcsim::ValidationError) */
  KVX_ENOMEM = 2,    /* device allocation failed */
  KVX_ECUDA = 3,     /* CUDA runtime/driver error, or no device */
  KVX_EABORTED = 4,  /* transfer source no longer resident (sim_engine.cpp:605-639) */
  KVX_EAGAIN = 5     /* not complete yet (kvx_transfer_query) */
} kvx_status;

#define KVX_KEY_EMPTY ((int64_t)(-0x7FFFFFFFFFFFFFFFLL - 1))      /* INT64_MIN */
#define KVX_KEY_TOMBSTONE ((int64_t)(-0x7FFFFFFFFFFFFFFFLL))      /* INT64_MIN + 1 */

int kvx_abi_version(void);
const char* kvx_last_error(void);
/* Number of kernels this library has launched in this process. */
uint64_t kvx_launch_count(void);
/* Host-blocking stream synchronise (convenience for C hosts). */
int kvx_sync(void* stream);

/* ---- stage 1a: block hashing ------------------------------------------ */

/* Scalar chain_hash (bit-identical to kvcsim::chain_hash, kvcache.cpp:14-23).
 * Pure function, usable on hosts without a GPU. */
int64_t kvx_chain_hash(int64_t prev_key, uint64_t content_hash);

/* Batched prefix block keys.  Request r owns tokens [tok_off[r], tok_off[r+1])
 * of d_tokens; its ceil(len/bs) keys go to d_keys[key_off[r] ...].
 * content_i = fold(chain_hash, block tokens as uint32, from 0);
 * key_i = chain_hash(key_{i-1}, content_i), key_{-1} = 0; the last block may
 * be partial.  d_key_off must be the exclusive scan of ceil(len/bs).
 * Block sizes that are multiples of 16 with a 16-byte aligned d_tokens run the
 * half-warp kernel (requests must be < 2^30 tokens each); others the
 * producer / fold kernel.  Both are bit-identical. */
int kvx_chain_hash_batch(const int32_t* d_tokens, const int64_t* d_tok_off, int64_t n_req,
                         int64_t bs, const int64_t* d_key_off, int64_t* d_keys, void* stream);
/* d_key_off[0..n_req] = exclusive scan of ceil((tok_off[r+1]-tok_off[r]) / bs)
 * (the key offsets kvx_chain_hash_batch takes), on the device. */
int kvx_key_offsets(const int64_t* d_tok_off, int64_t n_req, int64_t bs, int64_t* d_key_off,
                    void* stream);

/* ---- stage 1b: block index (GPU open-addressing table) + prefix match ---- */

typedef struct kvx_index kvx_index;

/* capacity_hint: expected resident keys; the table grows on demand. */
int kvx_index_create(int device, int64_t capacity_hint, kvx_index** out);
int kvx_index_destroy(kvx_index* idx);
int kvx_index_device(const kvx_index* idx);
/* Upsert keys (value = d_values[i], or the key's position i when NULL).
 * Reserved sentinel keys are skipped and counted as rejected. */
int kvx_index_insert(kvx_index* idx, const int64_t* d_keys, const int64_t* d_values, int64_t n,
                     void* stream);
int kvx_index_erase(kvx_index* idx, const int64_t* d_keys, int64_t n, void* stream);
/* Erase d_erase[0..ne) and upsert d_insert[0..ni) (values d_values, or the
 * position when NULL) in ONE kernel launch.  The two key sets must be
 * disjoint (the block manager's put: its victims and its new blocks). */
int kvx_index_update(kvx_index* idx, const int64_t* d_erase, int64_t ne, const int64_t* d_insert,
                     const int64_t* d_values, int64_t ni, void* stream);
/* Keep this index's key array resident in L2 for kernels launched on
 * `stream` (a persisting access-policy window over the table, sized to the
 * device's persisting-L2 carve-out, which this call raises if needed): the
 * prefix match probes it at random right after the hash streams the batch's
 * tokens.  on == 0 removes the stream's window.  The rebuilt table of a
 * later resize is not covered: call again after large inserts. */
int kvx_index_l2_pin(const kvx_index* idx, void* stream, int on);
/* d_values_out[i] = value of key i, or -1 when absent. */
int kvx_index_lookup(const kvx_index* idx, const int64_t* d_keys, int64_t n,
                     int64_t* d_values_out, void* stream);
int kvx_index_clear(kvx_index* idx, void* stream);
/* Rebuild the table (drops tombstones) sized for at least min_keys keys. */
int kvx_index_reserve(kvx_index* idx, int64_t min_keys, void* stream);
/* Host-blocking: live keys, tombstones, slots, rejected sentinel keys. */
int kvx_index_stats(kvx_index* idx, int64_t* live, int64_t* tombstones, int64_t* slots,
                    int64_t* rejected, void* stream);

/* Prefix match of n_req requests against n_inst instance indices (one
 * kvcsim prefill instance each), all on the stream's device.
 *   d_len_out[r*n_inst + i]  match_prefix of request r on instance i (optional)
 *   d_best_len[r], d_best_id[r]  find_best_prefix_match: longest match, ties to
 *                                the lowest inst_ids[i] (conductor.cpp:57-73)
 * n_inst == 0 is KVX_EINVAL (the reference throws on an empty pool).  d_keys
 * may be NULL when every chain is empty (key_off[n_req] == 0): an empty chain
 * matches 0 blocks everywhere and the best is (0, lowest id), as in the
 * reference.
 * inst_ids is a HOST array; n_inst <= KVX_MAX_INSTANCES. */
#define KVX_MAX_INSTANCES 64
int kvx_match_prefix_batch(const kvx_index* const* idx, const int32_t* inst_ids, int64_t n_inst,
                           const int64_t* d_keys, const int64_t* d_key_off, int64_t n_req,
                           int64_t* d_len_out, int64_t* d_best_len, int32_t* d_best_id,
                           void* stream);

/* Stage 1 in one call: kvx_chain_hash_batch, then kvx_match_prefix_batch on
 * the keys -- with the match of each request starting as soon as the hash
 * has stored that request's keys (a consumer kernel beside the hash works
 * through the hash's completion queue), so the batch's match hides under the
 * hash's long-request tail.  Same arguments and results as the two calls; d_keys
 * receives the keys.  Block sizes the half-warp hash does not take run the two
 * calls in sequence. */
int kvx_hash_match_batch(const int32_t* d_tokens, const int64_t* d_tok_off, int64_t n_req,
                         int64_t bs, const int64_t* d_key_off, int64_t* d_keys,
                         const kvx_index* const* idx, const int32_t* inst_ids, int64_t n_inst,
                         int64_t* d_len_out, int64_t* d_best_len, int32_t* d_best_id,
                         void* stream);
/* Host-blocking: KVX_ECUDA if a match task of kvx_hash_match_batch on the
 * device of `stream` gave up (5 s) waiting for a request the hash never
 * completed (a defect; its results are then missing), else KVX_OK. */
int kvx_hash_match_check(void* stream);

/* Same query, leaving per request the packed word (len << 32 | ~ordered(id))
 * whose MAXIMUM is the best match with the lowest-id tie-break: instances
 * held by different GPUs combine with one all-reduce(MAX) over these words
 * (SURVEY 8(e) case ii), then kvx_best_unpack. */
int kvx_match_prefix_packed(const kvx_index* const* idx, const int32_t* inst_ids, int64_t n_inst,
                            const int64_t* d_keys, const int64_t* d_key_off, int64_t n_req,
                            uint64_t* d_packed, void* stream);
int kvx_best_unpack(const uint64_t* d_packed, int64_t n_req, int64_t* d_best_len,
                    int32_t* d_best_id, void* stream);

/* Cross-GPU find_best_prefix_match WITHOUT a collective (SURVEY 8(e) case
 * ii; replaces kvx_match_prefix_packed + all-reduce(MAX) + kvx_best_unpack):
 * `world` processes, one per GPU, each holding some prefill instances.  Every
 * rank's match kernel atomically MAXes each request's packed word straight
 * into every rank's result buffer over NVLink (CUDA IPC mappings); stream-
 * ordered 64-bit flags then tell each rank that all ranks' atomics landed.
 * Setup: create on every rank, exchange the export blobs (any side channel),
 * connect each rank to every other.  kvx_xmatch_run is collective: every
 * rank calls it once per batch, same n_req, in the same order. */
#define KVX_MAX_PEERS 8
typedef struct kvx_xmatch kvx_xmatch;
int kvx_xmatch_create(int device, int rank, int world, int64_t max_req, kvx_xmatch** out);
int kvx_xmatch_destroy(kvx_xmatch* x);
int kvx_xmatch_export(kvx_xmatch* x, uint8_t* blob, int64_t cap, int64_t* len);
int kvx_xmatch_connect(kvx_xmatch* x, const uint8_t* blob, int64_t len);
int kvx_xmatch_run(kvx_xmatch* x, const kvx_index* const* idx, const int32_t* inst_ids,
                   int64_t n_inst, const int64_t* d_keys, const int64_t* d_key_off, int64_t n_req,
                   int64_t* d_best_len, int32_t* d_best_id, void* stream);
/* Request-sharded hashing for the same exchange.  kvx_xmatch_key_buffer
 * (before export/connect; same max_keys on every rank) allocates this rank's
 * copy of a batch-wide key buffer.  Per step each rank hashes ITS shard of the
 * requests straight into its copy (kvx_chain_hash_batch with its slice of the
 * batch's tok_off / key_off: keys land at their batch-wide positions), then
 * kvx_xmatch_share_keys pushes keys [key_lo, key_hi) into every peer's copy
 * with the copy engine (NVLink) and makes `stream` wait until every peer's
 * shard has landed here -- then kvx_xmatch_run on the whole batch, same
 * stream.  Collective: every rank calls share_keys then run once per step. */
int kvx_xmatch_key_buffer(kvx_xmatch* x, int64_t max_keys, int64_t** d_keys);
int kvx_xmatch_share_keys(kvx_xmatch* x, int64_t key_lo, int64_t key_hi, void* stream);
/* Request-sharded stage 1 with the key exchange inside the match kernel
 * (replaces chain_hash_batch + share_keys + run when every rank has its own
 * GPU): rank k hashes requests [shard_bounds[k], shard_bounds[k+1]) of the
 * batch (shard_bounds: host array of world + 1, from 0 to n_req, the same on
 * every rank; d_tok_off / d_key_off: the WHOLE batch's offsets) into its own
 * key buffer, and every rank's match kernel runs beside its hash and follows
 * the keys of the whole batch where they are produced -- local, or NVLink
 * loads of the owning peer's buffer (keys are preset to -1 and polled) --
 * against its instances, MAXing each request's packed best into every rank's
 * result buffer.  Stream-ordered flags order the steps (two key-buffer halves
 * by step parity); the host never blocks.  Collective, once per step, same
 * n_req, bs and bounds on every rank.  Needs kvx_xmatch_key_buffer (>= the
 * batch's keys), bs % 16 == 0, 16-byte aligned tokens; KVX_EINVAL if a peer
 * shares this GPU (its kernels would wait on ours).  *d_keys_out (may be
 * NULL): this rank's key buffer of the step (its own shard's keys).  Do not
 * interleave with kvx_xmatch_share_keys on the same exchange (both use the
 * key buffer's first half). */
int kvx_xmatch_hash_match(kvx_xmatch* x, const int32_t* d_tokens, const int64_t* d_tok_off,
                          const int64_t* shard_bounds, int64_t bs, const int64_t* d_key_off,
                          int64_t n_req, const kvx_index* const* idx, const int32_t* inst_ids,
                          int64_t n_inst, int64_t* d_best_len, int32_t* d_best_id,
                          int64_t** d_keys_out, void* stream);

/* ---- batched Conductor scoring (kvcache-centric schedule, FP64) -------- */

/* Mirrors of kvcsim::PerfModelParams (proj/include/kvcsim/perf_model.hpp:13-26),
 * the SLO / conductor knobs schedule() reads, and the two snapshot structs
 * (proj/include/kvcsim/conductor.hpp:41-55). */
typedef struct {
  double alpha_mlp, beta_attn, gamma_decode, delta_decode, epsilon_decode;
  double kv_bytes_per_token, link_bandwidth, load_bandwidth;
  int64_t prefill_chunk, cpp_group_size;
} kvx_perf_params;

typedef struct {
  double l_ttft_ms, l_tbt_ms, kvcache_balancing_threshold, now_ms;
  int64_t block_size;
} kvx_sched_params;

typedef struct {
  int32_t id;
  int32_t pad_;
  double busy_until_ms, sender_busy_until_ms, queued_work_ms;
} kvx_prefill_snapshot;

typedef struct {
  int32_t id;
  int32_t pad_;
  int64_t batch_size, resident_kv_tokens;
} kvx_decode_snapshot;

typedef struct {
  int32_t accepted;
  int32_t reject_reason; /* 0 none, 1 TTFT SLO, 2 TBT SLO (conductor.cpp:245-255) */
  int32_t prefill_id, decode_id;
  int64_t local_prefix_blocks, used_prefix_blocks;
  int64_t best_prefix_blocks;
  int32_t best_instance_id;
  int32_t migrate;         /* hot-spot migration planned (conductor.cpp:257-260) */
  int32_t migrate_source;
  int32_t pad_;
  int64_t migrate_prefix_blocks;
  double queue_ms, transfer_ms, exec_ms, ttft_ms, tbt_ms;
} kvx_sched_decision;

/* schedule() for kKvcacheCentric (proj/src/conductor.cpp:126-262) applied to
 * n_req requests against ONE snapshot: d_match_len is the n_req x n_prefill
 * matrix from kvx_match_prefix_batch (same instance order as d_prefill).  All
 * doubles are bit-identical to the reference's host arithmetic. */
int kvx_schedule_batch(const kvx_perf_params* perf, const kvx_sched_params* sp,
                       const kvx_prefill_snapshot* d_prefill, int64_t n_prefill,
                       const kvx_decode_snapshot* d_decode, int64_t n_decode,
                       const int64_t* d_input_len, const int64_t* d_match_len, int64_t n_req,
                       kvx_sched_decision* d_out, void* stream);

/* ---- paged KV pool ------------------------------------------------------ */

/* HBM layout: base[((layer*2 + kv)*slots + slot) * slab], slab =
 * block_size*heads*head_dim*dtype_bytes bytes (one block of one layer's K or
 * V).  Transfer buffers for layers [lo,hi) and n blocks are laid out
 * buf[(((l-lo)*2 + kv)*n + b) * slab]. */
typedef struct {
  int32_t layers;
  int32_t block_size;
  int32_t heads;
  int32_t head_dim;
  int32_t dtype_bytes;
  int64_t slots;
  int32_t device;
} kvx_pool_desc;

typedef struct kvx_pool kvx_pool;

int kvx_pool_create(const kvx_pool_desc* desc, kvx_pool** out);
/* Wrap memory the pool does not own (e.g. a peer pool mapped by kvx_ipc_open). */
int kvx_pool_create_view(const kvx_pool_desc* desc, void* d_base, kvx_pool** out);
int kvx_pool_destroy(kvx_pool* pool);
void* kvx_pool_base(const kvx_pool* pool);
int64_t kvx_pool_slab_bytes(const kvx_pool* pool);
int64_t kvx_pool_bytes(const kvx_pool* pool);
int kvx_pool_device(const kvx_pool* pool);
int32_t kvx_pool_layers(const kvx_pool* pool);

/* Synthetic content: 64-bit word w of slab (pool_id, layer, kv, slot) =
 * mix64(slab_seed + w) (oracle/kvx_oracle.c). */
int kvx_pool_fill_synthetic(kvx_pool* pool, uint32_t pool_id, void* stream);
/* Counts 64-bit words of dst slabs (dst_table[b], layers [lo,hi)) that differ
 * from the synthetic content of (src_pool_id, layer, kv, src_table[b]);
 * atomically ADDS the count to *d_mismatch (uint64). */
int kvx_pool_verify(const kvx_pool* dst, const int32_t* d_dst_table, uint32_t src_pool_id,
                    const int32_t* d_src_table, int64_t n, int32_t layer_lo, int32_t layer_hi,
                    uint64_t* d_mismatch, void* stream);

/* CPU-DRAM tier: a pool in pinned, device-mapped host memory (same layout).
 * desc->device is the GPU whose kernels access it; gather / scatter /
 * kvx_copy_paged accept it on either side and then run a small grid over
 * PCIe (zero copy).  Freed by kvx_pool_destroy. */
int kvx_pool_create_host(const kvx_pool_desc* desc, kvx_pool** out);
int kvx_pool_is_host(const kvx_pool* pool);

/* ---- stages 2 / 4 / fused ------------------------------------------------ */

int kvx_gather(const kvx_pool* pool, const int32_t* d_src_table, int64_t n, int32_t layer_lo,
               int32_t layer_hi, void* d_buf, void* stream);
int kvx_scatter(kvx_pool* pool, const int32_t* d_dst_table, int64_t n, int32_t layer_lo,
                int32_t layer_hi, const void* d_buf, void* stream);
/* dst[l][kv][dst_table[b]] = src[l][kv][src_table[b]].  dst may be a view of
 * a peer GPU's pool (stores go over NVLink); src must be local to `stream`. */
int kvx_copy_paged(const kvx_pool* src, const int32_t* d_src_table, kvx_pool* dst,
                   const int32_t* d_dst_table, int64_t n, int32_t layer_lo, int32_t layer_hi,
                   void* stream);
/* Copy-kernel variant selector (0 = LSU 128-bit, 1 = TMA bulk); default 0. */
int kvx_set_copy_impl(int impl);
/* Block-table bounds: gather / scatter / paged copy skip any (layer, K|V,
 * block) unit whose table entry is outside [0, slots) of its pool -- nothing
 * is written outside a pool -- and flag it on the device.  Synchronizes
 * `stream`, then returns KVX_EINVAL (and clears the flag) if an entry was out
 * of range since the last check on the device that owns `stream` (NULL: the
 * current device), KVX_ECUDA if a pull copy on it timed out, else KVX_OK. */
int kvx_copy_check(void* stream);

/* ---- stage 3: transfer engine ----------------------------------------- */

typedef struct kvx_xfer kvx_xfer;

/* One in-order copy-engine queue per source device (the reference's
 * per-sender FIFO, sim_engine.cpp:409-411). */
int kvx_xfer_create(int device, kvx_xfer** out);
int kvx_xfer_destroy(kvx_xfer* x);
void* kvx_xfer_stream(kvx_xfer* x);
/* Queue a copy of `bytes` from src to dst (either may be peer memory).  When
 * after_stream is non-NULL the copy starts only after the work already queued
 * on after_stream.  *ticket identifies the copy. */
int kvx_transfer_submit(kvx_xfer* x, void* dst, const void* src, int64_t bytes,
                        void* after_stream, uint64_t* ticket);
/* Host-blocking wait for a ticket. */
int kvx_transfer_wait(kvx_xfer* x, uint64_t ticket);
/* Device-side wait: work queued on `stream` after this call runs after the copy. */
int kvx_transfer_wait_stream(kvx_xfer* x, uint64_t ticket, void* stream);
/* KVX_OK when complete, KVX_EAGAIN when still in flight. */
int kvx_transfer_query(kvx_xfer* x, uint64_t ticket);
/* Queue a 64-bit flag store of `value` to d_flag (local or peer) on the
 * transfer queue, ordered after every copy submitted before it. */
int kvx_transfer_signal(kvx_xfer* x, void* d_flag, uint64_t value);

/* ---- layer-wise prefill -> decode stream (stages 2 -> 3 -> 4) ---------- */

/* Host C++ engine sequencing the kernels and copy engines above: one request
 * (or decode wave) is streamed as units of (block range, layer range), chunk-
 * major, the way chunked-pipeline prefill produces KV (perf_model.cpp:87-110,
 * sim_engine.cpp:455-470).  Ranks of a pair exchange kvx_streamer_export()
 * blobs (CUDA IPC handles) and kvx_streamer_connect() to each other. */
enum {
  KVX_STREAM_LOCAL_FUSED = 0,  /* one GPU: paged -> paged copy kernel */
  KVX_STREAM_LOCAL_STAGED = 1, /* one GPU: gather -> ring -> scatter */
  KVX_STREAM_PEER_FUSED = 2,   /* sender kernel stores into the receiver's pool */
  KVX_STREAM_PEER_CE = 3,      /* gather -> copy engine P2P -> scatter on the receiver */
  KVX_STREAM_PEER_PULL = 4,    /* receiver kernel loads the sender's pool (IPC view) over
                                  NVLink and stores locally; the prefill GPU's SMs stay free */
  KVX_STREAM_PEER_NCCL = 5     /* comparison: gather -> ncclSend / ncclRecv on the pair's own
                                  2-rank communicator (libnccl.so.2 loaded at run time,
                                  created in connect: both ends must connect) -> scatter */
};
enum { KVX_ROLE_LOCAL = 0, KVX_ROLE_SENDER = 1, KVX_ROLE_RECEIVER = 2 };

typedef struct {
  int32_t mode;
  int32_t role;
  int32_t ring;           /* staging slots (staged modes) */
  int32_t time_launches;  /* record CUDA events around each dominant launch */
  int64_t slot_bytes;     /* bytes per staging slot (>= the largest unit) */
} kvx_streamer_desc;

typedef struct kvx_streamer kvx_streamer;

int kvx_streamer_create(const kvx_streamer_desc* desc, kvx_pool* src, kvx_pool* dst,
                        kvx_streamer** out);
int kvx_streamer_destroy(kvx_streamer* s);
/* blob == NULL: *len = bytes needed. */
int kvx_streamer_export(kvx_streamer* s, uint8_t* blob, int64_t cap, int64_t* len);
/* peer_pool: the receiver's pool shape (PEER_FUSED sender only). */
int kvx_streamer_connect(kvx_streamer* s, const uint8_t* blob, int64_t len,
                         const kvx_pool_desc* peer_pool);
void* kvx_streamer_stream(kvx_streamer* s);
/* Sender / local: enqueue n blocks (device tables; dst table unused by PEER_CE
 * senders) in units of chunk_blocks x layers_per_chunk.  The units of ONE call
 * touch disjoint (chunk, layer) slabs and may run overlapped (programmatic
 * dependent launch in LOCAL_FUSED / PEER_FUSED, and in the PEER_PULL
 * receiver, whose pull kernels then wait for the sender's unit flag
 * themselves); the first unit of a call waits for all earlier work on the
 * streamer's queues, so successive calls stay ordered.  KVX_STREAM_PDL=0
 * turns the overlap off.  A destination table must not repeat a slot. */
int kvx_streamer_send(kvx_streamer* s, const int32_t* d_src_table, const int32_t* d_dst_table,
                      int64_t n, int64_t chunk_blocks, int32_t layer_lo, int32_t layer_hi,
                      int32_t layers_per_chunk);
/* Receiver: the matching units (same n / chunking / layer ranges); the source
 * table is read only by PEER_PULL (the receiver copies from the sender's pool). */
int kvx_streamer_recv(kvx_streamer* s, const int32_t* d_src_table, const int32_t* d_dst_table,
                      int64_t n, int64_t chunk_blocks, int32_t layer_lo, int32_t layer_hi,
                      int32_t layers_per_chunk);
/* End of a step; if stream != NULL it then waits for all queued work. */
int kvx_streamer_finish(kvx_streamer* s, void* stream);
/* The streamer's queues wait for work already queued on stream. */
int kvx_streamer_after(kvx_streamer* s, void* stream);
/* Time every stride-th dominant launch with CUDA events (0/1 = off/on). */
int kvx_streamer_set_timing(kvx_streamer* s, int on, int stride);
/* Host-blocking: timed dominant launches since the last reset. */
int kvx_streamer_launch_stats(kvx_streamer* s, int64_t* launches, double* avg_ms,
                              double* avg_bytes, int reset);
uint64_t kvx_streamer_units(const kvx_streamer* s);
/* Host-blocking: waits for the streamer's queues, then reports a failed unit
 * since the last check: KVX_ECUDA when a PEER_PULL unit gave up waiting for
 * the sender (20 s; its decode slots were NOT written and the sender saw bit
 * 62 in the step's "consumed" word), KVX_EINVAL for out-of-range block-table
 * entries (kvx_copy_check).  Receivers should call it after a step's finish
 * before using the decode slots. */
int kvx_streamer_check(kvx_streamer* s);
/* 1 when the connected peer process runs on this same GPU (device UUIDs
 * match): peer modes then wait only with stream memory operations, never
 * inside a kernel. */
int kvx_streamer_same_gpu(const kvx_streamer* s);
/* How a PEER_PULL receiver waits for the sender's units (default GATE, or
 * $KVX_PULL_GATE at connect; call after connect to override):
 *   GATE    a one-warp kernel waits, the copy follows it programmatically
 *           dependent -- near the link peak also for 8 MiB units; only one
 *           warp is resident while the prefill has not produced the layer
 *   INLINE  the copy's CTAs wait themselves (the whole next-unit grid stays
 *           resident while waiting; fastest for tiny units)
 *   STREAM  the stream front end waits (cuStreamWaitValue64), nothing is
 *           resident: the choice when the decode GPU runs whole-SM kernels
 *           (persistent GEMMs) that any co-resident CTA would delay
 * profiles/r02 and DESIGN.md section 5 have the measured trade-off. */
#define KVX_PULL_WAIT_GATE 0
#define KVX_PULL_WAIT_INLINE 1
#define KVX_PULL_WAIT_STREAM 2
int kvx_streamer_set_pull_wait(kvx_streamer* s, int mode);
/* CUDA-graph record / replay of one step (LOCAL_FUSED only): the sends issued
 * between record_begin and record_end are captured, not run; each replay runs
 * them again with one cudaGraphLaunch on the streamer's queue (tables are read
 * at replay time; same pointers and ranges).  Call finish(stream) after
 * record_end, not inside the recording. */
int kvx_streamer_record_begin(kvx_streamer* s);
int kvx_streamer_record_end(kvx_streamer* s);
int kvx_streamer_replay(kvx_streamer* s);

/* ---- layer-wise DRAM <-> HBM load / store ---------------
 * Replaces the reference's cache_load_time / layerwise_effective_prefill
 * model (proj/src/perf_model.cpp:73-85; load_bandwidth, config.cpp:218) with
 * the real transfer: "launch" queues a layer's copy on the object's load (or
 * store) queue, "wait" makes a stream wait for it.  Loads: host pool -> device
 * pool, one unit per layer in layer order, after the work on after_stream;
 * kvx_layer_load_wait(layer) before that layer's attention.  Stores: device
 * pool -> host pool, launched after the work on after_stream (the layer's
 * attention); kvx_layer_store_wait_all at the end (stream NULL: host-blocking).
 * Tables are device int32 arrays of n slot ids on each side. */
typedef struct kvx_layer_io kvx_layer_io;
int kvx_layer_io_create(int device, int32_t max_layers, kvx_layer_io** out);
int kvx_layer_io_destroy(kvx_layer_io* io);
void* kvx_layer_io_load_stream(kvx_layer_io* io);
void* kvx_layer_io_store_stream(kvx_layer_io* io);
int kvx_layer_load_launch(kvx_layer_io* io, const kvx_pool* host, const int32_t* d_host_table,
                          kvx_pool* dev, const int32_t* d_dev_table, int64_t n, int32_t layer_lo,
                          int32_t layer_hi, void* after_stream);
int kvx_layer_load_wait(kvx_layer_io* io, int32_t layer, void* stream);
int kvx_layer_store_launch(kvx_layer_io* io, const kvx_pool* dev, const int32_t* d_dev_table,
                           kvx_pool* host, const int32_t* d_host_table, int64_t n,
                           int32_t layer_lo, int32_t layer_hi, void* after_stream);
int kvx_layer_store_wait_all(kvx_layer_io* io, void* stream);
/* The same for CONTIGUOUS block runs: host slots [host_first, host_first+n)
 * <-> device slots [dev_first, dev_first+n).  Each (layer, K|V) plane is then
 * one contiguous range on both sides: two copy-engine copies per layer and
 * no kernel, so the SMs stay with the prefill (a register-heavy GEMM leaves
 * no room for a copy kernel to run beside it). */
int kvx_layer_load_range(kvx_layer_io* io, const kvx_pool* host, int64_t host_first,
                         kvx_pool* dev, int64_t dev_first, int64_t n, int32_t layer_lo,
                         int32_t layer_hi, void* after_stream);
int kvx_layer_store_range(kvx_layer_io* io, const kvx_pool* dev, int64_t dev_first,
                          kvx_pool* host, int64_t host_first, int64_t n, int32_t layer_lo,
                          int32_t layer_hi, void* after_stream);

/* ---- KVCache store of one instance + migration (hot-spot replication) ---- */

/* A store = paged pool + block index (key -> pool slot) + slot allocator.
 * put: index new keys at the lowest free slots (existing keys keep theirs);
 * get: slot per key or -1; evict: drop keys and free their slots.
 * migrate: copy the KV of keys resident in src into dst (every layer, K and
 * V), skipping keys dst already holds, and index them there -- the byte path
 * behind the reference's migration events (sim_engine.cpp:399-419,605-650).
 * If ANY key is not resident in src the call returns KVX_EABORTED and changes
 * nothing (the reference aborts when the source evicted part of the range).
 * All key/slot arrays are HOST arrays; put / get / evict / migrate are
 * host-blocking. */
typedef struct kvx_store kvx_store;
int kvx_store_create(const kvx_pool_desc* desc, kvx_store** out);
int kvx_store_destroy(kvx_store* s);
kvx_pool* kvx_store_pool(kvx_store* s);
kvx_index* kvx_store_index(kvx_store* s);
void* kvx_store_stream(kvx_store* s);
int kvx_store_put(kvx_store* s, const int64_t* keys, int64_t n, int32_t* slots_out);
int kvx_store_get(kvx_store* s, const int64_t* keys, int64_t n, int32_t* slots_out);
int kvx_store_evict(kvx_store* s, const int64_t* keys, int64_t n);
int kvx_store_migrate(kvx_store* src, kvx_store* dst, const int64_t* keys, int64_t n,
                      int64_t* n_copied);
/* Asynchronous migration, engine-driven (sim_engine.cpp:399-419,605-650).
 * Each SOURCE store has one in-order migration FIFO (the per-sender link,
 * sender_busy_until_ms, sim_engine.cpp:409-411).  submit queues the
 * migration (keys copied to the host-side FIFO) and returns a ticket; it
 * BEGINS when it reaches the head of the FIFO and the previous migration is
 * done: then the source is checked (any key not resident -> the ticket ends
 * KVX_EABORTED and nothing lands), destination slots are reserved and the copy
 * is launched after the work queued on the source store's stream and, if
 * after_stream != NULL, on after_stream at submit time.  Source slots stay
 * pinned until the copy is done (an eviction meanwhile drops the key but
 * defers the slot's reuse).  It is DONE when the copy finished: the keys land
 * in the destination index (blocks that became resident there meanwhile are
 * kept and the copied slot is freed).  Progress happens inside submit /
 * query / wait / progress calls on the source store (no threads):
 *   query: KVX_OK done, KVX_EAGAIN in flight or queued, KVX_EABORTED aborted;
 *   wait:  host-blocking until done; *n_copied = blocks landed; collects the
 *          ticket (a later query/wait of it is KVX_EINVAL).
 * kvx_store_migrate = submit + wait.  Destroy stores only after their
 * migrations are collected. */
int kvx_store_migrate_submit(kvx_store* src, kvx_store* dst, const int64_t* keys, int64_t n,
                             void* after_stream, uint64_t* ticket);
int kvx_store_migrate_query(kvx_store* src, uint64_t ticket);
int kvx_store_migrate_wait(kvx_store* src, uint64_t ticket, int64_t* n_copied);
int kvx_store_migrate_progress(kvx_store* src);

/* ---- decode block table: deterministic slot allocator (host) ---------- */

/* The decode instance's paged block table.  take() hands out the n lowest
 * free slots in ascending order (nothing is taken and KVX_ENOMEM returned
 * when fewer than n are free); the reference has no decode block table
 * (sim_engine.cpp:161-175 counts tokens only), so this is build-defined and
 * restated by oracle/kvx_oracle.c:kvo_alloc_lowest_free. */
typedef struct kvx_slot_alloc kvx_slot_alloc;
int kvx_slot_alloc_create(int64_t slots, kvx_slot_alloc** out);
int kvx_slot_alloc_destroy(kvx_slot_alloc* a);
int64_t kvx_slot_alloc_free_count(const kvx_slot_alloc* a);
int kvx_slot_alloc_take(kvx_slot_alloc* a, int64_t n, int32_t* table_out);
int kvx_slot_alloc_mark(kvx_slot_alloc* a, const int32_t* slots, int64_t n);
int kvx_slot_alloc_release(kvx_slot_alloc* a, const int32_t* slots, int64_t n);

/* ---- cross-process plumbing (one process per GPU) ---------------------- */

/* Raw device allocation (cudaMalloc: exportable with kvx_ipc_export). */
int kvx_device_alloc(int device, int64_t bytes, void** d_ptr);
int kvx_device_free(int device, void* d_ptr);

#define KVX_IPC_HANDLE_BYTES 64
int kvx_ipc_export(void* d_ptr, uint8_t handle[KVX_IPC_HANDLE_BYTES]);
int kvx_ipc_open(const uint8_t handle[KVX_IPC_HANDLE_BYTES], int device, void** d_ptr);
int kvx_ipc_close(void* d_ptr);
int kvx_enable_peer(int device, int peer_device);
/* Stream-ordered flag store / wait (no kernel spins: the stream front end
 * waits).  wait: proceeds once *(uint64*)d_flag >= value. */
int kvx_signal_write(void* stream, void* d_flag, uint64_t value);

/* Plumbing for C / C++ hosts that have no CUDA runtime of their own (the
 * drop-in libkvcsim_gpu.so calls only these and the entry points above):
 * a non-blocking stream; pinned, device-mapped host memory (kernels may read
 * and write it directly, e.g. query keys in and results out); an async copy;
 * a host-blocking wait until a pinned word the GPU writes reaches `target`
 * (signed >=; polling, no synchronise call; errors of `stream` and a stream
 * that went idle without writing are reported). */
int kvx_stream_create(int device, void** stream_out);
int kvx_stream_destroy(void* stream);
int kvx_host_alloc(int64_t bytes, void** host_ptr);
int kvx_host_free(void* host_ptr);
int kvx_memcpy_async(void* dst, const void* src, int64_t bytes, void* stream);
int kvx_wait_host_word(const volatile int64_t* word, int64_t target, void* stream);
int kvx_signal_wait(void* stream, const void* d_flag, uint64_t value);

#ifdef __cplusplus
}
#endif
#endif /* KVX_H_ */
