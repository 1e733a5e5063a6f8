/*
 * kvx_oracle.c -- CPU restatement of the KVCache hot path (TEST INFRASTRUCTURE).
 *
 * See kvx_oracle.h for the parity anchors.  Everything here is deliberately
 * plain: sorted arrays + binary search for residency, memcpy per slab for the
 * byte stages, so the checker is obviously correct rather than fast.  The
 * only concession to speed is optional pthread fan-out of the memcpy loops,
 * because the same loops are the CPU baseline timed by bench.py.
 */
#include "kvx_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* proj/src/kvcache.cpp:14-23 */
int64_t kvo_chain_hash(int64_t prev_key, uint64_t content_hash) {
  uint64_t x = (uint64_t)prev_key + 0x9E3779B97F4A7C15ull;
  x ^= content_hash + 0x9E3779B97F4A7C15ull + (x << 6) + (x >> 2);
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return (int64_t)(x & 0x7FFFFFFFFFFFFFFFull);
}

uint64_t kvo_content_hash(const int32_t* tokens, int64_t n_tokens) {
  int64_t h = 0;
  for (int64_t t = 0; t < n_tokens; ++t) h = kvo_chain_hash(h, (uint64_t)(uint32_t)tokens[t]);
  return (uint64_t)h;
}

void kvo_block_hash_batch(const int32_t* tokens, const int64_t* tok_off, int64_t n_req,
                          int64_t bs, const int64_t* key_off, int64_t* keys_out) {
  for (int64_t r = 0; r < n_req; ++r) {
    const int64_t lo = tok_off[r], hi = tok_off[r + 1];
    int64_t key = 0;
    int64_t k = key_off[r];
    for (int64_t t = lo; t < hi; t += bs) {
      const int64_t len = (hi - t) < bs ? (hi - t) : bs;
      key = kvo_chain_hash(key, kvo_content_hash(tokens + t, len));
      keys_out[k++] = key;
    }
  }
}

/* ---------------------------------------------------------------------- */

struct kvo_set {
  int64_t* keys;
  int64_t n;
};

static int cmp_i64(const void* a, const void* b) {
  const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

kvo_set* kvo_set_create(const int64_t* keys, int64_t n) {
  kvo_set* s = (kvo_set*)calloc(1, sizeof(kvo_set));
  s->keys = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  if (n > 0) memcpy(s->keys, keys, sizeof(int64_t) * (size_t)n);
  qsort(s->keys, (size_t)n, sizeof(int64_t), cmp_i64);
  /* dedupe */
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i)
    if (m == 0 || s->keys[m - 1] != s->keys[i]) s->keys[m++] = s->keys[i];
  s->n = m;
  return s;
}

void kvo_set_destroy(kvo_set* s) {
  if (!s) return;
  free(s->keys);
  free(s);
}

int kvo_set_contains(const kvo_set* s, int64_t key) {
  int64_t lo = 0, hi = s->n;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (s->keys[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo < s->n && s->keys[lo] == key;
}

/* proj/src/kvcache.cpp:150-154: stop at the first miss. */
int64_t kvo_match_prefix(const kvo_set* s, const int64_t* keys, int64_t n) {
  int64_t k = 0;
  while (k < n && kvo_set_contains(s, keys[k])) ++k;
  return k;
}

/* proj/src/conductor.cpp:57-73: the first instance seeds the best; a longer
 * match wins; an equal match goes to the lower instance id. */
void kvo_match_prefix_batch(const kvo_set* const* sets, const int32_t* inst_ids,
                            int64_t n_inst, const int64_t* keys, const int64_t* key_off,
                            int64_t n_req, int64_t* len_out, int64_t* best_len,
                            int32_t* best_id) {
  for (int64_t r = 0; r < n_req; ++r) {
    const int64_t* q = keys + key_off[r];
    const int64_t n = key_off[r + 1] - key_off[r];
    int64_t bl = 0;
    int32_t bid = n_inst > 0 ? inst_ids[0] : 0;
    for (int64_t i = 0; i < n_inst; ++i) {
      const int64_t len = kvo_match_prefix(sets[i], q, n);
      if (len_out) len_out[r * n_inst + i] = len;
      if (i == 0 || len > bl || (len == bl && inst_ids[i] < bid)) {
        bl = len;
        bid = inst_ids[i];
      }
    }
    if (best_len) best_len[r] = bl;
    if (best_id) best_id[r] = bid;
  }
}

/* ---------------------------------------------------------------------- */
/* Slab copies.  One unit = one (layer, kv, b) slab. */

typedef struct {
  const uint8_t* src;
  uint8_t* dst;
  int64_t src_slots, dst_slots, slab, n, layer_lo, layer_hi;
  const int32_t* src_table; /* NULL: contiguous buffer side */
  const int32_t* dst_table; /* NULL: contiguous buffer side */
  int64_t unit_begin, unit_end;
} copy_job;

static void copy_units(const copy_job* j) {
  for (int64_t u = j->unit_begin; u < j->unit_end; ++u) {
    const int64_t b = u % j->n;
    const int64_t lk = u / j->n; /* (l - lo)*2 + kv */
    const int64_t l = j->layer_lo + lk / 2, kv = lk % 2;
    const uint8_t* s;
    uint8_t* d;
    if (j->src_table) s = j->src + ((l * 2 + kv) * j->src_slots + j->src_table[b]) * j->slab;
    else s = j->src + u * j->slab;
    if (j->dst_table) d = j->dst + ((l * 2 + kv) * j->dst_slots + j->dst_table[b]) * j->slab;
    else d = j->dst + u * j->slab;
    memcpy(d, s, (size_t)j->slab);
  }
}

static void* copy_thread(void* arg) {
  copy_units((const copy_job*)arg);
  return NULL;
}

static void run_copy(copy_job base, int nthreads) {
  const int64_t units = (base.layer_hi - base.layer_lo) * 2 * base.n;
  if (nthreads <= 1 || units < 2) {
    base.unit_begin = 0;
    base.unit_end = units;
    copy_units(&base);
    return;
  }
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  copy_job jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    jobs[t] = base;
    jobs[t].unit_begin = units * t / nthreads;
    jobs[t].unit_end = units * (t + 1) / nthreads;
    pthread_create(&th[t], NULL, copy_thread, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}

void kvo_gather(const uint8_t* pool, int64_t slots, int64_t slab, const int32_t* src_table,
                int64_t n, int64_t layer_lo, int64_t layer_hi, uint8_t* buf, int nthreads) {
  copy_job j = {pool, buf, slots, 0, slab, n, layer_lo, layer_hi, src_table, NULL, 0, 0};
  run_copy(j, nthreads);
}

void kvo_scatter(uint8_t* pool, int64_t slots, int64_t slab, const int32_t* dst_table,
                 int64_t n, int64_t layer_lo, int64_t layer_hi, const uint8_t* buf,
                 int nthreads) {
  copy_job j = {buf, pool, 0, slots, slab, n, layer_lo, layer_hi, NULL, dst_table, 0, 0};
  run_copy(j, nthreads);
}

void kvo_copy_paged(const uint8_t* src_pool, int64_t src_slots, const int32_t* src_table,
                    uint8_t* dst_pool, int64_t dst_slots, const int32_t* dst_table,
                    int64_t slab, int64_t n, int64_t layer_lo, int64_t layer_hi,
                    int nthreads) {
  copy_job j = {src_pool, dst_pool, src_slots, dst_slots, slab, n, layer_lo, layer_hi,
                src_table, dst_table, 0, 0};
  run_copy(j, nthreads);
}

/* ---------------------------------------------------------------------- */
/* Synthetic KV content: splitmix64 finalizer over a per-slab seed + word. */

uint64_t kvo_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t kvo_slab_seed(uint32_t pool_id, uint32_t layer, uint32_t kv, uint32_t slot) {
  const uint64_t hi = ((uint64_t)(pool_id & 0xFFFFu) << 16) | ((uint64_t)(layer & 0x7FFFu) << 1) |
                      (uint64_t)(kv & 1u);
  return kvo_mix64((hi << 32) | (uint64_t)slot);
}

uint64_t kvo_kv_word(uint64_t slab_seed, uint64_t word) { return kvo_mix64(slab_seed + word); }

typedef struct {
  uint8_t* pool;
  uint32_t pool_id;
  int64_t slots, slab, unit_begin, unit_end;
} fill_job;

static void* fill_thread(void* arg) {
  const fill_job* j = (const fill_job*)arg;
  const int64_t words = j->slab / 8;
  for (int64_t u = j->unit_begin; u < j->unit_end; ++u) {
    const int64_t slot = u % j->slots, lk = u / j->slots;
    const uint64_t seed =
        kvo_slab_seed(j->pool_id, (uint32_t)(lk / 2), (uint32_t)(lk % 2), (uint32_t)slot);
    uint64_t* p = (uint64_t*)(j->pool + u * j->slab);
    for (int64_t w = 0; w < words; ++w) p[w] = kvo_kv_word(seed, (uint64_t)w);
  }
  return NULL;
}

void kvo_fill_pool(uint8_t* pool, uint32_t pool_id, int64_t layers, int64_t slots,
                   int64_t slab, int nthreads) {
  const int64_t units = layers * 2 * slots;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  fill_job jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    fill_job j = {pool, pool_id, slots, slab, units * t / nthreads, units * (t + 1) / nthreads};
    jobs[t] = j;
    if (nthreads == 1) fill_thread(&jobs[t]);
    else pthread_create(&th[t], NULL, fill_thread, &jobs[t]);
  }
  if (nthreads > 1)
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}

int64_t kvo_alloc_lowest_free(uint8_t* used, int64_t slots, int64_t n, int32_t* table_out) {
  int64_t got = 0;
  for (int64_t s = 0; s < slots && got < n; ++s)
    if (!used[s]) table_out[got++] = (int32_t)s;
  if (got < n) return got; /* exhausted: allocate nothing */
  for (int64_t i = 0; i < n; ++i) used[table_out[i]] = 1;
  return n;
}
