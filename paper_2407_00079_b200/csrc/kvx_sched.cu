// kvx_sched.cu -- batched Conductor scoring: the
// kvcache-centric prefill/decode choice for a whole batch of requests against
// one cluster snapshot, in FP64 on the GPU ("TTFTs are computed in parallel",
// PAPER.md:338).
//
// Per request, exactly the reference's schedule() for kKvcacheCentric
// (proj/src/conductor.cpp:126-262):
//   best      = find_best_prefix_match over the match matrix (longest, lowest id)
//   per prefill instance p (one lane each):
//     queue   = max(0, busy_until - now) + queued_work        (perf_model.cpp:47-49)
//     ratio   = balance_ratio(best, local_p)                  (conductor.cpp:118-122)
//     ratio <= threshold : ttft = queue + exec(input, min(local*bs, input))
//     otherwise          : ttft = transfer((best-local)*bs, best.sender_busy) + queue
//                                 + exec(input, min(best*bs, input))
//     exec    = max(cpp or plain prefill time, cache_load_time) (perf_model.cpp:112-126)
//   prefill   = argmin ttft, ties to the lowest id (conductor.cpp:220-224)
//   decode    = argmin decode_iteration_time(batch+1, kv+input), lowest id (:75-94)
//   reject    on ttft > l_ttft, then tbt > l_tbt (:245-255)
//   migration if balance_ratio(best, chosen local) > threshold (:257-260)
// The file is compiled with -fmad=false and keeps the reference's operation
// order, so every double is bit-identical to the host computation.
#include <cfloat>

#include "kvx_common.cuh"

namespace kvx {
namespace {

struct Perf {
  double alpha, beta, gamma, delta, epsilon, kv_bytes, link_bw, load_bw;
  int64_t chunk, stages;
};

__device__ double prefill_time(int64_t input, int64_t cached, const Perf& p) {
  const double uncached = static_cast<double>(input - cached);
  return p.alpha * uncached + p.beta * uncached * static_cast<double>(input);
}

__device__ double cpp_latency(int64_t uncached, int64_t cached_ctx, const Perf& p) {
  if (uncached == 0) return 0.0;
  double sum_ms = 0.0, max_ms = 0.0;
  int64_t done = 0;
  while (done < uncached) {
    const int64_t chunk = min(p.chunk, uncached - done);
    done += chunk;
    const int64_t context_end = cached_ctx + done;
    const double chunk_ms = p.alpha * static_cast<double>(chunk) +
                            p.beta * static_cast<double>(chunk) * static_cast<double>(context_end);
    sum_ms += chunk_ms;
    max_ms = fmax(max_ms, chunk_ms);
  }
  const double stages = static_cast<double>(p.stages);
  return sum_ms / stages + (stages - 1.0) * max_ms / stages;
}

__device__ double exec_ms(int64_t input, int64_t cached, const Perf& p) {
  const int64_t uncached = input - cached;
  const double compute = uncached > p.chunk ? cpp_latency(uncached, cached, p)
                                            : prefill_time(input, cached, p);
  const double load = static_cast<double>(cached) * p.kv_bytes / p.load_bw;
  return fmax(compute, load);
}

__device__ double balance_ratio(int64_t best, int64_t local) {
  if (best == 0) return 0.0;
  if (local == 0) return __longlong_as_double(0x7FF0000000000000LL);  // +inf
  return static_cast<double>(best) / static_cast<double>(local);
}

// (ttft, id) lexicographic min; NaN-free inputs.
__device__ __forceinline__ bool better(double t, int id, double bt, int bid) {
  return t < bt || (t == bt && id < bid);
}

__global__ void __launch_bounds__(128) schedule_kernel(
    const Perf p, double l_ttft, double l_tbt, double threshold, int64_t bs, double now,
    const kvx_prefill_snapshot* __restrict__ pre, int n_pre,
    const kvx_decode_snapshot* __restrict__ dec, int n_dec, const int64_t* __restrict__ input_len,
    const int64_t* __restrict__ match_len, int64_t n_req, kvx_sched_decision* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
       r < n_req; r += warps) {
    const int64_t input = input_len[r];
    const int64_t* lens = match_len + r * n_pre;
    // best prefix holder: longest, ties -> lowest id (the first instance seeds)
    int64_t best_len = -1;
    int best_id = 0, best_idx = 0;
    for (int i = lane; i < n_pre; i += 32) {
      const int64_t l = lens[i];
      const int id = pre[i].id;
      if (l > best_len || (l == best_len && id < best_id)) {
        best_len = l;
        best_id = id;
        best_idx = i;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const int64_t l2 = __shfl_xor_sync(0xffffffffu, best_len, o);
      const int id2 = __shfl_xor_sync(0xffffffffu, best_id, o);
      const int ix2 = __shfl_xor_sync(0xffffffffu, best_idx, o);
      if (l2 > best_len || (l2 == best_len && id2 < best_id)) {
        best_len = l2;
        best_id = id2;
        best_idx = ix2;
      }
    }
    const double best_sender = pre[best_idx].sender_busy_until_ms;
    // TTFT candidate per prefill instance
    double c_ttft = DBL_MAX, c_queue = 0, c_transfer = 0, c_exec = 0;
    int c_id = 0x7FFFFFFF, c_remote = 0;
    int64_t c_local = 0, c_used = 0;
    bool have = false;
    for (int i = lane; i < n_pre; i += 32) {
      const int64_t local = lens[i];
      const double queue = fmax(0.0, pre[i].busy_until_ms - now) + pre[i].queued_work_ms;
      const double ratio = balance_ratio(best_len, local);
      double ttft, transfer = 0.0, ex;
      int64_t used;
      int remote = 0;
      if (ratio <= threshold) {
        used = local;
        ex = exec_ms(input, min(local * bs, input), p);
        ttft = queue + ex;
      } else {
        remote = 1;
        used = best_len;
        const int64_t tokens = (best_len - local) * bs;
        transfer = fmax(0.0, best_sender - now) +
                   static_cast<double>(tokens) * p.kv_bytes / p.link_bw;
        ex = exec_ms(input, min(best_len * bs, input), p);
        ttft = transfer + queue + ex;
      }
      if (!have || better(ttft, pre[i].id, c_ttft, c_id)) {
        have = true;
        c_ttft = ttft;
        c_id = pre[i].id;
        c_queue = queue;
        c_transfer = transfer;
        c_exec = ex;
        c_local = local;
        c_used = used;
        c_remote = remote;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double t2 = __shfl_xor_sync(0xffffffffu, c_ttft, o);
      const int id2 = __shfl_xor_sync(0xffffffffu, c_id, o);
      const double q2 = __shfl_xor_sync(0xffffffffu, c_queue, o);
      const double tr2 = __shfl_xor_sync(0xffffffffu, c_transfer, o);
      const double ex2 = __shfl_xor_sync(0xffffffffu, c_exec, o);
      const int64_t lo2 = __shfl_xor_sync(0xffffffffu, c_local, o);
      const int64_t us2 = __shfl_xor_sync(0xffffffffu, c_used, o);
      const int rm2 = __shfl_xor_sync(0xffffffffu, c_remote, o);
      if (better(t2, id2, c_ttft, c_id)) {
        c_ttft = t2;
        c_id = id2;
        c_queue = q2;
        c_transfer = tr2;
        c_exec = ex2;
        c_local = lo2;
        c_used = us2;
        c_remote = rm2;
      }
    }
    // decode choice
    double d_tbt = DBL_MAX;
    int d_id = 0x7FFFFFFF;
    for (int i = lane; i < n_dec; i += 32) {
      const double tbt = p.gamma + p.delta * static_cast<double>(dec[i].batch_size + 1) +
                         p.epsilon * static_cast<double>(dec[i].resident_kv_tokens + input) /
                             1000.0;
      if (better(tbt, dec[i].id, d_tbt, d_id)) {
        d_tbt = tbt;
        d_id = dec[i].id;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double t2 = __shfl_xor_sync(0xffffffffu, d_tbt, o);
      const int id2 = __shfl_xor_sync(0xffffffffu, d_id, o);
      if (better(t2, id2, d_tbt, d_id)) {
        d_tbt = t2;
        d_id = id2;
      }
    }
    if (lane == 0) {
      kvx_sched_decision dd{};
      dd.prefill_id = c_id;
      dd.decode_id = d_id;
      dd.local_prefix_blocks = c_local;
      dd.used_prefix_blocks = c_used;
      dd.queue_ms = c_queue;
      dd.transfer_ms = c_transfer;
      dd.exec_ms = c_exec;
      dd.ttft_ms = c_ttft;
      dd.tbt_ms = d_tbt;
      dd.best_prefix_blocks = best_len;
      dd.best_instance_id = best_id;
      if (c_ttft > l_ttft) {
        dd.reject_reason = 1;
      } else if (d_tbt > l_tbt) {
        dd.reject_reason = 2;
      } else {
        dd.accepted = 1;
        if (balance_ratio(best_len, c_local) > threshold) {
          dd.migrate = 1;
          dd.migrate_source = best_id;
          dd.migrate_prefix_blocks = best_len;
        }
      }
      (void)c_remote;
      out[r] = dd;
    }
  }
}

}  // namespace
}  // namespace kvx

using namespace kvx;

extern "C" int kvx_schedule_batch(const kvx_perf_params* perf, const kvx_sched_params* sp,
                                  const kvx_prefill_snapshot* d_prefill, int64_t n_prefill,
                                  const kvx_decode_snapshot* d_decode, int64_t n_decode,
                                  const int64_t* d_input_len, const int64_t* d_match_len,
                                  int64_t n_req, kvx_sched_decision* d_out, void* stream) {
  KVX_REQUIRE(perf && sp, "kvx_schedule_batch: NULL parameters");
  KVX_REQUIRE(n_prefill >= 1, "schedule: empty prefill pool");
  KVX_REQUIRE(n_decode >= 1, "schedule: empty decoding pool");
  KVX_REQUIRE(n_prefill <= (1 << 20) && n_decode <= (1 << 20), "kvx_schedule_batch: pool too big");
  KVX_REQUIRE(perf->prefill_chunk >= 1 && perf->cpp_group_size >= 1 && perf->link_bandwidth > 0 &&
                  perf->load_bandwidth > 0,
              "kvx_schedule_batch: perf parameters out of range");
  KVX_REQUIRE(sp->block_size >= 1, "kvx_schedule_batch: block_size must be >= 1");
  if (n_req == 0) return KVX_OK;
  KVX_REQUIRE(d_prefill && d_decode && d_input_len && d_match_len && d_out,
              "kvx_schedule_batch: NULL array");
  int dev = 0;
  KVX_CUDA(cudaGetDevice(&dev));
  Perf p{perf->alpha_mlp,    perf->beta_attn,          perf->gamma_decode,
         perf->delta_decode, perf->epsilon_decode,     perf->kv_bytes_per_token,
         perf->link_bandwidth, perf->load_bandwidth,   perf->prefill_chunk,
         perf->cpp_group_size};
  const int64_t want = (n_req + 3) / 4;
  const int blocks = static_cast<int>(std::min<int64_t>(want, static_cast<int64_t>(sm_count(dev)) * 16));
  schedule_kernel<<<blocks, 128, 0, as_stream(stream)>>>(
      p, sp->l_ttft_ms, sp->l_tbt_ms, sp->kvcache_balancing_threshold, sp->block_size, sp->now_ms,
      d_prefill, static_cast<int>(n_prefill), d_decode, static_cast<int>(n_decode), d_input_len,
      d_match_len, n_req, d_out);
  KVX_LAUNCH_CHECK("schedule_kernel");
  return KVX_OK;
}
