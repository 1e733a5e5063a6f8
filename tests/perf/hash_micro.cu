// hash_micro.cu -- micro-measurements behind K1's design (run on a B200):
//   1. dependent latency of one chain_hash step (single thread, clock64)
//   2. the same with 2 and 4 independent chains interleaved in one thread
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../include -I../../paper_2407_00079_b200/csrc hash_micro.cu
#include <cstdio>

#include "kvx_common.cuh"

template <int CHAINS>
__global__ void chain_latency(int steps, long long* out_cycles, int64_t* sink) {
  int64_t h[CHAINS];
  for (int c = 0; c < CHAINS; ++c) h[c] = c + threadIdx.x;
  const long long t0 = clock64();
  for (int i = 0; i < steps; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) h[c] = kvx::chain_hash(h[c], static_cast<uint64_t>(i));
  }
  const long long t1 = clock64();
  int64_t acc = 0;
  for (int c = 0; c < CHAINS; ++c) acc ^= h[c];
  sink[threadIdx.x] = acc;
  if (threadIdx.x == 0) *out_cycles = t1 - t0;
}

int main() {
  long long* d_cyc;
  int64_t* d_sink;
  cudaMalloc(&d_cyc, sizeof(long long));
  cudaMalloc(&d_sink, 1024 * sizeof(int64_t));
  const int steps = 100000;
  long long cyc = 0;
  chain_latency<1><<<1, 1>>>(steps, d_cyc, d_sink);
  cudaMemcpy(&cyc, d_cyc, sizeof(cyc), cudaMemcpyDeviceToHost);
  std::printf("1 chain : %.1f cycles/step\n", double(cyc) / steps);
  chain_latency<2><<<1, 1>>>(steps, d_cyc, d_sink);
  cudaMemcpy(&cyc, d_cyc, sizeof(cyc), cudaMemcpyDeviceToHost);
  std::printf("2 chains: %.1f cycles/step (both)\n", double(cyc) / steps);
  chain_latency<4><<<1, 1>>>(steps, d_cyc, d_sink);
  cudaMemcpy(&cyc, d_cyc, sizeof(cyc), cudaMemcpyDeviceToHost);
  std::printf("4 chains: %.1f cycles/step (all)\n", double(cyc) / steps);
  chain_latency<1><<<1, 32>>>(steps, d_cyc, d_sink);
  cudaMemcpy(&cyc, d_cyc, sizeof(cyc), cudaMemcpyDeviceToHost);
  std::printf("1 chain x 32 lanes: %.1f cycles/step\n", double(cyc) / steps);
  chain_latency<1><<<1, 128>>>(steps, d_cyc, d_sink);
  cudaMemcpy(&cyc, d_cyc, sizeof(cyc), cudaMemcpyDeviceToHost);
  std::printf("1 chain x 4 warps: %.1f cycles/step\n", double(cyc) / steps);
  chain_latency<1><<<1, 512>>>(steps, d_cyc, d_sink);
  cudaMemcpy(&cyc, d_cyc, sizeof(cyc), cudaMemcpyDeviceToHost);
  std::printf("1 chain x 16 warps: %.1f cycles/step\n", double(cyc) / steps);
  return 0;
}
