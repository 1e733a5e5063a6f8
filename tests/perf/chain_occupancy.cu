// chain_occupancy.cu -- chain_hash throughput vs independent chains per thread
// (ILP) and resident warps per SM: what a hash kernel needs to saturate the
// ALU pipe (run on a B200).  One CTA per SM of W warps, C chains per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../include \
//        -I../../paper_2407_00079_b200/csrc chain_occupancy.cu -o chain_occupancy
#include <cstdio>
#include <cstdint>

#include "kvx_common.cuh"

template <int C>
__global__ void __launch_bounds__(1024, 1) chain_loop(int iters, const uint32_t* tok, int64_t* out) {
  int64_t h[C];
#pragma unroll
  for (int c = 0; c < C; ++c) h[c] = threadIdx.x + c * 977 + blockIdx.x;
  for (int i = 0; i < iters; ++i) {
    const uint32_t t = tok[i & 1023];
#pragma unroll
    for (int c = 0; c < C; ++c) h[c] = kvx::chain_hash(h[c], t + c);
  }
  int64_t acc = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) acc ^= h[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int C>
void run(int warps, int sms, const uint32_t* tok, int64_t* out) {
  const int iters = 2048 / C;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  chain_loop<C><<<sms, warps * 32>>>(iters, tok, out);
  cudaEventRecord(a);
  chain_loop<C><<<sms, warps * 32>>>(iters, tok, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double hashes = double(sms) * warps * 32 * iters * C;
  std::printf("chains/thread=%d warps/SM=%2d: %6.1f G chain_hash/s\n", C, warps,
              hashes / (ms * 1e-3) / 1e9);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* tok;
  int64_t* out;
  cudaMalloc(&tok, 4096);
  cudaMemset(tok, 7, 4096);
  cudaMalloc(&out, size_t(sms) * 1024 * 8);
  for (int w : {4, 8, 12, 16, 24, 32}) run<1>(w, sms, tok, out);
  for (int w : {4, 8, 12, 16, 24, 32}) run<2>(w, sms, tok, out);
  for (int w : {4, 8, 12, 16}) run<4>(w, sms, tok, out);
  return 0;
}
