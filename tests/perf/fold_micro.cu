// fold_micro.cu -- why is the per-request key fold slower than the chain_hash
// dependency latency?  4096 requests x 1024 blocks, contents pre-filled.
//   a) lane = request, strided 8-byte loads/stores (current design)
//   b) same, loads only (no stores)
//   c) warp = 32 requests, 32-block windows transposed through shared memory
//      (coalesced 256-byte rows in, coalesced rows out)
#include <cstdio>
#include <vector>

#include "kvx_common.cuh"

constexpr int kReq = 4096, kBlk = 1024;

__global__ void fold_strided(const int64_t* key_off, int64_t* keys, int n_req, int store) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_req) return;
  const int64_t k0 = key_off[r], k1 = key_off[r + 1];
  int64_t prev = 0, acc = 0;
  int64_t c[16];
  for (int j = 0; j < 16; ++j) c[j] = keys[k0 + j];
  for (int64_t k = k0; k < k1; k += 16) {
    int64_t nx[16];
    for (int j = 0; j < 16; ++j) nx[j] = (k + 16 + j < k1) ? keys[k + 16 + j] : 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      prev = kvx::chain_hash(prev, static_cast<uint64_t>(c[j]));
      if (store) keys[k + j] = prev; else acc ^= prev;
    }
    for (int j = 0; j < 16; ++j) c[j] = nx[j];
  }
  if (!store && acc == 42) keys[0] = acc;
}

__global__ void fold_transposed(const int64_t* key_off, int64_t* keys, int n_req) {
  __shared__ int64_t tile[32][33];
  const int lane = threadIdx.x;
  const int r0 = blockIdx.x * 32;
  const int r = r0 + lane;
  const int64_t my_k0 = key_off[r];
  const int64_t my_n = key_off[r + 1] - my_k0;
  int64_t prev = 0;
  for (int64_t w = 0; w < kBlk; w += 32) {
    for (int row = 0; row < 32; ++row) {  // coalesced row loads
      const int64_t k0 = key_off[r0 + row];
      tile[row][lane] = keys[k0 + w + lane];
    }
    __syncwarp();
#pragma unroll 8
    for (int j = 0; j < 32; ++j) {
      prev = kvx::chain_hash(prev, static_cast<uint64_t>(tile[lane][j]));
      tile[lane][j] = prev;
    }
    __syncwarp();
    for (int row = 0; row < 32; ++row) {
      const int64_t k0 = key_off[r0 + row];
      keys[k0 + w + lane] = tile[row][lane];
    }
    __syncwarp();
  }
  (void)my_n;
}

int main() {
  std::vector<int64_t> off(kReq + 1);
  for (int i = 0; i <= kReq; ++i) off[i] = static_cast<int64_t>(i) * kBlk;
  int64_t *d_off, *d_keys;
  cudaMalloc(&d_off, off.size() * 8);
  cudaMalloc(&d_keys, static_cast<size_t>(kReq) * kBlk * 8);
  cudaMemcpy(d_off, off.data(), off.size() * 8, cudaMemcpyHostToDevice);
  cudaMemset(d_keys, 1, static_cast<size_t>(kReq) * kBlk * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int v = 0; v < 3; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (v == 0) fold_strided<<<kReq / 32, 32>>>(d_off, d_keys, kReq, 1);
      if (v == 1) fold_strided<<<kReq / 32, 32>>>(d_off, d_keys, kReq, 0);
      if (v == 2) fold_transposed<<<kReq / 32, 32>>>(d_off, d_keys, kReq);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(&ms, a, b);
    const char* names[] = {"strided load+store", "strided load only", "smem transposed"};
    std::printf("%-20s %8.1f us  = %.1f cycles/step @1.965GHz\n", names[v], ms * 1e3,
                ms * 1e-3 * 1.965e9 / kBlk);
  }
  std::printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
