// fold_micro.cu -- why is the per-request key fold slower than the chain_hash
// dependency latency?  4096 requests x 1024 blocks, contents pre-filled.
//   a) lane = request, strided 8-byte loads/stores (current design)
//   b) same, loads only (no stores)
//   c) warp = 32 requests, 32-block windows transposed through shared memory
//      (coalesced 256-byte rows in, coalesced rows out)
//   d) the chain alone (contents in registers)   e) two requests per lane
//   f) 256-bit loads/stores, 8 or 16 entries per batch, 1 or 4 warps per SM
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

// d) the chain alone: contents from registers (no memory in the loop)
__global__ void fold_regs(const int64_t* key_off, int64_t* keys, int n_req) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_req) return;
  const int64_t k0 = key_off[r], k1 = key_off[r + 1];
  int64_t c[16];
  for (int j = 0; j < 16; ++j) c[j] = keys[k0 + j];
  int64_t prev = 0;
  for (int64_t k = k0; k < k1; k += 16) {
#pragma unroll
    for (int j = 0; j < 16; ++j) prev = kvx::chain_hash(prev, static_cast<uint64_t>(c[j]));
  }
  keys[k0] = prev;
}

// e) two requests per lane, chained interleaved (loads one batch ahead, stores)
__global__ void fold_two(const int64_t* key_off, int64_t* keys, int n_req) {
  const int r = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (r + 1 >= n_req + 1) return;
  const int64_t a0 = key_off[r], a1 = key_off[r + 1], b0 = key_off[r + 1], b1 = key_off[r + 2];
  const int64_t n = min(a1 - a0, b1 - b0);
  int64_t pa = 0, pb = 0;
  int64_t ca[8], cb[8];
  for (int j = 0; j < 8; ++j) { ca[j] = keys[a0 + j]; cb[j] = keys[b0 + j]; }
  for (int64_t k = 0; k < n; k += 8) {
    int64_t na[8], nb[8];
    for (int j = 0; j < 8; ++j) {
      na[j] = (k + 8 + j < n) ? keys[a0 + k + 8 + j] : 0;
      nb[j] = (k + 8 + j < n) ? keys[b0 + k + 8 + j] : 0;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      pa = kvx::chain_hash(pa, static_cast<uint64_t>(ca[j]));
      pb = kvx::chain_hash(pb, static_cast<uint64_t>(cb[j]));
      keys[a0 + k + j] = pa;
      keys[b0 + k + j] = pb;
    }
    for (int j = 0; j < 8; ++j) { ca[j] = na[j]; cb[j] = nb[j]; }
  }
}

// f) lane = request, 256-bit volatile loads one 16-batch ahead, 256-bit stores
__device__ __forceinline__ void ld4v(const int64_t* p, int64_t* v) {
  asm volatile("ld.volatile.global.v4.s64 {%0,%1,%2,%3}, [%4];"
               : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]) : "l"(p));
}
__device__ __forceinline__ void st4v(int64_t* p, const int64_t* v) {
  asm volatile("st.global.v4.s64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(v[0]), "l"(v[1]), "l"(v[2]),
               "l"(v[3]) : "memory");
}
template <int B>
__global__ void fold_vec(const int64_t* key_off, int64_t* keys, int n_req) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_req) return;
  const int64_t k0 = key_off[r], k1 = key_off[r + 1];
  int64_t prev = 0;
  int64_t c[B];
  for (int g = 0; g < B / 4; ++g) ld4v(keys + k0 + 4 * g, c + 4 * g);
  for (int64_t k = k0; k < k1; k += B) {
    int64_t nx[B];
    if (k + B < k1) {
#pragma unroll
      for (int g = 0; g < B / 4; ++g) ld4v(keys + k + B + 4 * g, nx + 4 * g);
    }
    int64_t o[B];
#pragma unroll
    for (int j = 0; j < B; ++j) {
      prev = kvx::chain_hash(prev, static_cast<uint64_t>(c[j]));
      o[j] = prev;
    }
#pragma unroll
    for (int g = 0; g < B / 4; ++g) st4v(keys + k + 4 * g, o + 4 * g);
#pragma unroll
    for (int j = 0; j < B; ++j) c[j] = nx[j];
  }
}

// Bandwidth hog for the "under load" variants: streams a large buffer on the
// other SMs (like the content producers streaming token ids).
__global__ void hog(const int4* __restrict__ a, int4* __restrict__ b, int64_t n, int reps) {
  for (int r = 0; r < reps; ++r)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
      b[i] = a[i];
}

// Same hog with L2 evict-first loads and streaming stores (does not displace the fold's keys).
__global__ void hog_ef(const int4* __restrict__ a, int4* __restrict__ b, int64_t n, int reps) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  for (int r = 0; r < reps; ++r)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
      int4 q;
      asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                   : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w) : "l"(a + i), "l"(pol));
      asm volatile("st.global.L2::cache_hint.v4.s32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(b + i), "r"(q.x),
                   "r"(q.y), "r"(q.z), "r"(q.w), "l"(pol) : "memory");
    }
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
  // hog: 2 x 1 GiB buffers, run on 116 SMs' worth of CTAs on a second stream
  const int64_t hn = (1LL << 30) / 16;
  int4 *ha, *hb;
  cudaMalloc(&ha, hn * 16);
  cudaMalloc(&hb, hn * 16);
  cudaStream_t hs;
  cudaStreamCreateWithFlags(&hs, cudaStreamNonBlocking);
  for (int v = 0; v < 16; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (v == 0) fold_strided<<<kReq / 32, 32>>>(d_off, d_keys, kReq, 1);
      if (v == 1) fold_strided<<<kReq / 32, 32>>>(d_off, d_keys, kReq, 0);
      if (v == 2) fold_transposed<<<kReq / 32, 32>>>(d_off, d_keys, kReq);
      if (v == 3) fold_regs<<<kReq / 32, 32>>>(d_off, d_keys, kReq);
      if (v == 4) fold_two<<<kReq / 64, 32>>>(d_off, d_keys, kReq);
      if (v == 5) fold_strided<<<kReq / 128, 128>>>(d_off, d_keys, kReq, 1);
      if (v == 6) fold_vec<8><<<kReq / 32, 32>>>(d_off, d_keys, kReq);
      if (v == 7) fold_vec<8><<<kReq / 128, 128>>>(d_off, d_keys, kReq);
      if (v == 8) fold_vec<16><<<kReq / 32, 32>>>(d_off, d_keys, kReq);
      if (v == 9) fold_vec<16><<<kReq / 128, 128>>>(d_off, d_keys, kReq);
      if (v >= 10) {
        // fold first (it takes the first 32 SMs), then the hog fills the rest
        cudaStream_t fs;
        cudaStreamCreateWithFlags(&fs, cudaStreamNonBlocking);
        cudaEventRecord(a, fs);
        // 200 KB of (unused) shared memory keeps the hog's CTAs off the folding SMs
        const int excl = 200 * 1024;
        cudaFuncSetAttribute(fold_vec<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, excl);
        cudaFuncSetAttribute(fold_strided, cudaFuncAttributeMaxDynamicSharedMemorySize, excl);
        if (v == 10 || v == 12 || v == 14) fold_vec<8><<<kReq / 128, 128, excl, fs>>>(d_off, d_keys, kReq);
        else fold_strided<<<kReq / 128, 128, excl, fs>>>(d_off, d_keys, kReq, 1);
        // v 10/11: hog saturates HBM; v 12/13: a light hog (~16 CTAs)
        if (v < 14) hog<<<v < 12 ? 116 * 4 : 16, 512, 0, hs>>>(ha, hb, hn, v < 12 ? 4 : 1);
        else hog_ef<<<16, 512, 0, hs>>>(ha, hb, hn, 1);
        cudaEventRecord(b, fs);
        cudaEventSynchronize(b);
        cudaStreamSynchronize(hs);
        cudaStreamDestroy(fs);
        continue;
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(&ms, a, b);
    const char* names[] = {"strided load+store", "strided load only", "smem transposed",
                           "registers only", "2 requests/lane", "a) 4 warps/CTA",
                           "f) vec8 1 warp/CTA", "f) vec8 4 warps/CTA", "f) vec16 1 warp/CTA",
                           "f) vec16 4 warps/CTA", "f) vec8 4w + HBM hog", "a) 4w + HBM hog",
                           "f) vec8 4w + light hog", "a) 4w + light hog",
                           "f) vec8 4w + light evict-first hog", "a) 4w + light evict-first hog"};
    std::printf("%-20s %8.1f us  = %.1f cycles/step @1.965GHz\n", names[v], ms * 1e3,
                ms * 1e-3 * 1.965e9 / kBlk);
  }
  std::printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
