// pipe_micro.cu -- per-instruction issue cost of the integer ops a 64-bit
// chain_hash step can be built from, and the throughput of chain_hash
// formulations that spread the step over the ALU and FMA pipes (run on a B200).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../include \
//        -I../../paper_2407_00079_b200/csrc pipe_micro.cu -o pipe_micro
//
// Each thread runs 8 independent dependency chains of one op (enough to hide
// the 4-5 cycle latency), 148 x 8 CTAs of 256 threads; reported as warp
// instructions per cycle per SM sub-partition (SMSP; 0.5 = rt 2).  Operands
// that would let ptxas fold the op into something else come from kernel
// arguments.  Check the SASS (cuobjdump -sass) before reading a number.
#include <cstdio>
#include <cstdint>

#include "kvx_common.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  std::printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int kChains = 8;

enum Op { kShf, kLop3, kImad, kImadHi, kImadWide, kLea, kIadd3, kMix, kAddc };

template <int OP>
__global__ void __launch_bounds__(256) op_loop(int iters, uint32_t a, uint32_t b, uint32_t* sink) {
  uint32_t x[kChains], y[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) { x[c] = threadIdx.x * 7 + c; y[c] = threadIdx.x ^ (c * 13); }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      if (OP == kShf) {
        x[c] = __funnelshift_r(x[c], y[c], a);
      } else if (OP == kLop3) {
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(y[c]), "r"(a));
      } else if (OP == kImad) {
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(y[c]));
      } else if (OP == kImadHi) {
        asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(x[c]) : "r"(a));
      } else if (OP == kImadWide) {
        uint64_t w = (static_cast<uint64_t>(y[c]) << 32) | x[c];
        asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w) : "r"(x[c]), "r"(a));
        x[c] = static_cast<uint32_t>(w);
        y[c] = static_cast<uint32_t>(w >> 32);
      } else if (OP == kMix) {  // one LOP3 + one IMAD per chain step: dual pipe
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(y[c]), "r"(a));
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(y[c]) : "r"(a), "r"(b));
      } else if (OP == kAddc) {  // 64-bit add: IADD3 + IADD3.X (2 instr)
        asm volatile("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, %3;"
                     : "+r"(x[c]), "+r"(y[c]) : "r"(a), "r"(b));
      } else if (OP == kLea) {
        x[c] = x[c] * 64u + y[c];  // LEA (ALU) or IMAD.SHL+add: see SASS
      } else {
        asm volatile("add.u32 %0, %0, %1;" : "+r"(x[c]) : "r"(y[c]));
      }
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc ^= x[c] ^ (y[c] * 3u);
  if (acc == 0x12345678u) sink[threadIdx.x] = acc;
}

// ---- chain_hash formulations ------------------------------------------------
// V1: the step's 64-bit shift-left-add and its high-word right shifts on the
// FMA pipe (mad.wide / mul.hi with register multipliers), the rest on ALU.
struct Mul {
  uint32_t s64, m2, m30, m27, m31;  // 64, 2^30, 2^2, 2^5, 2^1
  uint32_t one, dl, dh;             // 1, D = C + (C << 6) mod 2^64
};

__device__ __forceinline__ uint32_t lo32(uint64_t v) { return static_cast<uint32_t>(v); }
__device__ __forceinline__ uint32_t hi32(uint64_t v) { return static_cast<uint32_t>(v >> 32); }
__device__ __forceinline__ uint64_t mk64(uint32_t lo, uint32_t hi) {
  return (static_cast<uint64_t>(hi) << 32) | lo;
}
__device__ __forceinline__ uint64_t madw(uint32_t a, uint32_t b, uint64_t c) {
  uint64_t d;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint32_t mulhi(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t madlo(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// V3: a planned split, 16 ALU + 14 FMA-pipe instructions per step:
//   s = content + C + (x << 6) + (x >> 2) with x = prev + C is rewritten as
//   s = (content + D) + prev * 64 + (x >> 2),  D = C + (C << 6) mod 2^64,
// the content + D and prev * 64 terms on the FMA pipe (mad with register
// operands), the x >> 2 and the xor-shifts' funnels on ALU, the high words
// of the xor-shifts as mul.hi (FMA), the multiplies as three IMADs each.
__device__ __forceinline__ int64_t chain_v3(int64_t prev, uint64_t content, const Mul& m) {
  const uint32_t hl = lo32(prev), hh = hi32(prev);
  const uint32_t cl = lo32(content), ch = hi32(content);
  uint32_t xl, xh, cdl, cdh, tl, th, sl, sh;
  // cd = content + D (FMA: 64-bit cl * 1 + {dl, ch + dh})
  const uint32_t cdh0 = madlo(ch, m.one, m.dh);
  uint64_t cd = madw(cl, m.one, mk64(m.dl, cdh0));
  cdl = lo32(cd);
  cdh = hi32(cd);
  // t = cd + prev * 64 (FMA)
  uint64_t t = madw(hl, m.s64, mk64(cdl, cdh));
  tl = lo32(t);
  th = madlo(hh, m.s64, hi32(t));
  // x = prev + C (ALU)
  asm("add.cc.u32 %0, %2, 0x7F4A7C15;\n\taddc.u32 %1, %3, 0x9E3779B9;"
      : "=r"(xl), "=r"(xh) : "r"(hl), "r"(hh));
  // s = t + (x >> 2)
  const uint32_t rl = __funnelshift_r(xl, xh, 2);
  const uint32_t rh = mulhi(xh, m.m2);
  asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, %5;"
      : "=r"(sl), "=r"(sh) : "r"(tl), "r"(rl), "r"(th), "r"(rh));
  uint32_t yl = xl ^ sl, yh = xh ^ sh;
  // y ^= y >> 30
  {
    const uint32_t nl = __funnelshift_r(yl, yh, 30), nh = mulhi(yh, m.m30);
    yl ^= nl;
    yh ^= nh;
  }
  // y *= K1
  {
    const uint64_t p = madw(yl, 0x1CE4E5B9u, 0);
    const uint32_t ph = madlo(yh, 0x1CE4E5B9u, madlo(yl, 0xBF58476Du, hi32(p)));
    yl = lo32(p);
    yh = ph;
  }
  {
    const uint32_t nl = __funnelshift_r(yl, yh, 27), nh = mulhi(yh, m.m27);
    yl ^= nl;
    yh ^= nh;
  }
  {
    const uint64_t p = madw(yl, 0x133111EBu, 0);
    const uint32_t ph = madlo(yh, 0x133111EBu, madlo(yl, 0x94D049BBu, hi32(p)));
    yl = lo32(p);
    yh = ph;
  }
  {
    const uint32_t nl = __funnelshift_r(yl, yh, 31), nh = mulhi(yh, m.m31);
    yl ^= nl;
    yh = (yh ^ nh) & 0x7FFFFFFFu;
  }
  return static_cast<int64_t>(mk64(yl, yh));
}

// V4 / V5: IMAD.HI and IMAD.WIDE issue at half the IMAD rate (measured
// above), so only the prev * 64 term moves to the FMA pipe (one IMAD.WIDE +
// one IMAD replacing LEA + LEA.HI.X); V5 also moves the high word of x >> 2
// (one IMAD.HI).  ~17 ALU-pipe + ~10 FMA-pipe + 6 either-pipe adds per step.
template <int NHI>
__device__ __forceinline__ int64_t chain_v4(int64_t prev, uint64_t content, const Mul& m) {
  const uint32_t hl = lo32(prev), hh = hi32(prev);
  uint32_t cdl, cdh, xl, xh, sl, sh;
  asm("add.cc.u32 %0, %2, %4;\n\taddc.u32 %1, %3, %5;"
      : "=r"(cdl), "=r"(cdh) : "r"(lo32(content)), "r"(hi32(content)), "r"(m.dl), "r"(m.dh));
  const uint64_t t = madw(hl, m.s64, mk64(cdl, cdh));
  const uint32_t th = madlo(hh, m.s64, hi32(t));
  asm("add.cc.u32 %0, %2, 0x7F4A7C15;\n\taddc.u32 %1, %3, 0x9E3779B9;"
      : "=r"(xl), "=r"(xh) : "r"(hl), "r"(hh));
  const uint32_t rl = __funnelshift_r(xl, xh, 2);
  const uint32_t rh = NHI >= 1 ? mulhi(xh, m.m2) : (xh >> 2);
  asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, %5;"
      : "=r"(sl), "=r"(sh) : "r"(lo32(t)), "r"(rl), "r"(th), "r"(rh));
  uint64_t y = mk64(xl ^ sl, xh ^ sh);
  y ^= y >> 30;
  y *= 0xBF58476D1CE4E5B9ull;
  y ^= y >> 27;
  y *= 0x94D049BB133111EBull;
  y ^= y >> 31;
  return static_cast<int64_t>(y & 0x7FFFFFFFFFFFFFFFull);
}

template <int V>
__device__ __forceinline__ int64_t chain_v(int64_t prev, uint64_t content, const Mul& m) {
  if (V == 4) return chain_v4<0>(prev, content, m);
  if (V == 5) return chain_v4<1>(prev, content, m);
  if (V == 0) return kvx::chain_hash(prev, content);
  if (V == 3) return chain_v3(prev, content, m);
  constexpr uint64_t C = 0x9E3779B97F4A7C15ull;
  const uint64_t x = static_cast<uint64_t>(prev) + C;
  const uint32_t xl = lo32(x), xh = hi32(x);
  const uint64_t cc = content + C;
  // s = cc + (x << 6) + (x >> 2)
  uint64_t s = madw(xl, m.s64, cc);                  // cc + xl * 64
  s = mk64(lo32(s), madlo(xh, m.s64, hi32(s)));       // + xh * 64 << 32
  const uint32_t rl = __funnelshift_r(xl, xh, 2);
  const uint32_t rh = V == 2 ? mulhi(xh, m.m2) : (xh >> 2);
  s += mk64(rl, rh);
  uint64_t y = x ^ s;
  // y ^= y >> 30
  {
    const uint32_t l = lo32(y), h = hi32(y);
    const uint32_t nl = __funnelshift_r(l, h, 30);
    const uint32_t nh = V == 2 ? mulhi(h, m.m30) : (h >> 30);
    y = mk64(l ^ nl, h ^ nh);
  }
  y *= 0xBF58476D1CE4E5B9ull;
  {
    const uint32_t l = lo32(y), h = hi32(y);
    y = mk64(l ^ __funnelshift_r(l, h, 27), h ^ (V == 2 ? mulhi(h, m.m27) : (h >> 27)));
  }
  y *= 0x94D049BB133111EBull;
  {
    const uint32_t l = lo32(y), h = hi32(y);
    y = mk64(l ^ __funnelshift_r(l, h, 31), h ^ (V == 2 ? mulhi(h, m.m31) : (h >> 31)));
  }
  return static_cast<int64_t>(y & 0x7FFFFFFFFFFFFFFFull);
}

template <int V>
__global__ void __launch_bounds__(256) chain_loop(int iters, Mul m, const uint32_t* tok,
                                                  int64_t* out) {
  int64_t h[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) h[c] = threadIdx.x + c * 977 + blockIdx.x;
  for (int i = 0; i < iters; ++i) {
    const uint32_t t = tok[i & 1023];
#pragma unroll
    for (int c = 0; c < 4; ++c) h[c] = chain_v<V>(h[c], t + c, m);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = h[0] ^ h[1] ^ h[2] ^ h[3];
}

template <int V>
__global__ void chain_lat(int iters, Mul m, const uint32_t* tok, int64_t* out, long long* cyc) {
  int64_t h = threadIdx.x;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) h = chain_v<V>(h, tok[i & 1023], m);
  const long long t1 = clock64();
  out[threadIdx.x] = h;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <typename K>
static float time_kernel(K launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaEventRecord(a);
  launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  int dev = 0, clk_khz = 0, sms = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint32_t* sink;
  CK(cudaMalloc(&sink, 1 << 20));
  const int grid = sms * 8, threads = 256, iters = 4096;
  const double warp_instr = double(grid) * threads / 32 * iters * kChains;
  const char* names[] = {"SHF.R.U64 (funnel)", "LOP3", "IMAD", "IMAD.HI", "IMAD.WIDE (+xor)",
                         "x*64+y", "IADD3", "LOP3+IMAD (2 instr)", "IADD3+IADD3.X (2)"};
  // clocks: report per SMSP per cycle at the max clock (the loops run ~ms)
  const double hz = clk_khz * 1e3;
  auto report = [&](int op, float ms) {
    const double per_smsp_clk = warp_instr / (ms * 1e-3) / hz / (sms * 4.0);
    std::printf("%-20s %.3f warp-instr / clk / SMSP (rt %.2f)\n", names[op], per_smsp_clk,
                1.0 / per_smsp_clk);
  };
  report(kShf, time_kernel([&] { op_loop<kShf><<<grid, threads>>>(iters, 5, 7, sink); }));
  report(kLop3, time_kernel([&] { op_loop<kLop3><<<grid, threads>>>(iters, 5, 7, sink); }));
  report(kImad, time_kernel([&] { op_loop<kImad><<<grid, threads>>>(iters, 5, 7, sink); }));
  report(kImadHi, time_kernel([&] { op_loop<kImadHi><<<grid, threads>>>(iters, 0x9e3779b9u, 7, sink); }));
  report(kImadWide, time_kernel([&] { op_loop<kImadWide><<<grid, threads>>>(iters, 5, 7, sink); }));
  report(kLea, time_kernel([&] { op_loop<kLea><<<grid, threads>>>(iters, 5, 7, sink); }));
  report(kIadd3, time_kernel([&] { op_loop<kIadd3><<<grid, threads>>>(iters, 5, 7, sink); }));
  report(kMix, time_kernel([&] { op_loop<kMix><<<grid, threads>>>(iters, 5, 7, sink); }));
  report(kAddc, time_kernel([&] { op_loop<kAddc><<<grid, threads>>>(iters, 5, 7, sink); }));

  uint32_t* tok;
  int64_t *out, *out0;
  long long* cyc;
  CK(cudaMalloc(&tok, 1024 * 4));
  CK(cudaMalloc(&out, size_t(grid) * threads * 8));
  CK(cudaMalloc(&out0, size_t(grid) * threads * 8));
  CK(cudaMalloc(&cyc, 8));
  uint32_t htok[1024];
  for (int i = 0; i < 1024; ++i) htok[i] = 0x9e3779b9u * (i + 1) ^ (i << 7);
  CK(cudaMemcpy(tok, htok, sizeof(htok), cudaMemcpyHostToDevice));
  constexpr uint64_t C = 0x9E3779B97F4A7C15ull, D = C + (C << 6);
  const Mul m{64u, 1u << 30, 1u << 2, 1u << 5, 1u << 1, 1u, static_cast<uint32_t>(D),
              static_cast<uint32_t>(D >> 32)};
  const int citers = 1024;
  const double hashes = double(grid) * threads * citers * 4;
  int64_t* h0 = new int64_t[size_t(grid) * threads];
  int64_t* h1 = new int64_t[size_t(grid) * threads];
  for (int v = 0; v < 6; ++v) {
    float ms = 0;
    int64_t* o = v == 0 ? out0 : out;
    if (v == 0) ms = time_kernel([&] { chain_loop<0><<<grid, threads>>>(citers, m, tok, o); });
    if (v == 1) ms = time_kernel([&] { chain_loop<1><<<grid, threads>>>(citers, m, tok, o); });
    if (v == 2) ms = time_kernel([&] { chain_loop<2><<<grid, threads>>>(citers, m, tok, o); });
    if (v == 3) ms = time_kernel([&] { chain_loop<3><<<grid, threads>>>(citers, m, tok, o); });
    if (v == 4) ms = time_kernel([&] { chain_loop<4><<<grid, threads>>>(citers, m, tok, o); });
    if (v == 5) ms = time_kernel([&] { chain_loop<5><<<grid, threads>>>(citers, m, tok, o); });
    CK(cudaDeviceSynchronize());
    bool same = true;
    if (v > 0) {
      CK(cudaMemcpy(h0, out0, size_t(grid) * threads * 8, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(h1, out, size_t(grid) * threads * 8, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < size_t(grid) * threads; ++i) same = same && h0[i] == h1[i];
    }
    long long c = 0;
    if (v == 0) chain_lat<0><<<1, 1>>>(20000, m, tok, out, cyc);
    if (v == 1) chain_lat<1><<<1, 1>>>(20000, m, tok, out, cyc);
    if (v == 2) chain_lat<2><<<1, 1>>>(20000, m, tok, out, cyc);
    if (v == 3) chain_lat<3><<<1, 1>>>(20000, m, tok, out, cyc);
    if (v == 4) chain_lat<4><<<1, 1>>>(20000, m, tok, out, cyc);
    if (v == 5) chain_lat<5><<<1, 1>>>(20000, m, tok, out, cyc);
    CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    std::printf("chain_hash V%d: %.1f G/s full chip, %.1f cycles/step lone, bit-identical=%d\n", v,
                hashes / (ms * 1e-3) / 1e9, double(c) / 20000, int(same));
  }
  return 0;
}
