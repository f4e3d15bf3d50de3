// Issue throughput of the softmax instruction mix on B200 (instructions per
// SM per cycle), alone and mixed, to find which pipe each one shares.
// GPU-box tool:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tests/pipe_bench.cu -o /tmp/pipe && /tmp/pipe
#include <cstdint>
#include <cstdio>

#define EX2(x) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x))
#define CVT(r, x, y) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x), "f"(y))
#define FMA(x) asm volatile("fma.rn.f32 %0, %0, 0f3F800001, 0f3A000000;" : "+f"(x))
#define MAX3(x, y, z) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(x) : "f"(y), "f"(z))
#define PRMT(r, x, y) asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(x), "r"(y))
#define ADD(x, y) asm volatile("add.f32 %0, %0, %1;" : "+f"(x) : "f"(y))

#define FFMA2(x, s, n) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x) : "l"(s), "l"(n))
#define FADD2(x, y) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(y))
#define EX2LO(x) asm volatile("{.reg .f32 lo, hi; mov.b64 {lo, hi}, %0; ex2.approx.ftz.f32 lo, lo; ex2.approx.ftz.f32 hi, hi; mov.b64 %0, {lo, hi};}" : "+l"(x))

// 2^x for a pair on the FMA/ALU pipes (packed f32x2): clamp, round-to-int by
// the 1.5*2^23 trick, degree-3 polynomial of the fraction, exponent by shift+add.
__device__ __forceinline__ unsigned long long exp2_pair_poly(unsigned long long x) {
  float lo = __uint_as_float(uint32_t(x)), hi = __uint_as_float(uint32_t(x >> 32));
  lo = fmaxf(lo, -127.f);
  hi = fmaxf(hi, -127.f);
  float2 xv = make_float2(lo, hi);
  const float2 mg = make_float2(12582912.f, 12582912.f), nmg = make_float2(-12582912.f, -12582912.f);
  const float2 t = __fadd2_rn(xv, mg);
  const float2 f = __fadd2_rn(xv, __fmul2_rn(__fadd2_rn(t, nmg), make_float2(-1.f, -1.f)));
  float2 p = __ffma2_rn(f, make_float2(0.05500764772295952f, 0.05500764772295952f),
                        make_float2(0.24220800399780273f, 0.24220800399780273f));
  p = __ffma2_rn(p, f, make_float2(0.6932827234268188f, 0.6932827234268188f));
  p = __ffma2_rn(p, f, make_float2(1.f, 1.f));
  const uint32_t rl = __float_as_uint(p.x) + (__float_as_uint(t.x) << 23);
  const uint32_t rh = __float_as_uint(p.y) + (__float_as_uint(t.y) << 23);
  return (unsigned long long)rh << 32 | rl;
}

// MODE 8: packed softmax body per pair: FFMA2, 2x ex2, FADD2, cvt (one pair = 2 elements)
// MODE: 0 ex2 | 1 cvt | 2 ex2+cvt (2:1) | 3 fma | 4 max3 | 5 prmt | 6 ex2+fma (1:1)
//       7 ex2 + cvt + 2 fma (the softmax body per pair: 2 ex2, 1 cvt, 2 ffma, 2 fadd)
template <int MODE>
__global__ void k(uint32_t* out, int iters) {
  float a[8];
  uint32_t r[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = threadIdx.x * 1e-3f + 0.1f * i;
    r[i] = threadIdx.x + i;
  }
  unsigned long long pa[8], ps = 0, sc = 0x3F8000003F800000ull, ng = 0xBF000000BF000000ull;
#pragma unroll
  for (int i = 0; i < 8; ++i) pa[i] = (unsigned long long)(threadIdx.x + i) * 0x100000001ull;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 8 || (MODE >= 10 && MODE <= 14)) {
        FFMA2(pa[i], sc, ng);
        if (MODE >= 10 && i < MODE - 10) pa[i] = exp2_pair_poly(pa[i]);
        else EX2LO(pa[i]);
        FADD2(ps, pa[i]);
        CVT(r[i], __uint_as_float(uint32_t(pa[i])), __uint_as_float(uint32_t(pa[i] >> 32)));
      }
      if (MODE == 0) EX2(a[i]);
      if (MODE == 1) CVT(r[i], a[i], a[(i + 1) & 7]);
      if (MODE == 2) {
        EX2(a[i]);
        if (i & 1) CVT(r[i], a[i], a[i - 1]);
      }
      if (MODE == 3) FMA(a[i]);
      if (MODE == 4) MAX3(a[i], a[(i + 1) & 7], a[(i + 2) & 7]);
      if (MODE == 5) PRMT(r[i], r[(i + 1) & 7], r[(i + 2) & 7]);
      if (MODE == 6) {
        EX2(a[i]);
        FMA(a[(i + 4) & 7]);
      }
      if (MODE == 7) {
        FMA(a[i]);
        EX2(a[i]);
        ADD(a[(i + 3) & 7], a[i]);
        if (i & 1) CVT(r[i], a[i], a[i - 1]);
      }
    }
  }
  uint32_t x = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) x ^= __float_as_uint(a[i]) ^ r[i] ^ uint32_t(pa[i]);
  x ^= uint32_t(ps);
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

template <int MODE>
void run(const char* name, double insts_per_iter, int blocks = 148 * 8, int threads = 256) {
  uint32_t* d;
  const int iters = 2048;
  cudaMalloc(&d, sizeof(uint32_t) * blocks * threads);
  k<MODE><<<blocks, threads>>>(d, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<blocks, threads>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cycles = ms * 1e-3 * clk * 1e3;
  const double per_iter = double(blocks) * threads * iters;
  std::printf("[%4d warps/SM] %-40s %.3f ms  %.2f iters(x8)/SM/cycle  %.1f thread-insts/SM/cycle\n",
              blocks / 148 * threads / 32, name, ms,
              per_iter / 148 / cycles, per_iter * insts_per_iter / 148 / cycles);
  cudaFree(d);
}

int main() {
  run<0>("ex2", 8);
  run<1>("cvt.rn.bf16x2.f32", 8);
  run<2>("ex2 x8 + cvt x4", 12);
  run<3>("ffma", 8);
  run<4>("max3", 8);
  run<5>("prmt", 8);
  run<6>("ex2 x8 + ffma x8", 16);
  run<7>("softmax body: ffma,ex2,fadd x8 + cvt x4", 28);
  run<8>("packed body: ffma2,2 ex2,fadd2,cvt x8 (16 elems)", 40);
  run<11>("packed body, 1 of 8 pairs poly", 40);
  run<12>("packed body, 2 of 8 pairs poly", 40);
  run<13>("packed body, 3 of 8 pairs poly", 40);
  run<14>("packed body, 4 of 8 pairs poly", 40);
  run<11>("packed body, 1 of 8 pairs poly", 40, 148, 128);
  run<12>("packed body, 2 of 8 pairs poly", 40, 148, 128);
  run<13>("packed body, 3 of 8 pairs poly", 40, 148, 128);
  run<14>("packed body, 4 of 8 pairs poly", 40, 148, 128);
  run<12>("packed body, 2 of 8 pairs poly", 40, 148, 256);
  run<13>("packed body, 3 of 8 pairs poly", 40, 148, 256);
  run<14>("packed body, 4 of 8 pairs poly", 40, 148, 256);
  // one and two warps per SMSP: the two-stage kernel's softmax occupancy
  run<0>("ex2", 8, 148, 128);
  run<7>("softmax body: ffma,ex2,fadd x8 + cvt x4", 28, 148, 128);
  run<8>("packed body: ffma2,2 ex2,fadd2,cvt x8 (16 elems)", 40, 148, 128);
  run<7>("softmax body: ffma,ex2,fadd x8 + cvt x4", 28, 148, 256);
  run<8>("packed body: ffma2,2 ex2,fadd2,cvt x8 (16 elems)", 40, 148, 256);
  return 0;
}
