// Throughput of the softmax exp body per element on B200, f32 MUFU.EX2 vs the
// packed half-precision forms (ex2.approx.f16x2 / ex2.approx.ftz.bf16x2: two
// results per MUFU op).  Elements per SM per cycle, from clock64.
// GPU-box tool:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tests/ex2h_bench.cu -o /tmp/ex2h && /tmp/ex2h
#include <cstdint>
#include <cstdio>

#include <cuda_bf16.h>
#include <cuda_fp16.h>

// MODE 0: ex2.f32 alone (1 elem / op)            MODE 1: ex2.f16x2 alone (2 / op)
// MODE 2: ex2.bf16x2 alone (2 / op)
// MODE 3: f32 body  : ffma2, 2x ex2.f32, fadd2, cvt.bf16x2              (2 elems)
// MODE 4: f16 body  : ffma2, cvt.f16x2, ex2.f16x2, 2x cvt.f32.f16, fadd2, cvt.bf16x2
// MODE 5: bf16 body : ffma2, cvt.bf16x2, ex2.bf16x2, 2x unpack, fadd2   (P is the ex2 result)
template <int MODE>
__global__ void k(uint32_t* out, int iters, unsigned long long* cyc) {
  unsigned long long pa[8];
  uint32_t h[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    pa[i] = (unsigned long long)(threadIdx.x + i) * 0x100000001ull;
    h[i] = 0x3c003c00u + threadIdx.x + i;
  }
  float2 acc = make_float2(0.f, 0.f);
  uint32_t pk = 0;
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {
        asm volatile("{.reg .f32 lo, hi; mov.b64 {lo, hi}, %0; ex2.approx.ftz.f32 lo, lo; mov.b64 %0, {lo, hi};}"
                     : "+l"(pa[i]));
      } else if (MODE == 1) {
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h[i]));
      } else if (MODE == 2) {
        asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h[i]));
      } else {
        float2 x = make_float2(__uint_as_float(uint32_t(pa[i])), __uint_as_float(uint32_t(pa[i] >> 32)));
        x = __ffma2_rn(x, make_float2(0.999f, 0.999f), make_float2(-0.5f, -0.5f));
        float2 p;
        if (MODE == 3) {
          float a, b;
          asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(a) : "f"(x.x));
          asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(b) : "f"(x.y));
          p = make_float2(a, b);
          uint32_t r;
          asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(p.y), "f"(p.x));
          pk ^= r;
        } else if (MODE == 4) {
          uint32_t hh;
          asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(hh) : "f"(x.y), "f"(x.x));
          asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(hh));
          const __half2 hv = *reinterpret_cast<__half2*>(&hh);
          p = __half22float2(hv);
          uint32_t r;
          asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(p.y), "f"(p.x));
          pk ^= r;
        } else {
          uint32_t bb;
          asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(bb) : "f"(x.y), "f"(x.x));
          asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(bb));
          pk ^= bb;
          p = make_float2(__uint_as_float(bb << 16), __uint_as_float(bb & 0xffff0000u));
        }
        acc = __fadd2_rn(acc, p);
        pa[i] = (unsigned long long)__float_as_uint(x.y) << 32 | __float_as_uint(x.x);
      }
    }
  }
  const unsigned long long t1 = clock64();
  uint32_t s = pk ^ __float_as_uint(acc.x) ^ __float_as_uint(acc.y);
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= uint32_t(pa[i]) ^ h[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int threads) {
  const int blocks = 148, iters = 4096;
  uint32_t* d;
  unsigned long long* c;
  cudaMalloc(&d, blocks * threads * 4);
  cudaMalloc(&c, blocks * 8);
  k<MODE><<<blocks, threads>>>(d, 16, c);
  k<MODE><<<blocks, threads>>>(d, iters, c);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < blocks; ++i) avg += double(h[i]);
  avg /= blocks;
  const double elems_per_op = (MODE == 0) ? 1.0 : 2.0;  // per thread per inner step
  const double elems = double(threads) * iters * 8 * elems_per_op;
  std::printf("%-58s warps/SMSP=%2d  %6.2f elements/clk/SM  %s\n", name, threads / 128, elems / avg,
              cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(c);
}

int main() {
  for (int t : {256, 512}) {
    run<0>("ex2.approx.ftz.f32", t);
    run<1>("ex2.approx.f16x2", t);
    run<2>("ex2.approx.ftz.bf16x2", t);
    run<3>("body f32: ffma2, 2 ex2.f32, fadd2, cvt.bf16x2", t);
    run<4>("body f16: ffma2, cvt.f16x2, ex2.f16x2, 2 cvt.f32, fadd2, cvt", t);
    run<5>("body bf16: ffma2, cvt.bf16x2, ex2.bf16x2, unpack, fadd2", t);
  }
  return 0;
}
