// MUFU throughput on B200: ex2.approx.ftz.f32 vs ex2.approx.f16x2 vs
// ex2.approx.ftz.bf16x2 (results per SM per cycle).  GPU-box tool:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tests/mufu_bench.cu -o /tmp/mufu && /tmp/mufu
#include <cstdio>
#include <cstdint>

template <int MODE>
__global__ void k(float* out, int iters) {
  float a0 = threadIdx.x * 1e-3f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
  uint32_t h0 = 0x3c003c00u ^ threadIdx.x, h1 = h0 + 1, h2 = h0 + 2, h3 = h0 + 3;
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) {
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a0));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a1));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a2));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a3));
    } else if (MODE == 1) {
      asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h0));
      asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h1));
      asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h2));
      asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h3));
    } else {
      asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h0));
      asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h1));
      asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h2));
      asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h3));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + float(h0 ^ h1 ^ h2 ^ h3);
}

template <int MODE>
void run(const char* name) {
  float* d;
  const int blocks = 148 * 8, threads = 256, iters = 4096;
  cudaMalloc(&d, sizeof(float) * blocks * threads);
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
  const double insts = double(blocks) * threads * iters * 4;
  const double results = insts * (MODE == 0 ? 1 : 2);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cycles = ms * 1e-3 * clk * 1e3;
  std::printf("%-12s %.3f ms  %.1f results/SM/cycle (at %d MHz)\n", name, ms,
              results / 148 / cycles, clk / 1000);
  cudaFree(d);
}

int main() {
  run<0>("ex2.f32");
  run<1>("ex2.f16x2");
  run<2>("ex2.bf16x2");
  return 0;
}
