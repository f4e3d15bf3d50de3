// Microbenchmark of tcgen05.mma issue/throughput for the shapes K4 uses.
// Build+run on a B200: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20
//   -I../paper_2511_23113_b200/csrc tests/mma_bench.cu -o /tmp/mma_bench && /tmp/mma_bench
// Each CTA allocates 256 TMEM columns, fills 64 KB of smem with zeros and
// issues `rounds` groups of MMAs (one commit + wait per group); reports
// cycles per MMA instruction and the implied fraction of the tcgen05 floor
// (128*N/256 cycles for M=128).
#include <cstdio>
#include <cstdlib>

#include "ptx.cuh"

using namespace dbsp_dev;

template <int N, bool A_TMEM, int PER_GROUP>
__global__ void __launch_bounds__(128, 2) mma_kernel(int rounds, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (warp == 0) tmem_alloc(smem_u32(&tmem_slot), 256);
  if (threadIdx.x == 32) {
    mbar_init(smem_u32(&bar), 1);
    mbar_fence_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const uint32_t base = smem_u32(smem);
  unsigned long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_bf16(128, N, false, false);
    t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
      for (int k = 0; k < PER_GROUP; ++k) {
        const uint64_t bd = smem_desc_sw128(base + 32768 + (k & 3) * 32, 16, 1024);
        if (A_TMEM) {
          mma_ts(tmem + 128, tmem + (k & 7) * 8, bd, idesc, k > 0);
        } else {
          const uint64_t ad = smem_desc_sw128(base + (k & 3) * 32, 16, 1024);
          mma_ss(tmem, ad, bd, idesc, k > 0);
        }
      }
      tc_commit(smem_u32(&bar));
      mbar_wait(smem_u32(&bar), r & 1);
    }
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

template <int N, bool A_TMEM, int PER_GROUP>
void run(const char* name, int ctas_per_sm) {
  const int sms = 148, rounds = 2000;
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * sms * 2);
  auto k = mma_kernel<N, A_TMEM, PER_GROUP>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int grid = sms * ctas_per_sm;
  k<<<grid, 128, 65536>>>(10, d);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<grid, 128, 65536>>>(rounds, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[296];
  cudaMemcpy(h, d, sizeof(unsigned long long) * grid, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < grid; ++i) avg += double(h[i]);
  avg /= grid;
  const double per_mma = avg / (double(rounds) * PER_GROUP);
  const double floor = 128.0 * N / 256.0;
  const double flops = 2.0 * 128 * N * 16 * double(rounds) * PER_GROUP * grid;
  std::printf("%-28s ctas/SM=%d  cycles/MMA(per CTA)=%7.2f  floor=%5.1f  SM-level eff=%.3f  %.1f TFLOP/s  %s\n",
              name, ctas_per_sm, per_mma, floor, floor * ctas_per_sm / per_mma,
              flops / (ms * 1e-3) / 1e12, cudaGetErrorString(err));
  cudaFree(d);
}

int main() {
  for (int c : {1, 2}) {
    run<64, false, 8>("SS M128 N64 K16 x8", c);
    run<64, true, 8>("TS M128 N64 K16 x8", c);
    run<128, false, 4>("SS M128 N128 K16 x4", c);
    run<128, true, 4>("TS M128 N128 K16 x4", c);
    run<256, false, 4>("SS M128 N256 K16 x4", c);
    run<128, true, 64>("TS M128 N128 K16 x64", c);
    run<64, false, 64>("SS M128 N64 K16 x64", c);
    run<64, true, 64>("TS M128 N64 K16 x64", c);
    run<64, true, 4>("TS M128 N64 K16 x4", c);
    run<64, true, 1>("TS M128 N64 K16 x1", c);
  }
  return 0;
}
