// Microbenchmark of tcgen05.mma cta_group::2 (CTA pair, M=256) throughput for
// the shapes of the CTA-pair K4 kernels (attn_kernel_pd*.cuh), in isolation:
// only the leader's MMA thread runs, operands are zero-filled smem / TMEM.
// Build+run on a B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 \
//     -Ipaper_2511_23113_b200/csrc tests/mma2_bench.cu -o /tmp/mma2 -lcuda && /tmp/mma2
// Reports cycles per MMA instruction and the fraction of the tcgen05 floor
// (max(M,128)*N/(256*2) cycles per instruction for cta_group::2).
#include <cstdio>

#include "ptx.cuh"

using namespace dbsp_dev;

// mode 0: QK-like  SS, A K-major (smem), B K-major (smem)
// mode 1: PV-like  TS, A from TMEM,       B MN-major (smem)
// mode 2: PV-like  SS, A K-major (smem),  B MN-major (smem)
// mode 3: a full 128-key step: 8 x mode 0 then 8 x mode 1 (attn_kernel_pd2.cuh)
// mode 4: a full 128-key step: 8 x mode 0 then 8 x mode 2 (attn_kernel_pd3.cuh)
template <int N, int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mma2_kernel(int rounds, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32;
  const uint32_t rank = cluster_ctarank();
  for (int i = threadIdx.x; i < 98304 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (warp == 0) tmem_alloc_pair(smem_u32(&tmem_slot), 512);
  if (threadIdx.x == 32) {
    mbar_init(smem_u32(&bar), 1);
    mbar_fence_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const uint32_t base = smem_u32(smem);
  if (rank == 0 && threadIdx.x == 0) {
    constexpr uint32_t idesc_qk = idesc_bf16(256, N, false, false);
    constexpr uint32_t idesc_pv = idesc_bf16(256, N, false, true);
    auto qk = [&](int k) {
      const uint64_t ad = smem_desc_sw128(base + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
      const uint64_t bd = smem_desc_sw128(base + 32768 + (k >> 2) * 8192 + (k & 3) * 32, 16, 1024);
      mma_ss_pair(tmem, ad, bd, idesc_qk, k > 0);
    };
    auto pv_ts = [&](int k) {
      const uint64_t bd = smem_desc_sw128(base + 49152 + k * 2048, 16384, 1024);
      mma_ts_pair(tmem + 256, tmem + 128 + (k >> 2) * 64 + (k & 3) * 8, bd, idesc_pv, 1);
    };
    auto pv_ss = [&](int k) {
      const uint64_t ad = smem_desc_sw128(base + 65536 + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
      const uint64_t bd = smem_desc_sw128(base + 49152 + k * 2048, 16384, 1024);
      mma_ss_pair(tmem + 256, ad, bd, idesc_pv, 1);
    };
    const unsigned long long t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
      for (int k = 0; k < 8; ++k) {
        if (MODE == 0 || MODE == 3 || MODE == 4) qk(k);
        if (MODE == 1) pv_ts(k);
        if (MODE == 2) pv_ss(k);
      }
      if (MODE == 3)
        for (int k = 0; k < 8; ++k) pv_ts(k);
      if (MODE == 4)
        for (int k = 0; k < 8; ++k) pv_ss(k);
      tc_commit_pair(smem_u32(&bar), 0x3);
      mbar_wait(smem_u32(&bar), r & 1);
    }
    out[blockIdx.x / 2] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (warp == 0) tmem_dealloc_pair(tmem, 512);
}

template <int N, int MODE>
void run(const char* name) {
  const int pairs = 74, rounds = 2000;
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * pairs);
  auto k = mma2_kernel<N, MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304 + 1024);
  k<<<2 * pairs, 128, 98304 + 1024>>>(10, d);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<2 * pairs, 128, 98304 + 1024>>>(rounds, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[74];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < pairs; ++i) avg += double(h[i]);
  avg /= pairs;
  const int per_round = (MODE >= 3) ? 16 : 8;
  const double per_mma = avg / (double(rounds) * per_round);
  const double floor = 256.0 * N / 512.0;
  const double flops = 2.0 * 256 * N * 16 * double(rounds) * per_round * pairs;
  std::printf("%-40s cycles/MMA=%7.2f  floor=%5.1f  eff=%.3f  %.1f TFLOP/s  %s\n", name, per_mma, floor,
              floor / per_mma, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(err));
  cudaFree(d);
}

int main() {
  run<128, 0>("QK  SS  M256 N128 K16 x8");
  run<128, 1>("PV  TS  M256 N128 K16 x8 (B MN-major)");
  run<128, 2>("PV  SS  M256 N128 K16 x8 (B MN-major)");
  run<128, 3>("step: 8 QK SS + 8 PV TS");
  run<128, 4>("step: 8 QK SS + 8 PV SS");
  run<256, 0>("QK  SS  M256 N256 K16 x8");
  return 0;
}
