// Microbenchmark of K4's d=64 softmax step in isolation (no MMAs): each warp
// repeatedly loads a 32-lane x 64-column fp32 S tile from TMEM, takes the row
// max, runs the exp loop (3 of 8 pairs on the FMA pipe at {0,3,5}, packed
// FFMA2/FADD2, bf16 packing) and stores P (32 columns) back to TMEM -- the
// per-tile work of one softmax warp of attn_kernel.cuh, minus barriers.
// Varying the warps per SM sub-partition shows whether the softmax alone
// saturates a shared unit (MUFU, issue, TMEM) at the kernel's observed rate.
// softmax_split_kernel: the column-split layout (two warps per lane quarter,
// 32 columns each, partial row max exchanged through smem + a named barrier).
// Build+run on a B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 \
//     -Ipaper_2511_23113_b200/csrc tests/softmax_bench.cu -o tests/softmax_bench.bin && tests/softmax_bench.bin
#include <cstdio>

#include "attn_kernel.cuh"

using namespace dbsp_dev;

template <int WARPS, bool NOSUM = false, int PACK = 0, int PN = poly_pairs<64>()>
__global__ void __launch_bounds__(WARPS * 32, 1) softmax_kernel(int iters, float scale_log2,
                                                                 unsigned long long* out, float* sink) {
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(smem_u32(&tmem_slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  // Warp w works on lane quarter w % 4, in its own 96-column slice.
  const uint32_t lane_off = uint32_t((warp & 3) * 32) << 16;
  const uint32_t scol = tmem + lane_off + 96u * uint32_t(warp >> 2);  // S 64 + P 32 columns
  {  // deterministic S values
    uint32_t init[32];
    for (int i = 0; i < 32; ++i) init[i] = __float_as_uint(0.01f * float((lane * 7 + i * 13) % 97) - 0.3f);
    tmem_st32(scol, init);
    tmem_st32(scol + 32, init);
    tmem_st_wait();
  }
  float m = -INFINITY, l = 0.f;
  __syncwarp();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t sa[32], sb[32];
    tmem_ld32(scol, sa);
    tmem_ld32(scol + 32, sb);
    tmem_ld_wait();
    float v[64];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      v[i] = __uint_as_float(sa[i]);
      v[i + 32] = __uint_as_float(sb[i]);
    }
    float mx[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      mx[a] = fmax3f(v[8 * a], v[8 * a + 1], v[8 * a + 2]);
      mx[a] = fmax3f(mx[a], v[8 * a + 3], v[8 * a + 4]);
      mx[a] = fmax3f(mx[a], v[8 * a + 5], v[8 * a + 6]);
      mx[a] = fmaxf(mx[a], v[8 * a + 7]);
    }
    const float mt2 =
        fmaxf(fmax3f(mx[0], mx[1], mx[2]), fmax3f(fmax3f(mx[3], mx[4], mx[5]), mx[6], mx[7])) * scale_log2;
    if constexpr (PACK == 3) {  // speculative: exps with the running max, the max check after
      if (it == 0) m = mt2;
    } else if (mt2 > m + kRescaleThreshold) {
      l *= fast_exp2(m - mt2);
      m = mt2;
    }
    const float2 sc2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-m, -m);
    float2 acc2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    uint32_t pk[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float2 x = __ffma2_rn(make_float2(v[2 * i], v[2 * i + 1]), sc2, nm2);
      float2 pp;
      if constexpr (PACK == 2) {  // packed f16x2 ex2: cvt f32x2 -> f16x2, one MUFU for two exps
        uint32_t h, e;
        asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x.y), "f"(x.x));
        asm("ex2.approx.f16x2 %0, %1;" : "=r"(e) : "r"(h));
        pk[i] = e;
        continue;
      }
      if ((poly_mask(PN) >> (i & 7)) & 1)
        pp = exp2_poly3_pair(x);
      else
        pp = make_float2(fast_exp2(x.x), fast_exp2(x.y));
      if constexpr (!NOSUM) acc2[i & 1] = __fadd2_rn(acc2[i & 1], pp);
      if constexpr (PACK == 0 || PACK == 3) {
        pk[i] = pack_bf16x2(pp.x, pp.y);
      } else {  // truncate to bf16 with one byte permute (ALU pipe) instead of F2FP
        uint32_t r;
        asm("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(__float_as_uint(pp.x)), "r"(__float_as_uint(pp.y)));
        pk[i] = r;
      }
    }
    const float2 a2 = __fadd2_rn(acc2[0], acc2[1]);
    l += a2.x + a2.y;
    if constexpr (PACK == 3) {
      if (__any_sync(0xffffffffu, mt2 > m + kRescaleThreshold)) {  // never after the first step here
        l = 0.f;
        m = mt2;
      }
    }
    // P next to S, so S stays intact for the next iteration.
    tmem_st32(scol + 64, pk);
    tmem_st_wait();
    tc_fence_before();
    __syncwarp();
  }
  const unsigned long long t1 = clock64();
  if (lane == 0) out[blockIdx.x * WARPS + warp] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = l + m;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// TMEM read rate alone: each warp loads its 32 lanes x 64 columns repeatedly.
template <int WARPS, int COLS>
__global__ void __launch_bounds__(WARPS * 32, 1) tmem_ld_kernel(int iters, unsigned long long* out, float* sink) {
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(smem_u32(&tmem_slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const uint32_t col = tmem + (uint32_t((warp & 3) * 32) << 16) + 96u * uint32_t(warp >> 2);
  uint32_t accu = 0;
  __syncwarp();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t a[32];
#pragma unroll
    for (int c = 0; c < COLS / 32; ++c) {
      tmem_ld32(col + 32 * c, a);
      tmem_ld_wait();
      accu += a[0] ^ a[31];
    }
  }
  const unsigned long long t1 = clock64();
  if (lane == 0) out[blockIdx.x * WARPS + warp] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = float(accu);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int WARPS>
void run_ld() {
  const int sms = 148, iters = 4000;
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, sizeof(unsigned long long) * sms * WARPS);
  cudaMalloc(&sink, sizeof(float) * sms * WARPS * 32);
  tmem_ld_kernel<WARPS, 64><<<sms, WARPS * 32>>>(10, d, sink);
  cudaDeviceSynchronize();
  tmem_ld_kernel<WARPS, 64><<<sms, WARPS * 32>>>(iters, d, sink);
  cudaError_t err = cudaDeviceSynchronize();
  unsigned long long h[148 * 16];
  cudaMemcpy(h, d, sizeof(unsigned long long) * sms * WARPS, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms * WARPS; ++i) avg += double(h[i]);
  avg /= sms * WARPS;
  const double per = avg / iters;  // cycles per 64-column load (8 KB per warp)
  std::printf("tcgen05.ld only, warps/SM=%2d: %6.1f cycles per warp-load of 8 KB -> %6.1f B/clk per SM  %s\n", WARPS,
              per, 8192.0 * WARPS / per, cudaGetErrorString(err));
  cudaFree(d);
  cudaFree(sink);
}


// Column split: two warps share one lane quarter, each takes 32 of the 64
// columns, and they exchange their partial row max through shared memory and
// a 64-thread named barrier per tile.  WARPS softmax warps per SM.
template <int WARPS, int PN = poly_pairs<64>()>
__global__ void __launch_bounds__(WARPS * 32, 1) softmax_split_kernel(int iters, float scale_log2,
                                                                       unsigned long long* out, float* sink) {
  __shared__ uint32_t tmem_slot;
  __shared__ float xm[2][WARPS / 2][2][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(smem_u32(&tmem_slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const int quarter = warp & 3, half = (warp >> 2) & 1, slice = warp >> 3;
  const int pair = quarter + 4 * slice;
  const uint32_t lane_off = uint32_t(quarter * 32) << 16;
  const uint32_t scol = tmem + lane_off + 96u * uint32_t(slice) + 32u * half;
  {
    uint32_t init[32];
    for (int i = 0; i < 32; ++i) init[i] = __float_as_uint(0.01f * float((lane * 7 + i * 13 + half * 5) % 97) - 0.3f);
    tmem_st32(scol, init);
    tmem_st_wait();
  }
  float m = -INFINITY, l = 0.f;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t sa[32];
    tmem_ld32(scol, sa);
    tmem_ld_wait();
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(sa[i]);
    float mx[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      mx[a] = fmax3f(v[8 * a], v[8 * a + 1], v[8 * a + 2]);
      mx[a] = fmax3f(mx[a], v[8 * a + 3], v[8 * a + 4]);
      mx[a] = fmax3f(mx[a], v[8 * a + 5], v[8 * a + 6]);
      mx[a] = fmaxf(mx[a], v[8 * a + 7]);
    }
    float pm = fmaxf(fmax3f(mx[0], mx[1], mx[2]), mx[3]);
    xm[it & 1][pair][half][lane] = pm;
    named_bar_sync(1 + pair, 64);
    pm = fmaxf(pm, xm[it & 1][pair][half ^ 1][lane]);
    const float mt2 = pm * scale_log2;
    if (mt2 > m + kRescaleThreshold) {
      l *= fast_exp2(m - mt2);
      m = mt2;
    }
    const float2 sc2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-m, -m);
    float2 acc2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float2 x = __ffma2_rn(make_float2(v[2 * i], v[2 * i + 1]), sc2, nm2);
      float2 pp;
      if ((poly_mask(PN) >> (i & 7)) & 1)
        pp = exp2_poly3_pair(x);
      else
        pp = make_float2(fast_exp2(x.x), fast_exp2(x.y));
      acc2[i & 1] = __fadd2_rn(acc2[i & 1], pp);
      pk[i] = pack_bf16x2(pp.x, pp.y);
    }
    const float2 a2 = __fadd2_rn(acc2[0], acc2[1]);
    l += a2.x + a2.y;
    tmem_st16(scol + 64 - 32u * half + 16u * half, pk);
    tmem_st_wait();
    tc_fence_before();
    __syncwarp();
  }
  const unsigned long long t1 = clock64();
  if (lane == 0) out[blockIdx.x * WARPS + warp] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = l + m;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int WARPS, int PN = poly_pairs<64>()>
void run_split() {
  const int sms = 148, iters = 2000;
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, sizeof(unsigned long long) * sms * WARPS);
  cudaMalloc(&sink, sizeof(float) * sms * WARPS * 32);
  softmax_split_kernel<WARPS, PN><<<sms, WARPS * 32>>>(10, 0.18f, d, sink);
  cudaDeviceSynchronize();
  softmax_split_kernel<WARPS, PN><<<sms, WARPS * 32>>>(iters, 0.18f, d, sink);
  cudaError_t err = cudaDeviceSynchronize();
  unsigned long long h[148 * 16];
  cudaMemcpy(h, d, sizeof(unsigned long long) * sms * WARPS, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms * WARPS; ++i) avg += double(h[i]);
  avg /= sms * WARPS;
  const double per_step = avg / iters;  // cycles per half-row softmax step of one warp
  // One 128x64 tile = 8 half-warp-steps
  std::printf("column split poly %d/8 warps/SM=%2d (per SMSP %d): %7.1f cycles per warp-step, %7.1f SM cycles per 128x64 tile  %s\n",
              PN, WARPS, WARPS / 4, per_step, per_step * 8.0 / WARPS, cudaGetErrorString(err));
  cudaFree(d);
  cudaFree(sink);
}

template <int WARPS, bool NOSUM = false, int PACK = 0, int PN = poly_pairs<64>()>
void run() {
  const int sms = 148, iters = 2000;
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, sizeof(unsigned long long) * sms * WARPS);
  cudaMalloc(&sink, sizeof(float) * sms * WARPS * 32);
  softmax_kernel<WARPS, NOSUM, PACK, PN><<<sms, WARPS * 32>>>(10, 0.18f, d, sink);
  cudaDeviceSynchronize();
  softmax_kernel<WARPS, NOSUM, PACK, PN><<<sms, WARPS * 32>>>(iters, 0.18f, d, sink);
  cudaError_t err = cudaDeviceSynchronize();
  unsigned long long h[148 * 16];
  cudaMemcpy(h, d, sizeof(unsigned long long) * sms * WARPS, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms * WARPS; ++i) avg += double(h[i]);
  avg /= sms * WARPS;
  const double per_step = avg / iters;  // cycles per softmax step of one warp
  // One 128x64 tile = 4 warp-steps; SM throughput in tiles per cycle:
  const double sm_cycles_per_tile = per_step * 4.0 / WARPS;
  std::printf("poly %d/8 %s warps/SM=%2d (per SMSP %d): %7.1f cycles per warp-step, %7.1f SM cycles per 128x64 tile  %s\n",
              PN, PACK == 3 ? "spec max  " : PACK == 2 ? "f16x2 ex2 " : PACK ? "prmt pack " : NOSUM ? "no row sum" : "row sum   ", WARPS, WARPS / 4, per_step, sm_cycles_per_tile,
              cudaGetErrorString(err));
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  // exp pairs on the FMA pipe: 0, 2, 3, 4 of 8, at 2 and 4 softmax warps per SMSP
  run<8, false, 0, 0>();
  run<16, false, 0, 0>();
  run<8, false, 0, 2>();
  run<16, false, 0, 2>();
  run<8, false, 0, 3>();
  run<16, false, 0, 3>();
  run<8, false, 0, 4>();
  run<16, false, 0, 4>();
  run<8, true>();           // no row sum
  run<8, false, 1>();       // bf16 by byte permute instead of F2FP
  run<8, false, 2, 0>();    // ex2.approx.f16x2 (two exps per MUFU op)
  run<16, false, 2, 0>();
  run_ld<8>();
  run<8, false, 3, 3>();   // speculative exps (running max), max check off the critical path
  run<16, false, 3, 3>();
  run_split<16, 3>();
  run_split<16, 2>();
  run_split<8, 3>();
  return 0;
}
