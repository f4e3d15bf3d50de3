// Host side of the sm_100a attention path: TMA descriptors, schedule upload,
// launches of K4 (attn_kernel.cuh), the ring-accumulator init and K1 (exact
// mask statistics on device), all behind the C ABI of include/dbsp_b200.h.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/dbsp_b200.h"
#include <cstdlib>

#include "attn_kernel.cuh"
#include "attn_kernel_duo.cuh"
#include "attn_kernel_duo2.cuh"
#include "attn_kernel_quad.cuh"
#include "attn_kernel_quadp.cuh"
#include "attn_kernel_s32.cuh"
#include "attn_kernel_psmem.cuh"
#include "attn_kernel_pair.cuh"
#include "attn_kernel_pd.cuh"
#include "attn_kernel_pd2.cuh"
#include "attn_kernel_pd3.cuh"
#include "attn_kernel_pd4.cuh"
#include "attn_kernel_pd3p.cuh"
#include "attn_kernel_split.cuh"
#include "attn_kernel_wide.cuh"
#include "capi_util.hpp"
#include "core.hpp"
#include "schedule.hpp"

namespace dbsp_dev {

__global__ void accum_init_kernel(float* o, float* lse, size_t n_o, size_t n_lse) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_o; i += stride) o[i] = 0.f;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_lse; i += stride)
    lse[i] = -INFINITY;
}

// K1: exact per-head block counts, Q-row and KV-column marginals of the
// head-summed grid (planner.hpp:47-61, 160-167) from device mask words.
__global__ void mask_rows_kernel(const uint64_t* __restrict__ words, uint32_t heads, uint32_t nq,
                                 uint32_t wpr, unsigned long long* head_counts,
                                 unsigned long long* row_w) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= heads * nq) return;
  const uint64_t* w = words + size_t(r) * wpr;
  unsigned long long c = 0;
  for (uint32_t i = 0; i < wpr; ++i) c += __popcll(w[i]);
  if (c) {
    atomicAdd(head_counts + r / nq, c);
    atomicAdd(row_w + r % nq, c);
  }
}

__global__ void mask_cols_kernel(const uint64_t* __restrict__ words, uint32_t rows, uint32_t nk,
                                 uint32_t wpr, uint32_t rows_per_block,
                                 unsigned long long* col_w) {
  const uint32_t w = blockIdx.x;
  const uint32_t bit = threadIdx.x;  // 64 threads
  const uint32_t r0 = blockIdx.y * rows_per_block;
  const uint32_t r1 = min(rows, r0 + rows_per_block);
  unsigned long long c = 0;
  for (uint32_t r = r0; r < r1; ++r) c += (words[size_t(r) * wpr + w] >> bit) & 1ull;
  const uint32_t k = w * 64 + bit;
  if (c && k < nk) atomicAdd(col_w + k, c);
}

}  // namespace dbsp_dev

namespace {

using namespace dbsp_core;

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(kCuda, std::string(what) + ": " + cudaGetErrorString(e));
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    err = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
    if (err == cudaSuccess && q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  if (!fn) fail(kCuda, "cuTensorMapEncodeTiled unavailable: " + std::string(cudaGetErrorString(err)));
  return fn;
}

// [tokens, heads, d] bf16, box = 64 tokens x 1 head x 64 columns, 128B swizzle
// (the layout the UMMA SW128 descriptors of attn_kernel.cuh expect).
CUtensorMap make_tmap(const void* ptr, uint32_t tokens, uint32_t heads, uint32_t d,
                      uint32_t box_rows = 64) {
  CUtensorMap m;
  const cuuint64_t dims[3] = {d, heads, tokens};
  const cuuint64_t strides[2] = {cuuint64_t(d) * 2, cuuint64_t(heads) * d * 2};
  const cuuint32_t box[3] = {64, 1, box_rows};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr),
                                 dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(kCuda, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return m;
}

template <int D>
void launch_kernel(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                   const dbsp_dev::AttnParams& prm,
                   uint32_t items, cudaStream_t stream) {
  using C = dbsp_dev::KCfg<D>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(dbsp_dev::sparse_attn_fwd_kernel<D>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
  });
  cuda_check(attr_err, "cudaFuncSetAttribute");
  dbsp_dev::sparse_attn_fwd_kernel<D><<<items, dbsp_dev::kThreads, C::kSmemBytes, stream>>>(q, k, v, prm);
  cuda_check(cudaGetLastError(), "sparse_attn_fwd launch");
}

void launch_wide(const CUtensorMap& k, const CUtensorMap& v, const dbsp_dev::AttnParams& prm,
                 uint32_t items, cudaStream_t stream) {
  using C = dbsp_dev::WideCfg;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(dbsp_dev::sparse_attn_fwd_wide_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
  });
  cuda_check(attr_err, "cudaFuncSetAttribute(wide)");
  dbsp_dev::sparse_attn_fwd_wide_kernel<<<items, dbsp_dev::kThreads, C::kSmemBytes, stream>>>(k, v, prm);
  cuda_check(cudaGetLastError(), "sparse_attn_fwd_wide launch");
}

template <int D>
void launch_split(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                  const dbsp_dev::AttnParams& prm, uint32_t items, cudaStream_t stream) {
  using C = dbsp_dev::KCfg<D>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(dbsp_dev::sparse_attn_fwd_split_kernel<D>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
  });
  cuda_check(attr_err, "cudaFuncSetAttribute(split)");
  dbsp_dev::sparse_attn_fwd_split_kernel<D>
      <<<items, dbsp_dev::kThreadsSplit, C::kSmemBytes, stream>>>(q, k, v, prm);
  cuda_check(cudaGetLastError(), "sparse_attn_fwd_split launch");
}

// Softmax split across 8 warps (attn_kernel_split.cuh), opt-in (DBSP_K4_SPLIT=1):
// measured 15.2 ms vs 6.3 ms on the Wan layer (96-register cap at 640
// threads/SM spills the d=128 softmax) and 1.91 vs 1.85 ms on CogVideoX.
bool use_split() {
  static const bool split = [] {
    const char* e = std::getenv("DBSP_K4_SPLIT");
    return e && e[0] == '1';
  }();
  return split;
}

void launch_pair(const CUtensorMap& q, const CUtensorMap& k32, const CUtensorMap& v,
                 const dbsp_dev::AttnParams& prm, uint32_t items, cudaStream_t stream) {
  using C = dbsp_dev::PairCfg;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(dbsp_dev::sparse_attn_fwd_pair_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
  });
  cuda_check(attr_err, "cudaFuncSetAttribute(pair)");
  dbsp_dev::sparse_attn_fwd_pair_kernel<<<2 * items, dbsp_dev::kThreads, C::kSmemBytes, stream>>>(
      q, k32, v, prm);
  cuda_check(cudaGetLastError(), "sparse_attn_fwd_pair launch");
}

// exp2 pairs of every 8 on the FMA pipe in the CTA-pair split-KV kernels
// (DBSP_PD_POLY=0..3; default 0: attn_kernel_pd3.cuh measured 6.12 / 6.11 /
// 6.37 ms on Wan with 0 / 1 / 2 of 8, interleaved A/B, tests/ab_probe.py).
int pd_poly() {
  static const int n = [] {
    const char* e = std::getenv("DBSP_PD_POLY");
    return (e && e[0] >= '0' && e[0] <= '3') ? e[0] - '0' : 0;
  }();
  return n;
}

template <int kPoly>
void launch_pd_n(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                 const dbsp_dev::AttnParams& prm, uint32_t items, cudaStream_t stream) {
  using C = dbsp_dev::PdCfg;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(dbsp_dev::sparse_attn_fwd_pd_kernel<kPoly>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
  });
  cuda_check(attr_err, "cudaFuncSetAttribute(pd)");
  dbsp_dev::sparse_attn_fwd_pd_kernel<kPoly><<<2 * items, dbsp_dev::kThreadsPd, C::kSmemBytes, stream>>>(
      q, k, v, prm);
  cuda_check(cudaGetLastError(), "sparse_attn_fwd_pd launch");
}

template <int kPoly>
void launch_pd2_n(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                  const dbsp_dev::AttnParams& prm, uint32_t items, cudaStream_t stream) {
  using C = dbsp_dev::Pd2Cfg;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(dbsp_dev::sparse_attn_fwd_pd2_kernel<kPoly>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
  });
  cuda_check(attr_err, "cudaFuncSetAttribute(pd2)");
  dbsp_dev::sparse_attn_fwd_pd2_kernel<kPoly><<<2 * items, dbsp_dev::kThreadsPd2, C::kSmemBytes, stream>>>(
      q, k, v, prm);
  cuda_check(cudaGetLastError(), "sparse_attn_fwd_pd2 launch");
}

template <int kPoly, bool kAlt>
void launch_pd3_n(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                  const dbsp_dev::AttnParams& prm, uint32_t items, cudaStream_t stream) {
  using C = dbsp_dev::Pd3Cfg;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(dbsp_dev::sparse_attn_fwd_pd3_kernel<kPoly, kAlt>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
  });
  cuda_check(attr_err, "cudaFuncSetAttribute(pd3)");
  dbsp_dev::sparse_attn_fwd_pd3_kernel<kPoly, kAlt>
      <<<2 * items, dbsp_dev::kThreadsPd2, C::kSmemBytes, stream>>>(q, k, v, prm);
  cuda_check(cudaGetLastError(), "sparse_attn_fwd_pd3 launch");
}

// DBSP_PD_ALT=1: the two stages' exp phases strictly alternate (SmDone).
bool pd_alt() {
  static const bool v = [] {
    const char* e = std::getenv("DBSP_PD_ALT");
    return e && e[0] == '1';
  }();
  return v;
}

template <int kPoly>
void launch_pd4_n(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                  const dbsp_dev::AttnParams& prm, uint32_t items, cudaStream_t stream) {
  using C = dbsp_dev::Pd4Cfg;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(dbsp_dev::sparse_attn_fwd_pd4_kernel<kPoly>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
  });
  cuda_check(attr_err, "cudaFuncSetAttribute(pd4)");
  dbsp_dev::sparse_attn_fwd_pd4_kernel<kPoly><<<2 * items, dbsp_dev::kThreadsPd4, C::kSmemBytes, stream>>>(
      q, k, v, prm);
  cuda_check(cudaGetLastError(), "sparse_attn_fwd_pd4 launch");
}

void launch_pd3p(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                 const dbsp_dev::AttnParams& prm, uint32_t items, cudaStream_t stream) {
  using C = dbsp_dev::Pd3pCfg;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  static int sms = 148;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(dbsp_dev::sparse_attn_fwd_pd3p_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  });
  cuda_check(attr_err, "cudaFuncSetAttribute(pd3p)");
  const uint32_t clusters = std::min<uint32_t>(items, uint32_t(sms / 2));  // one persistent CTA pair per TPC
  dbsp_dev::sparse_attn_fwd_pd3p_kernel<<<2 * clusters, dbsp_dev::kThreadsPd2, C::kSmemBytes, stream>>>(
      q, k, v, prm, items);
  cuda_check(cudaGetLastError(), "sparse_attn_fwd_pd3p launch");
}

// Which CTA-pair split-KV kernel runs DBSP_SCHED_CTA_PAIR schedules
// (DBSP_PD_VARIANT): 1 one softmax warp per row (attn_kernel_pd.cuh),
// 2 two warps per row (attn_kernel_pd2.cuh), 3 two warps per row with P in
// shared memory (attn_kernel_pd3.cuh, the default).
int pd_variant() {
  static const int v = [] {
    const char* e = std::getenv("DBSP_PD_VARIANT");
    return (e && e[0] >= '1' && e[0] <= '4') ? e[0] - '0' : 3;
  }();
  return v;
}

void launch_pd(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
               const dbsp_dev::AttnParams& prm, uint32_t items, cudaStream_t stream) {
  if (pd_variant() == 4) {
    const int n = pd_poly();
    if (n == 0) launch_pd4_n<0>(q, k, v, prm, items, stream);
    else if (n == 1) launch_pd4_n<1>(q, k, v, prm, items, stream);
    else launch_pd4_n<2>(q, k, v, prm, items, stream);
    return;
  }
  if (pd_variant() == 3) {
    const int n = pd_poly();
    if (pd_alt()) {
      if (n == 0) launch_pd3_n<0, true>(q, k, v, prm, items, stream);
      else launch_pd3_n<2, true>(q, k, v, prm, items, stream);
    } else if (n == 1) {
      launch_pd3_n<1, false>(q, k, v, prm, items, stream);
    } else if (n >= 2) {
      launch_pd3_n<2, false>(q, k, v, prm, items, stream);
    } else {
      launch_pd3_n<0, false>(q, k, v, prm, items, stream);
    }
    return;
  }
  if (pd_variant() == 2) {
    switch (pd_poly()) {
      case 0: launch_pd2_n<0>(q, k, v, prm, items, stream); break;
      case 1: launch_pd2_n<1>(q, k, v, prm, items, stream); break;
      case 3: launch_pd2_n<3>(q, k, v, prm, items, stream); break;
      default: launch_pd2_n<2>(q, k, v, prm, items, stream); break;
    }
    return;
  }
  switch (pd_poly()) {
    case 0: launch_pd_n<0>(q, k, v, prm, items, stream); break;
    case 1: launch_pd_n<1>(q, k, v, prm, items, stream); break;
    case 3: launch_pd_n<3>(q, k, v, prm, items, stream); break;
    default: launch_pd_n<2>(q, k, v, prm, items, stream); break;
  }
}

template <int D>
void launch_duo(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                const dbsp_dev::AttnParams& prm, uint32_t items, cudaStream_t stream) {
  using C = dbsp_dev::DuoCfg<D>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(dbsp_dev::sparse_attn_fwd_duo_kernel<D>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
  });
  cuda_check(attr_err, "cudaFuncSetAttribute(duo)");
  dbsp_dev::sparse_attn_fwd_duo_kernel<D><<<items, dbsp_dev::kThreadsDuo, C::kSmemBytes, stream>>>(q, k, v, prm);
  cuda_check(cudaGetLastError(), "sparse_attn_fwd_duo launch");
}

template <int D>
void launch_duo2(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                 const dbsp_dev::AttnParams& prm, uint32_t items, cudaStream_t stream) {
  using C = dbsp_dev::Duo2Cfg<D>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(dbsp_dev::sparse_attn_fwd_duo2_kernel<D>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
  });
  cuda_check(attr_err, "cudaFuncSetAttribute(duo2)");
  dbsp_dev::sparse_attn_fwd_duo2_kernel<D><<<items, dbsp_dev::kThreadsDuo2, C::kSmemBytes, stream>>>(q, k, v, prm);
  cuda_check(cudaGetLastError(), "sparse_attn_fwd_duo2 launch");
}

void launch_quadp(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                  const dbsp_dev::AttnParams& prm, uint32_t items, cudaStream_t stream) {
  using C = dbsp_dev::QuadPCfg;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  static int sms = 148;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(dbsp_dev::sparse_attn_fwd_quadp_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  });
  cuda_check(attr_err, "cudaFuncSetAttribute(quadp)");
  const uint32_t grid = std::min<uint32_t>(items, uint32_t(sms));  // one persistent CTA per SM
  dbsp_dev::sparse_attn_fwd_quadp_kernel<<<grid, dbsp_dev::kThreadsQuadP, C::kSmemBytes, stream>>>(q, k, v, prm,
                                                                                                  items);
  cuda_check(cudaGetLastError(), "sparse_attn_fwd_quadp launch");
}

template <int D>
void launch_quad(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                 const dbsp_dev::AttnParams& prm, uint32_t items, cudaStream_t stream) {
  using C = dbsp_dev::QuadCfg<D>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(dbsp_dev::sparse_attn_fwd_quad_kernel<D>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
  });
  cuda_check(attr_err, "cudaFuncSetAttribute(quad)");
  dbsp_dev::sparse_attn_fwd_quad_kernel<D><<<items, dbsp_dev::kThreadsQuad, C::kSmemBytes, stream>>>(q, k, v, prm);
  cuda_check(cudaGetLastError(), "sparse_attn_fwd_quad launch");
}

// Quad schedules run the two-stage kernels (64-key steps, or 128-key steps
// with DBSP_SCHED_KEY128); DBSP_K4_PAIR=1 selects the
// CTA-pair kernel instead (d=128 only; measured 8.19 ms vs 6.34 ms for the
// pair-item kernel on the Wan layer).
bool use_pair() {
  static const bool pair = [] {
    const char* e = std::getenv("DBSP_K4_PAIR");
    return e && e[0] == '1';
  }();
  return pair;
}

void launch_s32(const CUtensorMap& k, const CUtensorMap& v, const dbsp_dev::AttnParams& prm, uint32_t items,
                cudaStream_t stream) {
  using C = dbsp_dev::S32Cfg;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(dbsp_dev::sparse_attn_fwd_s32_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
  });
  cuda_check(attr_err, "cudaFuncSetAttribute(s32)");
  dbsp_dev::sparse_attn_fwd_s32_kernel<<<items, dbsp_dev::kThreads, C::kSmemBytes, stream>>>(k, v, prm);
  cuda_check(cudaGetLastError(), "sparse_attn_fwd_s32 launch");
}

void launch_psmem(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v, const dbsp_dev::AttnParams& prm,
                  uint32_t items, cudaStream_t stream) {
  using C = dbsp_dev::PsmemCfg;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(dbsp_dev::sparse_attn_fwd_psmem_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
  });
  cuda_check(attr_err, "cudaFuncSetAttribute(psmem)");
  dbsp_dev::sparse_attn_fwd_psmem_kernel<<<items, dbsp_dev::kThreads, C::kSmemBytes, stream>>>(q, k, v, prm);
  cuda_check(cudaGetLastError(), "sparse_attn_fwd_psmem launch");
}

// d=128 with P staged in smem (attn_kernel_psmem.cuh), opt-in.
bool use_psmem() {
  static const bool on = [] {
    const char* e = std::getenv("DBSP_K4_PSMEM");
    return e && e[0] == '1';
  }();
  return on;
}

// d=128 with Q in TMEM and 32-key sub-steps (attn_kernel_s32.cuh), opt-in.
bool use_s32() {
  static const bool s32 = [] {
    const char* e = std::getenv("DBSP_K4_S32");
    return e && e[0] == '1';
  }();
  return s32;
}

// d=128 kernel choice.  The 128-key-step variant (one CTA/SM) measured 6.96 ms
// vs 6.36 ms for the 64-key, two-CTAs-per-SM kernel on the Wan layer: with a
// single softmax warp per SMSP its softmax cannot hide the MMA completion
// latency.  Kept selectable (DBSP_K4_WIDE=1) for further work.
bool use_wide() {
  static const bool wide = [] {
    const char* e = std::getenv("DBSP_K4_WIDE");
    return e && e[0] == '1';
  }();
  return wide;
}

unsigned long long* g_trace = nullptr;
unsigned long long* g_clock_probe = nullptr;

}  // namespace

struct dbsp_schedule {
  Schedule host;
  bool dirty = true;  // host schedule changed since the last upload
  size_t item_bytes = 0;
  void* dev = nullptr;
  size_t dev_bytes = 0;
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  cudaEvent_t uploaded = nullptr;
  bool pending = false;
  // device-built schedule (K2): items/entries live only in `dev`
  bool on_device = false;
  uint32_t dev_items = 0;
  void* view_dev = nullptr;  // head ids, q ids, present bitmap, kv_local table
  size_t view_bytes = 0;
  void* k2_scratch = nullptr;
  size_t k2_scratch_bytes = 0;
  unsigned int* item_counter = nullptr;  // persistent kernels: zeroed before each launch

  ~dbsp_schedule() {
    if (pending && uploaded) cudaEventSynchronize(uploaded);
    if (dev) cudaFree(dev);
    if (pinned) cudaFreeHost(pinned);
    if (uploaded) cudaEventDestroy(uploaded);
    if (view_dev) cudaFree(view_dev);
    if (k2_scratch) cudaFree(k2_scratch);
    if (item_counter) cudaFree(item_counter);
  }
};

namespace dbsp_k2 {
void build(const uint64_t* d_words, uint32_t nq_global, uint32_t nk_global,
           const dbsp_core::LocalView& v, uint32_t flags, const uint32_t* d_head_ids,
           const uint32_t* d_q_ids, const uint64_t* d_present, const int32_t* d_kv_local,
           dbsp_core::WorkItem* items_out, uint32_t* entries_out, void*& scratch,
           size_t& scratch_bytes, cudaStream_t stream);
}

using dbsp_capi::guard;

namespace {

// Copies items + entries to the device through a pinned staging buffer, on
// `stream`, only when the host schedule changed since the last upload.
void upload_schedule(dbsp_schedule* sched, cudaStream_t stream) {
  if (!sched->dirty) return;
  const Schedule& h = sched->host;
  const size_t item_bytes = h.items.size() * sizeof(WorkItem);
  const size_t bytes = item_bytes + h.entries.size() * sizeof(uint32_t);
  if (!sched->uploaded)
    cuda_check(cudaEventCreateWithFlags(&sched->uploaded, cudaEventDisableTiming), "event");
  if (sched->pending) {
    cuda_check(cudaEventSynchronize(sched->uploaded), "schedule upload sync");
    sched->pending = false;
  }
  if (sched->pinned_bytes < bytes) {
    if (sched->pinned) cudaFreeHost(sched->pinned);
    sched->pinned = nullptr;
    cuda_check(cudaMallocHost(&sched->pinned, bytes), "cudaMallocHost");
    sched->pinned_bytes = bytes;
  }
  if (sched->dev_bytes < bytes) {
    if (sched->dev) cudaFree(sched->dev);
    sched->dev = nullptr;
    cuda_check(cudaMalloc(&sched->dev, bytes), "cudaMalloc schedule");
    sched->dev_bytes = bytes;
  }
  std::memcpy(sched->pinned, h.items.data(), item_bytes);
  if (!h.entries.empty())
    std::memcpy(static_cast<uint8_t*>(sched->pinned) + item_bytes, h.entries.data(),
                h.entries.size() * sizeof(uint32_t));
  cuda_check(cudaMemcpyAsync(sched->dev, sched->pinned, bytes, cudaMemcpyHostToDevice, stream),
             "schedule upload");
  cuda_check(cudaEventRecord(sched->uploaded, stream), "event record");
  sched->pending = true;
  sched->item_bytes = item_bytes;
  sched->dirty = false;
}

}  // namespace

extern "C" {

int dbsp_schedule_create(dbsp_schedule** out) {
  return guard([&] {
    if (!out) fail(kContract, "null output");
    *out = new dbsp_schedule();
  });
}

void dbsp_schedule_destroy(dbsp_schedule* s) { delete s; }

int dbsp_schedule_build(dbsp_schedule* sched, const dbsp_mask_set* set,
                        const dbsp_local_view* view, int32_t flags) {
  return guard([&] {
    if (!sched || !set) fail(kContract, "null schedule or mask set");
    const MaskView m =
        make_view(set->heads, set->num_heads, set->num_q_blocks, set->num_kv_blocks, set->block_size);
    LocalView lv;
    if (view) {
      lv.heads = view->num_heads;
      lv.head_ids = view->head_ids;
      lv.q_blocks = view->num_q_blocks;
      lv.q_ids = view->q_block_ids;
      lv.kv_blocks = view->num_kv_blocks;
      lv.kv_ids = view->kv_block_ids;
      lv.kv_tokens_global = view->kv_tokens_global;
    } else {
      lv.heads = m.H;
      lv.q_blocks = m.nq;
      lv.kv_blocks = m.nk;
    }
    build_schedule(m, lv, uint32_t(flags), sched->host);
    sched->dirty = true;
    sched->on_device = false;
  });
}

int dbsp_schedule_build_device(dbsp_schedule* sched, const uint64_t* d_words, uint32_t heads,
                               uint32_t q_blocks, uint32_t kv_blocks, const dbsp_local_view* view,
                               int32_t flags, void* stream_ptr) {
  return guard([&] {
    if (!sched || !d_words) fail(kContract, "null schedule or mask words");
    if (heads == 0 || q_blocks == 0 || kv_blocks == 0) fail(kConfig, "mask dimensions must be positive");
    cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_ptr);
    LocalView lv;
    lv.heads = view ? view->num_heads : heads;
    lv.q_blocks = view ? view->num_q_blocks : q_blocks;
    lv.kv_blocks = view ? view->num_kv_blocks : kv_blocks;
    lv.kv_tokens_global = view ? view->kv_tokens_global : 0;
    if (lv.heads == 0 || lv.q_blocks == 0 || lv.kv_blocks == 0)
      fail(kConfig, "local view dimensions must be positive");
    const uint32_t wpr = (kv_blocks + 63) / 64;
    // Host-side view tables (small), uploaded with the build.
    std::vector<uint32_t> hid(lv.heads), qid(lv.q_blocks);
    std::vector<uint64_t> present(wpr, 0);
    std::vector<int32_t> kvl(kv_blocks, -1);
    for (uint32_t i = 0; i < lv.heads; ++i) {
      hid[i] = view && view->head_ids ? view->head_ids[i] : i;
      if (hid[i] >= heads) fail(kContract, "local head maps past the mask set");
    }
    for (uint32_t i = 0; i < lv.q_blocks; ++i) {
      qid[i] = view && view->q_block_ids ? view->q_block_ids[i] : i;
      if (qid[i] >= q_blocks) fail(kContract, "local Q block maps past the mask grid");
    }
    for (uint32_t i = 0; i < lv.kv_blocks; ++i) {
      const uint32_t k = view && view->kv_block_ids ? view->kv_block_ids[i] : i;
      if (k >= kv_blocks) fail(kContract, "local KV block maps past the mask grid");
      if (kvl[k] >= 0) fail(kContract, "KV block listed twice in the local view");
      kvl[k] = int32_t(i);
      present[k / 64] |= 1ull << (k % 64);
    }
    const size_t vb = hid.size() * 4 + qid.size() * 4 + present.size() * 8 + kvl.size() * 4 + 64;
    if (sched->view_bytes < vb) {
      if (sched->view_dev) cudaFree(sched->view_dev);
      sched->view_dev = nullptr;
      cuda_check(cudaMalloc(&sched->view_dev, vb), "cudaMalloc view");
      sched->view_bytes = vb;
    }
    uint8_t* vd = static_cast<uint8_t*>(sched->view_dev);
    uint64_t* d_present = reinterpret_cast<uint64_t*>(vd);  // 8-byte aligned first
    uint32_t* d_hid = reinterpret_cast<uint32_t*>(vd + present.size() * 8);
    uint32_t* d_qid = d_hid + hid.size();
    int32_t* d_kvl = reinterpret_cast<int32_t*>(d_qid + qid.size());
    cuda_check(cudaMemcpyAsync(d_present, present.data(), present.size() * 8, cudaMemcpyHostToDevice, stream), "view");
    cuda_check(cudaMemcpyAsync(d_hid, hid.data(), hid.size() * 4, cudaMemcpyHostToDevice, stream), "view");
    cuda_check(cudaMemcpyAsync(d_qid, qid.data(), qid.size() * 4, cudaMemcpyHostToDevice, stream), "view");
    cuda_check(cudaMemcpyAsync(d_kvl, kvl.data(), kvl.size() * 4, cudaMemcpyHostToDevice, stream), "view");
    const uint32_t step = (flags & kSchedPairQ) ? 2 : 1;
    const uint32_t n = lv.heads * ((lv.q_blocks + step - 1) / step);
    const size_t item_bytes = size_t(n) * sizeof(WorkItem);
    const size_t bytes = item_bytes + size_t(n) * lv.kv_blocks * sizeof(uint32_t);
    if (sched->pending) {
      cuda_check(cudaEventSynchronize(sched->uploaded), "schedule upload sync");
      sched->pending = false;
    }
    if (sched->dev_bytes < bytes) {
      if (sched->dev) cudaFree(sched->dev);
      sched->dev = nullptr;
      cuda_check(cudaMalloc(&sched->dev, bytes), "cudaMalloc schedule");
      sched->dev_bytes = bytes;
    }
    dbsp_k2::build(d_words, q_blocks, kv_blocks, lv, uint32_t(flags), d_hid, d_qid, d_present, d_kvl,
                   static_cast<WorkItem*>(sched->dev),
                   reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(sched->dev) + item_bytes),
                   sched->k2_scratch, sched->k2_scratch_bytes, stream);
    // Bounds for the launch-time checks; the host copy of the list is empty.
    sched->host.items.clear();
    sched->host.entries.clear();
    sched->host.tile_visits = sched->host.dense_tiles = 0;
    sched->host.max_head = lv.heads - 1;
    sched->host.max_q_block = lv.q_blocks - 1;
    sched->host.max_kv_block = lv.kv_blocks - 1;
    sched->on_device = true;
    sched->dirty = false;
    sched->dev_items = n;
    sched->item_bytes = item_bytes;
  });
}

int dbsp_schedule_stats(const dbsp_schedule* s, uint64_t* items, uint64_t* visits,
                        uint64_t* dense) {
  return guard([&] {
    if (!s) fail(kContract, "null schedule");
    if (!s->on_device) {
      if (items) *items = s->host.items.size();
      if (visits) *visits = s->host.tile_visits;
      if (dense) *dense = s->host.dense_tiles;
      return;
    }
    // Device-built: read the list back (synchronous; diagnostics only).
    cuda_check(cudaDeviceSynchronize(), "sync");
    std::vector<WorkItem> it(s->dev_items);
    cuda_check(cudaMemcpy(it.data(), s->dev, it.size() * sizeof(WorkItem), cudaMemcpyDeviceToHost), "d2h");
    uint64_t n = 0;
    for (const WorkItem& w : it) n += w.count;
    std::vector<uint32_t> e(n);
    if (n)
      cuda_check(cudaMemcpy(e.data(), static_cast<uint8_t*>(s->dev) + s->item_bytes, n * 4,
                            cudaMemcpyDeviceToHost), "d2h");
    uint64_t dn = 0;
    for (uint32_t x : e) dn += ((x & kEntryDenseA) != 0) + ((x & kEntryDenseB) != 0);
    if (items) *items = s->dev_items;
    if (visits) *visits = n;
    if (dense) *dense = dn;
  });
}

int dbsp_schedule_layout(const dbsp_schedule* s, uint32_t* flags) {
  return guard([&] {
    if (!s || !flags) fail(kContract, "null argument");
    *flags = s->on_device ? uint32_t(kSchedPairQ) : s->host.flags;  // K2 builds pair schedules
  });
}

int dbsp_schedule_download(const dbsp_schedule* s, void* items_out, uint32_t* entries_out,
                           uint64_t max_entries) {
  return guard([&] {
    if (!s || !items_out) fail(kContract, "null argument");
    if (!s->on_device) {
      std::memcpy(items_out, s->host.items.data(), s->host.items.size() * sizeof(WorkItem));
      if (s->host.entries.size() > max_entries) fail(kContract, "entries buffer too small");
      if (entries_out) std::memcpy(entries_out, s->host.entries.data(), s->host.entries.size() * 4);
      return;
    }
    cuda_check(cudaDeviceSynchronize(), "sync");
    cuda_check(cudaMemcpy(items_out, s->dev, size_t(s->dev_items) * sizeof(WorkItem), cudaMemcpyDeviceToHost), "d2h");
    uint64_t n = 0;
    for (uint32_t i = 0; i < s->dev_items; ++i) n += static_cast<const WorkItem*>(items_out)[i].count;
    if (n > max_entries) fail(kContract, "entries buffer too small");
    if (entries_out && n)
      cuda_check(cudaMemcpy(entries_out, static_cast<uint8_t*>(s->dev) + s->item_bytes, n * 4,
                            cudaMemcpyDeviceToHost), "d2h");
  });
}

int dbsp_schedule_upload(dbsp_schedule* sched, void* stream) {
  return guard([&] {
    if (!sched) fail(kContract, "null schedule");
    upload_schedule(sched, reinterpret_cast<cudaStream_t>(stream));
  });
}

int dbsp_schedule_upload_bytes(const dbsp_schedule* s, uint64_t* bytes) {
  return guard([&] {
    if (!s || !bytes) fail(kContract, "null argument");
    *bytes = s->host.items.size() * sizeof(WorkItem) + s->host.entries.size() * sizeof(uint32_t);
  });
}

namespace {
void attention_launch(dbsp_schedule* sched, const dbsp_attn_args* a, const dbsp_out_scatter* sc,
                      void* stream_ptr) {
  {
    if (!sched || !a) fail(kContract, "null schedule or args");
    if (a->head_dim != 64 && a->head_dim != 128) fail(kConfig, "head_dim must be 64 or 128");
    if (!a->q || !a->k || !a->v) fail(kContract, "null q/k/v");
    if (a->q_tokens == 0 || a->kv_tokens == 0 || a->heads == 0)
      fail(kConfig, "attention dimensions must be positive");
    if (reinterpret_cast<uintptr_t>(a->q) % 16) fail(kContract, "q must be 16-byte aligned");
    const bool acc = a->accumulate != 0;
    if (acc && (!a->o_accum || !a->lse_accum)) fail(kContract, "accumulate needs o_accum/lse_accum");
    if ((!acc || a->finalize) && !a->o && !sc) fail(kContract, "null output");
    if (sc && (!sc->out_peers || !sc->q_block_map || !sc->head_map || sc->out_heads == 0))
      fail(kContract, "incomplete output scatter");
    cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_ptr);
    const Schedule& h = sched->host;
    const uint32_t n_items = sched->on_device ? sched->dev_items : uint32_t(h.items.size());
    if (n_items == 0) return;
    const uint32_t q_blocks = (a->q_tokens + 63) / 64, kv_blocks = (a->kv_tokens + 63) / 64;
    if (h.max_head >= a->heads || h.max_q_block >= q_blocks)
      fail(kContract, "schedule addresses past the Q buffer");
    if ((sched->on_device || !h.entries.empty()) && h.max_kv_block >= kv_blocks)
      fail(kContract, "schedule addresses past the K/V buffers");
    if (!sched->on_device) upload_schedule(sched, stream);

    dbsp_dev::AttnParams prm;
    prm.items = static_cast<const WorkItem*>(sched->dev);
    prm.entries =
        reinterpret_cast<const uint32_t*>(static_cast<uint8_t*>(sched->dev) + sched->item_bytes);
    prm.q = static_cast<const __nv_bfloat16*>(a->q);
    prm.out = static_cast<__nv_bfloat16*>(a->o);
    prm.lse = a->lse;
    prm.o_acc = a->o_accum;
    prm.lse_acc = a->lse_accum;
    prm.q_tokens = a->q_tokens;
    prm.heads = a->heads;
    prm.mode = (acc ? dbsp_dev::kModeAccumulate : 0u) | (a->finalize ? dbsp_dev::kModeFinalize : 0u);
    const float scale = a->softmax_scale > 0.f ? a->softmax_scale : 1.0f / std::sqrt(float(a->head_dim));
    prm.scale_log2 = scale * 1.4426950408889634f;
    prm.trace = g_trace;
    prm.clock_probe = g_clock_probe;
    prm.out_peers = sc ? reinterpret_cast<__nv_bfloat16* const*>(sc->out_peers) : nullptr;
    prm.scatter_rows = sc ? sc->q_block_map : nullptr;
    prm.scatter_heads = sc ? sc->head_map : nullptr;
    prm.out_heads = sc ? sc->out_heads : 0;
    prm.item_counter = nullptr;
    const CUtensorMap tq = make_tmap(a->q, a->q_tokens, a->heads, a->head_dim);
    const CUtensorMap tk = make_tmap(a->k, a->kv_tokens, a->heads, a->head_dim);
    const CUtensorMap tv = make_tmap(a->v, a->kv_tokens, a->heads, a->head_dim);
    const bool quad = !sched->on_device && (h.flags & kSchedQuad);
    if (quad && use_pair() && a->head_dim != 128) fail(kConfig, "the CTA-pair kernel needs head_dim 128");
    if (sc && ((quad && use_pair()) || (!quad && (use_wide() || use_split()))))
      fail(kConfig, "the fused O return is not available in the opt-in pair/wide/split kernels");
    if (quad && use_pair())
      launch_pair(tq, make_tmap(a->k, a->kv_tokens, a->heads, a->head_dim, 32), tv, prm, n_items, stream);
    else if (quad && (h.flags & kSchedKey128) && (h.flags & kSchedCtaPair)) {
      if (a->head_dim != 128) fail(kConfig, "the CTA-pair split-KV kernel needs head_dim 128");
      if (h.flags & kSchedPersist) {
        if (!sched->item_counter)
          cuda_check(cudaMalloc(&sched->item_counter, sizeof(unsigned int)), "cudaMalloc item counter");
        cuda_check(cudaMemsetAsync(sched->item_counter, 0, sizeof(unsigned int), stream), "memset item counter");
        prm.item_counter = sched->item_counter;
        launch_pd3p(tq, tk, tv, prm, n_items, stream);
      } else {
        launch_pd(tq, tk, tv, prm, n_items, stream);
      }
    } else if (quad && (h.flags & kSchedKey128) && (h.flags & kSchedSplitSoftmax)) {
      if (a->head_dim == 128)
        launch_duo2<128>(tq, tk, tv, prm, n_items, stream);
      else
        launch_duo2<64>(tq, tk, tv, prm, n_items, stream);
    } else if (quad && (h.flags & kSchedKey128) && a->head_dim == 128)
      launch_duo<128>(tq, tk, tv, prm, n_items, stream);
    else if (quad && (h.flags & kSchedKey128))
      launch_duo<64>(tq, tk, tv, prm, n_items, stream);
    else if (quad && (h.flags & kSchedPersist) && a->head_dim == 128) {
      if (!sched->item_counter)
        cuda_check(cudaMalloc(&sched->item_counter, sizeof(unsigned int)), "cudaMalloc item counter");
      cuda_check(cudaMemsetAsync(sched->item_counter, 0, sizeof(unsigned int), stream), "memset item counter");
      prm.item_counter = sched->item_counter;
      launch_quadp(tq, tk, tv, prm, n_items, stream);
    }
    else if (quad && a->head_dim == 128)
      launch_quad<128>(tq, tk, tv, prm, n_items, stream);
    else if (quad)
      launch_quad<64>(tq, tk, tv, prm, n_items, stream);
    else if (a->head_dim == 128 && use_psmem())
      launch_psmem(tq, tk, tv, prm, n_items, stream);
    else if (a->head_dim == 128 && use_s32())
      launch_s32(tk, tv, prm, n_items, stream);
    else if (a->head_dim == 128 && use_wide())
      launch_wide(tk, tv, prm, n_items, stream);
    else if (use_split() && a->head_dim == 128)
      launch_split<128>(tq, tk, tv, prm, n_items, stream);
    else if (use_split())
      launch_split<64>(tq, tk, tv, prm, n_items, stream);
    else if (a->head_dim == 128)
      launch_kernel<128>(tq, tk, tv, prm, n_items, stream);
    else
      launch_kernel<64>(tq, tk, tv, prm, n_items, stream);
  }
}
}  // namespace

int dbsp_attention_launch(dbsp_schedule* sched, const dbsp_attn_args* a, void* stream) {
  return guard([&] { attention_launch(sched, a, nullptr, stream); });
}

int dbsp_attention_launch_scatter(dbsp_schedule* sched, const dbsp_attn_args* a,
                                  const dbsp_out_scatter* sc, void* stream) {
  return guard([&] {
    if (!sc) fail(kContract, "null output scatter");
    attention_launch(sched, a, sc, stream);
  });
}

int dbsp_sparse_attention(const dbsp_mask_set* set, const dbsp_attn_args* args, void* stream) {
  static thread_local dbsp_schedule* sched = nullptr;
  if (!sched) {
    const int rc = dbsp_schedule_create(&sched);
    if (rc) return rc;
  }
  dbsp_local_view v;
  std::memset(&v, 0, sizeof(v));
  if (set) {
    v.num_heads = set->num_heads;
    v.num_q_blocks = set->num_q_blocks;
    v.num_kv_blocks = set->num_kv_blocks;
    v.kv_tokens_global = args ? args->kv_tokens : 0;
  }
  // pair schedule; for d=128 the CTA-pair kernel where its quads stay dense
  const int32_t flags = (args && args->head_dim == 128) ? (DBSP_SCHED_PAIR_Q | DBSP_SCHED_AUTO_D128) : 1;
  const int rc = dbsp_schedule_build(sched, set, &v, flags);
  if (rc) return rc;
  return dbsp_attention_launch(sched, args, stream);
}

// Debug hook (not in the public header): device buffer of 16 blocks x 256
// tiles x 8 events u64 clock64 stamps, used by DBSP_TRACE builds.
int dbsp_debug_set_trace(unsigned long long* dev) {
  g_trace = dev;
  return 0;
}

// Debug hook (not in the public header): 4 x u64 device buffer that CTA 0 of
// the default kernel fills with {clock64, globaltimer} at start and end.
int dbsp_debug_set_clock_probe(unsigned long long* dev) {
  g_clock_probe = dev;
  return 0;
}

int dbsp_copy_2d(void* dst, uint64_t dst_pitch, const void* src, uint64_t src_pitch,
                 uint64_t width, uint64_t rows, int32_t to_device, void* stream) {
  return guard([&] {
    if (!dst || !src) fail(kContract, "null pointer");
    cuda_check(cudaMemcpy2DAsync(dst, dst_pitch, src, src_pitch, width, rows,
                                 to_device ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost,
                                 reinterpret_cast<cudaStream_t>(stream)),
               "cudaMemcpy2DAsync");
  });
}

int dbsp_accum_init(float* o_accum, float* lse_accum, uint32_t q_tokens, uint32_t heads,
                    uint32_t head_dim, void* stream) {
  return guard([&] {
    if (!o_accum || !lse_accum) fail(kContract, "null accumulators");
    const size_t n_o = size_t(q_tokens) * heads * head_dim, n_l = size_t(q_tokens) * heads;
    dbsp_dev::accum_init_kernel<<<592, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        o_accum, lse_accum, n_o, n_l);
    cuda_check(cudaGetLastError(), "accum_init launch");
  });
}

int dbsp_mask_stats_device(const uint64_t* d_words, uint32_t heads, uint32_t nq, uint32_t nk,
                           uint64_t* d_head_counts, uint64_t* d_row_weights,
                           uint64_t* d_col_weights, void* stream_ptr) {
  return guard([&] {
    if (!d_words || !d_head_counts || !d_row_weights || !d_col_weights)
      fail(kContract, "null device pointer");
    if (heads == 0 || nq == 0 || nk == 0) fail(kConfig, "mask dimensions must be positive");
    cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_ptr);
    const uint32_t wpr = (nk + 63) / 64;
    cuda_check(cudaMemsetAsync(d_head_counts, 0, sizeof(uint64_t) * heads, stream), "memset");
    cuda_check(cudaMemsetAsync(d_row_weights, 0, sizeof(uint64_t) * nq, stream), "memset");
    cuda_check(cudaMemsetAsync(d_col_weights, 0, sizeof(uint64_t) * nk, stream), "memset");
    const uint32_t rows = heads * nq;
    dbsp_dev::mask_rows_kernel<<<(rows + 255) / 256, 256, 0, stream>>>(
        d_words, heads, nq, wpr, reinterpret_cast<unsigned long long*>(d_head_counts),
        reinterpret_cast<unsigned long long*>(d_row_weights));
    cuda_check(cudaGetLastError(), "mask_rows launch");
    const uint32_t rpb = 256;
    dim3 grid(wpr, (rows + rpb - 1) / rpb);
    dbsp_dev::mask_cols_kernel<<<grid, 64, 0, stream>>>(
        d_words, rows, nk, wpr, rpb, reinterpret_cast<unsigned long long*>(d_col_weights));
    cuda_check(cudaGetLastError(), "mask_cols launch");
  });
}

}  // extern "C"
