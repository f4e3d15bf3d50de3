// K4: block-sparse FlashAttention forward for sm_100a (tcgen05 + TMEM + TMA).
//
// One CTA = one work item (schedule.hpp): a 128-row Q tile (two 64-row Q
// blocks of one head) against the union of their dense 64-key KV blocks.
// Warp roles (192 threads, two CTAs per SM so one CTA's softmax overlaps the
// other's MMAs):
//   warps 0-3  softmax + epilogue; thread t owns Q row t (TMEM lane t)
//   warp 4     TMA producer: Q once, then K (one tile ahead) and V per tile
//   warp 5     TMEM allocator + single-thread tcgen05.mma issuer
// Per KV tile j (S/P double-buffered in TMEM, O resident in TMEM):
//   S_j = Q K_j^T        tcgen05.mma SS, M=128 N=64 K=d   -> TMEM cols S[j&1]
//   P_j = exp2(S_j*c-m)  softmax warps, bf16, written back over S[j&1]
//   O  += P_j V_j        tcgen05.mma TS (A=P from TMEM), M=128 N=d K=64
// The online-softmax max is rescaled lazily (only when it grows by more than
// 2^8), so O in TMEM is touched by the softmax warps only on those rare steps.
// Mask semantics follow the reference BlockMask (mask.hpp:18-20): a tile is
// computed iff its bit is set; everything else contributes exactly zero.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/dbsp_b200.h"
#include "capi_util.hpp"
#include "core.hpp"
#include "ptx.cuh"
#include "schedule.hpp"

namespace dbsp_dev {

using dbsp_core::WorkItem;

enum : uint32_t { kModeAccumulate = 1, kModeFinalize = 2 };

struct AttnParams {
  const WorkItem* items;
  const uint32_t* entries;
  __nv_bfloat16* out;
  float* lse;
  float* o_acc;
  float* lse_acc;
  uint32_t q_tokens;
  uint32_t heads;
  uint32_t mode;
  float scale_log2;
  unsigned long long* trace;  // DBSP_TRACE builds only: clock64 per (block, tile, event)
};

// Event slots of the optional per-tile trace (DBSP_TRACE).
enum : int { kTrSoftStart = 0, kTrSoftEnd, kTrMmaS, kTrMmaPV, kTrSoftStartHi, kTrSoftEndHi,
             kTrLoadK, kTrLoadV, kTrEvents };
constexpr int kTraceBlocks = 16, kTraceTiles = 256;
#ifdef DBSP_TRACE
#define DBSP_TR(ev, j)                                                                         \
  do {                                                                                         \
    if (p.trace && blockIdx.x < kTraceBlocks && (j) < kTraceTiles)                             \
      p.trace[(size_t(blockIdx.x) * kTraceTiles + (j)) * kTrEvents + (ev)] = clock64();        \
  } while (0)
#else
#define DBSP_TR(ev, j) \
  do {                 \
  } while (0)
#endif

constexpr int kThreads = 192;
constexpr uint32_t kTmemCols = 256;
constexpr uint32_t kColO = 0;
constexpr uint32_t kColS0 = 128;
constexpr uint32_t kColS1 = 192;
constexpr float kRescaleThreshold = 8.0f;  // log2 domain
#ifndef DBSP_POLY_EVERY
#define DBSP_POLY_EVERY 4
#endif
constexpr int kPolyEvery = DBSP_POLY_EVERY;  // 1 in kPolyEvery exp2 pairs on the FMA pipe

template <int D>
struct KCfg {
  static constexpr int kChunks = D / 64;              // 128-byte swizzle atoms along d
  static constexpr uint32_t kQBytes = 128u * D * 2u;  // 128 rows
  static constexpr uint32_t kQChunk = 128u * 128u;    // one 64-column chunk of Q
  static constexpr uint32_t kTileBytes = 64u * D * 2u;
  static constexpr int kStages = D == 128 ? 2 : 4;
  static constexpr int kNumBars = 1 + 4 * kStages + 2 + 2 + 2;
  static constexpr uint32_t kDataBytes = kQBytes + 2u * kStages * kTileBytes;
  static constexpr uint32_t kSmemBytes = kDataBytes + 1024 + 8 * kNumBars + 16;
};

template <int D>
__global__ void __launch_bounds__(kThreads, 2)
    sparse_attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ,
                           const __grid_constant__ CUtensorMap tmK,
                           const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  using C = KCfg<D>;
  constexpr int NS = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);

  const uint32_t sQ = base;
  const uint32_t sK = sQ + C::kQBytes;
  const uint32_t sV = sK + NS * C::kTileBytes;
  const uint32_t sBar = sV + NS * C::kTileBytes;
  // Barrier slots.
  const uint32_t bQ = sBar;
  auto bKfull = [&](int s) { return sBar + 8u * (1 + s); };
  auto bVfull = [&](int s) { return sBar + 8u * (1 + NS + s); };
  auto bKempty = [&](int s) { return sBar + 8u * (1 + 2 * NS + s); };
  auto bVempty = [&](int s) { return sBar + 8u * (1 + 3 * NS + s); };
  auto bSfull = [&](int b) { return sBar + 8u * (1 + 4 * NS + b); };
  auto bPfull = [&](int b) { return sBar + 8u * (3 + 4 * NS + b); };
  const uint32_t bOdone = sBar + 8u * (5 + 4 * NS);   // one phase per PV_j
  const uint32_t bOfinal = sBar + 8u * (6 + 4 * NS);  // single phase: every PV done
  const uint32_t sTmemSlot = sBar + 8u * C::kNumBars;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const WorkItem it = p.items[blockIdx.x];
  const uint32_t count = it.count;

  if (threadIdx.x == 0) {
    mbar_init(bQ, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(bKfull(s), 1);
      mbar_init(bVfull(s), 1);
      mbar_init(bKempty(s), 1);
      mbar_init(bVempty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bSfull(b), 1);
      mbar_init(bPfull(b), 4);  // one arrive per softmax warp
    }
    mbar_init(bOdone, 1);
    mbar_init(bOfinal, 1);
    mbar_fence_init();
  }
  if (warp == 4 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
  }
  if (warp == 5) tmem_alloc(sTmemSlot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(gbase + (sTmemSlot - base));

  if (warp == 4) {
    // ------------------------------------------------------------ producer
    if (lane == 0 && count > 0) {
      const uint64_t pol_q = l2_policy_evict_first();
      const uint64_t pol_kv = l2_policy_evict_last();
      const int head = int(it.head);
      mbar_expect_tx(bQ, C::kQBytes);
      for (int c = 0; c < C::kChunks; ++c) {
        tma_load_3d(sQ + c * C::kQChunk, &tmQ, c * 64, head, int(it.qa) * 64, bQ, pol_q);
        tma_load_3d(sQ + c * C::kQChunk + 8192, &tmQ, c * 64, head, int(it.qb) * 64, bQ, pol_q);
      }
      const uint32_t* ent = p.entries + it.begin;
      auto load_tile = [&](const CUtensorMap* tm, uint32_t dst, uint32_t full, uint32_t j) {
        const int kv = int(__ldg(ent + j) & dbsp_core::kEntryKvMask);
        mbar_expect_tx(full, C::kTileBytes);
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_3d(dst + c * 8192, tm, c * 64, head, kv * 64, full, pol_kv);
      };
      auto load_k = [&](uint32_t j) {
        const int s = int(j % NS);
        mbar_wait(bKempty(s), ((j / NS) & 1) ^ 1);
        load_tile(&tmK, sK + s * C::kTileBytes, bKfull(s), j);
        DBSP_TR(kTrLoadK, j);
      };
      load_k(0);
      for (uint32_t j = 0; j < count; ++j) {
        if (j + 1 < count) load_k(j + 1);
        const int s = int(j % NS);
        mbar_wait(bVempty(s), ((j / NS) & 1) ^ 1);
        load_tile(&tmV, sV + s * C::kTileBytes, bVfull(s), j);
        DBSP_TR(kTrLoadV, j);
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0 && count > 0) {
      constexpr uint32_t kIdescQK = idesc_bf16(128, 64, false, false);
      constexpr uint32_t kIdescPV = idesc_bf16(128, D, false, true);
      auto pv = [&](uint32_t i) {
        const int b = int(i & 1);
        const int s = int(i % NS);
        mbar_wait(bPfull(b), (i >> 1) & 1);
        mbar_wait(bVfull(s), (i / NS) & 1);
        tc_fence_after();
        const uint32_t pcol = tmem + (b ? kColS1 : kColS0);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t bd = smem_desc_sw128(sV + s * C::kTileBytes + kk * 2048, 8192, 1024);
          mma_ts(tmem + kColO, pcol + kk * 8, bd, kIdescPV, (i > 0 || kk > 0) ? 1u : 0u);
        }
        tc_commit(bVempty(s));
        tc_commit(bOdone);
        DBSP_TR(kTrMmaPV, i);
      };
      mbar_wait(bQ, 0);
      tc_fence_after();
      for (uint32_t j = 0; j < count; ++j) {
        const int s = int(j % NS);
        // S_j overwrites the TMEM columns holding P_{j-2}, which PV_{j-2} (issued
        // just before) reads.  tcgen05.mma ops of one thread execute in issue
        // order, so the A-operand read precedes the later D write; measured
        // parity-identical with and without an explicit wait (DBSP_STRICT_WAR
        // re-enables it; completed PVs here are j-2 or j-1).
#ifdef DBSP_STRICT_WAR
        if (j >= 2) mbar_wait(bOdone, (j - 2) & 1);
#endif
        mbar_wait(bKfull(s), (j / NS) & 1);
        tc_fence_after();
        const uint32_t dcol = tmem + ((j & 1) ? kColS1 : kColS0);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t ad = smem_desc_sw128(sQ + (kk >> 2) * C::kQChunk + (kk & 3) * 32, 16, 1024);
          const uint64_t bd =
              smem_desc_sw128(sK + s * C::kTileBytes + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
          mma_ss(dcol, ad, bd, kIdescQK, kk > 0 ? 1u : 0u);
        }
        tc_commit(bKempty(s));
        tc_commit(bSfull(int(j & 1)));
        DBSP_TR(kTrMmaS, j);
        if (j > 0) pv(j - 1);
      }
      pv(count - 1);
      tc_commit(bOfinal);
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ softmax
    const int row = threadIdx.x;  // 0..127 == TMEM lane
    const bool upper = row >= 64;
    const uint32_t lane_off = uint32_t(warp * 32) << 16;
    const uint32_t dense_bit = upper ? dbsp_core::kEntryDenseB : dbsp_core::kEntryDenseA;
    const float sl2 = p.scale_log2;
    const uint32_t* ent = p.entries + it.begin;
    float m = -INFINITY, l = 0.f;
    for (uint32_t j = 0; j < count; ++j) {
      const uint32_t e = __ldg(ent + j);
      const bool dense = (e & dense_bit) != 0;  // warp-uniform (one half per warp)
      const uint32_t scol = tmem + lane_off + ((j & 1) ? kColS1 : kColS0);
      mbar_wait(bSfull(int(j & 1)), (j >> 1) & 1);
      if (lane == 0 && (warp == 0 || warp == 2)) DBSP_TR(warp == 0 ? kTrSoftStart : kTrSoftStartHi, j);
      tc_fence_after();
      uint32_t pk[32];
      if (dense) {
        uint32_t sa[32], sb[32];
        tmem_ld32(scol, sa);
        tmem_ld32(scol + 32, sb);
        tmem_ld_wait();
        const uint32_t valid = ((e >> dbsp_core::kEntryValidShift) & 63u) + 1u;
        float v[64];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          v[i] = __uint_as_float(sa[i]);
          v[i + 32] = __uint_as_float(sb[i]);
        }
        if (valid < 64) {  // partial last KV block (warp-uniform)
#pragma unroll
          for (int i = 0; i < 64; ++i)
            if (uint32_t(i) >= valid) v[i] = -INFINITY;
        }
        // Row max as a 3-input-max tree (FMNMX3): depth 5 instead of a 64-long chain.
        float mx[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          mx[a] = fmax3f(v[8 * a], v[8 * a + 1], v[8 * a + 2]);
          mx[a] = fmax3f(mx[a], v[8 * a + 3], v[8 * a + 4]);
          mx[a] = fmax3f(mx[a], v[8 * a + 5], v[8 * a + 6]);
          mx[a] = fmaxf(mx[a], v[8 * a + 7]);
        }
        const float mt = fmaxf(fmax3f(mx[0], mx[1], mx[2]),
                               fmax3f(fmax3f(mx[3], mx[4], mx[5]), mx[6], mx[7]));
        const float mt2 = mt * sl2;
        const bool resc = mt2 > m + kRescaleThreshold;
        const bool need_o = resc && (m != -INFINITY);
        float alpha = 1.f;
        if (resc) {
          alpha = fast_exp2(m - mt2);
          l *= alpha;
          m = mt2;
        }
        if (__any_sync(0xffffffffu, need_o)) {
          if (j > 0) {
            mbar_wait(bOdone, (j - 1) & 1);
            tc_fence_after();
          }
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            tmem_ld32(tmem + lane_off + kColO + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(tmem + lane_off + kColO + c * 32, o);
          }
        }
        // exp2 split between the MUFU (ex2.approx) and a degree-3 polynomial
        // on the FMA pipe for every kPolyEvery-th pair (FA4-style offload:
        // MUFU is 16/clk/SM, the FMA pipe is otherwise idle here).
        const float negm = -m;
        float sum4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float x0 = fmaf(v[2 * i], sl2, negm);
          const float x1 = fmaf(v[2 * i + 1], sl2, negm);
          float p0, p1;
          if ((i % kPolyEvery) == kPolyEvery - 1) {
            p0 = exp2_poly3(x0);
            p1 = exp2_poly3(x1);
          } else {
            p0 = fast_exp2(x0);
            p1 = fast_exp2(x1);
          }
          sum4[i & 3] += p0 + p1;
          pk[i] = pack_bf16x2(p0, p1);
        }
        l += (sum4[0] + sum4[1]) + (sum4[2] + sum4[3]);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) pk[i] = 0u;
      }
      tmem_st32(scol, pk);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bPfull(int(j & 1)));
      if (lane == 0 && (warp == 0 || warp == 2)) DBSP_TR(warp == 0 ? kTrSoftEnd : kTrSoftEndHi, j);
    }

    // ------------------------------------------------------------ epilogue
    if (count > 0) {
      // Not bOdone: up to two PV phases may still be outstanding here, and a
      // parity wait cannot tell phase count-1 from phase count-3.
      mbar_wait(bOfinal, 0);
      tc_fence_after();
    }
    const uint32_t qblk = upper ? it.qb : it.qa;
    const uint32_t token = qblk * 64u + uint32_t(row & 63);
    const bool live = !(upper && it.single) && token < p.q_tokens;
    const float inv_l = l > 0.f ? 1.f / l : 0.f;
    const float kLn2 = 0.6931471805599453f;
    const float lse_new = l > 0.f ? (m + log2f(l)) * kLn2 : -INFINITY;
    const size_t orow = (size_t(token) * p.heads + it.head) * D;
    const size_t lidx = size_t(it.head) * p.q_tokens + token;

    float c_old = 0.f, c_new = inv_l, lse_out = lse_new;
    const bool acc = (p.mode & kModeAccumulate) != 0;
    if (acc) {
      const float lse_old = live ? p.lse_acc[lidx] : -INFINITY;
      const float mx = fmaxf(lse_old, lse_new);
      if (mx == -INFINITY) {
        c_old = 0.f;
        c_new = 0.f;
        lse_out = -INFINITY;
      } else {
        const float w_old = __expf(lse_old - mx);
        const float w_new = __expf(lse_new - mx);
        const float den = w_old + w_new;
        c_old = w_old / den;
        c_new = w_new * inv_l / den;
        lse_out = mx + __logf(den);
      }
    }
    const bool write_bf16 = !acc || (p.mode & kModeFinalize);
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      uint32_t o[32];
      if (count > 0) {
        tmem_ld32(tmem + lane_off + kColO + c * 32, o);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) o[i] = 0u;
      }
      if (!live) continue;
      float r[32];
      if (acc) {
        float4* pa = reinterpret_cast<float4*>(p.o_acc + orow + c * 32);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float4 a = pa[i];
          a.x = a.x * c_old + __uint_as_float(o[4 * i + 0]) * c_new;
          a.y = a.y * c_old + __uint_as_float(o[4 * i + 1]) * c_new;
          a.z = a.z * c_old + __uint_as_float(o[4 * i + 2]) * c_new;
          a.w = a.w * c_old + __uint_as_float(o[4 * i + 3]) * c_new;
          pa[i] = a;
          r[4 * i + 0] = a.x;
          r[4 * i + 1] = a.y;
          r[4 * i + 2] = a.z;
          r[4 * i + 3] = a.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = __uint_as_float(o[i]) * inv_l;
      }
      if (write_bf16) {
        uint4* po = reinterpret_cast<uint4*>(p.out + orow + c * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          po[i] = make_uint4(pack_bf16x2(r[8 * i + 0], r[8 * i + 1]),
                             pack_bf16x2(r[8 * i + 2], r[8 * i + 3]),
                             pack_bf16x2(r[8 * i + 4], r[8 * i + 5]),
                             pack_bf16x2(r[8 * i + 6], r[8 * i + 7]));
      }
    }
    if (live) {
      if (acc)
        p.lse_acc[lidx] = lse_out;
      else if (p.lse)
        p.lse[lidx] = lse_new;
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 5) tmem_dealloc(tmem, kTmemCols);
}

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

// =====================================================================
// Host side
// =====================================================================
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

// [tokens, heads, d] bf16, box = 64 tokens x 1 head x 64 columns, 128B swizzle.
CUtensorMap make_tmap(const void* ptr, uint32_t tokens, uint32_t heads, uint32_t d) {
  CUtensorMap m;
  const cuuint64_t dims[3] = {d, heads, tokens};
  const cuuint64_t strides[2] = {cuuint64_t(d) * 2, cuuint64_t(heads) * d * 2};
  const cuuint32_t box[3] = {64, 1, 64};
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
                   const dbsp_dev::AttnParams& prm, uint32_t items, cudaStream_t stream) {
  using C = dbsp_dev::KCfg<D>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(dbsp_dev::sparse_attn_fwd_kernel<D>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
  });
  cuda_check(attr_err, "cudaFuncSetAttribute");
  dbsp_dev::sparse_attn_fwd_kernel<D>
      <<<items, dbsp_dev::kThreads, C::kSmemBytes, stream>>>(q, k, v, prm);
  cuda_check(cudaGetLastError(), "sparse_attn_fwd launch");
}

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

  ~dbsp_schedule() {
    if (pending && uploaded) cudaEventSynchronize(uploaded);
    if (dev) cudaFree(dev);
    if (pinned) cudaFreeHost(pinned);
    if (uploaded) cudaEventDestroy(uploaded);
  }
};

using dbsp_capi::guard;

namespace {

unsigned long long* g_trace = nullptr;

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

int dbsp_schedule_create(dbsp_schedule** out) {
  return guard([&] {
    if (!out) fail(kContract, "null output");
    *out = new dbsp_schedule();
  });
}

void dbsp_schedule_destroy(dbsp_schedule* s) { delete s; }

int dbsp_schedule_build(dbsp_schedule* sched, const dbsp_mask_set* set,
                        const dbsp_local_view* view, int32_t pair_q) {
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
    build_schedule(m, lv, pair_q != 0, sched->host);
    sched->dirty = true;
  });
}

int dbsp_schedule_stats(const dbsp_schedule* s, uint64_t* items, uint64_t* visits,
                        uint64_t* dense) {
  return guard([&] {
    if (!s) fail(kContract, "null schedule");
    if (items) *items = s->host.items.size();
    if (visits) *visits = s->host.tile_visits;
    if (dense) *dense = s->host.dense_tiles;
  });
}

int dbsp_attention_launch(dbsp_schedule* sched, const dbsp_attn_args* a, void* stream_ptr) {
  return guard([&] {
    if (!sched || !a) fail(kContract, "null schedule or args");
    if (a->head_dim != 64 && a->head_dim != 128) fail(kConfig, "head_dim must be 64 or 128");
    if (!a->q || !a->k || !a->v) fail(kContract, "null q/k/v");
    if (a->q_tokens == 0 || a->kv_tokens == 0 || a->heads == 0)
      fail(kConfig, "attention dimensions must be positive");
    const bool acc = a->accumulate != 0;
    if (acc && (!a->o_accum || !a->lse_accum)) fail(kContract, "accumulate needs o_accum/lse_accum");
    if ((!acc || a->finalize) && !a->o) fail(kContract, "null output");
    cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_ptr);
    const Schedule& h = sched->host;
    if (h.items.empty()) return;
    for (const WorkItem& it : h.items)
      if (it.head >= a->heads) fail(kContract, "schedule head past the buffer");
    upload_schedule(sched, stream);
    dbsp_dev::AttnParams prm;
    prm.items = static_cast<const WorkItem*>(sched->dev);
    prm.entries =
        reinterpret_cast<const uint32_t*>(static_cast<uint8_t*>(sched->dev) + sched->item_bytes);
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
    const CUtensorMap tq = make_tmap(a->q, a->q_tokens, a->heads, a->head_dim);
    const CUtensorMap tk = make_tmap(a->k, a->kv_tokens, a->heads, a->head_dim);
    const CUtensorMap tv = make_tmap(a->v, a->kv_tokens, a->heads, a->head_dim);
    if (a->head_dim == 128)
      launch_kernel<128>(tq, tk, tv, prm, uint32_t(h.items.size()), stream);
    else
      launch_kernel<64>(tq, tk, tv, prm, uint32_t(h.items.size()), stream);
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
  const int rc = dbsp_schedule_build(sched, set, &v, 1);
  if (rc) return rc;
  return dbsp_attention_launch(sched, args, stream);
}

// Debug hook (not in the public header): device buffer of
// 16 blocks x 256 tiles x 8 events u64 clock64 stamps, used by DBSP_TRACE builds.
int dbsp_debug_set_trace(unsigned long long* dev) {
  g_trace = dev;
  return 0;
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
