// K4, d=128 variant: 128-key S tiles, one CTA per SM.
//
// Same work items and mask semantics as attn_kernel.cuh, but each step covers
// TWO dense KV blocks of the item (entries 2t and 2t+1), so
//   S_t = Q [K_a; K_b]^T    tcgen05.mma TS, M=128 N=128 K=16 x 8 (A = Q in TMEM)
//   O  += P_t [V_a; V_b]    tcgen05.mma TS, M=128 N=128 K=16 x 8 (A = P in TMEM)
// Measured on B200 (tests/mma_bench.cu): SS-mode N=64 QK^T runs at 67% of the
// tcgen05 floor (6 KB smem per 32-cycle MMA > the 128 B/clk port) while TS-mode
// N=128 runs at 100%.  With Q in TMEM the smem traffic per step is K 32 KB + V
// 32 KB reads + 64 KB of TMA writes for 1024 MMA cycles.  TMEM (512 cols, the
// whole SM): Q [0,64) bf16, O [64,192) fp32, S/P double buffer [256,384),
// [384,512) -- S_{t+1} computes while the softmax works on S_t.
#pragma once

#include "attn_kernel.cuh"

namespace dbsp_dev {

struct WideCfg {
  static constexpr int D = 128;
  static constexpr uint32_t kColQ = 0, kColO = 64, kColS = 256;  // S buffer b at kColS + 128*b
  static constexpr uint32_t kHalfBytes = 64u * 128u * 2u;          // one 64-key block, all d (16 KB)
  static constexpr uint32_t kStepBytes = 2 * kHalfBytes;           // K (or V) of one step (32 KB)
  static constexpr uint32_t kChunk = 128u * 128u;                  // 128 rows x 128 B (16 KB)
  static constexpr int kStages = 3;
  static constexpr int kNumBars = 4 * kStages + 2 + 2 + 3;
  static constexpr uint32_t kSmemBytes = 2u * kStages * kStepBytes + 1024 + 8 * kNumBars + 16;
  static constexpr uint32_t kTmemCols = 512;
};

#ifndef DBSP_WIDE_POLY_EVERY
#define DBSP_WIDE_POLY_EVERY 4
#endif

__global__ void __launch_bounds__(kThreads, 1)
    sparse_attn_fwd_wide_kernel(const __grid_constant__ CUtensorMap tmK,
                                const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  using C = WideCfg;
  constexpr int NS = C::kStages;
  constexpr int kPoly = DBSP_WIDE_POLY_EVERY;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);

  const uint32_t sK = base;
  const uint32_t sV = sK + NS * C::kStepBytes;
  const uint32_t sBar = sV + NS * C::kStepBytes;
  auto bKfull = [&](int s) { return sBar + 8u * s; };
  auto bVfull = [&](int s) { return sBar + 8u * (NS + s); };
  auto bKempty = [&](int s) { return sBar + 8u * (2 * NS + s); };
  auto bVempty = [&](int s) { return sBar + 8u * (3 * NS + s); };
  auto bSfull = [&](int b) { return sBar + 8u * (4 * NS + b); };
  auto bPfull = [&](int b) { return sBar + 8u * (4 * NS + 2 + b); };
  const uint32_t bQready = sBar + 8u * (4 * NS + 4);
  const uint32_t bOdone = sBar + 8u * (4 * NS + 5);
  const uint32_t bOfinal = sBar + 8u * (4 * NS + 6);
  const uint32_t sTmemSlot = sBar + 8u * C::kNumBars;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const WorkItem it = p.items[blockIdx.x];
  const uint32_t count = it.count;
  const uint32_t steps = (count + 1) / 2;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(bKfull(s), 1);
      mbar_init(bVfull(s), 1);
      mbar_init(bKempty(s), 1);
      mbar_init(bVempty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bSfull(b), 1);
      mbar_init(bPfull(b), 4);
    }
    mbar_init(bQready, 4);
    mbar_init(bOdone, 1);
    mbar_init(bOfinal, 1);
    mbar_fence_init();
  }
  if (warp == 4 && lane == 0) {
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
  }
  if (warp == 5) tmem_alloc(sTmemSlot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(gbase + (sTmemSlot - base));
  const uint32_t* ent = p.entries + it.begin;

  if (warp == 4) {
    // ------------------------------------------------------------ producer
    if (lane == 0 && steps > 0) {
      const uint64_t pol_kv = l2_policy_evict_last();
      const int head = int(it.head);
      // One step = up to two 64-key blocks stacked in a 128-row operand; a
      // missing second block (odd count) is loaded as a copy of the first and
      // masked out by the softmax.
      auto load_step = [&](const CUtensorMap* tm, uint32_t dst, uint32_t full, uint32_t t) {
        const int kv0 = int(__ldg(ent + 2 * t) & dbsp_core::kEntryKvMask);
        const int kv1 = 2 * t + 1 < count ? int(__ldg(ent + 2 * t + 1) & dbsp_core::kEntryKvMask) : kv0;
        mbar_expect_tx(full, C::kStepBytes);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          tma_load_3d(dst + c * C::kChunk, tm, c * 64, head, kv0 * 64, full, pol_kv);
          tma_load_3d(dst + c * C::kChunk + 8192, tm, c * 64, head, kv1 * 64, full, pol_kv);
        }
      };
      auto load_k = [&](uint32_t t) {
        const int s = int(t % NS);
        mbar_wait(bKempty(s), ((t / NS) & 1) ^ 1);
        load_step(&tmK, sK + s * C::kStepBytes, bKfull(s), t);
      };
      load_k(0);
      for (uint32_t t = 0; t < steps; ++t) {
        if (t + 1 < steps) load_k(t + 1);
        const int s = int(t % NS);
        mbar_wait(bVempty(s), ((t / NS) & 1) ^ 1);
        load_step(&tmV, sV + s * C::kStepBytes, bVfull(s), t);
      }
    } else if (steps > 0) {
      mbar_wait(bOfinal, 0);
    }
    __syncwarp();
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0 && steps > 0) {
      constexpr uint32_t kIdesc = idesc_bf16(128, 128, false, false);
      constexpr uint32_t kIdescPV = idesc_bf16(128, 128, false, true);
      auto issue_s = [&](uint32_t t) {
        const int s = int(t % NS);
        mbar_wait(bKfull(s), (t / NS) & 1);
        tc_fence_after();
        const uint32_t dcol = tmem + C::kColS + 128u * (t & 1);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t bd =
              smem_desc_sw128(sK + s * C::kStepBytes + (kk >> 2) * C::kChunk + (kk & 3) * 32, 16, 1024);
          mma_ts(dcol, tmem + C::kColQ + kk * 8, bd, kIdesc, kk > 0 ? 1u : 0u);
        }
        tc_commit(bKempty(s));
        tc_commit(bSfull(int(t & 1)));
      };
      auto issue_pv = [&](uint32_t t) {
        const int b = int(t & 1);
        const int s = int(t % NS);
        mbar_wait(bPfull(b), (t >> 1) & 1);
        mbar_wait(bVfull(s), (t / NS) & 1);
        tc_fence_after();
        const uint32_t pcol = tmem + C::kColS + 128u * b;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t bd = smem_desc_sw128(sV + s * C::kStepBytes + kk * 2048, C::kChunk, 1024);
          mma_ts(tmem + C::kColO, pcol + kk * 8, bd, kIdescPV, (t > 0 || kk > 0) ? 1u : 0u);
        }
        tc_commit(bVempty(s));
        tc_commit(bOdone);
      };
      mbar_wait(bQready, 0);
      tc_fence_after();
      issue_s(0);
      if (steps > 1) issue_s(1);
      for (uint32_t t = 0; t < steps; ++t) {
        issue_pv(t);
        if (t + 2 < steps) issue_s(t + 2);  // reuses P_t's columns after PV_t (issue order)
      }
      tc_commit(bOfinal);
    } else if (steps > 0) {
      mbar_wait(bOfinal, 0);
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ Q -> TMEM
    const int row = threadIdx.x;
    const bool upper = row >= 64;
    const uint32_t lane_off = uint32_t(warp * 32) << 16;
    const uint32_t qblk = upper ? it.qb : it.qa;
    const uint32_t token = qblk * 64u + uint32_t(row & 63);
    if (steps > 0) {
      const bool in = token < p.q_tokens;
      const uint4* src = reinterpret_cast<const uint4*>(p.q + (size_t(token) * p.heads + it.head) * 128);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t w[32];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint4 x = in ? __ldg(src + c * 8 + i) : make_uint4(0, 0, 0, 0);
          w[4 * i + 0] = x.x;
          w[4 * i + 1] = x.y;
          w[4 * i + 2] = x.z;
          w[4 * i + 3] = x.w;
        }
        tmem_st32(tmem + lane_off + C::kColQ + c * 32, w);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bQready);
    }

    // ------------------------------------------------------------ softmax
    const uint32_t dense_bit = upper ? dbsp_core::kEntryDenseB : dbsp_core::kEntryDenseA;
    const float sl2 = p.scale_log2;
    float m = -INFINITY, l = 0.f;
    for (uint32_t t = 0; t < steps; ++t) {
      const uint32_t e0 = __ldg(ent + 2 * t);
      const bool has1 = 2 * t + 1 < count;
      const uint32_t e1 = has1 ? __ldg(ent + 2 * t + 1) : 0u;
      const bool d0 = (e0 & dense_bit) != 0;           // warp-uniform
      const bool d1 = has1 && (e1 & dense_bit) != 0;
      const int b = int(t & 1);
      const uint32_t scol = tmem + lane_off + C::kColS + 128u * b;
      mbar_wait(bSfull(b), (t >> 1) & 1);
      tc_fence_after();
      uint32_t pk[64];
      if (d0 || d1) {
        float v[128];
        {
          uint32_t r[32];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            tmem_ld32(scol + c * 32, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[c * 32 + i] = __uint_as_float(r[i]);
          }
        }
        const uint32_t valid0 = d0 ? ((e0 >> dbsp_core::kEntryValidShift) & 63u) + 1u : 0u;
        const uint32_t valid1 = d1 ? ((e1 >> dbsp_core::kEntryValidShift) & 63u) + 1u : 0u;
        if (valid0 < 64) {
#pragma unroll
          for (int i = 0; i < 64; ++i)
            if (uint32_t(i) >= valid0) v[i] = -INFINITY;
        }
        if (valid1 < 64) {
#pragma unroll
          for (int i = 0; i < 64; ++i)
            if (uint32_t(i) >= valid1) v[64 + i] = -INFINITY;
        }
        float mx[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          float x = fmax3f(v[16 * a], v[16 * a + 1], v[16 * a + 2]);
#pragma unroll
          for (int i = 3; i < 15; i += 2) x = fmax3f(x, v[16 * a + i], v[16 * a + i + 1]);
          mx[a] = fmaxf(x, v[16 * a + 15]);
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
          if (t > 0) {
            mbar_wait(bOdone, (t - 1) & 1);  // completed PVs here: t-1 or t
            tc_fence_after();
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t o[32];
            tmem_ld32(tmem + lane_off + C::kColO + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(tmem + lane_off + C::kColO + c * 32, o);
          }
        }
        const float negm = -m;
        float sum4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          const float x0 = fmaf(v[2 * i], sl2, negm);
          const float x1 = fmaf(v[2 * i + 1], sl2, negm);
          float p0, p1;
          if ((i % kPoly) == kPoly - 1) {
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
        for (int i = 0; i < 64; ++i) pk[i] = 0u;
      }
      tmem_st32(scol, *reinterpret_cast<uint32_t(*)[32]>(&pk[0]));
      tmem_st32(scol + 32, *reinterpret_cast<uint32_t(*)[32]>(&pk[32]));
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bPfull(b));
    }

    // ------------------------------------------------------------ epilogue
    if (steps > 0) {
      mbar_wait(bOfinal, 0);
      tc_fence_after();
    }
    const bool live = !(upper && it.single) && token < p.q_tokens;
    const float inv_l = l > 0.f ? 1.f / l : 0.f;
    const float kLn2 = 0.6931471805599453f;
    const float lse_new = l > 0.f ? (m + log2f(l)) * kLn2 : -INFINITY;
    const size_t orow = (size_t(token) * p.heads + it.head) * 128;
    const size_t lidx = size_t(it.head) * p.q_tokens + token;
    float c_old = 0.f, c_new = inv_l, lse_out = lse_new;
    const bool acc = (p.mode & kModeAccumulate) != 0;
    if (acc) {
      const float lse_old = live ? p.lse_acc[lidx] : -INFINITY;
      const float mxl = fmaxf(lse_old, lse_new);
      if (mxl == -INFINITY) {
        c_old = 0.f;
        c_new = 0.f;
        lse_out = -INFINITY;
      } else {
        const float w_old = __expf(lse_old - mxl);
        const float w_new = __expf(lse_new - mxl);
        const float den = w_old + w_new;
        c_old = w_old / den;
        c_new = w_new * inv_l / den;
        lse_out = mxl + __logf(den);
      }
    }
    const bool write_bf16 = !acc || (p.mode & kModeFinalize);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t o[32];
      if (steps > 0) {
        tmem_ld32(tmem + lane_off + C::kColO + c * 32, o);
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
  if (warp == 5) tmem_dealloc(tmem, C::kTmemCols);
}

}  // namespace dbsp_dev
