// K4, d=128 with Q in TMEM: the default kernel's structure (pair items, two
// CTAs per SM, two S buffers, one MMA issuer per CTA) with every 64-key KV
// tile processed as two 32-key sub-steps.
//
// Why: at d=128 the default kernel is bound by the shared-memory port.  Per
// 128x64 tile an SM moves Q 32 KB + K 16 KB + V 16 KB for the MMAs plus 32 KB
// of TMA writes (96 KB, 750 cycles at 128 B/clk; the trace measures 727).
// Q in TMEM (TS-mode QK^T) removes the 32 KB of Q reads, but 64 Q columns,
// two 64-column S buffers and 128 O columns exceed a CTA's 256 TMEM columns.
// With 32-key sub-steps the S buffers are 32 columns each:
//   Q [0,64)  S0 [64,96)  S1 [96,128)  O [128,256)
// and per tile the port moves 64 KB (500 cycles) against 512 cycles of MMA.
// The price is twice the barrier hand-offs per key.
// Mask semantics follow the reference BlockMask (mask.hpp:18-20).
#pragma once

#include "attn_kernel.cuh"

namespace dbsp_dev {

struct S32Cfg {
  static constexpr int D = 128;
  static constexpr uint32_t kTileBytes = 64u * D * 2u;  // one 64-key K or V tile
  static constexpr uint32_t kColQ = 0, kColS = 64, kColO = 128;
  static constexpr int kStages = 3;
  static constexpr int kNumBars = 4 * kStages + 2 * 2 + 3;
  static constexpr uint32_t kSmemBytes = 2u * kStages * kTileBytes + 1024 + 8 * kNumBars + 16;
};

__global__ void __launch_bounds__(kThreads, 2)
    sparse_attn_fwd_s32_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                               const AttnParams p) {
  using C = S32Cfg;
  constexpr int D = C::D;
  constexpr int NS = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);

  const uint32_t sK = base;
  const uint32_t sV = sK + NS * C::kTileBytes;
  const uint32_t sBar = sV + NS * C::kTileBytes;
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
  const uint32_t nsub = 2 * count;  // 32-key sub-steps
  clock_probe_mark(p, 0);

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
  if (warp == 5) tmem_alloc(sTmemSlot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(gbase + (sTmemSlot - base));
  const uint32_t* ent = p.entries + it.begin;

  if (warp == 4) {
    // ------------------------------------------------------------ producer (64-key tiles)
    if (lane == 0 && count > 0) {
      const uint64_t pol_kv = l2_policy_evict_last();
      const int head = int(it.head);
      auto load_tile = [&](const CUtensorMap* tm, uint32_t dst, uint32_t full, uint32_t j) {
        const int kv = int(__ldg(ent + j) & dbsp_core::kEntryKvMask);
        mbar_expect_tx(full, C::kTileBytes);
#pragma unroll
        for (int c = 0; c < 2; ++c) tma_load_3d(dst + c * 8192, tm, c * 64, head, kv * 64, full, pol_kv);
      };
      auto load_k = [&](uint32_t j) {
        const int s = int(j % NS);
        mbar_wait(bKempty(s), ((j / NS) & 1) ^ 1);
        load_tile(&tmK, sK + s * C::kTileBytes, bKfull(s), j);
      };
      load_k(0);
      for (uint32_t j = 0; j < count; ++j) {
        if (j + 1 < count) load_k(j + 1);
        const int s = int(j % NS);
        mbar_wait(bVempty(s), ((j / NS) & 1) ^ 1);
        load_tile(&tmV, sV + s * C::kTileBytes, bVfull(s), j);
      }
    } else if (count > 0) {
      mbar_wait(bOfinal, 0);
    }
    __syncwarp();
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer (32-key sub-steps)
    if (lane == 0 && count > 0) {
      constexpr uint32_t kIdescQK = idesc_bf16(128, 32, false, false);
      constexpr uint32_t kIdescPV = idesc_bf16(128, D, false, true);
      auto issue_s = [&](uint32_t js) {
        const uint32_t j = js >> 1, h = js & 1;
        const int s = int(j % NS);
        if (h == 0) {
          mbar_wait(bKfull(s), (j / NS) & 1);
          tc_fence_after();
        }
        const uint32_t dcol = tmem + C::kColS + 32u * (js & 1);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t bd = smem_desc_sw128(
              sK + s * C::kTileBytes + (kk >> 2) * 8192 + 4096 * h + (kk & 3) * 32, 16, 1024);
          mma_ts(dcol, tmem + C::kColQ + kk * 8, bd, kIdescQK, kk > 0 ? 1u : 0u);
        }
        tc_commit(bSfull(int(js & 1)));
        if (h == 1) tc_commit(bKempty(s));
      };
      auto issue_pv = [&](uint32_t js) {
        const uint32_t j = js >> 1, h = js & 1;
        const int s = int(j % NS);
        const int b = int(js & 1);
        mbar_wait(bPfull(b), (js >> 1) & 1);
        if (h == 0) mbar_wait(bVfull(s), (j / NS) & 1);
        tc_fence_after();
        const uint32_t pcol = tmem + C::kColS + 32u * b;
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const uint64_t bd = smem_desc_sw128(sV + s * C::kTileBytes + 4096 * h + kk * 2048, 8192, 1024);
          mma_ts(tmem + C::kColO, pcol + kk * 8, bd, kIdescPV, (js > 0 || kk > 0) ? 1u : 0u);
        }
        tc_commit(bOdone);
        if (h == 1) tc_commit(bVempty(s));
      };
      mbar_wait(bQready, 0);
      tc_fence_after();
      issue_s(0);
      issue_s(1);
      for (uint32_t js = 0; js < nsub; ++js) {
        issue_pv(js);
        if (js + 2 < nsub) issue_s(js + 2);
      }
      tc_commit(bOfinal);
    } else if (count > 0) {
      mbar_wait(bOfinal, 0);
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ Q -> TMEM, softmax, epilogue
    const int row = threadIdx.x;
    const bool upper = row >= 64;
    const uint32_t lane_off = uint32_t(warp * 32) << 16;
    const uint32_t qblk = upper ? it.qb : it.qa;
    const uint32_t token = qblk * 64u + uint32_t(row & 63);
    if (count > 0) {
      const bool in = token < p.q_tokens;
      const uint4* src = reinterpret_cast<const uint4*>(p.q + (size_t(token) * p.heads + it.head) * D);
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
    const uint32_t dense_bit = upper ? dbsp_core::kEntryDenseB : dbsp_core::kEntryDenseA;
    const float sl2 = p.scale_log2;
    const uint32_t ocol = tmem + lane_off + C::kColO;
    float m = -INFINITY, l = 0.f;
    for (uint32_t js = 0; js < nsub; ++js) {
      const uint32_t j = js >> 1, h = js & 1;
      const uint32_t e = __ldg(ent + j);
      const bool dense = (e & dense_bit) != 0;
      const int b = int(js & 1);
      const uint32_t scol = tmem + lane_off + C::kColS + 32u * b;
      mbar_wait(bSfull(b), (js >> 1) & 1);
      tc_fence_after();
      uint32_t pk[16];
      const uint32_t valid = ((e >> dbsp_core::kEntryValidShift) & 63u) + 1u;
      const int lim = int(valid) - int(32 * h);  // valid keys of this 32-key half
      if (dense && lim > 0) {
        float v[32];
        {
          uint32_t sa[32];
          tmem_ld32(scol, sa);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(sa[i]);
        }
        if (lim < 32) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (i >= lim) v[i] = -INFINITY;
        }
        float mx[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          mx[a] = fmax3f(v[8 * a], v[8 * a + 1], v[8 * a + 2]);
          mx[a] = fmax3f(mx[a], v[8 * a + 3], v[8 * a + 4]);
          mx[a] = fmax3f(mx[a], v[8 * a + 5], v[8 * a + 6]);
          mx[a] = fmaxf(mx[a], v[8 * a + 7]);
        }
        const float mt = fmaxf(fmax3f(mx[0], mx[1], mx[2]), mx[3]);
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
          // O quiescent: PV(js-1) complete (S(js) was issued after PV(js-2)).
          if (js > 0) {
            mbar_wait(bOdone, (js - 1) & 1);
            tc_fence_after();
          }
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            tmem_ld32(ocol + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(ocol + c * 32, o);
          }
        }
        const float2 sc2 = make_float2(sl2, sl2), nm2 = make_float2(-m, -m);
        float2 acc2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 x = __ffma2_rn(make_float2(v[2 * i], v[2 * i + 1]), sc2, nm2);
          const float2 pp = make_float2(fast_exp2(x.x), fast_exp2(x.y));
          acc2[i & 1] = __fadd2_rn(acc2[i & 1], pp);
          pk[i] = pack_bf16x2(pp.x, pp.y);
        }
        const float2 a2 = __fadd2_rn(acc2[0], acc2[1]);
        l += a2.x + a2.y;
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) pk[i] = 0u;
      }
      tmem_st16(scol, pk);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bPfull(b));
    }
    if (count > 0) {
      mbar_wait(bOfinal, 0);
      tc_fence_after();
    }
    finish_row<D>(p, ocol, count > 0, !(upper && it.single) && token < p.q_tokens, m, l, token, it.head);
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 5) tmem_dealloc(tmem, kTmemCols);
  clock_probe_mark(p, 1);
}

}  // namespace dbsp_dev
