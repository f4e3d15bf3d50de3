// K4, split-softmax variant: eight softmax warps per CTA.
//
// Same pipeline, TMEM/smem layout and work items as attn_kernel.cuh (two CTAs
// per SM, 64-key tiles, S double-buffered in TMEM), but each 128-row S tile
// is handled by two warps per 32-row lane group: warp w reads TMEM lanes
// 32*(w%4).. and columns 32*(w/4)..+31.  The row max is combined through a
// double-buffered smem slot and a 64-thread named barrier per warp pair; the
// row sums stay per half and are combined once in the epilogue; O rescale and
// the O epilogue are split by columns.  The per-tile softmax critical path
// (the quantity the clock64 trace showed the MMAs waiting on) roughly halves.
#pragma once

#include "attn_kernel.cuh"

namespace dbsp_dev {

constexpr int kThreadsSplit = 320;  // 8 softmax warps, producer (8), MMA (9)

__device__ __forceinline__ void pair_sync(int pair) {
  asm volatile("bar.sync %0, 64;" ::"r"(1 + pair) : "memory");
}

template <int D>
__global__ void __launch_bounds__(kThreadsSplit, 2)
    sparse_attn_fwd_split_kernel(const __grid_constant__ CUtensorMap tmQ,
                                 const __grid_constant__ CUtensorMap tmK,
                                 const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  using C = KCfg<D>;
  constexpr int NS = C::kStages;
  constexpr int NSB = C::kNSB;
  constexpr int kProducer = 8, kMma = 9;
  extern __shared__ uint8_t smem_raw[];
  __shared__ float red_max[2][2][128];  // [tile parity][column half][row]
  __shared__ float red_l[2][128];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);

  const uint32_t sQ = base;
  const uint32_t sK = base + C::kQBytes;
  const uint32_t sV = sK + NS * C::kTileBytes;
  const uint32_t sBar = sV + NS * C::kTileBytes;
  auto bKfull = [&](int s) { return sBar + 8u * s; };
  auto bVfull = [&](int s) { return sBar + 8u * (NS + s); };
  auto bKempty = [&](int s) { return sBar + 8u * (2 * NS + s); };
  auto bVempty = [&](int s) { return sBar + 8u * (3 * NS + s); };
  auto bSfull = [&](int b) { return sBar + 8u * (4 * NS + b); };
  auto bPfull = [&](int b) { return sBar + 8u * (4 * NS + NSB + b); };
  const uint32_t bQready = sBar + 8u * (4 * NS + 2 * NSB);
  const uint32_t bOdone = sBar + 8u * (4 * NS + 2 * NSB + 1);
  const uint32_t bOfinal = sBar + 8u * (4 * NS + 2 * NSB + 2);
  const uint32_t sTmemSlot = sBar + 8u * C::kNumBars;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const WorkItem it = p.items[blockIdx.x];
  const uint32_t count = it.count;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(bKfull(s), 1);
      mbar_init(bVfull(s), 1);
      mbar_init(bKempty(s), 1);
      mbar_init(bVempty(s), 1);
    }
    for (int b = 0; b < NSB; ++b) {
      mbar_init(bSfull(b), 1);
      mbar_init(bPfull(b), 8);
    }
    mbar_init(bQready, C::kQInTmem ? 8 : 1);
    mbar_init(bOdone, 1);
    mbar_init(bOfinal, 1);
    mbar_fence_init();
  }
  if (warp == kProducer && lane == 0) {
    if (!C::kQInTmem) tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
  }
  if (warp == kMma) tmem_alloc(sTmemSlot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(gbase + (sTmemSlot - base));

  if (warp == kProducer) {
    // ------------------------------------------------------------ producer
    if (lane == 0 && count > 0) {
      const uint64_t pol_kv = l2_policy_evict_last();
      const int head = int(it.head);
      const uint32_t* ent = p.entries + it.begin;
      if (!C::kQInTmem) {
        const uint64_t pol_q = l2_policy_evict_first();
        mbar_expect_tx(bQready, C::kQBytes);
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c) {
          tma_load_3d(sQ + c * C::kQChunk, &tmQ, c * 64, head, int(it.qa) * 64, bQready, pol_q);
          tma_load_3d(sQ + c * C::kQChunk + 8192, &tmQ, c * 64, head, int(it.qb) * 64, bQready,
                      pol_q);
        }
      }
      auto load_tile = [&](const CUtensorMap* tm, uint32_t dst, uint32_t full, uint32_t j) {
        const int kv = int(__ldg(ent + j) & dbsp_core::kEntryKvMask);
        mbar_expect_tx(full, C::kTileBytes);
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_3d(dst + c * 8192, tm, c * 64, head, kv * 64, full, pol_kv);
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
  } else if (warp == kMma) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0 && count > 0) {
      constexpr uint32_t kIdescQK = idesc_bf16(128, 64, false, false);
      constexpr uint32_t kIdescPV = idesc_bf16(128, D, false, true);
      auto issue_s = [&](uint32_t j) {
        const int s = int(j % NS);
        mbar_wait(bKfull(s), (j / NS) & 1);
        tc_fence_after();
        const uint32_t dcol = tmem + C::kColS + 64u * (j % NSB);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t bd =
              smem_desc_sw128(sK + s * C::kTileBytes + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
          if constexpr (C::kQInTmem) {
            mma_ts(dcol, tmem + C::kColQ + kk * 8, bd, kIdescQK, kk > 0 ? 1u : 0u);
          } else {
            const uint64_t ad =
                smem_desc_sw128(sQ + (kk >> 2) * C::kQChunk + (kk & 3) * 32, 16, 1024);
            mma_ss(dcol, ad, bd, kIdescQK, kk > 0 ? 1u : 0u);
          }
        }
        tc_commit(bKempty(s));
        tc_commit(bSfull(int(j % NSB)));
      };
      auto issue_pv = [&](uint32_t i) {
        const int b = int(i % NSB);
        const int s = int(i % NS);
        mbar_wait(bPfull(b), (i / NSB) & 1);
        mbar_wait(bVfull(s), (i / NS) & 1);
        tc_fence_after();
        const uint32_t pcol = tmem + C::kColS + 64u * b;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t bd = smem_desc_sw128(sV + s * C::kTileBytes + kk * 2048, 8192, 1024);
          mma_ts(tmem + C::kColO, pcol + kk * 8, bd, kIdescPV, (i > 0 || kk > 0) ? 1u : 0u);
        }
        tc_commit(bVempty(s));
        tc_commit(bOdone);
      };
      mbar_wait(bQready, 0);
      tc_fence_after();
      for (uint32_t j = 0; j < uint32_t(NSB) && j < count; ++j) issue_s(j);
      for (uint32_t j = 0; j < count; ++j) {
        issue_pv(j);
        if (j + NSB < count) issue_s(j + NSB);
      }
      tc_commit(bOfinal);
    } else if (count > 0) {
      mbar_wait(bOfinal, 0);
    }
    __syncwarp();
  } else {
    const int g = warp & 3;   // TMEM lane group
    const int ch = warp >> 2; // column half
    const int row = g * 32 + lane;
    const bool upper = row >= 64;
    const uint32_t lane_off = uint32_t(g * 32) << 16;
    const uint32_t qblk = upper ? it.qb : it.qa;
    const uint32_t token = qblk * 64u + uint32_t(row & 63);
    if (C::kQInTmem && count > 0) {
      // this warp's half of the row: D/2 bf16 = D/4 packed columns
      const bool in = token < p.q_tokens;
      const uint4* src =
          reinterpret_cast<const uint4*>(p.q + (size_t(token) * p.heads + it.head) * D + ch * (D / 2));
      uint32_t w[D / 4];
#pragma unroll
      for (int i = 0; i < D / 16; ++i) {
        const uint4 x = in ? __ldg(src + i) : make_uint4(0, 0, 0, 0);
        w[4 * i + 0] = x.x;
        w[4 * i + 1] = x.y;
        w[4 * i + 2] = x.z;
        w[4 * i + 3] = x.w;
      }
#pragma unroll
      for (int c = 0; c < D / 64; ++c) tmem_st16(tmem + lane_off + C::kColQ + ch * (D / 4) + c * 16, w + 16 * c);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bQready);
    }

    // ------------------------------------------------------------ softmax
    const uint32_t dense_bit = upper ? dbsp_core::kEntryDenseB : dbsp_core::kEntryDenseA;
    const float sl2 = p.scale_log2;
    const uint32_t* ent = p.entries + it.begin;
    float m = -INFINITY, l = 0.f;  // l: this warp's half of the row sum
    for (uint32_t j = 0; j < count; ++j) {
      const uint32_t e = __ldg(ent + j);
      const bool dense = (e & dense_bit) != 0;  // uniform across the warp pair
      const int b = int(j % NSB);
      const uint32_t scol = tmem + lane_off + C::kColS + 64u * b;
      mbar_wait(bSfull(b), (j / NSB) & 1);
      tc_fence_after();
      uint32_t pk[16];
      if (dense) {
        uint32_t sr[32];
        tmem_ld32(scol + ch * 32, sr);
        tmem_ld_wait();
        const uint32_t valid = ((e >> dbsp_core::kEntryValidShift) & 63u) + 1u;
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(sr[i]);
        if (valid < 64) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (uint32_t(ch * 32 + i) >= valid) v[i] = -INFINITY;
        }
        float mx[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          mx[a] = fmax3f(v[8 * a], v[8 * a + 1], v[8 * a + 2]);
          mx[a] = fmax3f(mx[a], v[8 * a + 3], v[8 * a + 4]);
          mx[a] = fmax3f(mx[a], v[8 * a + 5], v[8 * a + 6]);
          mx[a] = fmaxf(mx[a], v[8 * a + 7]);
        }
        red_max[j & 1][ch][row] = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
        pair_sync(g);
        const float mt = fmaxf(red_max[j & 1][0][row], red_max[j & 1][1][row]);
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
          if (NSB > 1 && j > 0) {
            mbar_wait(bOdone, (j - 1) & 1);
            tc_fence_after();
          }
#pragma unroll
          for (int c = 0; c < D / 64; ++c) {
            uint32_t o[32];
            const uint32_t oc = tmem + lane_off + C::kColO + ch * (D / 2) + c * 32;
            tmem_ld32(oc, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(oc, o);
          }
        }
        const float negm = -m;
        float s0 = 0.f, s1 = 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float p0 = fast_exp2(fmaf(v[2 * i], sl2, negm));
          const float p1 = fast_exp2(fmaf(v[2 * i + 1], sl2, negm));
          if (i & 1)
            s1 += p0 + p1;
          else
            s0 += p0 + p1;
          pk[i] = pack_bf16x2(p0, p1);
        }
        l += s0 + s1;
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) pk[i] = 0u;
      }
      tmem_st16(scol + ch * 16, pk);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bPfull(b));
    }

    // ------------------------------------------------------------ epilogue
    if (count > 0) {
      mbar_wait(bOfinal, 0);
      tc_fence_after();
    }
    const bool live = !(upper && it.single) && token < p.q_tokens;
    const size_t lidx = size_t(it.head) * p.q_tokens + token;
    const bool acc = (p.mode & kModeAccumulate) != 0;
    const float lse_old = (acc && live) ? p.lse_acc[lidx] : -INFINITY;  // read before any write
    red_l[ch][row] = l;
    pair_sync(g);
    const float lt = red_l[0][row] + red_l[1][row];
    const float inv_l = lt > 0.f ? 1.f / lt : 0.f;
    const float kLn2 = 0.6931471805599453f;
    const float lse_new = lt > 0.f ? (m + log2f(lt)) * kLn2 : -INFINITY;
    const size_t orow = (size_t(token) * p.heads + it.head) * D + ch * (D / 2);
    float c_old = 0.f, c_new = inv_l, lse_out = lse_new;
    if (acc) {
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
    for (int c = 0; c < D / 64; ++c) {
      uint32_t o[32];
      if (count > 0) {
        tmem_ld32(tmem + lane_off + C::kColO + ch * (D / 2) + c * 32, o);
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
    if (live && ch == 0) {
      if (acc)
        p.lse_acc[lidx] = lse_out;
      else if (p.lse)
        p.lse[lidx] = lse_new;
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kMma) tmem_dealloc(tmem, kTmemCols);
}

}  // namespace dbsp_dev
