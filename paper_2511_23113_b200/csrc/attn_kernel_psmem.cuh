// K4, d=128 with P staged in shared memory (SS-mode PV).
//
// The default kernel (attn_kernel.cuh) writes the bf16 P over S in TMEM, so
// the S buffer of tile j is busy until PV(j) has run, and QK^T(j+2) -- which
// reuses it -- waits behind PV(j): the softmax of j+2 then waits for S (about
// 500 of every 1450 cycles per tile in the trace).  Here the softmax warps
// release S(j) as soon as they have loaded it into registers (Sfree), write
// P(j) to a shared-memory tile in the 128-byte-swizzled K-major layout, and
// the MMA warp issues QK^T(j+2) right after Sfree(j), ahead of PV(j).
// Cost: 16 KB of P writes per tile and SS-mode PV (A = P from smem).
// Layout per CTA (two CTAs per SM): Q 32 KB | K 2x16 KB | V 2x16 KB | P 16 KB
// = 112 KB; TMEM: S0 [0,64) S1 [64,128) O [128,256).
// The K ring runs two tiles ahead of V (QK^T(j+2) precedes PV(j)).
// Mask semantics follow the reference BlockMask (mask.hpp:18-20).
#pragma once

#include "attn_kernel.cuh"

namespace dbsp_dev {

struct PsmemCfg {
  static constexpr int D = 128;
  static constexpr uint32_t kQBytes = 128u * D * 2u;
  static constexpr uint32_t kQChunk = 128u * 128u;
  static constexpr uint32_t kTileBytes = 64u * D * 2u;
  static constexpr uint32_t kPBytes = 128u * 64u * 2u;
  static constexpr int kStages = 2;
  static constexpr int kNumBars = 4 * kStages + 8;
  static constexpr uint32_t kUsed = kQBytes + 2u * kStages * kTileBytes + kPBytes + 8 * kNumBars + 16;
  // Two CTAs per SM: 2 * (dynamic + 1 KB reserved) <= 228 KB.  The layout
  // needs a 1024-byte aligned base; the slack covers a misaligned start.
  static constexpr uint32_t kSmemBytes = 115712;
  static_assert(kUsed <= kSmemBytes, "smem budget");
};

__global__ void __launch_bounds__(kThreads, 2)
    sparse_attn_fwd_psmem_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                                 const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  using C = PsmemCfg;
  constexpr int D = C::D;
  constexpr int NS = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  if (base + C::kUsed > raw + C::kSmemBytes) __trap();  // base too misaligned for the layout
  uint8_t* gbase = smem_raw + (base - raw);

  const uint32_t sQ = base;
  const uint32_t sK = sQ + C::kQBytes;
  const uint32_t sV = sK + NS * C::kTileBytes;
  const uint32_t sP = sV + NS * C::kTileBytes;
  const uint32_t sBar = sP + C::kPBytes;
  auto bKfull = [&](int s) { return sBar + 8u * s; };
  auto bVfull = [&](int s) { return sBar + 8u * (NS + s); };
  auto bKempty = [&](int s) { return sBar + 8u * (2 * NS + s); };
  auto bVempty = [&](int s) { return sBar + 8u * (3 * NS + s); };
  auto bSfull = [&](int b) { return sBar + 8u * (4 * NS + b); };
  auto bSfree = [&](int b) { return sBar + 8u * (4 * NS + 2 + b); };
  const uint32_t bPfull = sBar + 8u * (4 * NS + 4);  // one phase per tile
  const uint32_t bPfree = sBar + 8u * (4 * NS + 5);  // PV(j) done: P tile and O free
  const uint32_t bQready = sBar + 8u * (4 * NS + 6);
  const uint32_t bOfinal = sBar + 8u * (4 * NS + 7);
  const uint32_t sTmemSlot = sBar + 8u * C::kNumBars;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const WorkItem it = p.items[blockIdx.x];
  const uint32_t count = it.count;
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
      mbar_init(bSfree(b), 4);
    }
    mbar_init(bPfull, 4);
    mbar_init(bPfree, 1);
    mbar_init(bQready, 1);
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
  const uint32_t* ent = p.entries + it.begin;

  if (warp == 4) {
    // ------------------------------------------------------------ producer: Q, K two tiles ahead of V
    if (lane == 0 && count > 0) {
      const uint64_t pol_kv = l2_policy_evict_last();
      const uint64_t pol_q = l2_policy_evict_first();
      const int head = int(it.head);
      mbar_expect_tx(bQready, C::kQBytes);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        tma_load_3d(sQ + c * C::kQChunk, &tmQ, c * 64, head, int(it.qa) * 64, bQready, pol_q);
        tma_load_3d(sQ + c * C::kQChunk + 8192, &tmQ, c * 64, head, int(it.qb) * 64, bQready, pol_q);
      }
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
      for (uint32_t j = 0; j < 2 && j < count; ++j) load_k(j);
      for (uint32_t j = 0; j < count; ++j) {
        if (j + 2 < count) load_k(j + 2);
        const int s = int(j % NS);
        mbar_wait(bVempty(s), ((j / NS) & 1) ^ 1);
        load_tile(&tmV, sV + s * C::kTileBytes, bVfull(s), j);
      }
    } else if (count > 0) {
      mbar_wait(bOfinal, 0);
    }
    __syncwarp();
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0 && count > 0) {
      constexpr uint32_t kIdescQK = idesc_bf16(128, 64, false, false);
      constexpr uint32_t kIdescPV = idesc_bf16(128, D, false, true);
      auto issue_s = [&](uint32_t j) {
        const int s = int(j % NS);
        mbar_wait(bKfull(s), (j / NS) & 1);
        tc_fence_after();
        const uint32_t dcol = tmem + 64u * (j & 1);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t bd = smem_desc_sw128(sK + s * C::kTileBytes + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
          const uint64_t ad = smem_desc_sw128(sQ + (kk >> 2) * C::kQChunk + (kk & 3) * 32, 16, 1024);
          mma_ss(dcol, ad, bd, kIdescQK, kk > 0 ? 1u : 0u);
        }
        tc_commit(bKempty(s));
        tc_commit(bSfull(int(j & 1)));
      };
      auto issue_pv = [&](uint32_t j) {
        const int s = int(j % NS);
        mbar_wait(bPfull, j & 1);
        mbar_wait(bVfull(s), (j / NS) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t ad = smem_desc_sw128(sP + kk * 32, 16, 1024);
          const uint64_t bd = smem_desc_sw128(sV + s * C::kTileBytes + kk * 2048, 8192, 1024);
          mma_ss(tmem + 128, ad, bd, kIdescPV, (j > 0 || kk > 0) ? 1u : 0u);
        }
        tc_commit(bVempty(s));
        tc_commit(bPfree);
      };
      mbar_wait(bQready, 0);
      tc_fence_after();
      for (uint32_t j = 0; j < 2 && j < count; ++j) issue_s(j);
      for (uint32_t j = 0; j < count; ++j) {
        if (j + 2 < count) {  // QK^T(j+2) as soon as the softmax has read S(j)
          mbar_wait(bSfree(int(j & 1)), (j >> 1) & 1);
          issue_s(j + 2);
        }
        issue_pv(j);
      }
      tc_commit(bOfinal);
    } else if (count > 0) {
      mbar_wait(bOfinal, 0);
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ softmax + epilogue
    const int row = threadIdx.x;
    const bool upper = row >= 64;
    const uint32_t lane_off = uint32_t(warp * 32) << 16;
    const uint32_t token = (upper ? it.qb : it.qa) * 64u + uint32_t(row & 63);
    const uint32_t dense_bit = upper ? dbsp_core::kEntryDenseB : dbsp_core::kEntryDenseA;
    const float sl2 = p.scale_log2;
    const uint32_t ocol = tmem + lane_off + 128;
    uint8_t* prow = gbase + (sP - base) + row * 128;  // this row of the P tile
    float m = -INFINITY, l = 0.f;
    uint32_t e_next = count > 0 ? __ldg(ent) : 0u;
    for (uint32_t j = 0; j < count; ++j) {
      const uint32_t e = e_next;
      if (j + 1 < count) e_next = __ldg(ent + j + 1);
      const bool dense = (e & dense_bit) != 0;
      const int b = int(j & 1);
      const uint32_t scol = tmem + lane_off + 64u * b;
      mbar_wait(bSfull(b), (j >> 1) & 1);
      tc_fence_after();
      float v[64];
      if (dense) {
        uint32_t sa[32], sb[32];
        tmem_ld32(scol, sa);
        tmem_ld32(scol + 32, sb);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          v[i] = __uint_as_float(sa[i]);
          v[i + 32] = __uint_as_float(sb[i]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bSfree(b));  // S(j) is in registers: QK^T(j+2) may overwrite it
      uint32_t pk[32];
      bool pv_done = false;
      if (dense) {
        const uint32_t valid = ((e >> dbsp_core::kEntryValidShift) & 63u) + 1u;
        if (valid < 64) {
#pragma unroll
          for (int i = 0; i < 64; ++i)
            if (uint32_t(i) >= valid) v[i] = -INFINITY;
        }
        float mx[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          mx[a] = fmax3f(v[8 * a], v[8 * a + 1], v[8 * a + 2]);
          mx[a] = fmax3f(mx[a], v[8 * a + 3], v[8 * a + 4]);
          mx[a] = fmax3f(mx[a], v[8 * a + 5], v[8 * a + 6]);
          mx[a] = fmaxf(mx[a], v[8 * a + 7]);
        }
        const float mt = fmaxf(fmax3f(mx[0], mx[1], mx[2]), fmax3f(fmax3f(mx[3], mx[4], mx[5]), mx[6], mx[7]));
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
          // O quiescent: PV(j-1) complete.  PV(j-2) completed before P(j-1)
          // was written, so only phase j-1 of Pfree can be pending.
          if (j > 0) {
            mbar_wait(bPfree, (j - 1) & 1);
            tc_fence_after();
          }
          pv_done = true;
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            tmem_ld32(ocol + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(ocol + c * 32, o);
          }
          tmem_st_wait();
        }
        const float2 sc2 = make_float2(sl2, sl2), nm2 = make_float2(-m, -m);
        float2 acc2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float2 x = __ffma2_rn(make_float2(v[2 * i], v[2 * i + 1]), sc2, nm2);
          const float2 pp = make_float2(fast_exp2(x.x), fast_exp2(x.y));
          acc2[i & 1] = __fadd2_rn(acc2[i & 1], pp);
          pk[i] = pack_bf16x2(pp.x, pp.y);
        }
        const float2 a2 = __fadd2_rn(acc2[0], acc2[1]);
        l += a2.x + a2.y;
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) pk[i] = 0u;
      }
      // P(j) into the single smem P tile once PV(j-1) has read P(j-1).
      if (j > 0 && !pv_done) mbar_wait(bPfree, (j - 1) & 1);
#pragma unroll
      for (int c = 0; c < 8; ++c)
        *reinterpret_cast<uint4*>(prow + ((c ^ (row & 7)) << 4)) =
            make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bPfull);
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
