// K4, two-stage variant: one CTA per SM, two 128-row Q tiles ("stages") of
// one head sharing one KV stream, 128-key steps.
//
// Work item = a quad (schedule.hpp kSchedQuad): four 64-row Q blocks of one
// head, stage 0 = blocks 0,1 and stage 1 = blocks 2,3, against the union of
// their dense KV blocks.  Consecutive pairs of dense KV blocks form one
// 128-key step (the second slot of an odd tail re-loads the first block and is
// masked out), so every barrier round trip (tcgen05.commit -> mbarrier, ~350
// cycles measured) is paid once per 128 keys instead of per 64.
// Warp roles (320 threads):
//   warps 0-3 / 4-7   softmax + epilogue of stage 0 / 1 (thread = row = TMEM lane)
//   warp 8            TMA producer: Q once, then K and V steps through NS-deep rings
//   warp 9            TMEM allocator + single-thread tcgen05.mma issuer
// TMEM (512 columns, the whole SM):
//   d=128: S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512); Q in smem
//          (SS-mode QK^T at N=128: 8 KB per 64-cycle MMA = the 128 B/clk port)
//   d=64:  Q0 [0,32) Q1 [32,64) S0 [64,192) S1 [192,320) O0 [320,384) O1 [384,448)
// Per step t and stage s the MMA warp issues PV_s(t) then S_s(t+1): the bf16
// P_s(t) overwrites S_s(t) in TMEM, and tcgen05 ops of one thread execute in
// order, so S_s(t+1) is issued after the PV that reads P_s(t).  The two stages
// ping-pong: while stage 0's softmax runs, the tensor pipe executes stage 1's
// PV and QK^T, and vice versa.  Because S_s(t) completes after PV_s(t-1), a
// lazy O rescale in the softmax needs no extra wait.
// Mask semantics follow the reference BlockMask (mask.hpp:18-20).
#pragma once

#include "attn_kernel.cuh"

namespace dbsp_dev {

constexpr int kThreadsDuo = 320;
#ifdef DBSP_TRACE_FINE
#define DBSP_FINE 1
#else
#define DBSP_FINE 0
#endif

template <int D>
struct DuoCfg {
  static constexpr int kChunks = D / 64;
  static constexpr bool kQInTmem = D == 64;
  static constexpr uint32_t kQStageBytes = 128u * D * 2u;  // 128 rows of one stage
  static constexpr uint32_t kQBytes = kQInTmem ? 0u : 2u * kQStageBytes;
  static constexpr uint32_t kChunkBytes = 128u * 128u;  // 128 rows x 128 B (one d chunk)
  static constexpr uint32_t kStepBytes = 128u * D * 2u;  // one 128-key K or V step
  static constexpr uint32_t kColQ = 0;                  // d=64: stage s at s*32
  static constexpr uint32_t kColS = kQInTmem ? 64 : 0;  // stage s at kColS + 128 s
  static constexpr uint32_t kColO = kColS + 256;        // stage s at kColO + D s
  static_assert(kColO + 2 * D <= 512, "TMEM budget");
  static constexpr int kStages = D == 128 ? 2 : 4;
  static constexpr int kNumBars = 4 * kStages + 8;
  static constexpr uint32_t kSmemBytes = kQBytes + 2u * kStages * kStepBytes + 1024 + 8 * kNumBars + 16;
};

template <int D>
__global__ void __launch_bounds__(kThreadsDuo, 1)
    sparse_attn_fwd_duo_kernel(const __grid_constant__ CUtensorMap tmQ,
                               const __grid_constant__ CUtensorMap tmK,
                               const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  using C = DuoCfg<D>;
  constexpr int NS = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);

  const uint32_t sQ = base;
  const uint32_t sK = base + C::kQBytes;
  const uint32_t sV = sK + NS * C::kStepBytes;
  const uint32_t sBar = sV + NS * C::kStepBytes;
  auto bKfull = [&](int s) { return sBar + 8u * s; };
  auto bVfull = [&](int s) { return sBar + 8u * (NS + s); };
  auto bKempty = [&](int s) { return sBar + 8u * (2 * NS + s); };
  auto bVempty = [&](int s) { return sBar + 8u * (3 * NS + s); };
  auto bSfull = [&](int st) { return sBar + 8u * (4 * NS + st); };
  auto bPfull = [&](int st) { return sBar + 8u * (4 * NS + 2 + st); };
  auto bQready = [&](int st) { return sBar + 8u * (4 * NS + 4 + st); };
  auto bOfinal = [&](int st) { return sBar + 8u * (4 * NS + 6 + st); };
  const uint32_t sTmemSlot = sBar + 8u * C::kNumBars;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const WorkItem it = p.items[blockIdx.x];
  const uint32_t count = it.count;
  const uint32_t nsteps = (count + 1) / 2;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(bKfull(s), 1);
      mbar_init(bVfull(s), 1);
      mbar_init(bKempty(s), 1);
      mbar_init(bVempty(s), 1);
    }
    for (int st = 0; st < 2; ++st) {
      mbar_init(bSfull(st), 1);
      mbar_init(bPfull(st), 4);  // one arrive per softmax warp of the stage
      mbar_init(bQready(st), C::kQInTmem ? 4 : 1);
      mbar_init(bOfinal(st), 1);
    }
    mbar_fence_init();
  }
  if (warp == 8 && lane == 0) {
    if (!C::kQInTmem) tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
  }
  if (warp == 9) tmem_alloc(sTmemSlot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(gbase + (sTmemSlot - base));
  const uint32_t* ent = p.entries + it.begin;
  auto qblk = [&](int i) { return i == 0 ? it.qa : i == 1 ? it.qb : i == 2 ? it.pad0 : it.pad1; };

  if (warp == 8) {
    // ------------------------------------------------------------ producer
    if (lane == 0 && count > 0) {
      const uint64_t pol_kv = l2_policy_evict_last();
      const int head = int(it.head);
      if (!C::kQInTmem) {
        const uint64_t pol_q = l2_policy_evict_first();
#pragma unroll
        for (int st = 0; st < 2; ++st) {
          mbar_expect_tx(bQready(st), C::kQStageBytes);
#pragma unroll
          for (int c = 0; c < C::kChunks; ++c) {
            const uint32_t dst = sQ + st * C::kQStageBytes + c * C::kChunkBytes;
            tma_load_3d(dst, &tmQ, c * 64, head, int(qblk(2 * st)) * 64, bQready(st), pol_q);
            tma_load_3d(dst + 8192, &tmQ, c * 64, head, int(qblk(2 * st + 1)) * 64, bQready(st), pol_q);
          }
        }
      }
      // Both 64-key halves of step t; an odd tail re-loads the first block.
      auto load_step = [&](const CUtensorMap* tm, uint32_t dst, uint32_t full, uint32_t t) {
        const int kv0 = int(__ldg(ent + 2 * t) & dbsp_core::kEntryKvMask);
        const int kv1 = 2 * t + 1 < count ? int(__ldg(ent + 2 * t + 1) & dbsp_core::kEntryKvMask) : kv0;
        mbar_expect_tx(full, C::kStepBytes);
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c) {
          tma_load_3d(dst + c * C::kChunkBytes, tm, c * 64, head, kv0 * 64, full, pol_kv);
          tma_load_3d(dst + c * C::kChunkBytes + 8192, tm, c * 64, head, kv1 * 64, full, pol_kv);
        }
      };
      auto load_k = [&](uint32_t t) {
        const int s = int(t % NS);
        mbar_wait(bKempty(s), ((t / NS) & 1) ^ 1);
        load_step(&tmK, sK + s * C::kStepBytes, bKfull(s), t);
      };
      load_k(0);
      for (uint32_t t = 0; t < nsteps; ++t) {
        if (t + 1 < nsteps) load_k(t + 1);  // K runs one step ahead of V
        const int s = int(t % NS);
        mbar_wait(bVempty(s), ((t / NS) & 1) ^ 1);
        load_step(&tmV, sV + s * C::kStepBytes, bVfull(s), t);
      }
    } else if (count > 0) {
      mbar_wait(bOfinal(1), 0);
    }
    __syncwarp();
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0 && count > 0) {
      constexpr uint32_t kIdescQK = idesc_bf16(128, 128, false, false);
      constexpr uint32_t kIdescPV = idesc_bf16(128, D, false, true);
      auto issue_s = [&](int st, uint32_t t) {
        const int s = int(t % NS);
        if (st == 0) {
          mbar_wait(bKfull(s), (t / NS) & 1);
          tc_fence_after();
        }
        const uint32_t dcol = tmem + C::kColS + 128u * st;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t bd =
              smem_desc_sw128(sK + s * C::kStepBytes + (kk >> 2) * C::kChunkBytes + (kk & 3) * 32, 16, 1024);
          if constexpr (C::kQInTmem) {
            mma_ts(dcol, tmem + C::kColQ + 32u * st + kk * 8, bd, kIdescQK, kk > 0 ? 1u : 0u);
          } else {
            const uint64_t ad = smem_desc_sw128(
                sQ + st * C::kQStageBytes + (kk >> 2) * C::kChunkBytes + (kk & 3) * 32, 16, 1024);
            mma_ss(dcol, ad, bd, kIdescQK, kk > 0 ? 1u : 0u);
          }
        }
        tc_commit(bSfull(st));
        if (st == 1) tc_commit(bKempty(s));
#ifndef DBSP_TRACE_FINE
        DBSP_TR(4 + 2 * st, t);
#endif
      };
      auto issue_pv = [&](int st, uint32_t t) {
        const int s = int(t % NS);
        mbar_wait(bPfull(st), t & 1);
        if (st == 0) mbar_wait(bVfull(s), (t / NS) & 1);
        tc_fence_after();
#ifndef DBSP_TRACE_FINE
        DBSP_TR(5 + 2 * st, t);
#else
        if (st == 0) DBSP_TR(7, t);
#endif
        const uint32_t pcol = tmem + C::kColS + 128u * st;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t bd = smem_desc_sw128(sV + s * C::kStepBytes + kk * 2048, C::kChunkBytes, 1024);
          mma_ts(tmem + C::kColO + uint32_t(D) * st, pcol + kk * 8, bd, kIdescPV,
                 (t > 0 || kk > 0) ? 1u : 0u);
        }
        if (st == 1) tc_commit(bVempty(s));
      };
      if (C::kQInTmem) {
        mbar_wait(bQready(0), 0);
        mbar_wait(bQready(1), 0);
      } else {
        mbar_wait(bQready(0), 0);
      }
      tc_fence_after();
      issue_s(0, 0);
      if (!C::kQInTmem) {
        mbar_wait(bQready(1), 0);
        tc_fence_after();
      }
      issue_s(1, 0);
      for (uint32_t t = 0; t < nsteps; ++t) {
        const bool more = t + 1 < nsteps;
        issue_pv(0, t);
        if (more) issue_s(0, t + 1);
        else tc_commit(bOfinal(0));
        issue_pv(1, t);
        if (more) issue_s(1, t + 1);
        else tc_commit(bOfinal(1));
      }
    } else if (count > 0) {
      mbar_wait(bOfinal(1), 0);
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ softmax (+ Q -> TMEM for d=64)
    const int st = warp >> 2;
    const int row = threadIdx.x & 127;  // TMEM lane
    const uint32_t lane_off = uint32_t((warp & 3) * 32) << 16;
    const int bi = 2 * st + (row >> 6);  // quad row block 0..3 (warp-uniform)
    const uint32_t token = qblk(bi) * 64u + uint32_t(row & 63);
    const bool padded = (it.single >> bi) & 1u;
    if (C::kQInTmem && count > 0) {
      const bool in = !padded && token < p.q_tokens;
      const uint4* src = reinterpret_cast<const uint4*>(p.q + (size_t(token) * p.heads + it.head) * D);
      uint32_t w[32];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint4 x = in ? __ldg(src + i) : make_uint4(0, 0, 0, 0);
        w[4 * i + 0] = x.x;
        w[4 * i + 1] = x.y;
        w[4 * i + 2] = x.z;
        w[4 * i + 3] = x.w;
      }
      tmem_st32(tmem + lane_off + C::kColQ + 32u * st, w);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bQready(st));
    }

    const uint32_t dense_bit = 1u << (22 + bi);
    const float sl2 = p.scale_log2;
    const uint32_t scol = tmem + lane_off + C::kColS + 128u * st;
    const uint32_t ocol = tmem + lane_off + C::kColO + uint32_t(D) * st;
    float m = -INFINITY, l = 0.f;
    for (uint32_t t = 0; t < nsteps; ++t) {
      const uint32_t e0 = __ldg(ent + 2 * t);
      const uint32_t e1 = 2 * t + 1 < count ? __ldg(ent + 2 * t + 1) : 0u;
      const bool d0 = (e0 & dense_bit) != 0, d1 = (e1 & dense_bit) != 0;  // warp-uniform
      mbar_wait(bSfull(st), t & 1);
      tc_fence_after();
      if (lane == 0 && (warp & 3) == 0 && (!DBSP_FINE || st == 0)) DBSP_TR(2 * st, t);
      if (d0 || d1) {
        float v[128];
        {
          uint32_t a0[32], a1[32], a2[32], a3[32];
          tmem_ld32(scol, a0);
          tmem_ld32(scol + 32, a1);
          tmem_ld32(scol + 64, a2);
          tmem_ld32(scol + 96, a3);
          tmem_ld_wait();
#ifdef DBSP_TRACE_FINE
          if (lane == 0 && warp == 0) DBSP_TR(2, t);
#endif
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            v[i] = __uint_as_float(a0[i]);
            v[32 + i] = __uint_as_float(a1[i]);
            v[64 + i] = __uint_as_float(a2[i]);
            v[96 + i] = __uint_as_float(a3[i]);
          }
        }
        // Keys outside the row's dense set or past the sequence end -> -inf
        // (warp-uniform, rare: a half not dense for these rows, or the partial
        // last KV block).
        const uint32_t lim0 = d0 ? ((e0 >> dbsp_core::kQuadValidShift) & 63u) + 1u : 0u;
        const uint32_t lim1 = d1 ? ((e1 >> dbsp_core::kQuadValidShift) & 63u) + 1u : 0u;
        if (lim0 < 64 || lim1 < 64) {
#pragma unroll
          for (int i = 0; i < 64; ++i) {
            v[i] = uint32_t(i) < lim0 ? v[i] : -INFINITY;
            v[64 + i] = uint32_t(i) < lim1 ? v[64 + i] : -INFINITY;
          }
        }
        float mx[16];
#pragma unroll
        for (int a = 0; a < 16; ++a) {
          mx[a] = fmax3f(v[8 * a], v[8 * a + 1], v[8 * a + 2]);
          mx[a] = fmax3f(mx[a], v[8 * a + 3], v[8 * a + 4]);
          mx[a] = fmax3f(mx[a], v[8 * a + 5], v[8 * a + 6]);
          mx[a] = fmaxf(mx[a], v[8 * a + 7]);
        }
#pragma unroll
        for (int a = 0; a < 5; ++a) mx[a] = fmax3f(mx[3 * a], mx[3 * a + 1], mx[3 * a + 2]);
        const float mt = fmaxf(fmax3f(mx[0], mx[1], mx[2]), fmax3f(mx[3], mx[4], mx[15]));
        const float mt2 = mt * sl2;
#ifdef DBSP_TRACE_FINE
        if (lane == 0 && warp == 0) DBSP_TR(6, t);
#endif
        const bool resc = mt2 > m + kRescaleThreshold;
        const bool need_o = resc && (m != -INFINITY);
        float alpha = 1.f;
        if (resc) {
          alpha = fast_exp2(m - mt2);
          l *= alpha;
          m = mt2;
        }
        // P in two 64-key halves, each stored as soon as it is packed (keeps
        // 32 packed registers live, not 64); a half that is not dense for
        // these rows is all zeros.
        // Packed f32x2 FMA/add (FFMA2/FADD2) halve the non-MUFU issue slots
        // of the exp loop (tests/pipe_bench.cu: a lone warp runs the packed
        // body at 85% of the MUFU rate, the scalar one at 65%).
        const float2 sc2 = make_float2(sl2, sl2), nm2 = make_float2(-m, -m);
        float2 acc2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t pk[32];
          if (h == 0 ? d0 : d1) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float2 x = __ffma2_rn(make_float2(v[64 * h + 2 * i], v[64 * h + 2 * i + 1]), sc2, nm2);
              float2 pp;
              if ((i & 7) < poly_pairs<D>()) {
                pp = exp2_poly3_pair(x);
              } else {
                pp = make_float2(fast_exp2(x.x), fast_exp2(x.y));
              }
              acc2[i & 1] = __fadd2_rn(acc2[i & 1], pp);
              pk[i] = pack_bf16x2(pp.x, pp.y);
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) pk[i] = 0u;
          }
          tmem_st32(scol + 32 * h, pk);
#ifdef DBSP_TRACE_FINE
          if (lane == 0 && warp == 0) DBSP_TR(3 + h, t);
#endif
        }
        {
          const float2 a = __fadd2_rn(acc2[0], acc2[1]);
          l += a.x + a.y;
        }
        if (__any_sync(0xffffffffu, need_o)) {
          // O_s is quiescent: S_s(t) (complete) was issued after PV_s(t-1).
          // Done after P is packed, when the S registers are dead.
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
      } else {
        uint32_t pk[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) pk[i] = 0u;
        tmem_st32(scol, pk);
        tmem_st32(scol + 32, pk);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0 && (warp & 3) == 0 && (!DBSP_FINE || st == 0)) DBSP_TR(2 * st + 1, t);
      if (lane == 0) mbar_arrive(bPfull(st));
    }

    // ------------------------------------------------------------ epilogue
    if (count > 0) {
      mbar_wait(bOfinal(st), 0);
      tc_fence_after();
    }
    finish_row<D>(p, ocol, count > 0, !padded && token < p.q_tokens, m, l, token, it.head);
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 9) tmem_dealloc(tmem, 512);
}

}  // namespace dbsp_dev
