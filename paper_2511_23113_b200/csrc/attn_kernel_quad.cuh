// K4, quad variant: one CTA per SM runs two 128-row Q tiles ("stages") of one
// head against ONE shared stream of 64-key K/V tiles, each stage with two S
// buffers in TMEM.
//
// Why: the default kernel (attn_kernel.cuh, two CTAs per SM) is bound by the
// shared-memory port at d=128.  Per 128x64 tile an SM moves Q 32 KB + K 16 KB
// + V 16 KB through the port for the MMAs plus 32 KB of TMA writes (96 KB,
// 750 cycles at 128 B/clk; measured 727).  Here the two stages read the same
// K/V tile, so the TMA writes per Q tile halve: 80 KB per tile.  Unlike the
// 128-key two-stage kernel (attn_kernel_duo.cuh) each stage keeps two S
// buffers, so QK^T of tile j+1 overlaps the softmax of tile j.
// Work item = a quad (schedule.hpp kSchedQuad): stage 0 = Q blocks 0,1,
// stage 1 = blocks 2,3, KV list = union of the four rows.
// Warp roles (352 threads):
//   warps 0-3 / 4-7   softmax + epilogue of stage 0 / 1 (thread = row = TMEM lane)
//   warp 8            TMA producer: Q once, then K(j), V(j) through NS-deep rings
//   warps 9 / 10      tcgen05.mma issuer of stage 0 / 1 (warp 9 also owns TMEM)
// TMEM (512 columns):
//   d=128: S(stage s, buffer b) at 64(2s+b) in [0,256); O_s at 256+128s; Q in smem
//   d=64:  Q_s at 32s; S at 64+64(2s+b); O_s at 320+64s
// MMA order of stage s per tile j: PV_s(j), S_s(j+2).  S_s(j+2) reuses the
// columns of P_s(j), which PV_s(j) (issued just before, same thread) reads;
// tcgen05 ops of one thread execute in order.
// Mask semantics follow the reference BlockMask (mask.hpp:18-20).
#pragma once

#include "attn_kernel.cuh"

namespace dbsp_dev {

constexpr int kThreadsQuad = 352;

template <int D>
struct QuadCfg {
  static constexpr int kChunks = D / 64;
  static constexpr bool kQInTmem = D == 64;
  static constexpr uint32_t kQStageBytes = 128u * D * 2u;
  static constexpr uint32_t kQBytes = kQInTmem ? 0u : 2u * kQStageBytes;
  static constexpr uint32_t kQChunk = 128u * 128u;      // 128 rows x 128 B
  static constexpr uint32_t kTileBytes = 64u * D * 2u;  // one 64-key K or V tile
  static constexpr uint32_t kColQ = 0;
  static constexpr uint32_t kColS = kQInTmem ? 64 : 0;
  static constexpr uint32_t kColO = kColS + 256;
  static_assert(kColO + 2 * D <= 512, "TMEM budget");
  static constexpr int kStages = D == 128 ? 4 : 8;
  static constexpr int kNumBars = 4 * kStages + 4 + 4 + 2 + 2 + 2;
  static constexpr uint32_t kSmemBytes = kQBytes + 2u * kStages * kTileBytes + 1024 + 8 * kNumBars + 16;
};

template <int D>
__global__ void __launch_bounds__(kThreadsQuad, 1)
    sparse_attn_fwd_quad_kernel(const __grid_constant__ CUtensorMap tmQ,
                                const __grid_constant__ CUtensorMap tmK,
                                const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  using C = QuadCfg<D>;
  constexpr int NS = C::kStages;
  extern __shared__ uint8_t smem_raw[];
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
  auto bSfull = [&](int st, int b) { return sBar + 8u * (4 * NS + 2 * st + b); };
  auto bPfull = [&](int st, int b) { return sBar + 8u * (4 * NS + 4 + 2 * st + b); };
  auto bQready = [&](int st) { return sBar + 8u * (4 * NS + 8 + st); };
  auto bOdone = [&](int st) { return sBar + 8u * (4 * NS + 10 + st); };   // one phase per PV_s(j)
  auto bOfinal = [&](int st) { return sBar + 8u * (4 * NS + 12 + st); };  // single phase
  const uint32_t sTmemSlot = sBar + 8u * C::kNumBars;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const WorkItem it = p.items[blockIdx.x];
  const uint32_t count = it.count;
  clock_probe_mark(p, 0);
#ifdef DBSP_TRACE_CTA
  const unsigned long long c_start = clock64();
  if (threadIdx.x == 0 && p.trace) p.trace[4 * blockIdx.x] = globaltimer_ns();
#endif

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(bKfull(s), 1);
      mbar_init(bVfull(s), 1);
      mbar_init(bKempty(s), 2);  // one commit per stage's MMA thread
      mbar_init(bVempty(s), 2);
    }
    for (int st = 0; st < 2; ++st) {
      for (int b = 0; b < 2; ++b) {
        mbar_init(bSfull(st, b), 1);
        mbar_init(bPfull(st, b), 4);  // one arrive per softmax warp of the stage
      }
      mbar_init(bQready(st), C::kQInTmem ? 4 : 1);
      mbar_init(bOdone(st), 1);
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
            const uint32_t dst = sQ + st * C::kQStageBytes + c * C::kQChunk;
            tma_load_3d(dst, &tmQ, c * 64, head, int(qblk(2 * st)) * 64, bQready(st), pol_q);
            tma_load_3d(dst + 8192, &tmQ, c * 64, head, int(qblk(2 * st + 1)) * 64, bQready(st), pol_q);
          }
        }
      }
      auto load_tile = [&](const CUtensorMap* tm, uint32_t dst, uint32_t full, uint32_t j) {
        const int kv = int(__ldg(ent + j) & dbsp_core::kEntryKvMask);
        mbar_expect_tx(full, C::kTileBytes);
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c) tma_load_3d(dst + c * 8192, tm, c * 64, head, kv * 64, full, pol_kv);
      };
      auto load_k = [&](uint32_t j) {
        const int s = int(j % NS);
        mbar_wait(bKempty(s), ((j / NS) & 1) ^ 1);
        load_tile(&tmK, sK + s * C::kTileBytes, bKfull(s), j);
      };
      // Same order as the MMA warp consumes: K(0), K(1), then V(j), K(j+2).
      for (uint32_t j = 0; j < 2 && j < count; ++j) load_k(j);
      for (uint32_t j = 0; j < count; ++j) {
        const int s = int(j % NS);
        mbar_wait(bVempty(s), ((j / NS) & 1) ^ 1);
        load_tile(&tmV, sV + s * C::kTileBytes, bVfull(s), j);
        if (j + 2 < count) load_k(j + 2);
      }
    } else if (count > 0) {
      mbar_wait(bOfinal(1), 0);
    }
    __syncwarp();
  } else if (warp >= 9) {
    // ------------------------------------------------------------ MMA issuers
    // One issuing thread per stage (warp 9: stage 0, warp 10: stage 1), so a
    // late P of one stage never holds back the other stage's MMAs.  Both wait
    // on the shared K/V "full" barriers; the "empty" barriers count one commit
    // per stage.
    const int st = warp - 9;
    if (lane == 0 && count > 0) {
      constexpr uint32_t kIdescQK = idesc_bf16(128, 64, false, false);
      constexpr uint32_t kIdescPV = idesc_bf16(128, D, false, true);
      auto issue_s = [&](uint32_t j) {
        const int s = int(j % NS);
        mbar_wait(bKfull(s), (j / NS) & 1);
        tc_fence_after();
        const uint32_t dcol = tmem + C::kColS + 64u * (2 * st + (j & 1));
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t bd =
              smem_desc_sw128(sK + s * C::kTileBytes + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
          if constexpr (C::kQInTmem) {
            mma_ts(dcol, tmem + C::kColQ + 32u * st + kk * 8, bd, kIdescQK, kk > 0 ? 1u : 0u);
          } else {
            const uint64_t ad = smem_desc_sw128(
                sQ + st * C::kQStageBytes + (kk >> 2) * C::kQChunk + (kk & 3) * 32, 16, 1024);
            mma_ss(dcol, ad, bd, kIdescQK, kk > 0 ? 1u : 0u);
          }
        }
        tc_commit(bSfull(st, int(j & 1)));
        tc_commit(bKempty(s));
      };
      auto issue_pv = [&](uint32_t j) {
        const int s = int(j % NS);
        const int b = int(j & 1);
        mbar_wait(bPfull(st, b), (j >> 1) & 1);
        mbar_wait(bVfull(s), (j / NS) & 1);
        tc_fence_after();
        const uint32_t pcol = tmem + C::kColS + 64u * (2 * st + b);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t bd = smem_desc_sw128(sV + s * C::kTileBytes + kk * 2048, 8192, 1024);
          mma_ts(tmem + C::kColO + uint32_t(D) * st, pcol + kk * 8, bd, kIdescPV,
                 (j > 0 || kk > 0) ? 1u : 0u);
        }
        tc_commit(bOdone(st));
        tc_commit(bVempty(s));
      };
      mbar_wait(bQready(st), 0);
      tc_fence_after();
      for (uint32_t j = 0; j < 2 && j < count; ++j) issue_s(j);
      for (uint32_t j = 0; j < count; ++j) {
        issue_pv(j);
        if (j + 2 < count) issue_s(j + 2);
      }
      tc_commit(bOfinal(st));
    } else if (count > 0) {
      mbar_wait(bOfinal(st), 0);
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
    const uint32_t ocol = tmem + lane_off + C::kColO + uint32_t(D) * st;
    float m = -INFINITY, l = 0.f;
    for (uint32_t j = 0; j < count; ++j) {
      const uint32_t e = __ldg(ent + j);
      const bool dense = (e & dense_bit) != 0;  // warp-uniform
      const int b = int(j & 1);
      const uint32_t scol = tmem + lane_off + C::kColS + 64u * (2 * st + b);
      mbar_wait(bSfull(st, b), (j >> 1) & 1);
      tc_fence_after();
      uint32_t pk[32];
      if (dense) {
        float v[64];
        {
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
        const uint32_t valid = ((e >> dbsp_core::kQuadValidShift) & 63u) + 1u;
        if (valid < 64) {  // partial last KV block (warp-uniform)
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
          // O_s must be quiescent: PV_s(j-1) complete.  S_s(j) was issued
          // after PV_s(j-2), so phases up to j-2 are done and (j-1)&1 is
          // unambiguous.
          if (j > 0) {
            mbar_wait(bOdone(st), (j - 1) & 1);
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
        for (int i = 0; i < 32; ++i) {
          const float2 x = __ffma2_rn(make_float2(v[2 * i], v[2 * i + 1]), sc2, nm2);
          float2 pp;
          if ((i & 7) < poly_pairs<D>()) {
            pp = exp2_poly3_pair(x);
          } else {
            pp = make_float2(fast_exp2(x.x), fast_exp2(x.y));
          }
          acc2[i & 1] = __fadd2_rn(acc2[i & 1], pp);
          pk[i] = pack_bf16x2(pp.x, pp.y);
        }
        const float2 a2 = __fadd2_rn(acc2[0], acc2[1]);
        l += a2.x + a2.y;
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) pk[i] = 0u;
      }
      tmem_st32(scol, pk);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bPfull(st, b));
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
  clock_probe_mark(p, 1);
#ifdef DBSP_TRACE_CTA
  if (threadIdx.x == 0 && p.trace) {
    p.trace[4 * blockIdx.x + 1] = globaltimer_ns();
    p.trace[4 * blockIdx.x + 2] = smid();
    p.trace[4 * blockIdx.x + 3] = clock64() - c_start;
  }
#endif
}

}  // namespace dbsp_dev
