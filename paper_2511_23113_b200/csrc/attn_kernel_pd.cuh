// K4, d=128: CTA pair (tcgen05 cta_group::2) x two split-KV stages per CTA.
//
// A cluster of two CTAs on the two SMs of a TPC runs one quad work item
// (schedule.hpp kSchedQuad|kSchedKey128): four 64-row Q blocks of one head,
// CTA rank r owning blocks 2r, 2r+1 (128 rows), against the union of their
// dense KV blocks, walked in 128-key steps (two entries per step).  The steps
// alternate between two stages of each CTA -- stage 0 takes the even steps,
// stage 1 the odd ones -- each with its own S and O in TMEM and its own running
// (m, l); the epilogue merges the two partial results row by row.
//
// The leader CTA issues M=256 MMAs for both CTAs:
//   S_s = Q K^T   SS, M=256 N=128  A: each CTA's own Q (smem); B: CTA r holds
//                                 the 64 keys of entry 2t+r (one KV block)
//   O_s += P_s V  TS, M=256 N=128  A: each CTA's own P (TMEM); B: CTA r holds
//                                 columns [64r, 64r+64) of V for all 128 keys
// Per 128-key step an SM moves Q 32 KB + K 16 KB (QK^T) + V 16 KB (PV) + 32 KB
// of TMA writes = 96 KB through its smem port in 1024 tensor cycles (94 B/clk
// of the 128 B/clk port); the one-CTA kernels need 188 B/clk at N=64 (the
// measured limiter of attn_kernel.cuh) or 125 B/clk at N=128 (duo).  With two
// stages, one stage's softmax runs while the tensor pipe executes the other
// stage's PV and QK^T, and the per-stage chain softmax -> PV -> QK^T -> softmax
// is hidden by the other stage.  The exp work of a step equals its tensor work
// at d=128 (16384 exp2 / 16 per clock = 1024 cycles), so kPoly of every 8 exp2
// pairs run on the FMA pipe (exp2_poly3_pair).
// Warp roles (320 threads, one CTA per SM):
//   warps 0-3 / 4-7  softmax of stage 0 / 1 (thread = row = TMEM lane); epilogue
//   warp 8           TMA producer (both CTAs): Q once, K / V halves per step
//   warp 9           TMEM allocator; on the leader the single MMA-issuing thread
// TMEM (512 columns): S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512).
// Mask semantics follow the reference BlockMask (mask.hpp:18-20).
#pragma once

#include "attn_kernel.cuh"

namespace dbsp_dev {

constexpr int kThreadsPd = 320;
// DBSP_TRACE_FINE: stage-0 softmax phases (events 0 start, 2 S loaded, 6 max,
// 3 / 4 P halves stored, 5 before the P arrive, 1 after it, 7 PV_0 issued).
#if defined(DBSP_TRACE_MMA)
#define PD_TR(ev, j) \
  do {               \
  } while (0)
#define PD_TRC(ev, j) \
  do {                \
  } while (0)
#elif defined(DBSP_TRACE_FINE)
#define PD_TR(ev, j) DBSP_TR(ev, j)
#define PD_TRC(ev, j) \
  do {                \
  } while (0)
#else
#define PD_TR(ev, j) \
  do {               \
  } while (0)
#define PD_TRC(ev, j) DBSP_TR(ev, j)
#endif

struct PdCfg {
  static constexpr int D = 128;
  static constexpr uint32_t kQBytes = 128u * 128u * 2u;  // own 128 rows x 128 d
  static constexpr uint32_t kQChunk = 128u * 128u;       // 128 rows x 128 B (one 64-wide d chunk)
  static constexpr uint32_t kKStep = 64u * 128u * 2u;    // own 64 keys x 128 d
  static constexpr uint32_t kKChunk = 64u * 128u;        // 64 rows x 128 B
  static constexpr uint32_t kVStep = 128u * 64u * 2u;    // 128 keys x own 64 d
  static constexpr int kStages = 4;                      // K/V ring depth (steps)
  static constexpr uint32_t kColS = 0, kColO = 256;      // stage s: S at 128 s, O at 256 + 128 s
  static constexpr int kNumBars = 4 * kStages + 2 + 2 + 2 + 2;
  static constexpr uint32_t kSmemBytes =
      kQBytes + kStages * (kKStep + kVStep) + 1024 + 8 * kNumBars + 16 + 2 * 128 * 8;
};

template <int kPoly>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsPd, 1)
    sparse_attn_fwd_pd_kernel(const __grid_constant__ CUtensorMap tmQ,
                              const __grid_constant__ CUtensorMap tmK,
                              const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  using C = PdCfg;
  constexpr int NS = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);

  const uint32_t sQ = base;
  const uint32_t sK = sQ + C::kQBytes;
  const uint32_t sV = sK + NS * C::kKStep;
  const uint32_t sBar = sV + NS * C::kVStep;
  auto bKfull = [&](int s) { return sBar + 8u * s; };
  auto bVfull = [&](int s) { return sBar + 8u * (NS + s); };
  auto bKempty = [&](int s) { return sBar + 8u * (2 * NS + s); };
  auto bVempty = [&](int s) { return sBar + 8u * (3 * NS + s); };
  auto bSfull = [&](int st) { return sBar + 8u * (4 * NS + st); };
  auto bPfull = [&](int st) { return sBar + 8u * (4 * NS + 2 + st); };
  const uint32_t bQ = sBar + 8u * (4 * NS + 4);
  const uint32_t bOfinal = sBar + 8u * (4 * NS + 5);
  // exp phases run in step order across the two stages (one phase per step)
  auto bSmDone = [&](int st) { return sBar + 8u * (4 * NS + 6 + st); };
  const uint32_t sTmemSlot = sBar + 8u * C::kNumBars;
  // stage-1 (m, l) per row, read by the stage-0 thread of the same row
  float2* ml1 = reinterpret_cast<float2*>(gbase + (sTmemSlot + 16 - base));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const WorkItem it = p.items[blockIdx.x >> 1];
  const uint32_t count = it.count;
  const uint32_t nsteps = (count + 1) / 2;
  const uint32_t myq[2] = {rank ? it.pad0 : it.qa, rank ? it.pad1 : it.qb};  // quad rows 2r, 2r+1
  auto leader = [&](uint32_t local_bar) { return mapa_shared(local_bar, 0); };
  clock_probe_mark(p, 0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(bKfull(s), 1);
      mbar_init(bVfull(s), 1);
      mbar_init(bKempty(s), 1);
      mbar_init(bVempty(s), 1);
    }
    for (int st = 0; st < 2; ++st) {
      mbar_init(bSfull(st), 1);
      mbar_init(bPfull(st), 8);  // 4 softmax warps of the stage in each CTA of the pair
    }
    mbar_init(bQ, 1);
    mbar_init(bOfinal, 1);
    mbar_init(bSmDone(0), 4);  // the stage's softmax warps of this CTA
    mbar_init(bSmDone(1), 4);
    mbar_fence_init();
  }
  if (warp == 8 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
  }
  if (warp == 9) tmem_alloc_pair(sTmemSlot, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(gbase + (sTmemSlot - base));
  const uint32_t* ent = p.entries + it.begin;

  if (warp == 8) {
    // ------------------------------------------------------------ producer (both CTAs)
    if (lane == 0 && count > 0) {
      const uint64_t pol_q = l2_policy_evict_first();
      const uint64_t pol_kv = l2_policy_evict_last();
      const int head = int(it.head);
      if (rank == 0) mbar_expect_tx(bQ, 2 * C::kQBytes);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        tma_load_3d_pair(sQ + c * C::kQChunk, &tmQ, c * 64, head, int(myq[0]) * 64, leader(bQ), pol_q);
        tma_load_3d_pair(sQ + c * C::kQChunk + 8192, &tmQ, c * 64, head, int(myq[1]) * 64, leader(bQ),
                         pol_q);
      }
      // KV blocks of step t; an odd tail re-loads the first one (masked out).
      auto kv_of = [&](uint32_t t, uint32_t h) {
        const uint32_t j = 2 * t + h < count ? 2 * t + h : 2 * t;
        return int(__ldg(ent + j) & dbsp_core::kEntryKvMask);
      };
      auto load_k = [&](uint32_t t) {
        const int s = int(t % NS);
        mbar_wait(bKempty(s), ((t / NS) & 1) ^ 1);
        const int kv = kv_of(t, rank);
        if (rank == 0) mbar_expect_tx(bKfull(s), 2 * C::kKStep);
#pragma unroll
        for (int c = 0; c < 2; ++c)
          tma_load_3d_pair(sK + s * C::kKStep + c * C::kKChunk, &tmK, c * 64, head, kv * 64,
                           leader(bKfull(s)), pol_kv);
      };
      load_k(0);
      if (nsteps > 1) load_k(1);
      for (uint32_t t = 0; t < nsteps; ++t) {
        if (t + 2 < nsteps) load_k(t + 2);  // K runs two steps (one per stage) ahead of V
        const int s = int(t % NS);
        mbar_wait(bVempty(s), ((t / NS) & 1) ^ 1);
        if (rank == 0) mbar_expect_tx(bVfull(s), 2 * C::kVStep);
#pragma unroll
        for (int h = 0; h < 2; ++h)
          tma_load_3d_pair(sV + s * C::kVStep + h * 8192, &tmV, int(rank) * 64, head, kv_of(t, h) * 64,
                           leader(bVfull(s)), pol_kv);
      }
    }
    __syncwarp();
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer (leader only)
    if (rank == 0 && lane == 0 && count > 0) {
      constexpr uint32_t kIdescQK = idesc_bf16(256, 128, false, false);
      constexpr uint32_t kIdescPV = idesc_bf16(256, 128, false, true);
      auto issue_s = [&](uint32_t t) {
        const int s = int(t % NS);
        const uint32_t st = t & 1u;
        mbar_wait(bKfull(s), (t / NS) & 1);
        tc_fence_after();
        const uint32_t dcol = tmem + C::kColS + 128u * st;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t ad = smem_desc_sw128(sQ + (kk >> 2) * C::kQChunk + (kk & 3) * 32, 16, 1024);
          const uint64_t bd =
              smem_desc_sw128(sK + s * C::kKStep + (kk >> 2) * C::kKChunk + (kk & 3) * 32, 16, 1024);
          mma_ss_pair(dcol, ad, bd, kIdescQK, kk > 0 ? 1u : 0u);
        }
        tc_commit_pair(bKempty(s), 0x3);
        tc_commit_pair(bSfull(int(st)), 0x3);
        PD_TRC(4 + 2 * int(st), t >> 1);
      };
      auto issue_pv = [&](uint32_t t) {
        const int s = int(t % NS);
        const uint32_t st = t & 1u;
        mbar_wait(bPfull(int(st)), (t >> 1) & 1);
        mbar_wait(bVfull(s), (t / NS) & 1);
        tc_fence_after();
        PD_TRC(5 + 2 * int(st), t >> 1);
        if (st == 0) PD_TR(7, t >> 1);
        const uint32_t pcol = tmem + C::kColS + 128u * st;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t bd = smem_desc_sw128(sV + s * C::kVStep + kk * 2048, 16384, 1024);
          mma_ts_pair(tmem + C::kColO + 128u * st, pcol + kk * 8, bd, kIdescPV, (t >= 2 || kk > 0) ? 1u : 0u);
        }
        tc_commit_pair(bVempty(s), 0x3);
      };
      mbar_wait(bQ, 0);
      tc_fence_after();
      issue_s(0);
      if (nsteps > 1) issue_s(1);
      for (uint32_t t = 0; t < nsteps; ++t) {
        issue_pv(t);
        if (t + 2 < nsteps) issue_s(t + 2);  // S_s(t+2) overwrites P_s(t): in-order after PV_s(t)
      }
      tc_commit_pair(bOfinal, 0x3);
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ softmax (both CTAs)
    const int st = warp >> 2;
    const int row = threadIdx.x & 127;  // TMEM lane
    const uint32_t lane_off = uint32_t((warp & 3) * 32) << 16;
    const bool upper = row >= 64;
    const uint32_t dense_bit = 1u << (22 + 2 * rank + (upper ? 1 : 0));
    const uint32_t pfull_remote_base = rank ? leader(bPfull(0)) : 0u;
    const float sl2 = p.scale_log2;
    const uint32_t scol = tmem + lane_off + C::kColS + 128u * st;
    const uint32_t ocol = tmem + lane_off + C::kColO + 128u * st;
    float m = -INFINITY, l = 0.f;
    for (uint32_t t = st; t < nsteps; t += 2) {
      const uint32_t e0 = __ldg(ent + 2 * t);
      const uint32_t e1 = 2 * t + 1 < count ? __ldg(ent + 2 * t + 1) : 0u;
      const bool d0 = (e0 & dense_bit) != 0, d1 = (e1 & dense_bit) != 0;  // warp-uniform
      mbar_wait(bSfull(st), (t >> 1) & 1);
      tc_fence_after();
      if (lane == 0 && (warp & 3) == 0) PD_TRC(2 * st, t >> 1);
      const bool tr0 = lane == 0 && warp == 0;
      if (tr0) PD_TR(0, t >> 1);
      if (d0 || d1) {
        float v[128];
        {
          uint32_t a0[32], a1[32], a2[32], a3[32];
          tmem_ld32(scol, a0);
          tmem_ld32(scol + 32, a1);
          tmem_ld32(scol + 64, a2);
          tmem_ld32(scol + 96, a3);
          tmem_ld_wait();
          if (tr0) PD_TR(2, t >> 1);
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            v[i] = __uint_as_float(a0[i]);
            v[32 + i] = __uint_as_float(a1[i]);
            v[64 + i] = __uint_as_float(a2[i]);
            v[96 + i] = __uint_as_float(a3[i]);
          }
        }
        // Keys outside the row's dense set or past the sequence end -> -inf.
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
        if (tr0) PD_TR(6, t >> 1);
        const bool resc = mt2 > m + kRescaleThreshold;
        const bool need_o = resc && (m != -INFINITY);
        float alpha = 1.f;
        if (resc) {
          alpha = fast_exp2(m - mt2);
          l *= alpha;
          m = mt2;
        }
        // exp phases alternate between the stages in step order
        if (t > 0) mbar_wait(bSmDone(1 - st), ((t - 1) >> 1) & 1);
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
              if ((i & 7) < kPoly) {
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
          if (tr0) PD_TR(3 + h, t >> 1);
        }
        {
          const float2 a = __fadd2_rn(acc2[0], acc2[1]);
          l += a.x + a.y;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(bSmDone(st));
        if (__any_sync(0xffffffffu, need_o)) {
          // O_s is quiescent: S_s(t) (complete) was issued after PV_s(t-2).
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t o[32];
            tmem_ld32(ocol + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(ocol + c * 32, o);
          }
        }
      } else {
        if (t > 0) mbar_wait(bSmDone(1 - st), ((t - 1) >> 1) & 1);
        uint32_t pk[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) pk[i] = 0u;
        tmem_st32(scol, pk);
        tmem_st32(scol + 32, pk);
        __syncwarp();
        if (lane == 0) mbar_arrive(bSmDone(st));
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (tr0) PD_TR(5, t >> 1);
      if (lane == 0) {
        if (rank == 0)
          mbar_arrive(bPfull(st));
        else
          mbar_arrive_cluster(pfull_remote_base + 8u * st);
      }
      if (lane == 0 && (warp & 3) == 0) PD_TRC(2 * st + 1, t >> 1);
      if (tr0) PD_TR(1, t >> 1);
    }

    // ------------------------------------------------------------ epilogue: merge the stages
    if (count > 0) {
      mbar_wait(bOfinal, 0);
      tc_fence_after();
    }
    if (st == 1) ml1[row] = make_float2(m, l);
    named_bar_sync(1, 256);
    if (st == 0) {
      const uint32_t qi = 2 * rank + (upper ? 1 : 0);
      const uint32_t token = myq[upper ? 1 : 0] * 64u + uint32_t(row & 63);
      const bool live = !((it.single >> qi) & 1u) && token < p.q_tokens;
      const bool have1 = nsteps >= 2;  // stage 1 wrote O1
      const float2 o1 = ml1[row];
      const float mm = fmaxf(m, have1 ? o1.x : -INFINITY);
      float a0 = 0.f, a1 = 0.f, lm = 0.f;
      if (mm != -INFINITY) {
        a0 = m == -INFINITY ? 0.f : fast_exp2(m - mm);
        a1 = (!have1 || o1.x == -INFINITY) ? 0.f : fast_exp2(o1.x - mm);
        lm = l * a0 + (have1 ? o1.y * a1 : 0.f);
      }
      if (count > 0) {
        // O0 <- a0 O0 + a1 O1, then the shared row epilogue on O0.
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t x[32], y[32];
          tmem_ld32(ocol + c * 32, x);
          if (have1) tmem_ld32(ocol + 128 + c * 32, y);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            float r = __uint_as_float(x[i]) * a0;
            if (have1) r = fmaf(__uint_as_float(y[i]), a1, r);
            x[i] = __float_as_uint(r);
          }
          tmem_st32(ocol + c * 32, x);
        }
        tmem_st_wait();
      }
      finish_row<128>(p, ocol, count > 0, live, mm, lm, token, it.head);
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the leader's MMAs wrote into this CTA's TMEM / read its smem
  tc_fence_after();
  clock_probe_mark(p, 1);
  if (warp == 9) tmem_dealloc_pair(tmem, 512);
}

}  // namespace dbsp_dev
