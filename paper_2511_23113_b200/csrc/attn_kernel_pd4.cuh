// K4, d=128: CTA pair (tcgen05 cta_group::2) x two split-KV stages per CTA,
// ONE softmax warp per row, P staged in shared memory.
//
// attn_kernel_pd3.cuh with the pd (one warp per row) softmax: each thread
// holds its row's 128 scores of a step, so the row max needs no exchange
// between warps (pd3 pays a 64-thread named barrier and a second S read for
// it), and 10 warps leave ptxas 168 registers per thread.  S is released as
// soon as it is in registers; P goes to smem; the leader issues QK^T(t+2)
// ahead of PV(t) as in pd3.
// Warp roles (320 threads, one CTA per SM):
//   warps 0-3 / 4-7  softmax of stage 0 / 1 (thread = row = TMEM lane); epilogue
//   warp 8           TMA producer (both CTAs)
//   warp 9           TMEM allocator; on the leader the MMA-issuing warp
// Epilogue: the two threads of a row (stage 0 / 1) exchange (m, l); each writes
// 64 of the 128 output columns of O = (a0 O_0 + a1 O_1) / L.
// Mask semantics follow the reference BlockMask (mask.hpp:18-20).
#pragma once

#include "attn_kernel_pd3.cuh"

namespace dbsp_dev {

struct Pd4Cfg {
  static constexpr int D = 128;
  static constexpr uint32_t kQBytes = 128u * 128u * 2u;
  static constexpr uint32_t kQChunk = 128u * 128u;
  static constexpr uint32_t kKStep = 64u * 128u * 2u;
  static constexpr uint32_t kKChunk = 64u * 128u;
  static constexpr uint32_t kVStep = 128u * 64u * 2u;
  static constexpr uint32_t kPBytes = 128u * 128u * 2u;  // one stage's P: 2 chunks of 64 keys
  static constexpr int kStages = 3;
  static constexpr uint32_t kColS = 0, kColO = 256;
  static constexpr int kNumBars = 4 * kStages + 2 + 2 + 2 + 2 + 2 + 2;
  static constexpr uint32_t kXBytes = 0;
  static constexpr uint32_t kMlBytes = 2u * 128u * 8u;  // [stage][row] (m, l)
  static constexpr uint32_t kSmemBytes =
      kQBytes + kStages * (kKStep + kVStep) + 2 * kPBytes + kXBytes + kMlBytes + 1024 + 8 * kNumBars + 16;
};

constexpr int kThreadsPd4 = 320;

template <int kPoly>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsPd4, 1)
    sparse_attn_fwd_pd4_kernel(const __grid_constant__ CUtensorMap tmQ,
                               const __grid_constant__ CUtensorMap tmK,
                               const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  using C = Pd4Cfg;
  constexpr int NS = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);

  const uint32_t sQ = base;
  const uint32_t sK = sQ + C::kQBytes;
  const uint32_t sV = sK + NS * C::kKStep;
  const uint32_t sP = sV + NS * C::kVStep;  // stage st at sP + st * kPBytes
  float* xmax = reinterpret_cast<float*>(gbase + (sP + 2 * C::kPBytes - base));
  float2* mlbuf = reinterpret_cast<float2*>(xmax + C::kXBytes / 4);
  const uint32_t sBar = sP + 2 * C::kPBytes + C::kXBytes + C::kMlBytes;
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
  auto bSfree = [&](int st) { return sBar + 8u * (4 * NS + 8 + st); };   // S_st read (leader)
  auto bPempty = [&](int st) { return sBar + 8u * (4 * NS + 10 + st); };  // PV_st done (both CTAs)
  const uint32_t sTmemSlot = sBar + 8u * C::kNumBars;

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
    mbar_init(bSmDone(0), 4);
    mbar_init(bSmDone(1), 4);
    for (int st = 0; st < 2; ++st) {
      mbar_init(bSfree(st), 8);  // 4 softmax warps of the stage in each CTA of the pair
      mbar_init(bPempty(st), 1);
    }
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

  if (warp >= 8) {
    if (warp == 8) {
      // ---------------------------------------------------------- producer (both CTAs)
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
          if (t + 2 < nsteps) load_k(t + 2);
          const int s = int(t % NS);
          mbar_wait(bVempty(s), ((t / NS) & 1) ^ 1);
          if (rank == 0) mbar_expect_tx(bVfull(s), 2 * C::kVStep);
#pragma unroll
          for (int h = 0; h < 2; ++h)
            tma_load_3d_pair(sV + s * C::kVStep + h * 8192, &tmV, int(rank) * 64, head, kv_of(t, h) * 64,
                             leader(bVfull(s)), pol_kv);
        }
      }
    } else if (warp == 9) {
      // ---------------------------------------------------------- MMA issuer (leader only)
      // The whole warp runs the loop (warp-uniform control flow); one elected
      // lane issues.  Descriptors are a base plus per-k-step constants (the
      // 14-bit start-address field never carries), so each MMA costs two
      // uniform adds: with a lane-0 branch and full descriptor math the
      // issuing thread, which shares its SMSP with four softmax warps, took
      // ~90 cycles per MMA against the 64-cycle tensor floor.
      if (rank == 0 && count > 0) {
        constexpr uint32_t kIdescQK = idesc_bf16(256, 128, false, false);
        constexpr uint32_t kIdescPV = idesc_bf16(256, 128, false, true);
        const uint64_t dQ = smem_desc_sw128(sQ, 16, 1024);
        const uint64_t dK = smem_desc_sw128(sK, 16, 1024);
        const uint64_t dP = smem_desc_sw128(sP, 16, 1024);
        const uint64_t dV = smem_desc_sw128(sV, 16384, 1024);
        auto issue_s = [&](uint32_t t) {
          const int s = int(t % NS);
          const uint32_t st = t & 1u;
          mbar_wait(bKfull(s), (t / NS) & 1);
          if (t >= 2) PD_TRM(5, t - 2);
          tc_fence_after();
          const uint32_t dcol = tmem + C::kColS + 128u * st;
          const uint64_t bK = dK + ((uint32_t(s) * C::kKStep) >> 4);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              mma_ss_pair(dcol, dQ + (((kk >> 2) * C::kQChunk + (kk & 3) * 32) >> 4),
                          bK + (((kk >> 2) * C::kKChunk + (kk & 3) * 32) >> 4), kIdescQK, kk > 0 ? 1u : 0u);
            tc_commit_pair(bKempty(s), 0x3);
            tc_commit_pair(bSfull(int(st)), 0x3);
          }
          __syncwarp();
          PD_TRC(4 + 2 * int(st), t >> 1);
        };
        auto issue_pv = [&](uint32_t t) {
          const int s = int(t % NS);
          const uint32_t st = t & 1u;
          mbar_wait(bPfull(int(st)), (t >> 1) & 1);
          PD_TRM(2, t);
          mbar_wait(bVfull(s), (t / NS) & 1);
          PD_TRM(3, t);
          tc_fence_after();
          PD_TRC(5 + 2 * int(st), t >> 1);
          if (st == 0) PD_TR(7, t >> 1);
          const uint64_t aP = dP + ((st * C::kPBytes) >> 4);
          const uint64_t bV = dV + ((uint32_t(s) * C::kVStep) >> 4);
          const uint32_t ocol = tmem + C::kColO + 128u * st;
          const uint32_t acc0 = t >= 2 ? 1u : 0u;
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              mma_ss_pair(ocol, aP + (((kk >> 2) * 16384 + (kk & 3) * 32) >> 4), bV + ((kk * 2048) >> 4), kIdescPV,
                          kk > 0 ? 1u : acc0);
            tc_commit_pair(bVempty(s), 0x3);
            tc_commit_pair(bPempty(int(st)), 0x3);
          }
          __syncwarp();
          PD_TRM(4, t);
        };
        mbar_wait(bQ, 0);
        tc_fence_after();
        issue_s(0);
        if (nsteps > 1) issue_s(1);
        for (uint32_t t = 0; t < nsteps; ++t) {
          if (t + 2 < nsteps) {  // QK^T(t+2) as soon as the softmax has read S(t)
            mbar_wait(bSfree(int(t & 1)), (t >> 1) & 1);
            PD_TRM(0, t);
            issue_s(t + 2);
            PD_TRM(1, t);
          }
          issue_pv(t);
        }
        if (elect_one()) tc_commit_pair(bOfinal, 0x3);
        __syncwarp();
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ softmax: stage st, one warp per row
    const int st = warp >> 2;
    const int lg = warp & 3;
    const int row = lg * 32 + lane;  // TMEM lane = CTA row
    const bool upper = row >= 64;
    const uint32_t lane_off = uint32_t(lg * 32) << 16;
    const uint32_t scol = tmem + lane_off + C::kColS + 128u * st;
    const uint32_t ocol = tmem + lane_off + C::kColO + 128u * st;
    const uint32_t dense_bit = 1u << (22 + 2 * rank + (upper ? 1 : 0));
    const uint32_t pfull_remote_base = rank ? leader(bPfull(0)) : 0u;
    const uint32_t sfree_remote_base = rank ? leader(bSfree(0)) : 0u;
    uint8_t* const prow0 = gbase + (sP - base) + st * C::kPBytes + row * 128;  // + h * 16384
    const float sl2 = p.scale_log2;
    float m = -INFINITY, l = 0.f;
    for (uint32_t t = st; t < nsteps; t += 2) {
      const uint32_t e0 = __ldg(ent + 2 * t);
      const uint32_t e1 = 2 * t + 1 < count ? __ldg(ent + 2 * t + 1) : 0u;
      const bool d0 = (e0 & dense_bit) != 0, d1 = (e1 & dense_bit) != 0;  // warp-uniform
      mbar_wait(bSfull(st), (t >> 1) & 1);
      tc_fence_after();
      if (lane == 0 && lg == 0) PD_TRC(2 * st, t >> 1);
      // PV_st(t-2) must be done before P(t) overwrites its smem tile and O_st is
      // rescaled; waited before S is read so that no barrier sits between the
      // 128-value load and the exps (across one, ptxas parks S in local memory).
      if (t >= 2) {
        mbar_wait(bPempty(st), ((t >> 1) - 1) & 1);
        tc_fence_after();
      }
      float v[128];
      if (d0 || d1) {
        uint32_t a0[32], a1[32], a2[32], a3[32];
        tmem_ld32(scol, a0);
        tmem_ld32(scol + 32, a1);
        tmem_ld32(scol + 64, a2);
        tmem_ld32(scol + 96, a3);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          v[i] = __uint_as_float(a0[i]);
          v[32 + i] = __uint_as_float(a1[i]);
          v[64 + i] = __uint_as_float(a2[i]);
          v[96 + i] = __uint_as_float(a3[i]);
        }
      }
      bool need_o = false;
      float alpha = 1.f;
      if (d0 || d1) {
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
        const float mt2 = fmaxf(fmax3f(mx[0], mx[1], mx[2]), fmax3f(mx[3], mx[4], mx[15])) * sl2;
        if (mt2 > m + kRescaleThreshold) {
          need_o = m != -INFINITY;
          alpha = fast_exp2(m - mt2);
          l *= alpha;
          m = mt2;
        }
        const float2 sc2 = make_float2(sl2, sl2), nm2 = make_float2(-m, -m);
        float2 acc2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint8_t* const prow = prow0 + h * 16384;
          if (h == 0 ? d0 : d1) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {  // one 16-byte unit (8 keys) at a time: 4 live packed words
              uint32_t pk[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int j = 4 * u + i;
                const float2 x = __ffma2_rn(make_float2(v[64 * h + 2 * j], v[64 * h + 2 * j + 1]), sc2, nm2);
                float2 pp;
                if ((j & 7) < kPoly) {
                  pp = exp2_poly3_pair(x);
                } else {
                  pp = make_float2(fast_exp2(x.x), fast_exp2(x.y));
                }
                acc2[i & 1] = __fadd2_rn(acc2[i & 1], pp);
                pk[i] = pack_bf16x2(pp.x, pp.y);
              }
              *reinterpret_cast<uint4*>(prow + ((u ^ (row & 7)) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            }
          } else {
#pragma unroll
            for (int u = 0; u < 8; ++u)
              *reinterpret_cast<uint4*>(prow + ((u ^ (row & 7)) << 4)) = make_uint4(0, 0, 0, 0);
          }
        }
        const float2 a2 = __fadd2_rn(acc2[0], acc2[1]);
        l += a2.x + a2.y;
      } else {
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int u = 0; u < 8; ++u)
            *reinterpret_cast<uint4*>(prow0 + h * 16384 + ((u ^ (row & 7)) << 4)) = make_uint4(0, 0, 0, 0);
      }
      // S_st(t) has been consumed: QK^T(t+2) may overwrite it
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0)
          mbar_arrive(bSfree(st));
        else
          mbar_arrive_cluster(sfree_remote_base + 8u * st);
      }
      if (__any_sync(0xffffffffu, need_o)) {
        // O_s is quiescent: PV_s(t-2) completed (Pempty above).
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t o[32];
          tmem_ld32(ocol + c * 32, o);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st32(ocol + c * 32, o);
        }
        tmem_st_wait();
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // P (generic writes) -> tensor core
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0)
          mbar_arrive(bPfull(st));
        else
          mbar_arrive_cluster(pfull_remote_base + 8u * st);
      }
      if (lane == 0 && lg == 0) PD_TRC(2 * st + 1, t >> 1);
    }

    // ------------------------------------------------------------ epilogue: 64 columns per thread
    if (count > 0) {
      mbar_wait(bOfinal, 0);
      tc_fence_after();
    }
    mlbuf[st * 128 + row] = make_float2(m, l);
    named_bar_sync(1, 256);
    const float2 x0 = mlbuf[row], x1 = mlbuf[128 + row];
    const bool have1 = nsteps >= 2;  // stage 1 wrote O1
    const float m0 = x0.x, l0 = x0.y, m1 = x1.x, l1 = x1.y;
    const float mm = fmaxf(m0, have1 ? m1 : -INFINITY);
    float a0 = 0.f, a1 = 0.f, lt = 0.f;
    if (mm != -INFINITY) {
      a0 = m0 == -INFINITY ? 0.f : fast_exp2(m0 - mm);
      a1 = (!have1 || m1 == -INFINITY) ? 0.f : fast_exp2(m1 - mm);
      lt = l0 * a0 + (have1 ? l1 * a1 : 0.f);
    }
    const uint32_t qi = 2 * rank + (upper ? 1 : 0);
    const uint32_t token = myq[upper ? 1 : 0] * 64u + uint32_t(row & 63);
    const bool live = !((it.single >> qi) & 1u) && token < p.q_tokens;
    const float inv_l = lt > 0.f ? 1.f / lt : 0.f;
    const float lse_new = lt > 0.f ? (mm + log2f(lt)) * 0.6931471805599453f : -INFINITY;
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
      named_bar_sync(1, 256);  // both threads of the row read lse_acc before it is rewritten
    }
    bool live_out = live;
    __nv_bfloat16* const optr = out_row_ptr<128>(p, token, it.head, live_out);
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      const uint32_t col = 64u * st + 32u * cc;
      uint32_t x[32];
      if (count > 0) {
        uint32_t y[32];
        const uint32_t o0 = tmem + lane_off + C::kColO + col;
        tmem_ld32(o0, x);
        if (have1) tmem_ld32(o0 + 128, y);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          float r = __uint_as_float(x[i]) * a0;
          if (have1) r = fmaf(__uint_as_float(y[i]), a1, r);
          x[i] = __float_as_uint(r);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) x[i] = 0u;
      }
      if (!live) continue;
      const size_t orow = (size_t(token) * p.heads + it.head) * 128 + col;
      float r[32];
      if (acc) {
        float4* pa = reinterpret_cast<float4*>(p.o_acc + orow);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float4 a = pa[i];
          a.x = a.x * c_old + __uint_as_float(x[4 * i + 0]) * c_new;
          a.y = a.y * c_old + __uint_as_float(x[4 * i + 1]) * c_new;
          a.z = a.z * c_old + __uint_as_float(x[4 * i + 2]) * c_new;
          a.w = a.w * c_old + __uint_as_float(x[4 * i + 3]) * c_new;
          pa[i] = a;
          r[4 * i + 0] = a.x;
          r[4 * i + 1] = a.y;
          r[4 * i + 2] = a.z;
          r[4 * i + 3] = a.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = __uint_as_float(x[i]) * inv_l;
      }
      if ((!acc || (p.mode & kModeFinalize)) && live_out) {
        uint4* po = reinterpret_cast<uint4*>(optr + col);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          po[i] = make_uint4(pack_bf16x2(r[8 * i + 0], r[8 * i + 1]), pack_bf16x2(r[8 * i + 2], r[8 * i + 3]),
                             pack_bf16x2(r[8 * i + 4], r[8 * i + 5]), pack_bf16x2(r[8 * i + 6], r[8 * i + 7]));
      }
    }
    if (live && st == 0) {
      if (acc)
        p.lse_acc[lidx] = lse_out;
      else if (p.lse)
        p.lse[lidx] = lse_new;
    }
    if (p.out_peers) __threadfence_system();
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the leader's MMAs wrote into this CTA's TMEM / read its smem
  tc_fence_after();
  clock_probe_mark(p, 1);
  if (warp == 9) tmem_dealloc_pair(tmem, 512);
}

}  // namespace dbsp_dev
