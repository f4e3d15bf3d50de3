// K4, two-stage kernel with a split softmax (d=128): one CTA per SM, two
// 128-row Q tiles ("stages") of one head share one KV stream of 128-key steps
// (two dense 64-key blocks per tcgen05 QK^T), and every row's softmax is
// shared by TWO warps, one per 64-key block of the step.
//
// Why: in the two-stage kernel (attn_kernel_duo.cuh) each stage has one S
// buffer, so softmax -> PV -> next QK^T is a serial chain per stage, and its
// single softmax warp per SMSP ran at ~64% of the MUFU rate (2063 cycles per
// 128x128 step, profiles/r01_k4_analysis.md).  With two warps per SMSP on
// the same rows, the stage's softmax finishes in about half the time, so the
// other stage's MMAs (PV + QK^T, 1024+ cycles) cover it.
// Warp roles (640 threads, five warpgroups):
//   WG0..WG3 (warps 0-15)  softmax + epilogue; warp w: stage w/8, key half
//                          (w/4)%2, TMEM lanes 32*(w%4).  setmaxnreg 104.
//   WG4: warp 16 TMA producer, warp 17 MMA issuer of stage 0 (+ TMEM owner),
//        warp 18 MMA issuer of stage 1, warp 19 idle.  setmaxnreg 40.
// The two stages' exp phases alternate (SmDone barriers), so each runs alone
// on the MUFU while the tensor pipe works on the other stage.
// Row statistics: the two warps of a row exchange their partial row max
// through shared memory and a 64-thread named barrier each step, so both use
// the same running max m (and make the same lazy-rescale decision); each
// keeps the partial row sum of its half, added in the epilogue.
// TMEM: S_s [128s, 128s+128), O_s [256+128s, +128).  Warp half h writes its
// packed P over the first 32 of its own 64 S columns, so PV's A operand for
// k-step kk sits at column (kk/4)*64 + (kk%4)*8 of the stage's S region.
// Mask semantics follow the reference BlockMask (mask.hpp:18-20).
#pragma once

#include "attn_kernel.cuh"

namespace dbsp_dev {

constexpr int kThreadsDuo2 = 640;
#ifndef DBSP_DUO2_POLY
#define DBSP_DUO2_POLY 0
#endif
constexpr int kDuo2PolyPairs = DBSP_DUO2_POLY;  // exp2 pairs of every 8 on the FMA pipe

template <int kD>
struct Duo2Cfg {
  static constexpr int D = kD;
  static constexpr int kChunks = D / 64;          // 128-byte swizzle atoms along d
  static constexpr uint32_t kOHalf = D / 2;       // O columns per key-half warp
  static constexpr uint32_t kQStageBytes = 128u * D * 2u;
  static constexpr uint32_t kQBytes = 2u * kQStageBytes;
  static constexpr uint32_t kChunkBytes = 128u * 128u;  // 128 rows x 128 B
  static constexpr uint32_t kStepBytes = 128u * D * 2u;  // one 128-key K or V step
  static constexpr uint32_t kColS = 0, kColO = 256;  // O_s at kColO + D s
  static constexpr int kStages = 2;
  static constexpr int kNumBars = 4 * kStages + 10;
  static constexpr uint32_t kXBytes = 2u * 2u * 2u * 128u * 4u;  // [parity][stage][half][row] max
  static constexpr uint32_t kLBytes = 2u * 2u * 128u * 4u;        // [stage][half][row] sum / lse
  static constexpr uint32_t kSmemBytes =
      kQBytes + 2u * kStages * kStepBytes + kXBytes + kLBytes + 1024 + 8 * kNumBars + 16;
};

template <int kD>
__global__ void __launch_bounds__(kThreadsDuo2, 1)
    sparse_attn_fwd_duo2_kernel(const __grid_constant__ CUtensorMap tmQ,
                                const __grid_constant__ CUtensorMap tmK,
                                const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  using C = Duo2Cfg<kD>;
  constexpr int D = C::D;
  constexpr int NS = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);

  const uint32_t sQ = base;
  const uint32_t sK = base + C::kQBytes;
  const uint32_t sV = sK + NS * C::kStepBytes;
  float* xmax = reinterpret_cast<float*>(gbase + (sV + NS * C::kStepBytes - base));
  float* xsum = xmax + C::kXBytes / 4;
  const uint32_t sBar = sV + NS * C::kStepBytes + C::kXBytes + C::kLBytes;
  auto bKfull = [&](int s) { return sBar + 8u * s; };
  auto bVfull = [&](int s) { return sBar + 8u * (NS + s); };
  auto bKempty = [&](int s) { return sBar + 8u * (2 * NS + s); };
  auto bVempty = [&](int s) { return sBar + 8u * (3 * NS + s); };
  auto bSfull = [&](int st) { return sBar + 8u * (4 * NS + st); };
  auto bPfull = [&](int st) { return sBar + 8u * (4 * NS + 2 + st); };
  auto bQready = [&](int st) { return sBar + 8u * (4 * NS + 4 + st); };
  auto bOfinal = [&](int st) { return sBar + 8u * (4 * NS + 6 + st); };
  auto bSmDone = [&](int st) { return sBar + 8u * (4 * NS + 8 + st); };  // one phase per step
  const uint32_t sTmemSlot = sBar + 8u * C::kNumBars;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const WorkItem it = p.items[blockIdx.x];
  const uint32_t count = it.count;
  const uint32_t nsteps = (count + 1) / 2;
  clock_probe_mark(p, 0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(bKfull(s), 1);
      mbar_init(bVfull(s), 1);
      mbar_init(bKempty(s), 2);  // one commit per stage's MMA thread
      mbar_init(bVempty(s), 2);
    }
    for (int st = 0; st < 2; ++st) {
      mbar_init(bSfull(st), 1);
      mbar_init(bPfull(st), 8);  // 8 softmax warps per stage
      mbar_init(bQready(st), 1);
      mbar_init(bOfinal(st), 1);
      mbar_init(bSmDone(st), 8);
    }
    mbar_fence_init();
  }
  if (warp == 16 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
  }
  if (warp == 17) tmem_alloc(sTmemSlot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(gbase + (sTmemSlot - base));
  const uint32_t* ent = p.entries + it.begin;
  auto qblk = [&](int i) { return i == 0 ? it.qa : i == 1 ? it.qb : i == 2 ? it.pad0 : it.pad1; };

  if (warp >= 16) {
    setmaxnreg_dec<40>();
    if (warp == 16) {
      // ---------------------------------------------------------- producer
      if (lane == 0 && count > 0) {
        const uint64_t pol_kv = l2_policy_evict_last();
        const uint64_t pol_q = l2_policy_evict_first();
        const int head = int(it.head);
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
          if (t + 1 < nsteps) load_k(t + 1);
          const int s = int(t % NS);
          mbar_wait(bVempty(s), ((t / NS) & 1) ^ 1);
          load_step(&tmV, sV + s * C::kStepBytes, bVfull(s), t);
        }
      } else if (count > 0) {
        mbar_wait(bOfinal(1), 0);
      }
    } else if (warp <= 18) {
      // ---------------------------------------------------------- MMA issuer of stage (warp - 17)
      const int st = warp - 17;
      if (lane == 0 && count > 0) {
        constexpr uint32_t kIdescQK = idesc_bf16(128, 128, false, false);
        constexpr uint32_t kIdescPV = idesc_bf16(128, D, false, true);
        const uint32_t scol = tmem + C::kColS + 128u * st;
        const uint32_t ocol = tmem + C::kColO + uint32_t(D) * st;
        auto issue_s = [&](uint32_t t) {
          const int s = int(t % NS);
          mbar_wait(bKfull(s), (t / NS) & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint64_t bd = smem_desc_sw128(
                sK + s * C::kStepBytes + (kk >> 2) * C::kChunkBytes + (kk & 3) * 32, 16, 1024);
            const uint64_t ad = smem_desc_sw128(
                sQ + st * C::kQStageBytes + (kk >> 2) * C::kChunkBytes + (kk & 3) * 32, 16, 1024);
            mma_ss(scol, ad, bd, kIdescQK, kk > 0 ? 1u : 0u);
          }
          tc_commit(bSfull(st));
          tc_commit(bKempty(s));
          DBSP_TR(4 + 2 * st, t);
        };
        auto issue_pv = [&](uint32_t t) {
          const int s = int(t % NS);
          mbar_wait(bPfull(st), t & 1);
          mbar_wait(bVfull(s), (t / NS) & 1);
          tc_fence_after();
          DBSP_TR(5 + 2 * st, t);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint64_t bd = smem_desc_sw128(sV + s * C::kStepBytes + kk * 2048, C::kChunkBytes, 1024);
            mma_ts(ocol, scol + (kk >> 2) * 64 + (kk & 3) * 8, bd, kIdescPV, (t > 0 || kk > 0) ? 1u : 0u);
          }
          tc_commit(bVempty(s));
        };
        mbar_wait(bQready(st), 0);
        tc_fence_after();
        issue_s(0);
        for (uint32_t t = 0; t < nsteps; ++t) {
          issue_pv(t);
          if (t + 1 < nsteps) issue_s(t + 1);
        }
        tc_commit(bOfinal(st));
      } else if (count > 0) {
        mbar_wait(bOfinal(st), 0);
      }
    }
    __syncwarp();
  } else {
    // Registers come from the CTA's own pool (96/thread at launch): the 16
    // softmax warps may take only what WG4 gives back, 16*(104-96) <= 4*(96-40).
    setmaxnreg_inc<104>();
    // ------------------------------------------------------------ softmax: stage st, key half hf
    const int st = warp >> 3;
    const int hf = (warp >> 2) & 1;
    const int lg = warp & 3;
    const int row = lg * 32 + lane;      // TMEM lane = stage row
    const int bi = 2 * st + (row >> 6);  // quad row block (warp-uniform)
    const uint32_t token = qblk(bi) * 64u + uint32_t(row & 63);
    const bool padded = (it.single >> bi) & 1u;
    const uint32_t lane_off = uint32_t(lg * 32) << 16;
    const uint32_t scol = tmem + lane_off + C::kColS + 128u * st + 64u * hf;
    const uint32_t ocol = tmem + lane_off + C::kColO + uint32_t(D) * st + C::kOHalf * hf;
    const uint32_t bar_id = 1u + 4u * st + lg;  // the two warps (hf 0/1) of these rows
    const uint32_t dense_bit = 1u << (22 + bi);
    const float sl2 = p.scale_log2;
    float m = -INFINITY, l = 0.f;
    for (uint32_t t = 0; t < nsteps; ++t) {
      const uint32_t idx = 2 * t + hf;
      const uint32_t e = idx < count ? __ldg(ent + idx) : 0u;
      const bool dense = (e & dense_bit) != 0;  // warp-uniform: this warp's 64-key block
      mbar_wait(bSfull(st), t & 1);
      tc_fence_after();
      if (lane == 0 && hf == 0 && lg == 0) DBSP_TR(2 * st, t);
      // Pass 1: this half's row max.  S stays in TMEM and is read again for
      // the exps after the exchange, so no 64-value array lives across the
      // named barrier (that spilled).
      const uint32_t valid = ((e >> dbsp_core::kQuadValidShift) & 63u) + 1u;
      auto load_s = [&](float (&v)[64]) {
        uint32_t a0[32], a1[32];
        tmem_ld32(scol, a0);
        tmem_ld32(scol + 32, a1);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          v[i] = __uint_as_float(a0[i]);
          v[32 + i] = __uint_as_float(a1[i]);
        }
        if (valid < 64) {
#pragma unroll
          for (int i = 0; i < 64; ++i)
            if (uint32_t(i) >= valid) v[i] = -INFINITY;
        }
      };
      float lmax = -INFINITY;
      if (dense) {
        float v[64];
        load_s(v);
        float mx[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          mx[a] = fmax3f(v[8 * a], v[8 * a + 1], v[8 * a + 2]);
          mx[a] = fmax3f(mx[a], v[8 * a + 3], v[8 * a + 4]);
          mx[a] = fmax3f(mx[a], v[8 * a + 5], v[8 * a + 6]);
          mx[a] = fmaxf(mx[a], v[8 * a + 7]);
        }
        lmax = fmaxf(fmax3f(mx[0], mx[1], mx[2]), fmax3f(fmax3f(mx[3], mx[4], mx[5]), mx[6], mx[7]));
      }
      // exchange the partial max with the other half's warp (same rows)
      float* xm = xmax + ((t & 1) * 2 + st) * 256;
      xm[hf * 128 + row] = lmax;
      named_bar_sync(bar_id, 64);
      const float mt2 = fmaxf(lmax, xm[(1 - hf) * 128 + row]) * sl2;
      const bool resc = mt2 > m + kRescaleThreshold;
      const bool need_o = resc && (m != -INFINITY);
      float alpha = 1.f;
      if (resc) {
        alpha = fast_exp2(m - mt2);
        l *= alpha;
        m = mt2;
      }
      // Ping-pong of the exp phase: stage 1's exps of step t follow stage 0's,
      // and stage 0's of step t+1 follow stage 1's of step t, so the two never
      // share the SMSPs' MUFU; loads and row max overlap the other stage.
      if (st == 1)
        mbar_wait(bSmDone(0), t & 1);
      else if (t > 0)
        mbar_wait(bSmDone(1), (t - 1) & 1);
      if (dense) {
        float v[64];
        load_s(v);  // pass 2
        const float2 sc2 = make_float2(sl2, sl2), nm2 = make_float2(-m, -m);
        float2 acc2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int j = 16 * c + i;
            const float2 x = __ffma2_rn(make_float2(v[2 * j], v[2 * j + 1]), sc2, nm2);
            float2 pp;
            if ((j & 7) < kDuo2PolyPairs) {
              pp = exp2_poly3_pair(x);
            } else {
              pp = make_float2(fast_exp2(x.x), fast_exp2(x.y));
            }
            acc2[i & 1] = __fadd2_rn(acc2[i & 1], pp);
            pk[i] = pack_bf16x2(pp.x, pp.y);
          }
          tmem_st16(scol + 16 * c, pk);
        }
        const float2 a2 = __fadd2_rn(acc2[0], acc2[1]);
        l += a2.x + a2.y;
      } else {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) pk[i] = 0u;
        tmem_st16(scol, pk);
        tmem_st16(scol + 16, pk);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(bSmDone(st));
      if (__any_sync(0xffffffffu, need_o)) {
        // O_s is quiescent: S_s(t) (complete) was issued after PV_s(t-1).
#pragma unroll
        for (int c = 0; c < int(C::kOHalf / 32); ++c) {
          uint32_t o[32];
          tmem_ld32(ocol + c * 32, o);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st32(ocol + c * 32, o);
        }
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0 && hf == 0 && lg == 0) DBSP_TR(2 * st + 1, t);
      if (lane == 0) mbar_arrive(bPfull(st));
    }

    // ------------------------------------------------------------ epilogue (this warp's 64 columns)
    if (count > 0) {
      mbar_wait(bOfinal(st), 0);
      tc_fence_after();
    }
    float* xs = xsum + st * 256;
    xs[hf * 128 + row] = l;
    named_bar_sync(bar_id, 64);
    const float lt = l + xs[(1 - hf) * 128 + row];
    const bool live = !padded && token < p.q_tokens;
    const float inv_l = lt > 0.f ? 1.f / lt : 0.f;
    const float lse_new = lt > 0.f ? (m + log2f(lt)) * 0.6931471805599453f : -INFINITY;
    const size_t orow = (size_t(token) * p.heads + it.head) * D + C::kOHalf * hf;
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
      named_bar_sync(bar_id, 64);  // both halves read lse_acc before half 0 rewrites it
    }
    bool live_out = live;
    __nv_bfloat16* const optr = out_row_ptr<D>(p, token, it.head, live_out) + C::kOHalf * hf;
    const bool write_bf16 = !acc || (p.mode & kModeFinalize);
#pragma unroll
    for (int c = 0; c < int(C::kOHalf / 32); ++c) {
      uint32_t o[32];
      if (count > 0) {
        tmem_ld32(ocol + c * 32, o);
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
      if (write_bf16 && live_out) {
        uint4* po = reinterpret_cast<uint4*>(optr + c * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          po[i] = make_uint4(pack_bf16x2(r[8 * i + 0], r[8 * i + 1]), pack_bf16x2(r[8 * i + 2], r[8 * i + 3]),
                             pack_bf16x2(r[8 * i + 4], r[8 * i + 5]), pack_bf16x2(r[8 * i + 6], r[8 * i + 7]));
      }
    }
    if (live && hf == 0) {
      if (acc)
        p.lse_acc[lidx] = lse_out;
      else if (p.lse)
        p.lse[lidx] = lse_new;
    }
    if (p.out_peers) __threadfence_system();
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 17) tmem_dealloc(tmem, 512);
  clock_probe_mark(p, 1);
}

}  // namespace dbsp_dev
