// K4, d=128: CTA pair (tcgen05 cta_group::2) x two split-KV stages per CTA,
// two softmax warps per row, P staged in shared memory.
//
// A cluster of two CTAs on the two SMs of a TPC runs one quad work item
// (schedule.hpp kSchedQuad|kSchedKey128|kSchedCtaPair): four 64-row Q blocks
// of one head, CTA rank r owning blocks 2r, 2r+1 (128 rows), against the union
// of their dense KV blocks, walked in 128-key steps (two entries per step).
// The steps alternate between two stages of each CTA -- stage 0 takes the even
// steps, stage 1 the odd ones -- each with its own S and O in TMEM and its own
// running (m, l); the epilogue merges the two partial results row by row.
//
// The leader CTA issues M=256 N=128 MMAs for both CTAs:
//   S_s = Q K^T   SS  A: each CTA's own Q (smem); B: CTA r holds the 64 keys
//                     of entry 2t+r (one KV block)
//   O_s += P_s V  SS  A: each CTA's own P (smem, written by the softmax);
//                     B: CTA r holds columns [64r, 64r+64) of V, 128 keys
// Each SM stages only its half of every K / V step, so the B operand bytes per
// SM are half those of a one-CTA M=128 tile.
//
// The softmax warps release S(t) as soon as they have read it (Sfree), write
// P(t) to a shared-memory tile in the 128-byte-swizzled K-major layout, and
// the leader issues QK^T(t+2) right after Sfree(t), ahead of PV(t).  The MMAs
// leave the per-stage chain; what remains per stage is the softmax.  The O
// rescale and the P(t) store wait for PV(t-2) (Pempty), which S(t)'s
// completion no longer implies.
//
// Every row's softmax is shared by two warps (one per 64-key block of the
// step).  They exchange their partial row max through shared memory and a
// 64-thread named barrier, so both use the same running max m (same lazy
// rescale decision); each keeps the partial row sum of its half.
// Warp roles (640 threads, five warpgroups, one CTA per SM):
//   WG0..WG3 (warps 0-15)  softmax + epilogue; warp w: stage w/8, key half
//                          (w/4)%2, TMEM lanes 32*(w%4).  setmaxnreg 104.
//   WG4: warp 16 TMA producer (both CTAs), warp 17 TMEM owner + MMA issuer
//        (leader), warps 18-19 idle.  setmaxnreg 64.
// Epilogue: the four threads of a row (stage x half) exchange (m, l) and each
// writes 32 of the 128 output columns of O = (a0 O_0 + a1 O_1) / L.
// TMEM (512 columns): S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512).
// The design history (one warp per row, P over S in TMEM, persistence, ...)
// with the measured numbers of each rejected variant is in DESIGN.md §3 and
// profiles/README.md.
// Mask semantics follow the reference BlockMask (mask.hpp:18-20).
#pragma once

#include "attn_kernel.cuh"

namespace dbsp_dev {

constexpr int kThreadsPd3 = 640;

// DBSP_TRACE builds (tests/trace_kernel.py): DBSP_TRACE_FINE records the
// stage-0 softmax phases, DBSP_TRACE_MMA the leader's MMA thread, the default
// trace the per-stage step boundaries.
#if defined(DBSP_TRACE_MMA)
#define PD_TR(ev, j) \
  do {               \
  } while (0)
#define PD_TRC(ev, j) \
  do {                \
  } while (0)
#define PD_TRM(ev, j) DBSP_TR(ev, j)
#elif defined(DBSP_TRACE_FINE)
#define PD_TR(ev, j) DBSP_TR(ev, j)
#define PD_TRC(ev, j) \
  do {                \
  } while (0)
#define PD_TRM(ev, j) \
  do {                \
  } while (0)
#else
#define PD_TR(ev, j) \
  do {               \
  } while (0)
#define PD_TRC(ev, j) DBSP_TR(ev, j)
#define PD_TRM(ev, j) \
  do {                \
  } while (0)
#endif

struct Pd3Cfg {
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
  static constexpr uint32_t kXBytes = 2u * 2u * 2u * 128u * 4u;  // [parity][stage][half][row] partial max
  static constexpr uint32_t kMlBytes = 2u * 2u * 128u * 8u;      // [stage][half][row] (m, l)
  static constexpr uint32_t kSmemBytes =
      kQBytes + kStages * (kKStep + kVStep) + 2 * kPBytes + kXBytes + kMlBytes + 1024 + 8 * kNumBars + 16;
};

template <int kPoly>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsPd3, 1)
    sparse_attn_fwd_pd3_kernel(const __grid_constant__ CUtensorMap tmQ,
                               const __grid_constant__ CUtensorMap tmK,
                               const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  using C = Pd3Cfg;
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
  // slots 4*NS+6, 4*NS+7 are unused (kept so the barrier layout matches the traces in profiles/)
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
#ifdef DBSP_TRACE_CTA
  const unsigned long long c_start = clock64();
  if (threadIdx.x == 0 && rank == 0 && p.trace) p.trace[4 * (blockIdx.x >> 1)] = globaltimer_ns();
#endif

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(bKfull(s), 1);
      mbar_init(bVfull(s), 1);
      mbar_init(bKempty(s), 1);
      mbar_init(bVempty(s), 1);
    }
    for (int st = 0; st < 2; ++st) {
      mbar_init(bSfull(st), 1);
      mbar_init(bPfull(st), 16);  // 8 softmax warps of the stage in each CTA of the pair
    }
    mbar_init(bQ, 1);
    mbar_init(bOfinal, 1);
    for (int st = 0; st < 2; ++st) {
      mbar_init(bSfree(st), 16);  // 8 softmax warps of the stage in each CTA of the pair
      mbar_init(bPempty(st), 1);
    }
    mbar_fence_init();
  }
  if (warp == 16 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
  }
  if (warp == 17) tmem_alloc_pair(sTmemSlot, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(gbase + (sTmemSlot - base));
  const uint32_t* ent = p.entries + it.begin;

  if (warp >= 16) {
    // Registers come from the CTA's own pool (96/thread at launch): the 16
    // softmax warps may take only what WG4 gives back, 16*(104-96) <= 4*(96-64);
    // 64 (not less) keeps the MMA issuer's descriptors out of local memory.
    setmaxnreg_dec<64>();
    if (warp == 16) {
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
    } else if (warp == 17) {
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
    setmaxnreg_inc<104>();
    // ------------------------------------------------------------ softmax: stage st, key half hf
    const int st = warp >> 3;
    const int hf = (warp >> 2) & 1;
    const int lg = warp & 3;
    const int row = lg * 32 + lane;  // TMEM lane = CTA row
    const bool upper = row >= 64;
    const uint32_t lane_off = uint32_t(lg * 32) << 16;
    const uint32_t scol = tmem + lane_off + C::kColS + 128u * st + 64u * hf;
    const uint32_t ocol = tmem + lane_off + C::kColO + 128u * st + 64u * hf;
    const uint32_t bar_id = 1u + 4u * st + lg;  // the two warps (hf 0/1) of these rows
    const uint32_t dense_bit = 1u << (22 + 2 * rank + (upper ? 1 : 0));
    const uint32_t pfull_remote_base = rank ? leader(bPfull(0)) : 0u;
    const uint32_t sfree_remote_base = rank ? leader(bSfree(0)) : 0u;
    uint8_t* const prow0 = gbase + (sP - base) + hf * 16384 + row * 128;  // + st * kPBytes
    const float sl2 = p.scale_log2;
    float m = -INFINITY, l = 0.f;
    for (uint32_t t = st; t < nsteps; t += 2) {
      const uint32_t idx = 2 * t + hf;
      const uint32_t e = idx < count ? __ldg(ent + idx) : 0u;
      const bool dense = (e & dense_bit) != 0;  // warp-uniform: this warp's 64-key block
      mbar_wait(bSfull(st), (t >> 1) & 1);
      tc_fence_after();
      if (lane == 0 && hf == 0 && lg == 0) PD_TRC(2 * st, t >> 1);
      // DBSP_TRACE_FINE (warp 0): 0 start, 2 S loaded, 6 max exchanged, 3 S reloaded
      // and released, 5 exps done, 4 P stored (after the PV(t-2) wait), 1 P arrived
      const bool tr0 = lane == 0 && warp == 0;
      if (tr0) PD_TR(0, t >> 1);
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
      auto release_s = [&]() {  // S_st(t) is in registers: QK^T(t+2) may overwrite it
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (rank == 0)
            mbar_arrive(bSfree(st));
          else
            mbar_arrive_cluster(sfree_remote_base + 8u * st);
        }
      };
      // PV_st(t-2) must be done before P(t) overwrites its smem tile and
      // before O_st is rescaled.
      auto wait_pv = [&]() {
        if (t >= 2) {
          mbar_wait(bPempty(st), ((t >> 1) - 1) & 1);
          tc_fence_after();
        }
      };
      // Pass 1 reads S for the row max, pass 2 again for the exps: holding the
      // 64 values across the max exchange instead (one read, S released before
      // the exchange) spills at 104 registers and measured 1.8x slower.
      float v[64];
      float lmax = -INFINITY;
      if (dense) {
        load_s(v);
        if (tr0) PD_TR(2, t >> 1);
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
      float* xm = xmax + (((t >> 1) & 1) * 2 + st) * 256;
      xm[hf * 128 + row] = lmax;
      named_bar_sync(bar_id, 64);
      const float mt2 = fmaxf(lmax, xm[(1 - hf) * 128 + row]) * sl2;
      if (tr0) PD_TR(6, t >> 1);
      const bool resc = mt2 > m + kRescaleThreshold;
      const bool need_o = resc && (m != -INFINITY);
      float alpha = 1.f;
      if (resc) {
        alpha = fast_exp2(m - mt2);
        l *= alpha;
        m = mt2;
      }
      uint8_t* const prow = prow0 + st * C::kPBytes;
      if (dense) {
        load_s(v);  // pass 2
        release_s();
        if (tr0) PD_TR(3, t >> 1);
#ifdef DBSP_PD3_EARLY_PVWAIT
        wait_pv();
#endif
        // The exps run BEFORE the wait for PV(t-2): only the P store and the O
        // rescale need it, so the wait overlaps the MUFU work instead of
        // preceding it (P stays in registers, 32 packed words).
        const float2 sc2 = make_float2(sl2, sl2), nm2 = make_float2(-m, -m);
        float2 acc2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        uint32_t pk[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float2 x = __ffma2_rn(make_float2(v[2 * j], v[2 * j + 1]), sc2, nm2);
          float2 pp;
          if ((j & 7) < kPoly) {
            pp = exp2_poly3_pair(x);
          } else {
            pp = make_float2(fast_exp2(x.x), fast_exp2(x.y));
          }
          acc2[j & 1] = __fadd2_rn(acc2[j & 1], pp);
          pk[j] = pack_bf16x2(pp.x, pp.y);
        }
        if (tr0) PD_TR(5, t >> 1);
#ifndef DBSP_PD3_EARLY_PVWAIT
        wait_pv();
#endif
#pragma unroll
        for (int u = 0; u < 8; ++u)
          *reinterpret_cast<uint4*>(prow + ((u ^ (row & 7)) << 4)) =
              make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        const float2 a2 = __fadd2_rn(acc2[0], acc2[1]);
        l += a2.x + a2.y;
      } else {
        release_s();
        if (tr0) PD_TR(3, t >> 1);
        wait_pv();
#pragma unroll
        for (int u = 0; u < 8; ++u) *reinterpret_cast<uint4*>(prow + ((u ^ (row & 7)) << 4)) = make_uint4(0, 0, 0, 0);
      }
      __syncwarp();
      if (tr0) PD_TR(4, t >> 1);
      if (__any_sync(0xffffffffu, need_o)) {
        // O_s is quiescent: PV_s(t-2) completed (wait_pv).
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t o[32];
          tmem_ld32(ocol + c * 32, o);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st32(ocol + c * 32, o);
        }
        tmem_st_wait();  // the only TMEM stores of the step
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
      if (lane == 0 && hf == 0 && lg == 0) PD_TRC(2 * st + 1, t >> 1);
      if (tr0) PD_TR(1, t >> 1);
    }

    // ------------------------------------------------------------ epilogue: 32 columns per thread
    if (count > 0) {
      mbar_wait(bOfinal, 0);
      tc_fence_after();
    }
    mlbuf[(st * 2 + hf) * 128 + row] = make_float2(m, l);
    const uint32_t ebar = 9u + lg;  // the four warps (stage x half) of these rows
    named_bar_sync(ebar, 128);
    const float2 x00 = mlbuf[0 * 128 + row], x01 = mlbuf[1 * 128 + row];
    const float2 x10 = mlbuf[2 * 128 + row], x11 = mlbuf[3 * 128 + row];
    const float m0 = x00.x, l0 = x00.y + x01.y, m1 = x10.x, l1 = x10.y + x11.y;
    const bool have1 = nsteps >= 2;  // stage 1 wrote O1
    const float mm = fmaxf(m0, have1 ? m1 : -INFINITY);
    float a0 = 0.f, a1 = 0.f, lt = 0.f;
    if (mm != -INFINITY) {
      a0 = m0 == -INFINITY ? 0.f : fast_exp2(m0 - mm);
      a1 = (!have1 || m1 == -INFINITY) ? 0.f : fast_exp2(m1 - mm);
      lt = l0 * a0 + (have1 ? l1 * a1 : 0.f);
    }
    const uint32_t cc = 2u * st + hf;  // this thread's 32-column chunk of the row
    const uint32_t qi = 2 * rank + (upper ? 1 : 0);
    const uint32_t token = myq[upper ? 1 : 0] * 64u + uint32_t(row & 63);
    const bool live = !((it.single >> qi) & 1u) && token < p.q_tokens;
    const float inv_l = lt > 0.f ? 1.f / lt : 0.f;
    const float lse_new = lt > 0.f ? (mm + log2f(lt)) * 0.6931471805599453f : -INFINITY;
    const size_t orow = (size_t(token) * p.heads + it.head) * 128 + 32u * cc;
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
      named_bar_sync(ebar, 128);  // every thread of the row read lse_acc before it is rewritten
    }
    uint32_t x[32];
    if (count > 0) {
      uint32_t y[32];
      const uint32_t o0 = tmem + lane_off + C::kColO + 32u * cc;
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
    if (live) {
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
      bool live_out = live;
      __nv_bfloat16* const optr = out_row_ptr<128>(p, token, it.head, live_out) + 32u * cc;
      if ((!acc || (p.mode & kModeFinalize)) && live_out) {
        uint4* po = reinterpret_cast<uint4*>(optr);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          po[i] = make_uint4(pack_bf16x2(r[8 * i + 0], r[8 * i + 1]), pack_bf16x2(r[8 * i + 2], r[8 * i + 3]),
                             pack_bf16x2(r[8 * i + 4], r[8 * i + 5]), pack_bf16x2(r[8 * i + 6], r[8 * i + 7]));
      }
      if (cc == 0) {
        if (acc)
          p.lse_acc[lidx] = lse_out;
        else if (p.lse)
          p.lse[lidx] = lse_new;
      }
    }
    if (p.out_peers) __threadfence_system();
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the leader's MMAs wrote into this CTA's TMEM / read its smem
  tc_fence_after();
  clock_probe_mark(p, 1);
#ifdef DBSP_TRACE_CTA
  if (threadIdx.x == 0 && rank == 0 && p.trace) {
    p.trace[4 * (blockIdx.x >> 1) + 1] = globaltimer_ns();
    p.trace[4 * (blockIdx.x >> 1) + 2] = smid();
    p.trace[4 * (blockIdx.x >> 1) + 3] = clock64() - c_start;
  }
#endif
  if (warp == 17) tmem_dealloc_pair(tmem, 512);
}

}  // namespace dbsp_dev
