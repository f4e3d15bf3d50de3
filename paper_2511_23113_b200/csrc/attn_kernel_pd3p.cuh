// K4, d=128: persistent form of attn_kernel_pd3.cuh (CTA pair x two split-KV
// stages, P in smem).  Each cluster loops over quad items taken from a global
// counter in the schedule's heavy-first order, so the next item's Q load, K/V
// loads and first QK^T overlap the current item's epilogue; the one-item-per-
// cluster kernel exposes them (the same change took the single-CTA quad kernel
// from 6.67 to 6.28 ms on Wan, interleaved A/B).
// Hand-off: the leader's producer fetches the item id and publishes it in a
// 2-slot ring in both CTAs (remote store + release.cluster arrive); every role
// of both CTAs reads the ids in order and releases the slot (ItemEmpty, in the
// leader).  Barrier phases run on cumulative counters: K/V ring steps, per-
// stage S/P uses, and non-empty items (Q full, Qfree after an item's last
// QK^T, Ofinal after its last PV, Odrained after both CTAs' epilogues read O).
// Warp roles, TMEM and the epilogue are those of attn_kernel_pd3.cuh; setmaxnreg
// 112/32 (at 104 the item-loop state spills the softmax: 9.4 ms on Wan).
// Status: parity-green, opt-in (schedule flags 217).  With the softmax warps'
// item state in shared memory: Wan 6.19 vs 6.26 ms for the non-persistent
// kernel (short items gain), HunyuanVideo 46.2 vs 45.3 (long items lose).
// Mask semantics follow the reference BlockMask (mask.hpp:18-20).
#pragma once

#include "attn_kernel_pd3.cuh"

namespace dbsp_dev {

struct Pd3pCfg {
  static constexpr int D = 128;
  static constexpr uint32_t kQBytes = 128u * 128u * 2u;
  static constexpr uint32_t kQChunk = 128u * 128u;
  static constexpr uint32_t kKStep = 64u * 128u * 2u;
  static constexpr uint32_t kKChunk = 64u * 128u;
  static constexpr uint32_t kVStep = 128u * 64u * 2u;
  static constexpr uint32_t kPBytes = 128u * 128u * 2u;  // one stage's P: 2 chunks of 64 keys
  static constexpr int kStages = 3;
  static constexpr uint32_t kColS = 0, kColO = 256;
  static constexpr int kItemSlots = 2;
  static constexpr int kNumBars = 4 * kStages + 2 + 2 + 2 + 2 + 2 + 2 + 2 + 2 * kItemSlots;
  static constexpr uint32_t kXBytes = 2u * 2u * 2u * 128u * 4u;  // [parity][stage][half][row] partial max
  static constexpr uint32_t kMlBytes = 2u * 2u * 2u * 128u * 8u;  // [item parity][stage][half][row] (m, l)
  static constexpr uint32_t kSmemBytes =
      kQBytes + kStages * (kKStep + kVStep) + 2 * kPBytes + kXBytes + kMlBytes + 1024 + 8 * kNumBars + 16 + 8 * kItemSlots +
      16 * 16;  // per softmax warp: {item count, item id, non-empty items}
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsPd2, 1)
    sparse_attn_fwd_pd3p_kernel(const __grid_constant__ CUtensorMap tmQ,
                                const __grid_constant__ CUtensorMap tmK,
                                const __grid_constant__ CUtensorMap tmV, const AttnParams p,
                                uint32_t n_items) {
  constexpr int kPoly = 0;
  constexpr bool kAltExp = false;
  using C = Pd3pCfg;
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
  const uint32_t bQfree = sBar + 8u * (4 * NS + 12);      // an item's last QK^T done (both CTAs)
  const uint32_t bOdrained = sBar + 8u * (4 * NS + 13);   // both CTAs' epilogues read O (leader)
  auto bItemEmpty = [&](int k) { return sBar + 8u * (4 * NS + 14 + C::kItemSlots + k); };  // leader
  const uint32_t sTmemSlot = sBar + 8u * C::kNumBars;
  const uint32_t sRing = sTmemSlot + 16;  // kItemSlots x {item id, sequence}
  const uint32_t sWst = sRing + 8u * C::kItemSlots;  // softmax warps' item-loop state

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  auto leader = [&](uint32_t local_bar) { return mapa_shared(local_bar, 0); };
  // Consumers' side of the item ring: slot k holds {id, k + 1} written by the
  // leader's producer with one 64-bit store (local and, for the peer, remote),
  // so the sequence number and the id arrive together and no release.cluster
  // fence is needed; consumers spin on the sequence, read the id and release
  // the slot (ItemEmpty, in the leader).
  auto take_item = [&](uint32_t k) -> uint32_t {
    const int slot = int(k % C::kItemSlots);
    uint32_t id, seq;
    for (;;) {
      uint64_t w;
      asm volatile("ld.volatile.shared.b64 %0, [%1];" : "=l"(w) : "r"(sRing + 8u * slot) : "memory");
      id = uint32_t(w);
      seq = uint32_t(w >> 32);
      if (seq == k + 1) break;
      __nanosleep(32);
    }
    __syncwarp();
    if (lane == 0) {
      if (rank == 0)
        mbar_arrive(bItemEmpty(slot));
      else
        mbar_arrive_cluster(leader(bItemEmpty(slot)));
    }
    return id;
  };
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
      mbar_init(bPfull(st), 16);  // 8 softmax warps of the stage in each CTA of the pair
    }
    mbar_init(bQ, 1);
    mbar_init(bOfinal, 1);
    mbar_init(bSmDone(0), 8);  // the stage's softmax warps of this CTA
    mbar_init(bSmDone(1), 8);
    mbar_init(bQfree, 1);
    mbar_init(bOdrained, 32);  // 16 softmax warps in each CTA of the pair
    for (int k = 0; k < C::kItemSlots; ++k) {
      mbar_init(bItemEmpty(k), 34);  // 16 + 16 softmax warps, the MMA warp, the peer's producer
      asm volatile("st.shared.b64 [%0], %1;" ::"r"(sRing + 8u * k), "l"(0ull) : "memory");
    }
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

  if (warp >= 16) {
    // Registers come from the CTA's own pool (96/thread at launch): the 16
    // softmax warps may take only what WG4 gives back, 16*(104-96) <= 4*(96-64);
    // 64 (not less) keeps the MMA issuer's descriptors out of local memory.
    setmaxnreg_dec<32>();
    if (warp == 16) {
      // ---------------------------------------------------------- producer (both CTAs)
      if (lane == 0) {
        const uint64_t pol_q = l2_policy_evict_first();
        const uint64_t pol_kv = l2_policy_evict_last();
        uint32_t gs = 0, nz = 0;  // K/V ring steps and non-empty items so far
        for (uint32_t k = 0;; ++k) {
          const int slot = int(k % C::kItemSlots);
          uint32_t id;
          if (rank == 0) {
            mbar_wait(bItemEmpty(slot), ((k / C::kItemSlots) & 1) ^ 1);
            id = atomicAdd(p.item_counter, 1u);
            const uint32_t a = sRing + 8u * slot;
            const uint64_t w = uint64_t(k + 1) << 32 | id;  // one single-copy-atomic 64-bit word
            asm volatile("st.shared.b64 [%0], %1;" ::"r"(a), "l"(w) : "memory");
            asm volatile("st.shared::cluster.b64 [%0], %1;" ::"r"(mapa_shared(a, 1)), "l"(w) : "memory");
          } else {
            uint32_t seq;
            for (;;) {
              uint64_t w;
              asm volatile("ld.volatile.shared.b64 %0, [%1];" : "=l"(w) : "r"(sRing + 8u * slot) : "memory");
              id = uint32_t(w);
              seq = uint32_t(w >> 32);
              if (seq == k + 1) break;
              __nanosleep(32);
            }
            mbar_arrive_cluster(leader(bItemEmpty(slot)));
          }
          if (id >= n_items) break;
          const WorkItem it = p.items[id];
          const uint32_t count = it.count;
          if (count == 0) continue;
          const uint32_t nsteps = (count + 1) / 2;
          const uint32_t myq[2] = {rank ? it.pad0 : it.qa, rank ? it.pad1 : it.qb};
          const uint32_t* ent = p.entries + it.begin;
          const int head = int(it.head);
          auto kv_of = [&](uint32_t t, uint32_t h) {
            const uint32_t j = 2 * t + h < count ? 2 * t + h : 2 * t;
            return int(__ldg(ent + j) & dbsp_core::kEntryKvMask);
          };
          auto load_k = [&](uint32_t t) {
            const uint32_t g = gs + t;
            const int s = int(g % NS);
            mbar_wait(bKempty(s), ((g / NS) & 1) ^ 1);
            const int kv = kv_of(t, rank);
            if (rank == 0) mbar_expect_tx(bKfull(s), 2 * C::kKStep);
#pragma unroll
            for (int c = 0; c < 2; ++c)
              tma_load_3d_pair(sK + s * C::kKStep + c * C::kKChunk, &tmK, c * 64, head, kv * 64,
                               leader(bKfull(s)), pol_kv);
          };
          load_k(0);
          if (nsteps > 1) load_k(1);
          if (nz > 0) mbar_wait(bQfree, (nz - 1) & 1);  // the previous item's QK^T are done
          if (rank == 0) mbar_expect_tx(bQ, 2 * C::kQBytes);
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            tma_load_3d_pair(sQ + c * C::kQChunk, &tmQ, c * 64, head, int(myq[0]) * 64, leader(bQ), pol_q);
            tma_load_3d_pair(sQ + c * C::kQChunk + 8192, &tmQ, c * 64, head, int(myq[1]) * 64, leader(bQ),
                             pol_q);
          }
          for (uint32_t t = 0; t < nsteps; ++t) {
            if (t + 2 < nsteps) load_k(t + 2);
            const uint32_t g = gs + t;
            const int s = int(g % NS);
            mbar_wait(bVempty(s), ((g / NS) & 1) ^ 1);
            if (rank == 0) mbar_expect_tx(bVfull(s), 2 * C::kVStep);
#pragma unroll
            for (int h = 0; h < 2; ++h)
              tma_load_3d_pair(sV + s * C::kVStep + h * 8192, &tmV, int(rank) * 64, head, kv_of(t, h) * 64,
                               leader(bVfull(s)), pol_kv);
          }
          gs += nsteps;
          ++nz;
        }
      }
    } else if (warp == 17) {
      // ---------------------------------------------------------- MMA issuer (leader only)
      if (rank == 0) {
        constexpr uint32_t kIdescQK = idesc_bf16(256, 128, false, false);
        constexpr uint32_t kIdescPV = idesc_bf16(256, 128, false, true);
        const uint64_t dQ = smem_desc_sw128(sQ, 16, 1024);
        const uint64_t dK = smem_desc_sw128(sK, 16, 1024);
        const uint64_t dP = smem_desc_sw128(sP, 16, 1024);
        const uint64_t dV = smem_desc_sw128(sV, 16384, 1024);
        uint32_t gs = 0, nz = 0, gu[2] = {0, 0};  // ring steps, non-empty items, per-stage S/P uses
        for (uint32_t k = 0;; ++k) {
          const uint32_t id = take_item(k);
          if (id >= n_items) break;
          const uint32_t count = p.items[id].count;
          if (count == 0) continue;
          const uint32_t nsteps = (count + 1) / 2;
          auto issue_s = [&](uint32_t t) {
            const uint32_t g = gs + t;
            const int s = int(g % NS);
            const uint32_t st = t & 1u;
            mbar_wait(bKfull(s), (g / NS) & 1);
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
              if (t + 1 == nsteps) tc_commit_pair(bQfree, 0x3);  // the item's last QK^T: Q may be replaced
            }
            __syncwarp();
          };
          auto issue_pv = [&](uint32_t t) {
            const uint32_t g = gs + t;
            const int s = int(g % NS);
            const uint32_t st = t & 1u;
            const uint32_t u = gu[st] + (t >> 1);
            mbar_wait(bPfull(int(st)), u & 1);
            mbar_wait(bVfull(s), (g / NS) & 1);
            if (t == 0 && nz > 0) mbar_wait(bOdrained, (nz - 1) & 1);  // the previous item's O was read
            tc_fence_after();
            const uint64_t aP = dP + ((st * C::kPBytes) >> 4);
            const uint64_t bV = dV + ((uint32_t(s) * C::kVStep) >> 4);
            const uint32_t ocol = tmem + C::kColO + 128u * st;
            const uint32_t acc0 = t >= 2 ? 1u : 0u;
            if (elect_one()) {
#pragma unroll
              for (int kk = 0; kk < 8; ++kk)
                mma_ss_pair(ocol, aP + (((kk >> 2) * 16384 + (kk & 3) * 32) >> 4), bV + ((kk * 2048) >> 4),
                            kIdescPV, kk > 0 ? 1u : acc0);
              tc_commit_pair(bVempty(s), 0x3);
              tc_commit_pair(bPempty(int(st)), 0x3);
            }
            __syncwarp();
          };
          mbar_wait(bQ, nz & 1);
          tc_fence_after();
#pragma unroll
          for (uint32_t t0 = 0; t0 < 2; ++t0) {
            if (t0 >= nsteps) break;
            if (gu[t0] > 0) mbar_wait(bSfree(int(t0)), (gu[t0] - 1) & 1);  // last use of S_t0 released
            issue_s(t0);
          }
          for (uint32_t t = 0; t < nsteps; ++t) {
            if (t + 2 < nsteps) {  // QK^T(t+2) as soon as the softmax has read S(t)
              mbar_wait(bSfree(int(t & 1)), (gu[t & 1] + (t >> 1)) & 1);
              issue_s(t + 2);
            }
            issue_pv(t);
          }
          if (elect_one()) tc_commit_pair(bOfinal, 0x3);
          __syncwarp();
          gs += nsteps;
          gu[0] += (nsteps + 1) / 2;
          gu[1] += nsteps / 2;
          ++nz;
        }
      }
    }
    __syncwarp();
  } else {
    setmaxnreg_inc<112>();
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
    // Item-loop state other than gu lives in shared memory (wst: item count k,
    // item id, non-empty items nz) so that it holds no registers across the step
    // loop; at 112 registers the softmax has none to spare.
    volatile uint32_t* const wst = reinterpret_cast<volatile uint32_t*>(gbase + (sWst - base)) + 4 * warp;
    if (lane == 0) {
      wst[0] = 0;
      wst[1] = 0;
      wst[2] = 0;
    }
    __syncwarp();
    uint32_t gu = 0;  // this stage's cumulative S/P uses
    for (;;) {
    const uint32_t id = take_item(wst[0]);
    if (id >= n_items) break;
    if (lane == 0) wst[1] = id;
    // only what the step loop needs stays live; the epilogue re-reads the item
    const uint32_t count = __ldg(&p.items[id].count);
    const uint32_t nsteps = (count + 1) / 2;
    const uint32_t* ent = p.entries + __ldg(&p.items[id].begin);
    float m = -INFINITY, l = 0.f;
    for (uint32_t t = st; t < nsteps; t += 2) {
      const uint32_t u = gu + (t >> 1);  // this stage's use index of S_st / P_st
      const uint32_t idx = 2 * t + hf;
      const uint32_t e = idx < count ? __ldg(ent + idx) : 0u;
      const bool dense = (e & dense_bit) != 0;  // warp-uniform: this warp's 64-key block
      mbar_wait(bSfull(st), u & 1);
      tc_fence_after();
      // DBSP_TRACE_FINE (warp 0): 0 start, 2 S loaded, 6 max exchanged, 3 exp start,
      // 4 P stored, 5 before the P arrive, 1 after it
      const bool tr0 = lane == 0 && warp == 0;
      if (false && tr0) PD_TR(0, t >> 1);
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
        if (u >= 1) {
          mbar_wait(bPempty(st), (u - 1) & 1);
          tc_fence_after();
        }
      };
      // Optional strict alternation of the two stages' exp phases.
      auto wait_turn = [&]() {
        if (kAltExp && t > 0) mbar_wait(bSmDone(1 - st), ((t - 1) >> 1) & 1);
        if (false && tr0) PD_TR(3, t >> 1);
      };
      // Pass 1 reads S for the row max, pass 2 again for the exps: holding the
      // 64 values across the max exchange instead (one read, S released before
      // the exchange) spills at 104 registers and measured 1.8x slower.
      float v[64];
      float lmax = -INFINITY;
      if (dense) {
        load_s(v);
        if (false && tr0) PD_TR(2, t >> 1);
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
      float* xm = xmax + ((u & 1) * 2 + st) * 256;
      xm[hf * 128 + row] = lmax;
      named_bar_sync(bar_id, 64);
      const float mt2 = fmaxf(lmax, xm[(1 - hf) * 128 + row]) * sl2;
      if (false && tr0) PD_TR(6, t >> 1);
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
        wait_turn();
        wait_pv();
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
            if ((j & 7) < kPoly) {
              pp = exp2_poly3_pair(x);
            } else {
              pp = make_float2(fast_exp2(x.x), fast_exp2(x.y));
            }
            acc2[i & 1] = __fadd2_rn(acc2[i & 1], pp);
            pk[i] = pack_bf16x2(pp.x, pp.y);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            *reinterpret_cast<uint4*>(prow + (((4 * c + u) ^ (row & 7)) << 4)) =
                make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        }
        const float2 a2 = __fadd2_rn(acc2[0], acc2[1]);
        l += a2.x + a2.y;
      } else {
        release_s();
        wait_turn();
        wait_pv();
#pragma unroll
        for (int u = 0; u < 8; ++u) *reinterpret_cast<uint4*>(prow + ((u ^ (row & 7)) << 4)) = make_uint4(0, 0, 0, 0);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(bSmDone(st));
      if (false && tr0) PD_TR(4, t >> 1);
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
      if (false && tr0) PD_TR(5, t >> 1);
      if (lane == 0) {
        if (rank == 0)
          mbar_arrive(bPfull(st));
        else
          mbar_arrive_cluster(pfull_remote_base + 8u * st);
      }

      if (false && tr0) PD_TR(1, t >> 1);
    }

    // ------------------------------------------------------------ epilogue: 32 columns per thread
    if (count > 0) {
      mbar_wait(bOfinal, wst[2] & 1);
      tc_fence_after();
    }
    __syncwarp();
    const WorkItem it = p.items[wst[1]];
    const uint32_t myq[2] = {rank ? it.pad0 : it.qa, rank ? it.pad1 : it.qb};  // quad rows 2r, 2r+1
    float2* const mlk = mlbuf + (wst[0] & 1u) * 512;  // by item parity: a partner may still read the last one
    mlk[(st * 2 + hf) * 128 + row] = make_float2(m, l);
    const uint32_t ebar = 9u + lg;  // the four warps (stage x half) of these rows
    named_bar_sync(ebar, 128);
    const float2 x00 = mlk[0 * 128 + row], x01 = mlk[1 * 128 + row];
    const float2 x10 = mlk[2 * 128 + row], x11 = mlk[3 * 128 + row];
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
    if (count > 0) {
      // this thread's O reads are complete (tcgen05.wait::ld above): the next item's PVs may run
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0)
          mbar_arrive(bOdrained);
        else
          mbar_arrive_cluster(leader(bOdrained));
      }
    }
    __syncwarp();
    if (lane == 0) {
      wst[0] = wst[0] + 1;
      if (count > 0) wst[2] = wst[2] + 1;
    }
    __syncwarp();
    gu += (nsteps + 1 - uint32_t(st)) / 2;
    }  // item loop
    if (p.out_peers) __threadfence_system();
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the leader's MMAs wrote into this CTA's TMEM / read its smem
  tc_fence_after();
  clock_probe_mark(p, 1);
  if (warp == 17) tmem_dealloc_pair(tmem, 512);
}

}  // namespace dbsp_dev
