// K4, persistent quad kernel (d=128).
//
// The quad kernel (attn_kernel_quad.cuh: one CTA per SM, two 128-row Q tiles
// of one head share one stream of 64-key K/V tiles, two S buffers per stage,
// one MMA issuer per stage) with each CTA looping over work items, taken
// dynamically from a global counter in the LPT (heavy-first) order.  The non-persistent quad kernel paid a
// non-overlapped 5.5 us per item (CTA exit + launch, barrier init, TMEM
// alloc, Q load latency, epilogue); here the next item's K/V loads, Q load
// and first QK^T overlap the current item's epilogue.
// Barrier phases run on global counters: step index gj (K/V ring slots, S/P
// buffers, PV completions) and nonempty-item index nz.  Hand-over barriers:
//   Qfree      both stages' last QK^T of an item done -> producer may load the next Q
//   Ofinal_s   all PV_s of an item done               -> epilogue may read O_s
//   Odrained_s epilogue read O_s                      -> next item's first PV_s may run
// Warp roles (352 threads): warps 0-3 / 4-7 softmax + epilogue of stage 0 / 1,
// warp 8 TMA producer, warps 9 / 10 MMA issuer of stage 0 / 1 (9 owns TMEM).
// TMEM: S(stage s, buffer b) at 64(2s+b), O_s at 256 + 128s.
// Mask semantics follow the reference BlockMask (mask.hpp:18-20).
#pragma once

#include "attn_kernel.cuh"

namespace dbsp_dev {

constexpr int kThreadsQuadP = 352;

struct QuadPCfg {
  static constexpr int D = 128;
  static constexpr uint32_t kQStageBytes = 128u * D * 2u;
  static constexpr uint32_t kQBytes = 2u * kQStageBytes;
  static constexpr uint32_t kQChunk = 128u * 128u;
  static constexpr uint32_t kTileBytes = 64u * D * 2u;
  static constexpr uint32_t kColS = 0, kColO = 256;
  static constexpr int kStages = 4;
  static constexpr int kItemSlots = 4;  // item ids the producer publishes ahead
  static constexpr int kNumBars = 4 * kStages + 17 + 2 * kItemSlots;
  static constexpr uint32_t kSmemBytes = kQBytes + 2u * kStages * kTileBytes + 1024 + 8 * kNumBars + 16 + 16;
};

__global__ void __launch_bounds__(kThreadsQuadP, 1)
    sparse_attn_fwd_quadp_kernel(const __grid_constant__ CUtensorMap tmQ,
                                 const __grid_constant__ CUtensorMap tmK,
                                 const __grid_constant__ CUtensorMap tmV, const AttnParams p,
                                 uint32_t n_items) {
  using C = QuadPCfg;
  constexpr int D = C::D;
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
  auto bOdone = [&](int st) { return sBar + 8u * (4 * NS + 10 + st); };
  auto bOfinal = [&](int st) { return sBar + 8u * (4 * NS + 12 + st); };
  auto bOdrained = [&](int st) { return sBar + 8u * (4 * NS + 14 + st); };
  const uint32_t bQfree = sBar + 8u * (4 * NS + 16);
  auto bItemFull = [&](int k) { return sBar + 8u * (4 * NS + 17 + k); };
  auto bItemEmpty = [&](int k) { return sBar + 8u * (4 * NS + 17 + C::kItemSlots + k); };
  const uint32_t sTmemSlot = sBar + 8u * C::kNumBars;
  volatile uint32_t* item_ring = reinterpret_cast<volatile uint32_t*>(gbase + (sTmemSlot + 16 - base));
  // Item hand-out: the producer takes the next item id from the global counter
  // (dynamic LPT over the heavy-first list, like the hardware CTA scheduler of
  // the non-persistent kernels) and publishes it in a 4-slot ring; the two
  // MMA threads and the eight softmax warps read every id in the same order.
  auto next_item = [&](uint32_t k) -> uint32_t {  // consumers
    const int s = int(k % C::kItemSlots);
    mbar_wait(bItemFull(s), (k / C::kItemSlots) & 1);
    const uint32_t id = item_ring[s];
    __syncwarp(__activemask());  // MMA warps run this on lane 0 only
    if ((threadIdx.x & 31) == 0) mbar_arrive(bItemEmpty(s));
    return id;
  };

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  clock_probe_mark(p, 0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(bKfull(s), 1);
      mbar_init(bVfull(s), 1);
      mbar_init(bKempty(s), 2);
      mbar_init(bVempty(s), 2);
    }
    for (int st = 0; st < 2; ++st) {
      for (int b = 0; b < 2; ++b) {
        mbar_init(bSfull(st, b), 1);
        mbar_init(bPfull(st, b), 4);
      }
      mbar_init(bQready(st), 1);
      mbar_init(bOdone(st), 1);
      mbar_init(bOfinal(st), 1);
      mbar_init(bOdrained(st), 4);
    }
    mbar_init(bQfree, 2);
    for (int k = 0; k < C::kItemSlots; ++k) {
      mbar_init(bItemFull(k), 1);
      mbar_init(bItemEmpty(k), 10);  // 2 MMA warps + 8 softmax warps
    }
    mbar_fence_init();
  }
  if (warp == 8 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
  }
  if (warp == 9) tmem_alloc(sTmemSlot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(gbase + (sTmemSlot - base));

  if (warp == 8) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      const uint64_t pol_kv = l2_policy_evict_last();
      const uint64_t pol_q = l2_policy_evict_first();
      uint32_t gj = 0, nz = 0;
      for (uint32_t k = 0;; ++k) {
        const int slot = int(k % C::kItemSlots);
        mbar_wait(bItemEmpty(slot), ((k / C::kItemSlots) & 1) ^ 1);
        const uint32_t i = atomicAdd(p.item_counter, 1u);
        item_ring[slot] = i;
        mbar_arrive(bItemFull(slot));
        if (i >= n_items) break;
        const WorkItem it = p.items[i];
        const uint32_t count = it.count;
        if (count == 0) continue;
        const int head = int(it.head);
        const uint32_t* ent = p.entries + it.begin;
        auto load_tile = [&](const CUtensorMap* tm, uint32_t dst, uint32_t full, uint32_t j) {
          const int kv = int(__ldg(ent + j) & dbsp_core::kEntryKvMask);
          mbar_expect_tx(full, C::kTileBytes);
#pragma unroll
          for (int c = 0; c < 2; ++c) tma_load_3d(dst + c * 8192, tm, c * 64, head, kv * 64, full, pol_kv);
        };
        auto load_k = [&](uint32_t j) {
          const uint32_t g = gj + j;
          const int s = int(g % NS);
          mbar_wait(bKempty(s), ((g / NS) & 1) ^ 1);
          load_tile(&tmK, sK + s * C::kTileBytes, bKfull(s), j);
        };
        for (uint32_t j = 0; j < 2 && j < count; ++j) load_k(j);
        if (nz > 0) mbar_wait(bQfree, (nz - 1) & 1);  // the previous item's QK^T are done
        const uint32_t qb[4] = {it.qa, it.qb, it.pad0, it.pad1};
#pragma unroll
        for (int st = 0; st < 2; ++st) {
          mbar_expect_tx(bQready(st), C::kQStageBytes);
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const uint32_t dst = sQ + st * C::kQStageBytes + c * C::kQChunk;
            tma_load_3d(dst, &tmQ, c * 64, head, int(qb[2 * st]) * 64, bQready(st), pol_q);
            tma_load_3d(dst + 8192, &tmQ, c * 64, head, int(qb[2 * st + 1]) * 64, bQready(st), pol_q);
          }
        }
        for (uint32_t j = 0; j < count; ++j) {
          const uint32_t g = gj + j;
          const int s = int(g % NS);
          mbar_wait(bVempty(s), ((g / NS) & 1) ^ 1);
          load_tile(&tmV, sV + s * C::kTileBytes, bVfull(s), j);
          if (j + 2 < count) load_k(j + 2);
        }
        gj += count;
        ++nz;
      }
    }
    __syncwarp();
  } else if (warp >= 9) {
    // ------------------------------------------------------------ MMA issuer of stage warp-9
    const int st = warp - 9;
    if (lane == 0) {
      constexpr uint32_t kIdescQK = idesc_bf16(128, 64, false, false);
      constexpr uint32_t kIdescPV = idesc_bf16(128, D, false, true);
      uint32_t gj = 0, nz = 0;
      for (uint32_t k = 0;; ++k) {
        const uint32_t i = next_item(k);
        if (i >= n_items) break;
        const uint32_t count = p.items[i].count;
        if (count == 0) continue;
        auto issue_s = [&](uint32_t j) {
          const uint32_t g = gj + j;
          const int s = int(g % NS);
          mbar_wait(bKfull(s), (g / NS) & 1);
          tc_fence_after();
          const uint32_t dcol = tmem + C::kColS + 64u * (2 * st + (g & 1));
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint64_t bd =
                smem_desc_sw128(sK + s * C::kTileBytes + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
            const uint64_t ad = smem_desc_sw128(
                sQ + st * C::kQStageBytes + (kk >> 2) * C::kQChunk + (kk & 3) * 32, 16, 1024);
            mma_ss(dcol, ad, bd, kIdescQK, kk > 0 ? 1u : 0u);
          }
          tc_commit(bSfull(st, int(g & 1)));
          tc_commit(bKempty(s));
          if (j + 1 == count) tc_commit(bQfree);  // this stage no longer reads Q
        };
        auto issue_pv = [&](uint32_t j) {
          const uint32_t g = gj + j;
          const int s = int(g % NS);
          const int b = int(g & 1);
          mbar_wait(bPfull(st, b), (g >> 1) & 1);
          mbar_wait(bVfull(s), (g / NS) & 1);
          if (j == 0 && nz > 0) mbar_wait(bOdrained(st), (nz - 1) & 1);  // O_s free again
          tc_fence_after();
          const uint32_t pcol = tmem + C::kColS + 64u * (2 * st + b);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t bd = smem_desc_sw128(sV + s * C::kTileBytes + kk * 2048, 8192, 1024);
            mma_ts(tmem + C::kColO + uint32_t(D) * st, pcol + kk * 8, bd, kIdescPV, (j > 0 || kk > 0) ? 1u : 0u);
          }
          tc_commit(bOdone(st));
          tc_commit(bVempty(s));
        };
        mbar_wait(bQready(st), nz & 1);
        tc_fence_after();
        for (uint32_t j = 0; j < 2 && j < count; ++j) issue_s(j);
        for (uint32_t j = 0; j < count; ++j) {
          issue_pv(j);
          if (j + 2 < count) issue_s(j + 2);
        }
        tc_commit(bOfinal(st));
        gj += count;
        ++nz;
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ softmax + epilogue of stage st
    const int st = warp >> 2;
    const int row = threadIdx.x & 127;
    const uint32_t lane_off = uint32_t((warp & 3) * 32) << 16;
    const int bi = 2 * st + (row >> 6);
    const uint32_t dense_bit = 1u << (22 + bi);
    const float sl2 = p.scale_log2;
    const uint32_t ocol = tmem + lane_off + C::kColO + uint32_t(D) * st;
    uint32_t gj = 0, nz = 0;
    for (uint32_t k = 0;; ++k) {
      const uint32_t i = next_item(k);
      if (i >= n_items) break;
      const WorkItem it = p.items[i];
      const uint32_t count = it.count;
      const uint32_t qblk = bi == 0 ? it.qa : bi == 1 ? it.qb : bi == 2 ? it.pad0 : it.pad1;
      const uint32_t token = qblk * 64u + uint32_t(row & 63);
      const bool padded = (it.single >> bi) & 1u;
      if (count == 0) {  // no KV tile: zeros and LSE -inf, no barrier traffic
        finish_row<D>(p, ocol, false, !padded && token < p.q_tokens, -INFINITY, 0.f, token, it.head);
        continue;
      }
      const uint32_t* ent = p.entries + it.begin;
      float m = -INFINITY, l = 0.f;
      for (uint32_t j = 0; j < count; ++j) {
        const uint32_t g = gj + j;
        const uint32_t e = __ldg(ent + j);
        const bool dense = (e & dense_bit) != 0;
        const int b = int(g & 1);
        const uint32_t scol = tmem + lane_off + C::kColS + 64u * (2 * st + b);
        mbar_wait(bSfull(st, b), (g >> 1) & 1);
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
            for (int k2 = 0; k2 < 32; ++k2) {
              v[k2] = __uint_as_float(sa[k2]);
              v[k2 + 32] = __uint_as_float(sb[k2]);
            }
          }
          const uint32_t valid = ((e >> dbsp_core::kQuadValidShift) & 63u) + 1u;
          if (valid < 64) {
#pragma unroll
            for (int k2 = 0; k2 < 64; ++k2)
              if (uint32_t(k2) >= valid) v[k2] = -INFINITY;
          }
          float mx[8];
#pragma unroll
          for (int a = 0; a < 8; ++a) {
            mx[a] = fmax3f(v[8 * a], v[8 * a + 1], v[8 * a + 2]);
            mx[a] = fmax3f(mx[a], v[8 * a + 3], v[8 * a + 4]);
            mx[a] = fmax3f(mx[a], v[8 * a + 5], v[8 * a + 6]);
            mx[a] = fmaxf(mx[a], v[8 * a + 7]);
          }
          const float mt =
              fmaxf(fmax3f(mx[0], mx[1], mx[2]), fmax3f(fmax3f(mx[3], mx[4], mx[5]), mx[6], mx[7]));
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
            // O_s quiescent: PV_s(g-1) complete (phases <= g-2 are done, see quad)
            if (j > 0) {
              mbar_wait(bOdone(st), (g - 1) & 1);
              tc_fence_after();
            }
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
              uint32_t o[32];
              tmem_ld32(ocol + c * 32, o);
              tmem_ld_wait();
#pragma unroll
              for (int k2 = 0; k2 < 32; ++k2) o[k2] = __float_as_uint(__uint_as_float(o[k2]) * alpha);
              tmem_st32(ocol + c * 32, o);
            }
          }
          const float2 sc2 = make_float2(sl2, sl2), nm2 = make_float2(-m, -m);
          float2 acc2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
          for (int k2 = 0; k2 < 32; ++k2) {
            const float2 x = __ffma2_rn(make_float2(v[2 * k2], v[2 * k2 + 1]), sc2, nm2);
            const float2 pp = make_float2(fast_exp2(x.x), fast_exp2(x.y));
            acc2[k2 & 1] = __fadd2_rn(acc2[k2 & 1], pp);
            pk[k2] = pack_bf16x2(pp.x, pp.y);
          }
          const float2 a2 = __fadd2_rn(acc2[0], acc2[1]);
          l += a2.x + a2.y;
        } else {
#pragma unroll
          for (int k2 = 0; k2 < 32; ++k2) pk[k2] = 0u;
        }
        tmem_st32(scol, pk);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bPfull(st, b));
      }
      mbar_wait(bOfinal(st), nz & 1);
      tc_fence_after();
      finish_row<D>(p, ocol, true, !padded && token < p.q_tokens, m, l, token, it.head);
      tc_fence_before();  // the O reads above precede the next item's first PV_s
      __syncwarp();
      if (lane == 0) mbar_arrive(bOdrained(st));
      gj += count;
      ++nz;
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 9) tmem_dealloc(tmem, 512);
  clock_probe_mark(p, 1);
}

}  // namespace dbsp_dev
