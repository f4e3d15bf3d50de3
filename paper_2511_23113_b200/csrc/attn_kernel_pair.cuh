// K4, d=128, CTA-pair variant (tcgen05 cta_group::2).
//
// A cluster of two CTAs on the two SMs of a TPC runs one "quad" work item:
// four 64-row Q blocks of one head (CTA rank r owns blocks 2r, 2r+1 = 128
// rows) against the union of their dense KV blocks.  The leader (rank 0)
// issues M=256 MMAs for both:
//   S = Q K^T   SS, M=256 N=64   A: each CTA's own Q (smem); B: each CTA holds
//                                half the keys of the K block (32 rows)
//   O += P V    TS, M=256 N=128  A: each CTA's own P (TMEM); B: each CTA holds
//                                half the head dim of the V block (64 columns)
// so each SM stages and streams through its smem port only half of every K/V
// tile.  Per 64-key tile an SM now moves 40 KB (QK) + 8 KB (PV) + 16 KB of TMA
// writes = 64 KB = 512 port cycles, the MMA time; the 2-CTA-per-SM single-CTA
// kernel moved 96 KB (measured port-bound, tests/mma_bench.cu).  Cost: the KV
// list is the union of four rows (96% dense on the Wan masks vs 99% for two).
// Softmax, lazy rescale and epilogue are the per-CTA code of attn_kernel.cuh.
#pragma once

#include "attn_kernel.cuh"

namespace dbsp_dev {

struct PairCfg {
  static constexpr int D = 128;
  static constexpr uint32_t kQBytes = 128u * 128u * 2u;  // own 128 rows
  static constexpr uint32_t kQChunk = 128u * 128u;
  static constexpr uint32_t kKHalf = 32u * 128u * 2u;    // 32 keys x 128 d (8 KB)
  static constexpr uint32_t kKChunk = 32u * 128u;        // 32 rows x 128 B
  static constexpr uint32_t kVHalf = 64u * 64u * 2u;     // 64 keys x 64 d (8 KB)
  static constexpr int kStages = 4;
  static constexpr uint32_t kColS = 0, kColO = 128;      // S double buffer [0,128), O [128,256)
  static constexpr int kNumBars = 4 * kStages + 2 + 2 + 4;
  static constexpr uint32_t kSmemBytes =
      kQBytes + kStages * (kKHalf + kVHalf) + 1024 + 8 * kNumBars + 16;
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 2)
    sparse_attn_fwd_pair_kernel(const __grid_constant__ CUtensorMap tmQ,
                                const __grid_constant__ CUtensorMap tmK32,
                                const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  using C = PairCfg;
  constexpr int NS = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);

  const uint32_t sQ = base;
  const uint32_t sK = sQ + C::kQBytes;
  const uint32_t sV = sK + NS * C::kKHalf;
  const uint32_t sBar = sV + NS * C::kVHalf;
  auto bKfull = [&](int s) { return sBar + 8u * s; };
  auto bVfull = [&](int s) { return sBar + 8u * (NS + s); };
  auto bKempty = [&](int s) { return sBar + 8u * (2 * NS + s); };
  auto bVempty = [&](int s) { return sBar + 8u * (3 * NS + s); };
  auto bSfull = [&](int b) { return sBar + 8u * (4 * NS + b); };
  auto bPfull = [&](int b) { return sBar + 8u * (4 * NS + 2 + b); };
  const uint32_t bQ = sBar + 8u * (4 * NS + 4);
  const uint32_t bOdone = sBar + 8u * (4 * NS + 5);
  const uint32_t bOfinal = sBar + 8u * (4 * NS + 6);
  const uint32_t sTmemSlot = sBar + 8u * C::kNumBars;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const WorkItem it = p.items[blockIdx.x >> 1];
  const uint32_t count = it.count;
  const uint32_t myq[2] = {rank ? it.pad0 : it.qa, rank ? it.pad1 : it.qb};  // quad rows 2r, 2r+1
  auto leader = [&](uint32_t local_bar) { return mapa_shared(local_bar, 0); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(bKfull(s), 1);
      mbar_init(bVfull(s), 1);
      mbar_init(bKempty(s), 1);
      mbar_init(bVempty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bSfull(b), 1);
      mbar_init(bPfull(b), 8);  // 4 softmax warps in each CTA of the pair
    }
    mbar_init(bQ, 1);
    mbar_init(bOdone, 1);
    mbar_init(bOfinal, 1);
    mbar_fence_init();
  }
  if (warp == 4 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK32);
    tma_prefetch_desc(&tmV);
  }
  if (warp == 5) tmem_alloc_pair(sTmemSlot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(gbase + (sTmemSlot - base));

  if (warp == 4) {
    // ------------------------------------------------------------ producer (both CTAs)
    if (lane == 0 && count > 0) {
      const uint64_t pol_q = l2_policy_evict_first();
      const uint64_t pol_kv = l2_policy_evict_last();
      const int head = int(it.head);
      const uint32_t* ent = p.entries + it.begin;
      if (rank == 0) mbar_expect_tx(bQ, 2 * C::kQBytes);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        tma_load_3d_pair(sQ + c * C::kQChunk, &tmQ, c * 64, head, int(myq[0]) * 64, leader(bQ), pol_q);
        tma_load_3d_pair(sQ + c * C::kQChunk + 8192, &tmQ, c * 64, head, int(myq[1]) * 64, leader(bQ),
                         pol_q);
      }
      auto load_k = [&](uint32_t j) {
        const int s = int(j % NS);
        mbar_wait(bKempty(s), ((j / NS) & 1) ^ 1);
        const int kv = int(__ldg(ent + j) & dbsp_core::kEntryKvMask);
        if (rank == 0) mbar_expect_tx(bKfull(s), 2 * C::kKHalf);
#pragma unroll
        for (int c = 0; c < 2; ++c)
          tma_load_3d_pair(sK + s * C::kKHalf + c * C::kKChunk, &tmK32, c * 64, head,
                           kv * 64 + int(rank) * 32, leader(bKfull(s)), pol_kv);
      };
      load_k(0);
      for (uint32_t j = 0; j < count; ++j) {
        if (j + 1 < count) load_k(j + 1);
        const int s = int(j % NS);
        mbar_wait(bVempty(s), ((j / NS) & 1) ^ 1);
        const int kv = int(__ldg(ent + j) & dbsp_core::kEntryKvMask);
        if (rank == 0) mbar_expect_tx(bVfull(s), 2 * C::kVHalf);
        tma_load_3d_pair(sV + s * C::kVHalf, &tmV, int(rank) * 64, head, kv * 64, leader(bVfull(s)),
                         pol_kv);
      }
    } else if (count > 0) {
      mbar_wait(bOfinal, 0);
    }
    __syncwarp();
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer (leader only)
    if (rank == 0 && lane == 0 && count > 0) {
      constexpr uint32_t kIdescQK = idesc_bf16(256, 64, false, false);
      constexpr uint32_t kIdescPV = idesc_bf16(256, 128, false, true);
      auto issue_s = [&](uint32_t j) {
        const int s = int(j % NS);
        mbar_wait(bKfull(s), (j / NS) & 1);
        tc_fence_after();
        const uint32_t dcol = tmem + C::kColS + 64u * (j & 1);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t ad = smem_desc_sw128(sQ + (kk >> 2) * C::kQChunk + (kk & 3) * 32, 16, 1024);
          const uint64_t bd =
              smem_desc_sw128(sK + s * C::kKHalf + (kk >> 2) * C::kKChunk + (kk & 3) * 32, 16, 1024);
          mma_ss_pair(dcol, ad, bd, kIdescQK, kk > 0 ? 1u : 0u);
        }
        tc_commit_pair(bKempty(s), 0x3);
        tc_commit_pair(bSfull(int(j & 1)), 0x3);
        DBSP_TR(kTrMmaS, j);
      };
      auto issue_pv = [&](uint32_t i) {
        const int b = int(i & 1);
        const int s = int(i % NS);
        mbar_wait(bPfull(b), (i >> 1) & 1);
        mbar_wait(bVfull(s), (i / NS) & 1);
        tc_fence_after();
        const uint32_t pcol = tmem + C::kColS + 64u * b;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t bd = smem_desc_sw128(sV + s * C::kVHalf + kk * 2048, 8192, 1024);
          mma_ts_pair(tmem + C::kColO, pcol + kk * 8, bd, kIdescPV, (i > 0 || kk > 0) ? 1u : 0u);
        }
        tc_commit_pair(bVempty(s), 0x3);
        tc_commit_pair(bOdone, 0x3);
        DBSP_TR(kTrMmaPV, i);
      };
      mbar_wait(bQ, 0);
      tc_fence_after();
      issue_s(0);
      if (count > 1) issue_s(1);
      for (uint32_t j = 0; j < count; ++j) {
        issue_pv(j);
        if (j + 2 < count) issue_s(j + 2);
      }
      tc_commit_pair(bOfinal, 0x3);
    } else if (count > 0) {
      mbar_wait(bOfinal, 0);
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ softmax (both CTAs)
    const int row = threadIdx.x;
    const bool upper = row >= 64;
    const uint32_t lane_off = uint32_t(warp * 32) << 16;
    const uint32_t dense_bit = 1u << (22 + 2 * rank + (upper ? 1 : 0));
    const uint32_t pfull_remote_base = rank ? leader(bPfull(0)) : 0u;
    const float sl2 = p.scale_log2;
    const uint32_t* ent = p.entries + it.begin;
    float m = -INFINITY, l = 0.f;
    for (uint32_t j = 0; j < count; ++j) {
      const uint32_t e = __ldg(ent + j);
      const bool dense = (e & dense_bit) != 0;  // warp-uniform
      const int b = int(j & 1);
      const uint32_t scol = tmem + lane_off + C::kColS + 64u * b;
      mbar_wait(bSfull(b), (j >> 1) & 1);
      tc_fence_after();
      if (lane == 0 && warp == 0) DBSP_TR(rank ? kTrSoftStartHi : kTrSoftStart, j);
      uint32_t pk[32];
      if (dense) {
        uint32_t sa[32], sb[32];
        tmem_ld32(scol, sa);
        tmem_ld32(scol + 32, sb);
        tmem_ld_wait();
        const uint32_t valid = ((e >> dbsp_core::kQuadValidShift) & 63u) + 1u;
        float v[64];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          v[i] = __uint_as_float(sa[i]);
          v[i + 32] = __uint_as_float(sb[i]);
        }
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
        const float mt = fmaxf(fmax3f(mx[0], mx[1], mx[2]),
                               fmax3f(fmax3f(mx[3], mx[4], mx[5]), mx[6], mx[7]));
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
          if (j > 0) {
            mbar_wait(bOdone, (j - 1) & 1);  // completed PVs here: j-1 or j
            tc_fence_after();
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t o[32];
            tmem_ld32(tmem + lane_off + C::kColO + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(tmem + lane_off + C::kColO + c * 32, o);
          }
        }
        const float negm = -m;
        float sum4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float p0 = fast_exp2(fmaf(v[2 * i], sl2, negm));
          const float p1 = fast_exp2(fmaf(v[2 * i + 1], sl2, negm));
          sum4[i & 3] += p0 + p1;
          pk[i] = pack_bf16x2(p0, p1);
        }
        l += (sum4[0] + sum4[1]) + (sum4[2] + sum4[3]);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) pk[i] = 0u;
      }
      tmem_st32(scol, pk);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0 && warp == 0) DBSP_TR(rank ? kTrSoftEndHi : kTrSoftEnd, j);
      if (lane == 0) {
        if (rank == 0)
          mbar_arrive(bPfull(b));
        else
          mbar_arrive_cluster(pfull_remote_base + 8u * b);
      }
    }

    // ------------------------------------------------------------ epilogue
    if (count > 0) {
      mbar_wait(bOfinal, 0);
      tc_fence_after();
    }
    const uint32_t qblk = myq[upper ? 1 : 0];
    const uint32_t token = qblk * 64u + uint32_t(row & 63);
    const bool live = !((it.single >> (2 * rank + (upper ? 1 : 0))) & 1u) && token < p.q_tokens;
    const float inv_l = l > 0.f ? 1.f / l : 0.f;
    const float kLn2 = 0.6931471805599453f;
    const float lse_new = l > 0.f ? (m + log2f(l)) * kLn2 : -INFINITY;
    const size_t orow = (size_t(token) * p.heads + it.head) * 128;
    const size_t lidx = size_t(it.head) * p.q_tokens + token;
    float c_old = 0.f, c_new = inv_l, lse_out = lse_new;
    const bool acc = (p.mode & kModeAccumulate) != 0;
    if (acc) {
      const float lse_old = live ? p.lse_acc[lidx] : -INFINITY;
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
    for (int c = 0; c < 4; ++c) {
      uint32_t o[32];
      if (count > 0) {
        tmem_ld32(tmem + lane_off + C::kColO + c * 32, o);
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
    if (live) {
      if (acc)
        p.lse_acc[lidx] = lse_out;
      else if (p.lse)
        p.lse[lidx] = lse_new;
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the leader's MMAs wrote into this CTA's TMEM / read its smem
  tc_fence_after();
  if (warp == 5) tmem_dealloc_pair(tmem, kTmemCols);
}

}  // namespace dbsp_dev
