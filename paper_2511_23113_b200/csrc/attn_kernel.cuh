// K4: block-sparse FlashAttention forward for sm_100a (tcgen05 + TMEM + TMA).
//
// One CTA = one work item (schedule.hpp): a 128-row Q tile (two 64-row Q
// blocks of one head) against the union of their dense 64-key KV blocks.
// Two CTAs per SM, so one CTA's softmax overlaps the other's MMAs.
// Warp roles (192 threads):
//   warps 0-3  Q -> TMEM at start; softmax; epilogue.  Thread t owns Q row t
//              (TMEM lane t).
//   warp 4     TMA producer: K and V tiles through an NS-deep smem ring.
//   warp 5     TMEM allocator + single-thread tcgen05.mma issuer.
// Per KV tile j:
//   S_j = Q K_j^T        tcgen05.mma TS: A = Q from TMEM, B = K (smem, SW128),
//                        M=128 N=64 K=d -> TMEM S[j % NSB]
//   P_j = exp2(S_j*c-m)  softmax warps; bf16 P written over S[j % NSB]
//   O  += P_j V_j        tcgen05.mma TS: A = P from TMEM, B = V (smem, MN-major)
// Q lives in TMEM rather than shared memory: an SS-mode QK^T with N=64 reads
// 6 KB of smem per 32-cycle MMA (192 B/clk, above the 128 B/clk smem port),
// which capped the first version at ~55% tensor activity.  With A in TMEM the
// per-tile smem traffic is K + V reads + their TMA writes = 64 KB / 512 MMA
// cycles.  The online-softmax max is rescaled lazily (only when it grows by
// more than 2^8), so O in TMEM is touched by the softmax warps only rarely.
// Mask semantics follow the reference BlockMask (mask.hpp:18-20): a tile is
// computed iff its bit is set; everything else contributes exactly zero.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "schedule.hpp"

namespace dbsp_dev {

using dbsp_core::WorkItem;

enum : uint32_t { kModeAccumulate = 1, kModeFinalize = 2 };

struct AttnParams {
  const WorkItem* items;
  const uint32_t* entries;
  const __nv_bfloat16* q;  // [q_tokens, heads, D]
  __nv_bfloat16* out;
  float* lse;
  float* o_acc;
  float* lse_acc;
  uint32_t q_tokens;
  uint32_t heads;
  uint32_t mode;
  float scale_log2;
  unsigned long long* trace;  // DBSP_TRACE builds only: clock64 per (block, tile, event)
  // Optional: CTA 0 writes {clock64, globaltimer} at start and end, so the host
  // can read the SM clock the kernel actually ran at (power capping).
  unsigned long long* clock_probe;
  // Fused O return (reverse all-to-all in the epilogue).  Non-null: the bf16
  // row (local token t, local head h) goes to out_peers[rank] -- the home
  // rank's [home tokens, out_heads, D] buffer, a peer pointer over NVLink --
  // at row scatter_rows[3*(t/64)+1] + t%64 and head scatter_heads[h];
  // scatter_rows[3*b] is the home rank, [3*b+2] the valid rows of block b.
  __nv_bfloat16* const* out_peers;
  const uint32_t* scatter_rows;
  const uint32_t* scatter_heads;
  uint32_t out_heads;
};

// Where the bf16 output row of (local token, local head) goes: the local
// buffer, or its home rank's buffer when the O return is fused (out_peers).
template <int D>
__device__ __forceinline__ __nv_bfloat16* out_row_ptr(const AttnParams& p, uint32_t token, uint32_t head,
                                                     bool& live) {
  if (p.out_peers == nullptr) return p.out + (size_t(token) * p.heads + head) * D;
  const uint32_t* e = p.scatter_rows + 3 * (token >> 6);
  const uint32_t r = token & 63u;
  live = live && r < e[2];
  return p.out_peers[e[0]] + (size_t(e[1] + r) * p.out_heads + p.scatter_heads[head]) * D;
}

__device__ __forceinline__ void clock_probe_mark(const AttnParams& p, int slot) {
  if (p.clock_probe && blockIdx.x == 0 && threadIdx.x == 0) {
    p.clock_probe[2 * slot] = clock64();
    p.clock_probe[2 * slot + 1] = globaltimer_ns();
  }
}

// Event slots of the optional per-tile trace (DBSP_TRACE).
enum : int { kTrSoftStart = 0, kTrSoftEnd, kTrMmaS, kTrMmaPV, kTrSoftStartHi, kTrSoftEndHi,
             kTrLoadK, kTrLoadV, kTrEvents };
#ifdef DBSP_TRACE_EXPS
// Exp-phase overlap of co-resident CTAs (tests/trace_kernel.py --exps): every
// CTA of the first wave; per step, each softmax warp w stamps the start and end
// of its exp loop into slots 2w, 2w+1; tile slot kTraceTiles-1 holds the
// warps' %warpid (slots 0-3) and %smid (slot 4).
constexpr int kTraceBlocks = 296, kTraceTiles = 128;
#else
constexpr int kTraceBlocks = 16, kTraceTiles = 256;
#endif
#ifdef DBSP_TRACE
#define DBSP_TR(ev, j)                                                                         \
  do {                                                                                         \
    if (p.trace && blockIdx.x < kTraceBlocks && (j) < kTraceTiles)                             \
      p.trace[(size_t(blockIdx.x) * kTraceTiles + (j)) * kTrEvents + (ev)] = clock64();        \
  } while (0)
#else
#define DBSP_TR(ev, j) \
  do {                 \
  } while (0)
#endif
// DBSP_TRACE_FINE1 (tests/trace_kernel.py --fine1 [--warp W]): softmax warp W
// stamps the phases of its step into slots 4-7 -- S loaded, max known, exps
// done, P stored -- instead of the hi-half and load events.
#if defined(DBSP_TRACE) && defined(DBSP_TRACE_EXPS)
#define DBSP_TRF(ev, j) \
  do {                  \
  } while (0)
#define DBSP_TRC(ev, j) \
  do {                  \
  } while (0)
#elif defined(DBSP_TRACE) && defined(DBSP_TRACE_FINE1)
#ifndef DBSP_TRACE_WARP
#define DBSP_TRACE_WARP 0
#endif
#define DBSP_TRF(ev, j)                                        \
  do {                                                         \
    if (warp == DBSP_TRACE_WARP && lane == 0) DBSP_TR(ev, j); \
  } while (0)
#define DBSP_TRC(ev, j)         \
  do {                          \
    if ((ev) < 4) DBSP_TR(ev, j); \
  } while (0)
#else
#define DBSP_TRF(ev, j) \
  do {                  \
  } while (0)
#define DBSP_TRC(ev, j) DBSP_TR(ev, j)
#endif

constexpr int kThreads = 192;
constexpr uint32_t kTmemCols = 256;
constexpr float kRescaleThreshold = 8.0f;  // log2 domain
// exp2 pairs (of every 8) computed on the FMA pipe (exp2_poly3_pair) instead
// of MUFU.  Measured: d=64 is MUFU-bound -- on the CogVideoX layer 1.94 ms
// with none (round 1, tests/kernel_sweep.py), and per launch (ncu cycles,
// tests/variant_cycles.py, round 2) 3.07 M cycles with 2 of 8 vs 2.99 M with
// 3 of 8 (4 of 8 is slower again, profiles/r02_d64_poly_sweep.log); d=128 is
// smem-port and power bound and only slows down (Wan: 5.71 / 5.97 / 6.32 ms
// for 0 / 1 / 2 of 8).
// With the row sum on the tensor core (d=64, KCfg::kColL) 2 of 8 beat 3 of 8:
// 2.787 M vs 2.800 M cycles, and 1.3% in sustained runs.
// Which pairs of every 8 go to the FMA pipe: spread out, so the compiler
// interleaves the polynomial chains with the MUFU stream (3 of 8 at {0,3,5}:
// 2.94 M vs 2.98 M cycles for {0,1,2} on CogVideoX, tests/variant_cycles.py).
__host__ __device__ constexpr uint32_t poly_mask(int n) {
  return n <= 0 ? 0u : n == 1 ? 0x01u : n == 2 ? 0x11u : n == 3 ? 0x29u : n == 4 ? 0x55u : (1u << n) - 1u;
}
template <int D>
__host__ __device__ constexpr int poly_pairs() {
#ifdef DBSP_POLY_N
  return DBSP_POLY_N;
#else
  return D == 64 ? 2 : 0;
#endif
}


template <int D>
struct KCfg {
  static constexpr int kChunks = D / 64;  // 128-byte swizzle atoms along d
  static constexpr uint32_t kTileBytes = 64u * D * 2u;
  // Where Q lives.  d=64: in TMEM (TS-mode QK^T; 32 cols) -- measured 1.17x
  // faster on the CogVideoX layer.  d=128: Q in TMEM (64 cols) would leave
  // room for only one S buffer next to the 128-col O, which serialises
  // softmax and MMA inside a CTA (measured 1.24x slower than Q in smem with
  // two S buffers), so Q stays in smem (SS-mode QK^T) there.
  // (Round 1 also measured d=64 with Q in smem and a third S buffer in the
  // freed columns: within 1% -- profiles/r01_k4_analysis.md.)
  static constexpr bool kQInTmem = D == 64;
  static constexpr int kNSB = 2;
  static constexpr uint32_t kQBytes = kQInTmem ? 0u : 128u * D * 2u;
  static constexpr uint32_t kQChunk = 128u * 128u;  // one 64-column chunk of a 128-row Q tile
  // TMEM columns (256 per CTA): [Q], NSB S/P buffers of 64 cols, O (fp32, D
  // cols); regions 64-column aligned.  d=64: Q 0-31, row sum l 32-47 (kColL).
  static constexpr uint32_t kColQ = 0;
  static constexpr uint32_t kColS = kQInTmem ? 64 : 0;
  static constexpr uint32_t kColO = kColS + 64 * kNSB;
  static_assert(kColO + D <= kTmemCols, "TMEM budget");
  static constexpr int kStages = D == 128 ? 2 : (kQInTmem ? 6 : 5);  // K/V smem ring depth
  static constexpr int kNumBars = 4 * kStages + 2 * kNSB + 4;
  // d=64: the row sum l comes from the tensor core -- one more MMA per PV,
  // P x (64 keys x 16 ones) into 16 TMEM columns beside Q (kColL) -- so the
  // softmax warps skip 32 FADD2 per row and tile (8% of the kernel's
  // instructions).  The ones block is one 64-key x 64-column bf16 tile in
  // smem, read like a V tile.  l then sums the bf16 P the PV MMA consumes.
  // With 2 of 8 exp pairs on the FMA pipe (poly_pairs): CogVideoX 2.787 M vs
  // 2.807 M cycles (ncu) and 1.723-1.730 vs 1.751-1.755 ms in sustained
  // interleaved runs (tests/ab_probe.py --sustained --rounds 20, x3).  At
  // d=128 TMEM is full (S 128 + O 128 columns).
  static constexpr uint32_t kColL = 32;
  static constexpr uint32_t kOnesBytes = kQInTmem ? 64u * 64u * 2u : 0u;
  static constexpr uint32_t kDataBytes = kQBytes + 2u * kStages * kTileBytes + kOnesBytes;
  static constexpr uint32_t kSmemBytes = kDataBytes + 1024 + 8 * kNumBars + 16;
};

template <int D, int POLY = poly_pairs<D>(), bool LMMA = D == 64>
__global__ void __launch_bounds__(kThreads, 2)
    sparse_attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ,
                           const __grid_constant__ CUtensorMap tmK,
                           const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  using C = KCfg<D>;
  constexpr int NS = C::kStages;
  constexpr int NSB = C::kNSB;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);

  const uint32_t sQ = base;  // only when !kQInTmem
  const uint32_t sK = base + C::kQBytes;
  const uint32_t sV = sK + NS * C::kTileBytes;
  const uint32_t sOnes = sV + NS * C::kTileBytes;  // kOnesBytes, LMMA only
  const uint32_t sBar = sOnes + C::kOnesBytes;
  static_assert(!LMMA || C::kQInTmem, "the tensor-core row sum needs the d=64 TMEM layout");
  auto bKfull = [&](int s) { return sBar + 8u * s; };
  auto bVfull = [&](int s) { return sBar + 8u * (NS + s); };
  auto bKempty = [&](int s) { return sBar + 8u * (2 * NS + s); };
  auto bVempty = [&](int s) { return sBar + 8u * (3 * NS + s); };
  auto bSfull = [&](int b) { return sBar + 8u * (4 * NS + b); };
  auto bPfull = [&](int b) { return sBar + 8u * (4 * NS + NSB + b); };
  const uint32_t bQready = sBar + 8u * (4 * NS + 2 * NSB);      // Q in TMEM / smem
  // PV_j commits bOdone(j & 1): with NSB=3, S_j completes after PV_{j-3}, so
  // two PVs may be pending and a single barrier's parity would alias.
  auto bOdone = [&](uint32_t j) { return sBar + 8u * (4 * NS + 2 * NSB + 1 + (j & 1)); };
  const uint32_t bOfinal = sBar + 8u * (4 * NS + 2 * NSB + 3);  // single phase: all PVs done
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
      mbar_init(bKempty(s), 1);
      mbar_init(bVempty(s), 1);
    }
    for (int b = 0; b < NSB; ++b) {
      mbar_init(bSfull(b), 1);
      mbar_init(bPfull(b), 4);  // one arrive per softmax warp
    }
    mbar_init(bQready, C::kQInTmem ? 4 : 1);  // 4 softmax warps, or the TMA tx arrive
    mbar_init(bOdone(0), 1);
    mbar_init(bOdone(1), 1);
    mbar_init(bOfinal, 1);
    mbar_fence_init();
  }
  if (warp == 4 && lane == 0) {
    if (!C::kQInTmem) tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
  }
  if (warp == 5) tmem_alloc(sTmemSlot, kTmemCols);
  if constexpr (LMMA) {
    uint4* ones = reinterpret_cast<uint4*>(gbase + (sOnes - base));
    for (uint32_t i = threadIdx.x; i < C::kOnesBytes / 16; i += kThreads)
      ones[i] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);  // bf16 1.0
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(gbase + (sTmemSlot - base));

  if (warp == 4) {
    // ------------------------------------------------------------ producer
    // The whole warp runs the loop (warp-uniform waits); one elected lane
    // issues the copies.
    if (count > 0) {
      const uint64_t pol_kv = l2_policy_evict_last();
      const int head = int(it.head);
      const uint32_t* ent = p.entries + it.begin;
      if (!C::kQInTmem) {  // both 64-row Q blocks of the tile, via TMA
        if (elect_one()) {
          const uint64_t pol_q = l2_policy_evict_first();
          mbar_expect_tx(bQready, C::kQBytes);
#pragma unroll
          for (int c = 0; c < C::kChunks; ++c) {
            tma_load_3d(sQ + c * C::kQChunk, &tmQ, c * 64, head, int(it.qa) * 64, bQready, pol_q);
            tma_load_3d(sQ + c * C::kQChunk + 8192, &tmQ, c * 64, head, int(it.qb) * 64, bQready,
                        pol_q);
          }
        }
        __syncwarp();
      }
      auto load_tile = [&](const CUtensorMap* tm, uint32_t dst, uint32_t full, uint32_t j) {
        const int kv = int(__ldg(ent + j) & dbsp_core::kEntryKvMask);
        if (elect_one()) {
          mbar_expect_tx(full, C::kTileBytes);
#pragma unroll
          for (int c = 0; c < C::kChunks; ++c)
            tma_load_3d(dst + c * 8192, tm, c * 64, head, kv * 64, full, pol_kv);
        }
        __syncwarp();
      };
      auto load_k = [&](uint32_t j) {
        const int s = int(j % NS);
        mbar_wait(bKempty(s), ((j / NS) & 1) ^ 1);
        load_tile(&tmK, sK + s * C::kTileBytes, bKfull(s), j);
        if (lane == 0) DBSP_TRC(kTrLoadK, j);
      };
      load_k(0);
      for (uint32_t j = 0; j < count; ++j) {
        if (j + 1 < count) load_k(j + 1);  // K runs one tile ahead of V
        const int s = int(j % NS);
        mbar_wait(bVempty(s), ((j / NS) & 1) ^ 1);
        load_tile(&tmV, sV + s * C::kTileBytes, bVfull(s), j);
        if (lane == 0) DBSP_TRC(kTrLoadV, j);
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    // Warp-uniform loop, one elected lane issues, descriptors precomputed (a
    // base plus per-stage / per-k-step constants that never carry out of the
    // 14-bit address field).  The first version issued from a lane-0 branch
    // while lanes 1-31 spun on an mbarrier in the same warp: each group of
    // four MMAs took 650-860 cycles to issue and PV(j) left 1,300 cycles
    // after P(j) was ready (tests/trace_kernel.py --workload cogvideox).
    if (count > 0) {
      constexpr uint32_t kIdescQK = idesc_bf16(128, 64, false, false);
      constexpr uint32_t kIdescPV = idesc_bf16(128, D, false, true);
      const uint64_t dK = smem_desc_sw128(sK, 16, 1024);
      const uint64_t dQ = smem_desc_sw128(sQ, 16, 1024);  // used only when !kQInTmem
      const uint64_t dV = smem_desc_sw128(sV, 8192, 1024);
      constexpr uint32_t kIdescL = idesc_bf16(128, 16, false, true);
      const uint64_t dOnes = smem_desc_sw128(sOnes, 8192, 1024);
      auto issue_s = [&](uint32_t j) {
        const int s = int(j % NS);
        mbar_wait(bKfull(s), (j / NS) & 1);
        tc_fence_after();
        const uint32_t dcol = tmem + C::kColS + 64u * (j % NSB);
        const uint64_t bK = dK + ((uint32_t(s) * C::kTileBytes) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint64_t bd = bK + (((kk >> 2) * 8192 + (kk & 3) * 32) >> 4);
            if constexpr (C::kQInTmem) {
              mma_ts(dcol, tmem + C::kColQ + kk * 8, bd, kIdescQK, kk > 0 ? 1u : 0u);
            } else {
              mma_ss(dcol, dQ + (((kk >> 2) * C::kQChunk + (kk & 3) * 32) >> 4), bd, kIdescQK, kk > 0 ? 1u : 0u);
            }
          }
          tc_commit(bKempty(s));
          tc_commit(bSfull(int(j % NSB)));
          DBSP_TRC(kTrMmaS, j);
        }
        __syncwarp();
      };
      auto issue_pv = [&](uint32_t i) {
        const int b = int(i % NSB);
        const int s = int(i % NS);
        mbar_wait(bPfull(b), (i / NSB) & 1);
        mbar_wait(bVfull(s), (i / NS) & 1);
        tc_fence_after();
        const uint32_t pcol = tmem + C::kColS + 64u * b;
        const uint64_t bV = dV + ((uint32_t(s) * C::kTileBytes) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_ts(tmem + C::kColO, pcol + kk * 8, bV + ((kk * 2048) >> 4), kIdescPV, (i > 0 || kk > 0) ? 1u : 0u);
          tc_commit(bVempty(s));
          if constexpr (LMMA) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_ts(tmem + C::kColL, pcol + kk * 8, dOnes + ((kk * 2048) >> 4), kIdescL, (i > 0 || kk > 0) ? 1u : 0u);
          }
          tc_commit(bOdone(i));
          DBSP_TRC(kTrMmaPV, i);
        }
        __syncwarp();
      };
      mbar_wait(bQready, 0);
      tc_fence_after();
      // S runs NSB tiles ahead of PV.  S_{j+NSB} reuses the TMEM columns of
      // P_j, which PV_j (issued just before) reads: tcgen05.mma ops of one
      // thread execute in issue order, so that read precedes the later write
      // (DBSP_STRICT_WAR adds an explicit completion wait).  elect.sync picks
      // the same lane every time (the lowest active one), so every MMA of the
      // kernel comes from one thread.
      for (uint32_t j = 0; j < uint32_t(NSB) && j < count; ++j) issue_s(j);
      for (uint32_t j = 0; j < count; ++j) {
        issue_pv(j);
        if (j + NSB < count) {
#ifdef DBSP_STRICT_WAR
          mbar_wait(bOdone(j), (j >> 1) & 1);
#endif
          issue_s(j + NSB);
        }
      }
      if (elect_one()) tc_commit(bOfinal);
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ Q -> TMEM
    const int row = threadIdx.x;  // 0..127 == TMEM lane
    const bool upper = row >= 64;
    const uint32_t lane_off = uint32_t(warp * 32) << 16;
    const uint32_t qblk = upper ? it.qb : it.qa;
    const uint32_t token = qblk * 64u + uint32_t(row & 63);
    if (C::kQInTmem && count > 0) {
      const bool in = token < p.q_tokens;
      const uint4* src = reinterpret_cast<const uint4*>(p.q + (size_t(token) * p.heads + it.head) * D);
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        uint32_t w[32];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint4 x = in ? __ldg(src + c * 8 + i) : make_uint4(0, 0, 0, 0);
          w[4 * i + 0] = x.x;
          w[4 * i + 1] = x.y;
          w[4 * i + 2] = x.z;
          w[4 * i + 3] = x.w;
        }
        tmem_st32(tmem + lane_off + C::kColQ + c * 32, w);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bQready);
    }

#ifdef DBSP_TRACE_EXPS
    if (lane == 0 && p.trace && blockIdx.x < kTraceBlocks) {
      unsigned long long* hdr = p.trace + (size_t(blockIdx.x) * kTraceTiles + kTraceTiles - 1) * kTrEvents;
      uint32_t wid;
      asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
      hdr[warp] = wid;
      if (warp == 0) hdr[4] = smid();
    }
#endif
    // ------------------------------------------------------------ softmax
    const uint32_t dense_bit = upper ? dbsp_core::kEntryDenseB : dbsp_core::kEntryDenseA;
    const float sl2 = p.scale_log2;
    const uint32_t* ent = p.entries + it.begin;
    float m = -INFINITY, l = 0.f;
    // Entries are read one step ahead: when S_j is already waiting, the
    // global load of entry j would otherwise sit on the softmax chain.
    uint32_t e_next = count > 0 ? __ldg(ent) : 0u;
    // Unrolled by the S-buffer count: 2% fewer instructions (buffer index and
    // phase become constants), CogVideoX 2.804 M vs 2.821 M cycles (ncu).
#pragma unroll 2
    for (uint32_t j = 0; j < count; ++j) {
      const uint32_t e = e_next;
      if (j + 1 < count) e_next = __ldg(ent + j + 1);
      const bool dense = (e & dense_bit) != 0;  // warp-uniform (one half per warp)
      const int b = int(j % NSB);
      const uint32_t scol = tmem + lane_off + C::kColS + 64u * b;
      mbar_wait(bSfull(b), (j / NSB) & 1);
      tc_fence_after();
#if defined(DBSP_TRACE) && defined(DBSP_TRACE_FINE1)
      DBSP_TRF(kTrSoftStart, j);
#else
      if (lane == 0 && (warp == 0 || warp == 2)) DBSP_TRC(warp == 0 ? kTrSoftStart : kTrSoftStartHi, j);
#endif
      if (dense) {
        uint32_t sa[32], sb[32];
        tmem_ld32(scol, sa);
        tmem_ld32(scol + 32, sb);
        tmem_ld_wait();
        DBSP_TRF(4, j);
        const uint32_t valid = ((e >> dbsp_core::kEntryValidShift) & 63u) + 1u;
        float v[64];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          v[i] = __uint_as_float(sa[i]);
          v[i + 32] = __uint_as_float(sb[i]);
        }
        if (valid < 64) {  // partial last KV block (warp-uniform)
#pragma unroll
          for (int i = 0; i < 64; ++i)
            if (uint32_t(i) >= valid) v[i] = -INFINITY;
        }
        // Row max (log2 domain) as a 3-input-max tree (FMNMX3): depth 5, not a
        // 64-long chain.
        auto row_max2 = [&]() {
          float mx[8];
#pragma unroll
          for (int a = 0; a < 8; ++a) {
            mx[a] = fmax3f(v[8 * a], v[8 * a + 1], v[8 * a + 2]);
            mx[a] = fmax3f(mx[a], v[8 * a + 3], v[8 * a + 4]);
            mx[a] = fmax3f(mx[a], v[8 * a + 5], v[8 * a + 6]);
            mx[a] = fmaxf(mx[a], v[8 * a + 7]);
          }
          return fmaxf(fmax3f(mx[0], mx[1], mx[2]), fmax3f(fmax3f(mx[3], mx[4], mx[5]), mx[6], mx[7])) * sl2;
        };
        // Raise the running max to mt2 when it grows by more than the
        // threshold; O and l are rescaled by the same factor.
        auto raise_max = [&](float mt2) {
          const bool resc = mt2 > m + kRescaleThreshold;
          const bool need_o = resc && (m != -INFINITY);
          float alpha = 1.f;
          if (resc) {
            alpha = fast_exp2(m - mt2);
            if constexpr (!LMMA) l *= alpha;
            m = mt2;
          }
          if (__any_sync(0xffffffffu, need_o)) {
            // O must be quiescent.  With one S buffer, S_j was issued after
            // PV_{j-1}, so its completion (seen above) implies PV_{j-1}'s.
            if (NSB > 1 && j > 0) {
              mbar_wait(bOdone(j - 1), ((j - 1) >> 1) & 1);
              tc_fence_after();
            }
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
              uint32_t o[32];
              tmem_ld32(tmem + lane_off + C::kColO + c * 32, o);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
              tmem_st32(tmem + lane_off + C::kColO + c * 32, o);
            }
            if constexpr (LMMA) {  // l: the first of its 16 (equal) columns is the one read
              const uint32_t lv = tmem_ld1(tmem + lane_off + C::kColL);
              tmem_ld_wait();
              tmem_st1(tmem + lane_off + C::kColL, __float_as_uint(__uint_as_float(lv) * alpha));
            }
          }
        };
        // P = 2^(S*scale - m) as packed bf16; returns the row sum (0 when the
        // tensor core sums the rows, LMMA).  Packed
        // f32x2 FMA/add (FFMA2/FADD2): half the non-MUFU issue slots.
        uint32_t pk[32];
        auto exps = [&]() {
          const float2 sc2 = make_float2(sl2, sl2), nm2 = make_float2(-m, -m);
          float2 acc2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float2 x = __ffma2_rn(make_float2(v[2 * i], v[2 * i + 1]), sc2, nm2);
            float2 pp;
            if ((poly_mask(POLY) >> (i & 7)) & 1) {  // FA4-style MUFU offload
              pp = exp2_poly3_pair(x);
            } else {
              pp = make_float2(fast_exp2(x.x), fast_exp2(x.y));
            }
            if constexpr (!LMMA) acc2[i & 1] = __fadd2_rn(acc2[i & 1], pp);
            pk[i] = pack_bf16x2(pp.x, pp.y);
          }
          if constexpr (LMMA) return 0.f;
          const float2 a2 = __fadd2_rn(acc2[0], acc2[1]);
          return a2.x + a2.y;
        };
        const float mt2 = row_max2();
        DBSP_TRF(5, j);
        raise_max(mt2);
#ifdef DBSP_TRACE_EXPS
        if (lane == 0 && j + 1 < uint32_t(kTraceTiles)) DBSP_TR(2 * warp, j);
#endif
        l += exps();
#ifdef DBSP_TRACE_EXPS
        if (lane == 0 && j + 1 < uint32_t(kTraceTiles)) DBSP_TR(2 * warp + 1, j);
#endif
        DBSP_TRF(6, j);
        tmem_st32(scol, pk);
      } else {  // this half's rows have no keys in the block: P = 0
        uint32_t z[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) z[i] = 0u;
        tmem_st32(scol, z);
      }
      tmem_st_wait();
      DBSP_TRF(7, j);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bPfull(b));
#if defined(DBSP_TRACE) && defined(DBSP_TRACE_FINE1)
      DBSP_TRF(kTrSoftEnd, j);
#else
      if (lane == 0 && (warp == 0 || warp == 2)) DBSP_TRC(warp == 0 ? kTrSoftEnd : kTrSoftEndHi, j);
#endif
    }

    // ------------------------------------------------------------ epilogue
    if (count > 0) {
      // Not bOdone: up to two PV phases may still be outstanding here, and a
      // parity wait cannot tell phase count-1 from phase count-3.
      mbar_wait(bOfinal, 0);
      tc_fence_after();
      if constexpr (LMMA) {
        const uint32_t lv = tmem_ld1(tmem + lane_off + C::kColL);
        tmem_ld_wait();
        l = __uint_as_float(lv);
      }
    }
    const bool live = !(upper && it.single) && token < p.q_tokens;
    const float inv_l = l > 0.f ? 1.f / l : 0.f;
    const float kLn2 = 0.6931471805599453f;
    const float lse_new = l > 0.f ? (m + log2f(l)) * kLn2 : -INFINITY;
    const size_t orow = (size_t(token) * p.heads + it.head) * D;
    const size_t lidx = size_t(it.head) * p.q_tokens + token;
    bool live_out = live;
    __nv_bfloat16* const orow_ptr = out_row_ptr<D>(p, token, it.head, live_out);

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
    }
    const bool write_bf16 = !acc || (p.mode & kModeFinalize);
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
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
      if (write_bf16 && live_out) {
        uint4* po = reinterpret_cast<uint4*>(orow_ptr + c * 32);
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
    if (p.out_peers) __threadfence_system();  // peer stores complete before the kernel ends
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 5) tmem_dealloc(tmem, kTmemCols);
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
