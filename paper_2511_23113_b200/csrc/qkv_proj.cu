// K6: the DiT QKV projection with the sequence-parallel all-to-all(v) fused
// into its epilogue ("fuse the QKV projection
// epilogue with the Ulysses a2a send").
//
// Y = X W^T (+ b) on one rank's home tokens: X [T, C] bf16 (C = hidden),
// W [3*H*d, C] bf16 (nn.Linear layout: rows = q | k | v, each head-major),
// fp32 accumulation in TMEM.  Instead of writing Y home and running the
// exchange afterwards (sp.py step 1), every output row segment goes straight
// to the rank that consumes it under the plan -- Q rows of block b, head h to
// GPU u(h)*y + q_assign[b]; K/V rows to GPU u(h)*y + kv_assign[b] (the ring
// rank that holds group kv_assign[b] in period 0) -- at that rank's local
// buffer position, through peer pointers over NVLink.  The stores of each
// tile overlap the MMAs of the next one (two CTAs per SM).
//
// Tile: 128 tokens x 256 outputs, K step 64; tcgen05.mma kind::f16 M=128
// N=256 (SS, both operands TMA-staged with 128-byte swizzle), accumulator in
// 256 TMEM columns.  Warp roles as in K4: warps 0-3 epilogue (thread = row),
// warp 4 TMA producer, warp 5 TMEM owner + MMA issuer.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/dbsp_b200.h"
#include "capi_util.hpp"
#include "core.hpp"
#include "ptx.cuh"

namespace dbsp_dev {

constexpr int kQkvThreads = 192;
constexpr int kQkvStages = 2;
constexpr uint32_t kQkvA = 128u * 64u * 2u;  // 16 KB: 128 tokens x 64 k
constexpr uint32_t kQkvB = 256u * 64u * 2u;  // 32 KB: 256 outputs x 64 k
constexpr uint32_t kQkvSmem = kQkvStages * (kQkvA + kQkvB) + 1024 + 8 * (2 * kQkvStages + 1) + 16;

struct QkvParams {
  uint32_t T, C, H, d;  // home tokens, hidden, heads, head dim
  const __nv_bfloat16* bias;  // [3*H*d] or null
  __nv_bfloat16* out;         // local [T, 3*H*d] (no scatter) or null
  // scatter (null peers: write `out`)
  __nv_bfloat16* const* q_peers;  // [G] dest rank -> its local Q buffer [nq_loc*64, Hu, d]
  __nv_bfloat16* const* k_peers;
  __nv_bfloat16* const* v_peers;
  const uint32_t* blk;    // per home block b: {q dest ring rank, q local pos, kv group, kv local pos}
  const uint32_t* head;   // per head h: {u, local head index}
  const uint32_t* heads_of;  // per dest rank: local head count (Hu)
  uint32_t y;
};

// Tile order: groups of kGroupM consecutive M tiles sweep all N tiles, so the
// CTAs resident at any time share ~16 X row-bands and a few W row-bands in
// L2 (a plain M-fast order re-streams X from HBM once per N tile: at 32K
// tokens that is 20 GB per call).
constexpr uint32_t kGroupM = 16;
__device__ __forceinline__ void tile_of(uint32_t L, uint32_t nM, uint32_t nN, uint32_t& mt, uint32_t& nt) {
  const uint32_t per_group = kGroupM * nN;
  const uint32_t g = L / per_group, r = L % per_group;
  const uint32_t gm = min(kGroupM, nM - g * kGroupM);  // last group may be short
  mt = g * kGroupM + r % gm;
  nt = r / gm;
}

// Epilogue of one 128x256 tile (thread = row = TMEM lane): bias, bf16, and the
// store -- home [T, 3*H*d], or the consuming rank's local Q/K/V buffer.
__device__ __forceinline__ void qkv_epilogue(const QkvParams& p, uint32_t tmem, uint32_t m0, uint32_t n0, int warp,
                                             int lane, uint32_t bAcc) {
  const uint32_t row = uint32_t(warp * 32 + lane);
  const uint32_t t = m0 + row;
  const uint32_t lane_off = uint32_t(warp * 32) << 16;
  const uint32_t HD = p.H * p.d;
  mbar_wait(bAcc, 0);
  tc_fence_after();
  const bool live = t < p.T;
  const uint32_t* bk = p.blk + 4 * (t >> 6);
#pragma unroll 1
  for (int c = 0; c < 8; ++c) {
    uint32_t o[32];
    tmem_ld32(tmem + lane_off + c * 32, o);
    tmem_ld_wait();
    const uint32_t n = n0 + c * 32;
    if (!live || n >= 3 * HD) continue;
    const uint32_t which = n / HD, h = (n % HD) / p.d, dd = n % p.d;
    float r[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) r[i] = __uint_as_float(o[i]);
    if (p.bias) {
      const uint4* bb = reinterpret_cast<const uint4*>(p.bias + n);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint4 b4 = __ldg(bb + i);
        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b4);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = __bfloat1622float2(b2[j]);
          r[8 * i + 2 * j] += f.x;
          r[8 * i + 2 * j + 1] += f.y;
        }
      }
    }
    __nv_bfloat16* dst;
    if (p.q_peers) {
      const uint32_t u = p.head[2 * h], hl = p.head[2 * h + 1];
      const uint32_t rr = which == 0 ? bk[0] : bk[2];
      const uint32_t pos = which == 0 ? bk[1] : bk[3];
      const uint32_t dest = u * p.y + rr;
      __nv_bfloat16* const* peers = which == 0 ? p.q_peers : which == 1 ? p.k_peers : p.v_peers;
      dst = peers[dest] + ((size_t(pos) * 64 + (t & 63)) * p.heads_of[dest] + hl) * p.d + dd;
    } else {
      dst = p.out + size_t(t) * 3 * HD + n;
    }
    uint4* po = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int i = 0; i < 4; ++i)
      po[i] = make_uint4(pack_bf16x2(r[8 * i + 0], r[8 * i + 1]), pack_bf16x2(r[8 * i + 2], r[8 * i + 3]),
                         pack_bf16x2(r[8 * i + 4], r[8 * i + 5]), pack_bf16x2(r[8 * i + 6], r[8 * i + 7]));
  }
  if (p.q_peers) __threadfence_system();
}

__global__ void __launch_bounds__(kQkvThreads, 2)
    qkv_proj_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                    const QkvParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t sA = base, sB = base + kQkvStages * kQkvA;
  const uint32_t sBar = sB + kQkvStages * kQkvB;
  auto bFull = [&](int s) { return sBar + 8u * s; };
  auto bEmpty = [&](int s) { return sBar + 8u * (kQkvStages + s); };
  const uint32_t bAcc = sBar + 8u * (2 * kQkvStages);
  const uint32_t sTmemSlot = sBar + 8u * (2 * kQkvStages + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t mt, nt;
  tile_of(blockIdx.x, (p.T + 127) / 128, (3 * p.H * p.d) / 256, mt, nt);
  const uint32_t m0 = mt * 128u, n0 = nt * 256u;
  const uint32_t ksteps = (p.C + 63) / 64;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kQkvStages; ++s) {
      mbar_init(bFull(s), 1);
      mbar_init(bEmpty(s), 1);
    }
    mbar_init(bAcc, 1);
    mbar_fence_init();
  }
  if (warp == 4 && lane == 0) {
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmW);
  }
  if (warp == 5) tmem_alloc(sTmemSlot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(gbase + (sTmemSlot - base));

  if (warp == 4) {
    if (lane == 0) {
      const uint64_t pol_x = l2_policy_evict_last();   // X tile rows are reused by all N tiles
      const uint64_t pol_w = l2_policy_evict_last();
      for (uint32_t k = 0; k < ksteps; ++k) {
        const int s = int(k % kQkvStages);
        mbar_wait(bEmpty(s), ((k / kQkvStages) & 1) ^ 1);
        mbar_expect_tx(bFull(s), kQkvA + kQkvB);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
            " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(sA + s * kQkvA),
            "l"(reinterpret_cast<uint64_t>(&tmX)), "r"(int(k * 64)), "r"(int(m0)), "r"(bFull(s)), "l"(pol_x)
            : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
            " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(sB + s * kQkvB),
            "l"(reinterpret_cast<uint64_t>(&tmW)), "r"(int(k * 64)), "r"(int(n0)), "r"(bFull(s)), "l"(pol_w)
            : "memory");
      }
    } else {
      mbar_wait(bAcc, 0);
    }
    __syncwarp();
  } else if (warp == 5) {
    if (lane == 0) {
      constexpr uint32_t kIdesc = idesc_bf16(128, 256, false, false);
      for (uint32_t k = 0; k < ksteps; ++k) {
        const int s = int(k % kQkvStages);
        mbar_wait(bFull(s), (k / kQkvStages) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t ad = smem_desc_sw128(sA + s * kQkvA + kk * 32, 16, 1024);
          const uint64_t bd = smem_desc_sw128(sB + s * kQkvB + kk * 32, 16, 1024);
          mma_ss(tmem, ad, bd, kIdesc, (k > 0 || kk > 0) ? 1u : 0u);
        }
        tc_commit(bEmpty(s));
      }
      tc_commit(bAcc);
    } else {
      mbar_wait(bAcc, 0);
    }
    __syncwarp();
  } else {
    qkv_epilogue(p, tmem, m0, n0, warp, lane, bAcc);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 5) tmem_dealloc(tmem, 256);
}


// The same tile loop with a CTA pair (tcgen05 cta_group::2): a cluster of two
// CTAs on two SMs computes a 256x256 tile; each CTA stages its own 128 token
// rows and HALF of the 256 weight rows, and the leader issues M=256 MMAs.
// Per SM the smem port moves A 4 KB + B 4 KB per 128-cycle MMA plus 32 KB of
// TMA writes per K step, 128 B/clk, against 190 B/clk for the one-SM tile
// (profiles: 1272 vs 1551 TFLOP/s of cuBLAS on a home shard).
constexpr int kQkvPStages = 3;
constexpr uint32_t kQkvPB = 128u * 64u * 2u;  // 16 KB: this CTA's half of the 256 weight rows
constexpr uint32_t kQkvPSmem = kQkvPStages * (kQkvA + kQkvPB) + 1024 + 8 * (2 * kQkvPStages + 1) + 16;

__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const void* tmap, int c0, int c1, uint32_t bar,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(bar), "l"(policy)
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kQkvThreads, 2)
    qkv_proj_pair_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                         const QkvParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t sA = base, sB = base + kQkvPStages * kQkvA;
  const uint32_t sBar = sB + kQkvPStages * kQkvPB;
  auto bFull = [&](int s) { return sBar + 8u * s; };
  auto bEmpty = [&](int s) { return sBar + 8u * (kQkvPStages + s); };
  const uint32_t bAcc = sBar + 8u * (2 * kQkvPStages);
  const uint32_t sTmemSlot = sBar + 8u * (2 * kQkvPStages + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  uint32_t mt, nt;
  tile_of(blockIdx.x >> 1, (p.T + 255) / 256, (3 * p.H * p.d) / 256, mt, nt);
  const uint32_t m0 = mt * 256u + rank * 128u, n0 = nt * 256u;
  const uint32_t ksteps = (p.C + 63) / 64;
  auto leader = [&](uint32_t local_bar) { return mapa_shared(local_bar, 0); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kQkvPStages; ++s) {
      mbar_init(bFull(s), 1);
      mbar_init(bEmpty(s), 1);
    }
    mbar_init(bAcc, 1);
    mbar_fence_init();
  }
  if (warp == 4 && lane == 0) {
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmW);
  }
  if (warp == 5) tmem_alloc_pair(sTmemSlot, 256);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(gbase + (sTmemSlot - base));

  if (warp == 4) {
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_last();
      for (uint32_t k = 0; k < ksteps; ++k) {
        const int s = int(k % kQkvPStages);
        mbar_wait(bEmpty(s), ((k / kQkvPStages) & 1) ^ 1);
        if (rank == 0) mbar_expect_tx(bFull(s), 2 * (kQkvA + kQkvPB));
        tma_load_2d_pair(sA + s * kQkvA, &tmX, int(k * 64), int(m0), leader(bFull(s)), pol);
        tma_load_2d_pair(sB + s * kQkvPB, &tmW, int(k * 64), int(n0 + rank * 128), leader(bFull(s)), pol);
      }
    } else {
      mbar_wait(bAcc, 0);
    }
    __syncwarp();
  } else if (warp == 5) {
    if (lane == 0 && rank == 0) {
      constexpr uint32_t kIdesc = idesc_bf16(256, 256, false, false);
      for (uint32_t k = 0; k < ksteps; ++k) {
        const int s = int(k % kQkvPStages);
        mbar_wait(bFull(s), (k / kQkvPStages) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t ad = smem_desc_sw128(sA + s * kQkvA + kk * 32, 16, 1024);
          const uint64_t bd = smem_desc_sw128(sB + s * kQkvPB + kk * 32, 16, 1024);
          mma_ss_pair(tmem, ad, bd, kIdesc, (k > 0 || kk > 0) ? 1u : 0u);
        }
        tc_commit_pair(bEmpty(s), 0x3);
      }
      tc_commit_pair(bAcc, 0x3);
    } else {
      mbar_wait(bAcc, 0);
    }
    __syncwarp();
  } else {
    qkv_epilogue(p, tmem, m0, n0, warp, lane, bAcc);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the leader's MMAs wrote this CTA's TMEM and read its smem
  tc_fence_after();
  if (warp == 5) tmem_dealloc_pair(tmem, 256);
}

}  // namespace dbsp_dev

namespace {

using namespace dbsp_core;

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(kCuda, std::string(what) + ": " + cudaGetErrorString(e));
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(ptr);
  });
  if (!fn) fail(kCuda, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// Row-major [rows, cols] bf16, box = 64 cols x box_rows rows, 128-byte swizzle.
CUtensorMap tmap2d(const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {64, box_rows};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(kCuda, "cuTensorMapEncodeTiled (qkv) failed: " + std::to_string(int(r)));
  return m;
}

}  // namespace

extern "C" {

int dbsp_qkv_project(const dbsp_qkv_args* a, const dbsp_qkv_scatter* sc, void* stream) {
  return dbsp_capi::guard([&] {
    if (!a || !a->x || !a->w) fail(kContract, "null qkv arguments");
    if (a->tokens == 0 || a->hidden == 0 || a->heads == 0) fail(kConfig, "qkv dimensions must be positive");
    if (a->head_dim != 64 && a->head_dim != 128) fail(kConfig, "head_dim must be 64 or 128");
    if (a->hidden % 64) fail(kConfig, "hidden must be a multiple of 64");
    const uint64_t N = 3ull * a->heads * a->head_dim;
    if (N % 256) fail(kConfig, "3 * heads * head_dim must be a multiple of 256");
    if (!sc && !a->out) fail(kContract, "null output");
    if (sc && (a->tokens % 64)) fail(kContract, "the fused scatter needs whole 64-token blocks");
    if (sc && (!sc->q_peers || !sc->k_peers || !sc->v_peers || !sc->block_map || !sc->head_map || !sc->heads_of))
      fail(kContract, "incomplete qkv scatter");
    dbsp_dev::QkvParams p;
    p.T = a->tokens;
    p.C = a->hidden;
    p.H = a->heads;
    p.d = a->head_dim;
    p.bias = static_cast<const __nv_bfloat16*>(a->bias);
    p.out = static_cast<__nv_bfloat16*>(a->out);
    p.q_peers = sc ? reinterpret_cast<__nv_bfloat16* const*>(sc->q_peers) : nullptr;
    p.k_peers = sc ? reinterpret_cast<__nv_bfloat16* const*>(sc->k_peers) : nullptr;
    p.v_peers = sc ? reinterpret_cast<__nv_bfloat16* const*>(sc->v_peers) : nullptr;
    p.blk = sc ? sc->block_map : nullptr;
    p.head = sc ? sc->head_map : nullptr;
    p.heads_of = sc ? sc->heads_of : nullptr;
    p.y = sc ? sc->ring : 1;
    static const bool single = [] {
      const char* e = std::getenv("DBSP_K6_SINGLE");
      return e && e[0] == '1';
    }();
    const CUtensorMap tx = tmap2d(a->x, a->tokens, a->hidden, 128);
    if (!single) {  // CTA-pair kernel: each CTA stages half of the 256 weight rows
      const CUtensorMap tw = tmap2d(a->w, N, a->hidden, 128);
      static std::once_flag once2;
      static cudaError_t attr2 = cudaSuccess;
      std::call_once(once2, [] {
        attr2 = cudaFuncSetAttribute(dbsp_dev::qkv_proj_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     dbsp_dev::kQkvPSmem);
      });
      ck(attr2, "cudaFuncSetAttribute(qkv pair)");
      const dim3 grid(2 * ((a->tokens + 255) / 256) * uint32_t(N / 256));
      dbsp_core::count_launch();
      dbsp_dev::qkv_proj_pair_kernel<<<grid, dbsp_dev::kQkvThreads, dbsp_dev::kQkvPSmem,
                                       reinterpret_cast<cudaStream_t>(stream)>>>(tx, tw, p);
      ck(cudaGetLastError(), "qkv_proj_pair launch");
      return;
    }
    const CUtensorMap tw = tmap2d(a->w, N, a->hidden, 256);
    static std::once_flag once;
    static cudaError_t attr = cudaSuccess;
    std::call_once(once, [] {
      attr = cudaFuncSetAttribute(dbsp_dev::qkv_proj_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  dbsp_dev::kQkvSmem);
    });
    ck(attr, "cudaFuncSetAttribute(qkv)");
    const dim3 grid(((a->tokens + 127) / 128) * uint32_t(N / 256));
    dbsp_core::count_launch();
    dbsp_dev::qkv_proj_kernel<<<grid, dbsp_dev::kQkvThreads, dbsp_dev::kQkvSmem,
                                reinterpret_cast<cudaStream_t>(stream)>>>(tx, tw, p);
    ck(cudaGetLastError(), "qkv_proj launch");
  });
}

}  // extern "C"
