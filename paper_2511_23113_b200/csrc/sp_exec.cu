// Sequence-parallel execution of one block-sparse attention call in C++:
// the C-ABI form of paper_2511_23113_b200/sp.py (SURVEY.md §8(b) "new
// attention call": SpContext + sparse_attention over NCCL).
//
// GPU g = u*y + r (metrics.hpp:116).  One call under strategy UxRy and plan
// (head, q, kv assignments):
//   1. one fused all-to-all(v) over all G ranks (Ulysses head scatter C1 and
//      the db-SP balancing moves C2): rank (u,r) receives Q blocks
//      {q : q_assign = r} and KV blocks of its initial ring group {k : kv = r}
//      for heads {h : head = u}, from each home rank, in ascending block order;
//   2. y ring periods (C3): in period p the rank holds KV group (r+p) mod y
//      (metrics.hpp:131-132), runs K4 in accumulate mode (K5 merge in the
//      epilogue) while the next group arrives from ring rank r+1 on the
//      communication stream (double-buffered);
//   3. the reverse all-to-all(v) returns O to the home layout.
// Two drivers share the per-rank code: NCCL (one process per GPU,
// dbsp_sp_attention) and an in-process one that runs all G ranks on this GPU
// with device copies as the transport (dbsp_sp_attention_simulated), which
// is how the multi-rank logic is tested on one GPU.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>

#include <chrono>
#include <thread>

#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <optional>
#include <string>
#include <vector>

#include "../../include/dbsp_b200.h"
#include "capi_util.hpp"
#include "core.hpp"

using namespace dbsp_core;
using dbsp_capi::guard;

namespace {

// NCCL is resolved at run time (dlopen of libnccl.so.2) rather than linked: a
// process that already loaded torch's bundled NCCL gets that same library
// back, so there is never a second NCCL in the process.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
};

const NcclApi& N() {
  static NcclApi api;
  static std::string err;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load NCCL: ") + dlerror();
      return;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn && err.empty()) err = std::string("NCCL symbol missing: ") + name;
    };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.Send, "ncclSend");
    sym(api.Recv, "ncclRecv");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    sym(api.GetErrorString, "ncclGetErrorString");
    sym(api.CommGetAsyncError, "ncclCommGetAsyncError");
    sym(api.CommAbort, "ncclCommAbort");
  });
  if (!err.empty()) dbsp_core::fail(dbsp_core::kCuda, err);
  return api;
}

}  // namespace

namespace dbsp_dev {
// dst[(i*nh + j)*d + c] = src[row(i)*H*d + heads[j]*d + c], row(i) = (blocks[i/64] - lo)*64 + i%64.
__global__ void sp_gather_kernel(const uint4* __restrict__ src, uint32_t H, uint32_t d16,
                                 const uint32_t* __restrict__ blocks, uint32_t lo,
                                 const uint32_t* __restrict__ heads, uint32_t nh, uint32_t nrows,
                                 uint4* __restrict__ dst) {
  const size_t total = size_t(nrows) * nh * d16;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += size_t(gridDim.x) * blockDim.x) {
    const uint32_t c = uint32_t(i % d16);
    const size_t rj = i / d16;
    const uint32_t j = uint32_t(rj % nh), r = uint32_t(rj / nh);
    const size_t srow = size_t(blocks[r >> 6] - lo) * 64 + (r & 63);
    dst[i] = src[(srow * H + heads[j]) * d16 + c];
  }
}
// The inverse: out[row(i)*H*d + heads[j]*d + c] = src[(i*nh + j)*d + c].
__global__ void sp_scatter_kernel(const uint4* __restrict__ src, uint32_t H, uint32_t d16,
                                  const uint32_t* __restrict__ blocks, uint32_t lo,
                                  const uint32_t* __restrict__ heads, uint32_t nh, uint32_t nrows,
                                  uint4* __restrict__ out) {
  const size_t total = size_t(nrows) * nh * d16;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += size_t(gridDim.x) * blockDim.x) {
    const uint32_t c = uint32_t(i % d16);
    const size_t rj = i / d16;
    const uint32_t j = uint32_t(rj % nh), r = uint32_t(rj / nh);
    const size_t orow = size_t(blocks[r >> 6] - lo) * 64 + (r & 63);
    out[(orow * H + heads[j]) * d16 + c] = src[i];
  }
}
// A ring whose final period holds an empty KV group launches no K4 there:
// the merged fp32 accumulator (already normalised, see the K4 epilogue) is
// written out as bf16 instead.
__global__ void sp_finalize_kernel(const float4* __restrict__ acc, uint2* __restrict__ out, size_t n4) {
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += size_t(gridDim.x) * blockDim.x) {
    const float4 a = acc[i];
    __nv_bfloat162 lo = __floats2bfloat162_rn(a.x, a.y), hi = __floats2bfloat162_rn(a.z, a.w);
    out[i] = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
  }
}
}  // namespace dbsp_dev

namespace {

// NVTX ranges for nsys / ncu --nvtx (header-only NVTX v3; no-ops without a tool).
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(kCuda, std::string(what) + ": " + cudaGetErrorString(e));
}
void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(kCuda, std::string(what) + ": " + N().GetErrorString(r));
}
void rc(int code) {
  if (code != 0) fail(code, dbsp_last_error());
}

std::pair<uint32_t, uint32_t> home_range(uint32_t rank, uint32_t world, uint32_t nb) {
  return {uint32_t(uint64_t(rank) * nb / world), uint32_t(uint64_t(rank + 1) * nb / world)};
}

struct Layout {
  uint32_t rank = 0, u = 0, r = 0, y = 1;
  std::vector<uint32_t> heads, q_blocks;
  std::vector<std::vector<uint32_t>> groups;  // per ring group: KV blocks ascending
  uint32_t period_group(uint32_t p) const { return (r + p) % y; }
};

std::vector<Layout> rank_layouts(Strategy s, const Plan& plan, uint32_t nq, uint32_t nk) {
  std::vector<std::vector<uint32_t>> groups(s.y);
  for (uint32_t k = 0; k < nk; ++k) groups[plan.kv[k]].push_back(k);
  std::vector<Layout> out;
  for (uint32_t u = 0; u < s.x; ++u)
    for (uint32_t r = 0; r < s.y; ++r) {
      Layout L;
      L.rank = u * s.y + r;
      L.u = u;
      L.r = r;
      L.y = s.y;
      for (uint32_t h = 0; h < plan.head.size(); ++h)
        if (plan.head[h] == u) L.heads.push_back(h);
      for (uint32_t q = 0; q < nq; ++q)
        if (plan.q[q] == r) L.q_blocks.push_back(q);
      L.groups = groups;
      out.push_back(std::move(L));
    }
  return out;
}

std::vector<uint32_t> in_range(const std::vector<uint32_t>& v, uint32_t lo, uint32_t hi) {
  std::vector<uint32_t> o;
  for (uint32_t b : v)
    if (b >= lo && b < hi) o.push_back(b);
  return o;
}

// Device copy of a host u32 list (kept alive by the owner).
struct DevList {
  uint32_t* p = nullptr;
  uint32_t n = 0;
  void set(const std::vector<uint32_t>& v, cudaStream_t s) {
    n = uint32_t(v.size());
    if (p) cudaFree(p);
    p = nullptr;
    if (n) {
      ck(cudaMalloc(&p, n * 4), "cudaMalloc list");
      ck(cudaMemcpyAsync(p, v.data(), n * 4, cudaMemcpyHostToDevice, s), "list h2d");
    }
  }
  ~DevList() {
    if (p) cudaFree(p);
  }
};

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void* get(size_t n) {
    if (n > bytes) {
      if (p) cudaFree(p);
      p = nullptr;
      ck(cudaMalloc(&p, std::max<size_t>(n, 16)), "cudaMalloc sp buffer");
      bytes = std::max<size_t>(n, 16);
    }
    return p;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

void launch_gather(const void* src, uint32_t H, uint32_t d, const DevList& blocks, uint32_t lo,
                   const DevList& heads, void* dst, cudaStream_t s) {
  const uint32_t nrows = blocks.n * 64;
  if (!nrows || !heads.n) return;
  const size_t total = size_t(nrows) * heads.n * (d / 8);
  const uint32_t grid = uint32_t(std::min<size_t>((total + 255) / 256, 148 * 16));
  dbsp_core::count_launch();
  dbsp_dev::sp_gather_kernel<<<grid, 256, 0, s>>>(static_cast<const uint4*>(src), H, d / 8, blocks.p, lo, heads.p,
                                                  heads.n, nrows, static_cast<uint4*>(dst));
  ck(cudaGetLastError(), "sp_gather launch");
}

void launch_scatter(const void* src, uint32_t H, uint32_t d, const DevList& blocks, uint32_t lo,
                    const DevList& heads, void* out, cudaStream_t s) {
  const uint32_t nrows = blocks.n * 64;
  if (!nrows || !heads.n) return;
  const size_t total = size_t(nrows) * heads.n * (d / 8);
  const uint32_t grid = uint32_t(std::min<size_t>((total + 255) / 256, 148 * 16));
  dbsp_core::count_launch();
  dbsp_dev::sp_scatter_kernel<<<grid, 256, 0, s>>>(static_cast<const uint4*>(src), H, d / 8, blocks.p, lo, heads.p,
                                                   heads.n, nrows, static_cast<uint4*>(out));
  ck(cudaGetLastError(), "sp_scatter launch");
}

uint64_t fnv1a(uint64_t h, const void* p, size_t n) {
  const uint8_t* b = static_cast<const uint8_t*>(p);
  for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  return h;
}

// Identity of one call's inputs to the per-rank planning: the plan, the
// strategy, the shapes and the mask words (FNV-1a over 64-bit words).
uint64_t call_key(const dbsp_mask_set* set, Strategy s, const Plan& p, uint32_t tokens, uint32_t d) {
  uint64_t h = 1469598103934665603ull;
  const uint32_t dims[6] = {s.x, s.y, tokens, d, set->num_heads, set->num_kv_blocks};
  h = fnv1a(h, dims, sizeof(dims));
  h = fnv1a(h, p.head.data(), p.head.size() * 4);
  h = fnv1a(h, p.q.data(), p.q.size() * 4);
  h = fnv1a(h, p.kv.data(), p.kv.size() * 4);
  const size_t wpr = (size_t(set->num_kv_blocks) + 63) / 64;
  for (uint32_t hd = 0; hd < set->num_heads; ++hd) {
    const uint64_t* w = set->heads[hd];
    for (size_t i = 0; i < size_t(set->num_q_blocks) * wpr; ++i) h = (h ^ w[i]) * 1099511628211ull;
  }
  return h;
}

// Everything one rank needs for one call: its layout, what it exchanges with
// each peer, its local buffers and its per-group K4 schedules.
struct RankExec {
  uint64_t key = 0;  // call_key of the prepared state (0 = none)
  uint32_t G = 1, rank = 0, H = 0, d = 0, S = 0, nb = 0;
  Layout me;
  std::vector<Layout> all;
  // forward exchange, per peer: my home blocks it needs (send) and counts I get (recv)
  std::vector<DevList> send_q, send_kv, peer_heads;
  std::vector<std::vector<uint32_t>> send_q_h, send_kv_h;
  std::vector<uint32_t> recv_q, recv_kv;
  // reverse exchange: per peer, my local O rows homed at the peer (offset, blocks) and,
  // receiving, the peer's rows homed here
  std::vector<uint32_t> oslice_off, oslice_n;
  std::vector<DevList> back_blocks, back_heads;
  DevList my_heads;
  size_t row_bytes = 0;  // bytes of one token row of the local buffers (Hu * d * 2)
  DevBuf q_loc, kbuf[2], vbuf[2], o_loc, o_acc, lse_acc;
  std::vector<DevBuf> sendq, sendk, sendv, recvo;
  DevBuf sendo;
  DevBuf words;  // the call's mask words on the device (K2 input)
  std::vector<dbsp_schedule*> sched;  // per ring group
  dbsp_mask_set set{};

  ~RankExec() {
    for (dbsp_schedule* s : sched)
      if (s) dbsp_schedule_destroy(s);
  }

  void plan(const dbsp_mask_set* mset, Strategy s, const Plan& p, uint32_t world, uint32_t r, uint32_t tokens,
            uint32_t head_dim, cudaStream_t st) {
    G = world;
    rank = r;
    H = mset->num_heads;
    d = head_dim;
    S = tokens;
    nb = mset->num_q_blocks;
    set = *mset;
    all = rank_layouts(s, p, mset->num_q_blocks, mset->num_kv_blocks);
    me = all[rank];
    row_bytes = size_t(me.heads.size()) * d * 2;
    const auto [lo, hi] = home_range(rank, G, nb);
    send_q.resize(G);
    send_kv.resize(G);
    peer_heads.resize(G);
    send_q_h.assign(G, {});
    send_kv_h.assign(G, {});
    recv_q.assign(G, 0);
    recv_kv.assign(G, 0);
    for (uint32_t dst = 0; dst < G; ++dst) {
      const Layout& D = all[dst];
      send_q_h[dst] = in_range(D.q_blocks, lo, hi);
      send_kv_h[dst] = in_range(D.groups[D.r], lo, hi);
      send_q[dst].set(send_q_h[dst], st);
      send_kv[dst].set(send_kv_h[dst], st);
      peer_heads[dst].set(D.heads, st);
      const auto [slo, shi] = home_range(dst, G, nb);
      recv_q[dst] = uint32_t(in_range(me.q_blocks, slo, shi).size());
      recv_kv[dst] = uint32_t(in_range(me.groups[me.r], slo, shi).size());
    }
    my_heads.set(me.heads, st);
    // reverse: my local Q rows are ascending by global block, so the rows homed
    // at each peer form one contiguous slice
    oslice_off.assign(G, 0);
    oslice_n.assign(G, 0);
    uint32_t off = 0;
    for (uint32_t s2 = 0; s2 < G; ++s2) {
      oslice_off[s2] = off;
      oslice_n[s2] = recv_q[s2];
      off += recv_q[s2];
    }
    back_blocks.resize(G);
    back_heads.resize(G);
    for (uint32_t src = 0; src < G; ++src) {
      back_blocks[src].set(in_range(all[src].q_blocks, lo, hi), st);
      back_heads[src].set(all[src].heads, st);
    }
    // per-group K4 schedules over this rank's local view, built on the GPU (K2)
    // from the call's mask words: a new plan or new masks cost one 1.3 MB copy
    // (Wan layer) and a few small kernels, no host pass over the masks
    for (dbsp_schedule* sc : sched)
      if (sc) dbsp_schedule_destroy(sc);
    sched.assign(me.y, nullptr);
    const size_t wpr = (size_t(mset->num_kv_blocks) + 63) / 64, per_head = size_t(mset->num_q_blocks) * wpr;
    uint64_t* dw = nullptr;
    if (!me.heads.empty() && !me.q_blocks.empty()) {
      dw = static_cast<uint64_t*>(words.get(per_head * H * 8));
      for (uint32_t h = 0; h < H; ++h)
        ck(cudaMemcpyAsync(dw + h * per_head, mset->heads[h], per_head * 8, cudaMemcpyHostToDevice, st),
           "mask words h2d");
    }
    if (!me.heads.empty() && !me.q_blocks.empty())
      for (uint32_t g = 0; g < me.y; ++g) {
        if (me.groups[g].empty()) continue;
        rc(dbsp_schedule_create(&sched[g]));
        dbsp_local_view v;
        v.num_heads = uint32_t(me.heads.size());
        v.head_ids = me.heads.data();
        v.num_q_blocks = uint32_t(me.q_blocks.size());
        v.q_block_ids = me.q_blocks.data();
        v.num_kv_blocks = uint32_t(me.groups[g].size());
        v.kv_block_ids = me.groups[g].data();
        v.kv_tokens_global = tokens;
        // the pair schedule (DBSP_SCHED_AUTO_D128 resolves to it for d=128)
        rc(dbsp_schedule_build_device(sched[g], dw, H, mset->num_q_blocks, mset->num_kv_blocks, &v,
                                      d == 128 ? (DBSP_SCHED_PAIR_Q | DBSP_SCHED_AUTO_D128) : DBSP_SCHED_PAIR_Q,
                                      st));
      }
    // buffers
    size_t max_g = 1;
    for (const auto& g : me.groups) max_g = std::max(max_g, g.size());
    const size_t nq_loc = me.q_blocks.size();
    q_loc.get(nq_loc * 64 * row_bytes);
    o_loc.get(nq_loc * 64 * row_bytes);
    for (int i = 0; i < 2; ++i) {
      kbuf[i].get(max_g * 64 * row_bytes);
      vbuf[i].get(max_g * 64 * row_bytes);
    }
    if (me.y > 1) {
      o_acc.get(nq_loc * 64 * me.heads.size() * d * 4);
      lse_acc.get(nq_loc * 64 * me.heads.size() * 4);
    }
    sendq.resize(G);
    sendk.resize(G);
    sendv.resize(G);
    recvo.resize(G);
    for (uint32_t dst = 0; dst < G; ++dst) {
      const size_t pb = size_t(all[dst].heads.size()) * d * 2 * 64;
      sendq[dst].get(send_q_h[dst].size() * pb);
      sendk[dst].get(send_kv_h[dst].size() * pb);
      sendv[dst].get(send_kv_h[dst].size() * pb);
      recvo[dst].get(back_blocks[dst].n * pb);
    }
  }

  // byte offsets of peer pieces in my local Q / KV buffers (peer order)
  size_t q_off(uint32_t s2) const {
    size_t o = 0;
    for (uint32_t i = 0; i < s2; ++i) o += recv_q[i];
    return o * 64 * row_bytes;
  }
  size_t kv_off(uint32_t s2) const {
    size_t o = 0;
    for (uint32_t i = 0; i < s2; ++i) o += recv_kv[i];
    return o * 64 * row_bytes;
  }
  size_t piece_bytes(uint32_t dst, size_t blocks) const { return blocks * 64 * all[dst].heads.size() * d * 2; }

  void pack_forward(const void* q_home, const void* k_home, const void* v_home, cudaStream_t st) {
    const uint32_t lo = home_range(rank, G, nb).first;
    for (uint32_t dst = 0; dst < G; ++dst) {
      launch_gather(q_home, H, d, send_q[dst], lo, peer_heads[dst], sendq[dst].p, st);
      launch_gather(k_home, H, d, send_kv[dst], lo, peer_heads[dst], sendk[dst].p, st);
      launch_gather(v_home, H, d, send_kv[dst], lo, peer_heads[dst], sendv[dst].p, st);
    }
  }

  // K4 for ring period p on the buffer `cur`.
  void compute(uint32_t p, int cur, cudaStream_t st) {
    const uint32_t y = me.y;
    const uint32_t g = me.period_group(p);
    const size_t nq_loc = me.q_blocks.size();
    if (me.heads.empty() || nq_loc == 0) return;
    const uint32_t hl = uint32_t(me.heads.size());
    if (p == 0 && y > 1) rc(dbsp_accum_init(static_cast<float*>(o_acc.p), static_cast<float*>(lse_acc.p),
                                            uint32_t(nq_loc * 64), hl, d, st));
    if (!sched[g]) {  // empty KV group (or no dense tile reachable): nothing to attend to
      if (y == 1) {
        ck(cudaMemsetAsync(o_loc.p, 0, nq_loc * 64 * row_bytes, st), "memset o");
      } else if (p == y - 1) {
        const size_t n4 = nq_loc * 64 * hl * d / 4;
        dbsp_core::count_launch();
        dbsp_dev::sp_finalize_kernel<<<uint32_t(std::min<size_t>((n4 + 255) / 256, 148 * 8)), 256, 0, st>>>(
            static_cast<const float4*>(o_acc.p), static_cast<uint2*>(o_loc.p), n4);
        ck(cudaGetLastError(), "sp_finalize launch");
      }
      return;
    }
    dbsp_attn_args a;
    std::memset(&a, 0, sizeof(a));
    a.q = q_loc.p;
    a.k = kbuf[cur].p;
    a.v = vbuf[cur].p;
    a.o = o_loc.p;
    a.q_tokens = uint32_t(nq_loc * 64);
    a.kv_tokens = uint32_t(me.groups[g].size() * 64);
    a.heads = hl;
    a.head_dim = d;
    if (y > 1) {
      a.o_accum = static_cast<float*>(o_acc.p);
      a.lse_accum = static_cast<float*>(lse_acc.p);
      a.accumulate = 1;
      a.finalize = p == y - 1;
    }
    rc(dbsp_attention_launch(sched[g], &a, st));
  }

  void pack_reverse(cudaStream_t st) {
    (void)st;  // O slices are contiguous in o_loc: sent in place
  }
  void unpack_reverse(void* o_home, cudaStream_t st) {
    const uint32_t lo = home_range(rank, G, nb).first;
    for (uint32_t src = 0; src < G; ++src)
      launch_scatter(recvo[src].p, H, d, back_blocks[src], lo, back_heads[src], o_home, st);
  }
  const uint8_t* oslice(uint32_t s2) const {
    return static_cast<const uint8_t*>(o_loc.p) + size_t(oslice_off[s2]) * 64 * row_bytes;
  }
};

}  // namespace

struct dbsp_sp_context {
  ncclComm_t comm = nullptr;
  bool aborted = false;
  uint32_t rank = 0, world = 1;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_ready[2] = {nullptr, nullptr}, ev_done = nullptr;
  std::unique_ptr<RankExec> ex;
  // per-period K4 timing of the last call (dbsp_sp_set_timing)
  bool timing = false;
  std::vector<cudaEvent_t> ev_k;  // 2 per period
  uint32_t timed_periods = 0;
  ~dbsp_sp_context() {
    for (cudaEvent_t e : ev_k) cudaEventDestroy(e);
    if (comm && !aborted) N().CommDestroy(comm);
    if (comm_stream) cudaStreamDestroy(comm_stream);
    for (cudaEvent_t e : ev_ready)
      if (e) cudaEventDestroy(e);
    if (ev_done) cudaEventDestroy(ev_done);
  }
};

namespace {

Plan plan_from(const dbsp_mask_set* set, const dbsp_plan* p) {
  if (!set || !p || !p->head_assignment || !p->q_assignment || !p->kv_assignment)
    fail(kContract, "null mask set or plan");
  Plan o;
  o.head.assign(p->head_assignment, p->head_assignment + set->num_heads);
  o.q.assign(p->q_assignment, p->q_assignment + set->num_q_blocks);
  o.kv.assign(p->kv_assignment, p->kv_assignment + set->num_kv_blocks);
  return o;
}

// A failed or aborted communicator fails every later call loudly.
void check_comm(dbsp_sp_context* ctx) {
  if (ctx->aborted) fail(kCuda, "the NCCL communicator was aborted after an error or a timeout");
  ncclResult_t r = ncclSuccess;
  nck(N().CommGetAsyncError(ctx->comm, &r), "ncclCommGetAsyncError");
  if (r != ncclSuccess && r != ncclInProgress) {
    N().CommAbort(ctx->comm);
    ctx->aborted = true;
    fail(kCuda, std::string("NCCL asynchronous error, communicator aborted: ") + N().GetErrorString(r));
  }
}

void check_call(const dbsp_mask_set* set, dbsp_strategy s, const Plan& p, uint32_t world, uint32_t tokens,
                uint32_t head_dim) {
  if (!set) fail(kContract, "null mask set");
  if (s.ulysses * s.ring != world) fail(kConfig, "strategy does not match the number of ranks");
  if (tokens % 64 || tokens / 64 != set->num_q_blocks || set->num_q_blocks != set->num_kv_blocks)
    fail(kContract, "the SP path needs tokens = 64 * blocks and a square block grid");
  if (head_dim != 64 && head_dim != 128) fail(kConfig, "head_dim must be 64 or 128");
  MaskView m = make_view(set->heads, set->num_heads, set->num_q_blocks, set->num_kv_blocks, set->block_size);
  validate_plan(m, Strategy{s.ulysses, s.ring}, p.head.data(), p.q.data(), p.kv.data());
  // Empty ring groups are allowed (a plan may leave a ring rank without KV
  // blocks): such a period exchanges nothing and launches nothing, and if it
  // is a rank's last period the accumulator is finalised by sp_finalize_kernel.
}

}  // namespace

extern "C" {

int dbsp_nccl_unique_id(uint8_t* out, uint32_t size) {
  return guard([&] {
    if (!out || size < sizeof(ncclUniqueId)) fail(kContract, "unique id buffer too small");
    ncclUniqueId id;
    nck(N().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof(id));
  });
}

int dbsp_sp_context_create(uint32_t rank, uint32_t world, const uint8_t* nccl_id, dbsp_sp_context** out) {
  return guard([&] {
    if (!out || !nccl_id) fail(kContract, "null argument");
    if (world == 0 || rank >= world) fail(kConfig, "rank must be < world");
    auto ctx = std::make_unique<dbsp_sp_context>();
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    nck(N().CommInitRank(&ctx->comm, int(world), id, int(rank)), "ncclCommInitRank");
    ctx->rank = rank;
    ctx->world = world;
    ck(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking), "comm stream");
    for (cudaEvent_t& e : ctx->ev_ready) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&ctx->ev_done, cudaEventDisableTiming), "event");
    *out = ctx.release();
  });
}

void dbsp_sp_context_destroy(dbsp_sp_context* ctx) { delete ctx; }

int dbsp_sp_attention(dbsp_sp_context* ctx, const dbsp_mask_set* set, dbsp_strategy s, const dbsp_plan* plan,
                      const void* q_home, const void* k_home, const void* v_home, void* o_home, uint32_t tokens,
                      uint32_t head_dim, void* stream_ptr) {
  return guard([&] {
    if (!ctx) fail(kContract, "null context");
    if (!q_home || !k_home || !v_home || !o_home) fail(kContract, "null home buffer");
    Nvtx r_call("dbsp.sp_attention");
    check_comm(ctx);
    const Plan p = plan_from(set, plan);
    check_call(set, s, p, ctx->world, tokens, head_dim);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_ptr);
    if (!ctx->ex) ctx->ex = std::make_unique<RankExec>();
    RankExec& E = *ctx->ex;
    // Layouts, device lists, buffers and K4 schedules are rebuilt only when the
    // plan or the masks change (a static-mask layer reuses them every step).
    const uint64_t key = call_key(set, Strategy{s.ulysses, s.ring}, p, tokens, head_dim);
    if (key != E.key) {
      Nvtx r_plan("dbsp.sp_plan");
      E.plan(set, Strategy{s.ulysses, s.ring}, p, ctx->world, ctx->rank, tokens, head_dim, st);
      E.key = key;
    }
    const uint32_t G = ctx->world, me = ctx->rank;
    if (ctx->timing && ctx->ev_k.size() < 2 * size_t(s.ring)) {
      const size_t old = ctx->ev_k.size();
      ctx->ev_k.resize(2 * size_t(s.ring));
      for (size_t i = old; i < ctx->ev_k.size(); ++i) ck(cudaEventCreate(&ctx->ev_k[i]), "timing event");
    }
    ctx->timed_periods = ctx->timing ? s.ring : 0;
    // 1. fused all-to-all(v) on the compute stream (it gates everything after it)
    std::optional<Nvtx> r_fwd;
    r_fwd.emplace("dbsp.a2av_forward");
    E.pack_forward(q_home, k_home, v_home, st);
    nck(N().GroupStart(), "group");
    for (uint32_t x = 0; x < G; ++x) {
      const size_t bq = E.piece_bytes(x, E.send_q_h[x].size()), bkv = E.piece_bytes(x, E.send_kv_h[x].size());
      uint8_t* qd = static_cast<uint8_t*>(E.q_loc.p) + E.q_off(x);
      uint8_t* kd = static_cast<uint8_t*>(E.kbuf[0].p) + E.kv_off(x);
      uint8_t* vd = static_cast<uint8_t*>(E.vbuf[0].p) + E.kv_off(x);
      const size_t rq = size_t(E.recv_q[x]) * 64 * E.row_bytes, rkv = size_t(E.recv_kv[x]) * 64 * E.row_bytes;
      if (x == me) {
        if (bq) ck(cudaMemcpyAsync(qd, E.sendq[x].p, bq, cudaMemcpyDeviceToDevice, st), "self q");
        if (bkv) {
          ck(cudaMemcpyAsync(kd, E.sendk[x].p, bkv, cudaMemcpyDeviceToDevice, st), "self k");
          ck(cudaMemcpyAsync(vd, E.sendv[x].p, bkv, cudaMemcpyDeviceToDevice, st), "self v");
        }
        continue;
      }
      if (bq) nck(N().Send(E.sendq[x].p, bq, ncclUint8, int(x), ctx->comm, st), "send q");
      if (bkv) {
        nck(N().Send(E.sendk[x].p, bkv, ncclUint8, int(x), ctx->comm, st), "send k");
        nck(N().Send(E.sendv[x].p, bkv, ncclUint8, int(x), ctx->comm, st), "send v");
      }
      if (rq) nck(N().Recv(qd, rq, ncclUint8, int(x), ctx->comm, st), "recv q");
      if (rkv) {
        nck(N().Recv(kd, rkv, ncclUint8, int(x), ctx->comm, st), "recv k");
        nck(N().Recv(vd, rkv, ncclUint8, int(x), ctx->comm, st), "recv v");
      }
    }
    nck(N().GroupEnd(), "group");
    r_fwd.reset();
    // 2. ring periods: K4 on the held group while the next one arrives on the comm stream
    const Layout& L = E.me;
    const uint32_t y = L.y;
    const uint32_t nxt = L.u * y + (L.r + 1) % y, prv = L.u * y + (L.r + y - 1) % y;
    int cur = 0;
    for (uint32_t pd = 0; pd < y; ++pd) {
      Nvtx r_period("dbsp.ring_period");
      if (pd + 1 < y) {
        const size_t n = L.groups[L.period_group(pd)].size() * 64 * E.row_bytes;
        const size_t nn = L.groups[L.period_group(pd + 1)].size() * 64 * E.row_bytes;
        ck(cudaEventRecord(ctx->ev_ready[cur], st), "event");  // the held group is in place
        ck(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_ready[cur], 0), "wait");
        nck(N().GroupStart(), "group");
        if (n && E.row_bytes) {
          nck(N().Send(E.kbuf[cur].p, n, ncclUint8, int(prv), ctx->comm, ctx->comm_stream), "ring send k");
          nck(N().Send(E.vbuf[cur].p, n, ncclUint8, int(prv), ctx->comm, ctx->comm_stream), "ring send v");
        }
        if (nn && E.row_bytes) {
          nck(N().Recv(E.kbuf[1 - cur].p, nn, ncclUint8, int(nxt), ctx->comm, ctx->comm_stream), "ring recv k");
          nck(N().Recv(E.vbuf[1 - cur].p, nn, ncclUint8, int(nxt), ctx->comm, ctx->comm_stream), "ring recv v");
        }
        nck(N().GroupEnd(), "group");
      }
      if (ctx->timing) ck(cudaEventRecord(ctx->ev_k[2 * pd], st), "timing event");
      {
        Nvtx r_k4("dbsp.k4");
        E.compute(pd, cur, st);
      }
      if (ctx->timing) ck(cudaEventRecord(ctx->ev_k[2 * pd + 1], st), "timing event");
      if (pd + 1 < y) {
        ck(cudaEventRecord(ctx->ev_done, ctx->comm_stream), "event");
        ck(cudaStreamWaitEvent(st, ctx->ev_done, 0), "wait");  // next group arrived, held one sent
      }
      cur = 1 - cur;
    }
    // 3. reverse all-to-all(v): O slices go home, then land in the home layout
    Nvtx r_rev("dbsp.a2av_reverse");
    nck(N().GroupStart(), "group");
    for (uint32_t x = 0; x < G; ++x) {
      const size_t sb = size_t(E.oslice_n[x]) * 64 * E.row_bytes;
      const size_t rb = size_t(E.back_blocks[x].n) * 64 * E.all[x].heads.size() * head_dim * 2;
      if (x == me) {
        if (sb) ck(cudaMemcpyAsync(E.recvo[x].p, E.oslice(x), sb, cudaMemcpyDeviceToDevice, st), "self o");
        continue;
      }
      if (sb) nck(N().Send(E.oslice(x), sb, ncclUint8, int(x), ctx->comm, st), "send o");
      if (rb) nck(N().Recv(E.recvo[x].p, rb, ncclUint8, int(x), ctx->comm, st), "recv o");
    }
    nck(N().GroupEnd(), "group");
    E.unpack_reverse(o_home, st);
  });
}

int dbsp_sp_set_timing(dbsp_sp_context* ctx, int32_t on) {
  return guard([&] {
    if (!ctx) fail(kContract, "null context");
    ctx->timing = on != 0;
  });
}

int dbsp_sp_period_ms(dbsp_sp_context* ctx, float* ms, uint32_t cap, uint32_t* n) {
  return guard([&] {
    if (!ctx || !n) fail(kContract, "null argument");
    *n = ctx->timed_periods;
    if (ctx->timed_periods > cap || (ctx->timed_periods && !ms)) fail(kContract, "period buffer too small");
    for (uint32_t p = 0; p < ctx->timed_periods; ++p) {
      ck(cudaEventSynchronize(ctx->ev_k[2 * p + 1]), "timing sync");
      ck(cudaEventElapsedTime(&ms[p], ctx->ev_k[2 * p], ctx->ev_k[2 * p + 1]), "elapsed");
    }
  });
}

int dbsp_sp_synchronize(dbsp_sp_context* ctx, void* stream_ptr, uint32_t timeout_ms) {
  return guard([&] {
    if (!ctx) fail(kContract, "null context");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_ptr);
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
      const cudaError_t a = cudaStreamQuery(st), b = cudaStreamQuery(ctx->comm_stream);
      if (a == cudaSuccess && b == cudaSuccess) break;
      if (a != cudaErrorNotReady && a != cudaSuccess) ck(a, "compute stream");
      if (b != cudaErrorNotReady && b != cudaSuccess) ck(b, "communication stream");
      check_comm(ctx);  // aborts the communicator on an asynchronous NCCL error
      const auto el = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0);
      if (timeout_ms && el.count() > int64_t(timeout_ms)) {
        N().CommAbort(ctx->comm);
        ctx->aborted = true;
        fail(kCuda, "sequence-parallel call did not finish within " + std::to_string(timeout_ms) +
                        " ms; NCCL communicator aborted");
      }
      std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
    check_comm(ctx);
  });
}

// All G ranks of UxRy on this GPU, with device copies as the transport: the
// same per-rank plans, packing, ring rotation and reverse exchange as
// dbsp_sp_attention.  q/k/v/o_homes: G home shards [home tokens_g, H, d].
int dbsp_sp_attention_simulated(const dbsp_mask_set* set, dbsp_strategy s, const dbsp_plan* plan,
                                const void* const* q_homes, const void* const* k_homes,
                                const void* const* v_homes, void* const* o_homes, uint32_t tokens,
                                uint32_t head_dim, void* stream_ptr) {
  return guard([&] {
    if (!q_homes || !k_homes || !v_homes || !o_homes) fail(kContract, "null home buffers");
    const uint32_t G = s.ulysses * s.ring;
    const Plan p = plan_from(set, plan);
    check_call(set, s, p, G, tokens, head_dim);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_ptr);
    std::vector<std::unique_ptr<RankExec>> R;
    for (uint32_t r = 0; r < G; ++r) {
      R.push_back(std::make_unique<RankExec>());
      R.back()->plan(set, Strategy{s.ulysses, s.ring}, p, G, r, tokens, head_dim, st);
      R.back()->pack_forward(q_homes[r], k_homes[r], v_homes[r], st);
    }
    // forward exchange: src's piece for dst lands at dst's offset for src
    for (uint32_t src = 0; src < G; ++src)
      for (uint32_t dst = 0; dst < G; ++dst) {
        RankExec& S = *R[src];
        RankExec& D = *R[dst];
        const size_t bq = S.piece_bytes(dst, S.send_q_h[dst].size()), bkv = S.piece_bytes(dst, S.send_kv_h[dst].size());
        if (bq != size_t(D.recv_q[src]) * 64 * D.row_bytes || bkv != size_t(D.recv_kv[src]) * 64 * D.row_bytes)
          fail(kInternal, "exchange sizes disagree between sender and receiver");
        if (bq)
          ck(cudaMemcpyAsync(static_cast<uint8_t*>(D.q_loc.p) + D.q_off(src), S.sendq[dst].p, bq,
                             cudaMemcpyDeviceToDevice, st), "copy q");
        if (bkv) {
          ck(cudaMemcpyAsync(static_cast<uint8_t*>(D.kbuf[0].p) + D.kv_off(src), S.sendk[dst].p, bkv,
                             cudaMemcpyDeviceToDevice, st), "copy k");
          ck(cudaMemcpyAsync(static_cast<uint8_t*>(D.vbuf[0].p) + D.kv_off(src), S.sendv[dst].p, bkv,
                             cudaMemcpyDeviceToDevice, st), "copy v");
        }
      }
    // ring periods: every rank computes, then rank r takes the group ring rank r+1 held
    const uint32_t y = s.ring;
    int cur = 0;
    for (uint32_t pd = 0; pd < y; ++pd) {
      for (uint32_t r = 0; r < G; ++r) R[r]->compute(pd, cur, st);
      if (pd + 1 < y)
        for (uint32_t r = 0; r < G; ++r) {
          RankExec& D = *R[r];
          const RankExec& N = *R[D.me.u * y + (D.me.r + 1) % y];
          const size_t nn = D.me.groups[D.me.period_group(pd + 1)].size() * 64 * D.row_bytes;
          if (nn) {
            ck(cudaMemcpyAsync(D.kbuf[1 - cur].p, N.kbuf[cur].p, nn, cudaMemcpyDeviceToDevice, st), "ring k");
            ck(cudaMemcpyAsync(D.vbuf[1 - cur].p, N.vbuf[cur].p, nn, cudaMemcpyDeviceToDevice, st), "ring v");
          }
        }
      cur = 1 - cur;
    }
    // reverse exchange
    for (uint32_t home = 0; home < G; ++home) {
      RankExec& Hm = *R[home];
      for (uint32_t src = 0; src < G; ++src) {
        const RankExec& Sr = *R[src];
        const size_t sb = size_t(Sr.oslice_n[home]) * 64 * Sr.row_bytes;
        if (sb) ck(cudaMemcpyAsync(Hm.recvo[src].p, Sr.oslice(home), sb, cudaMemcpyDeviceToDevice, st), "copy o");
      }
      Hm.unpack_reverse(o_homes[home], st);
    }
    ck(cudaStreamSynchronize(st), "simulated sp sync");  // R's buffers die here
  });
}

}  // extern "C"
