// Host side of the sm_100a attention path: TMA descriptors, schedule upload,
// launches of K4 (attn_kernel.cuh), the ring-accumulator init and K1 (exact
// mask statistics on device), all behind the C ABI of include/dbsp_b200.h.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/dbsp_b200.h"
#include <cstdlib>

#include "attn_kernel.cuh"
#include "attn_kernel_pd3.cuh"
#include "capi_util.hpp"
#include "core.hpp"
#include "schedule.hpp"

namespace dbsp_dev {

__global__ void accum_init_kernel(float* o, float* lse, size_t n_o, size_t n_lse) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_o; i += stride) o[i] = 0.f;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_lse; i += stride)
    lse[i] = -INFINITY;
}

// K1: exact per-head block counts, Q-row and KV-column marginals of the
// head-summed grid (planner.hpp:47-61, 160-167) from device mask words.
__global__ void mask_rows_kernel(const uint64_t* __restrict__ words, uint32_t heads, uint32_t nq,
                                 uint32_t wpr, unsigned long long* head_counts,
                                 unsigned long long* row_w) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= heads * nq) return;
  const uint64_t* w = words + size_t(r) * wpr;
  unsigned long long c = 0;
  for (uint32_t i = 0; i < wpr; ++i) c += __popcll(w[i]);
  if (c) {
    atomicAdd(head_counts + r / nq, c);
    atomicAdd(row_w + r % nq, c);
  }
}

__global__ void mask_cols_kernel(const uint64_t* __restrict__ words, uint32_t rows, uint32_t nk,
                                 uint32_t wpr, uint32_t rows_per_block,
                                 unsigned long long* col_w) {
  const uint32_t w = blockIdx.x;
  const uint32_t bit = threadIdx.x;  // 64 threads
  const uint32_t r0 = blockIdx.y * rows_per_block;
  const uint32_t r1 = min(rows, r0 + rows_per_block);
  unsigned long long c = 0;
  for (uint32_t r = r0; r < r1; ++r) c += (words[size_t(r) * wpr + w] >> bit) & 1ull;
  const uint32_t k = w * 64 + bit;
  if (c && k < nk) atomicAdd(col_w + k, c);
}

}  // namespace dbsp_dev

namespace {

using namespace dbsp_core;

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(kCuda, std::string(what) + ": " + cudaGetErrorString(e));
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    err = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
    if (err == cudaSuccess && q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  if (!fn) fail(kCuda, "cuTensorMapEncodeTiled unavailable: " + std::string(cudaGetErrorString(err)));
  return fn;
}

// [tokens, heads, d] bf16, box = 64 tokens x 1 head x 64 columns, 128B swizzle
// (the layout the UMMA SW128 descriptors of attn_kernel.cuh expect).
CUtensorMap make_tmap(const void* ptr, uint32_t tokens, uint32_t heads, uint32_t d,
                      uint32_t box_rows = 64) {
  CUtensorMap m;
  const cuuint64_t dims[3] = {d, heads, tokens};
  const cuuint64_t strides[2] = {cuuint64_t(d) * 2, cuuint64_t(heads) * d * 2};
  const cuuint32_t box[3] = {64, 1, box_rows};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr),
                                 dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(kCuda, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return m;
}

template <int D>
void launch_kernel(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                   const dbsp_dev::AttnParams& prm,
                   uint32_t items, cudaStream_t stream) {
  using C = dbsp_dev::KCfg<D>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(dbsp_dev::sparse_attn_fwd_kernel<D>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
  });
  cuda_check(attr_err, "cudaFuncSetAttribute");
  dbsp_core::count_launch();
  dbsp_dev::sparse_attn_fwd_kernel<D><<<items, dbsp_dev::kThreads, C::kSmemBytes, stream>>>(q, k, v, prm);
  cuda_check(cudaGetLastError(), "sparse_attn_fwd launch");
}

// The CTA-pair split-KV kernel (attn_kernel_pd3.cuh): one cluster of two CTAs
// per quad item.  No exp2 runs on the FMA pipe at d=128 (kPoly 0): 1 and 2 of
// 8 pairs measured 6.11 and 6.37 ms against 6.12 ms on Wan (tests/ab_probe.py).
#ifndef DBSP_PD3_POLY
#define DBSP_PD3_POLY 0
#endif
void launch_pd3(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                const dbsp_dev::AttnParams& prm, uint32_t items, cudaStream_t stream) {
  using C = dbsp_dev::Pd3Cfg;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(dbsp_dev::sparse_attn_fwd_pd3_kernel<DBSP_PD3_POLY>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
  });
  cuda_check(attr_err, "cudaFuncSetAttribute(pd3)");
  dbsp_core::count_launch();
  dbsp_dev::sparse_attn_fwd_pd3_kernel<DBSP_PD3_POLY><<<2 * items, dbsp_dev::kThreadsPd3, C::kSmemBytes, stream>>>(
      q, k, v, prm);
  cuda_check(cudaGetLastError(), "sparse_attn_fwd_pd3 launch");
}

unsigned long long* g_trace = nullptr;
unsigned long long* g_clock_probe = nullptr;

}  // namespace

struct dbsp_schedule {
  Schedule host;
  bool dirty = true;  // host schedule changed since the last upload
  size_t item_bytes = 0;
  void* dev = nullptr;
  size_t dev_bytes = 0;
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  cudaEvent_t uploaded = nullptr;
  bool pending = false;
  // device-built schedule (K2): items/entries live only in `dev`.
  bool on_device = false;
  bool dev_quad = false;  // the list is the CTA-pair (quad) layout
  uint32_t dev_items = 0;
  void* view_dev = nullptr;  // present bitmap, head ids, q ids, kv_local table
  size_t view_bytes = 0;
  // Host image of the view tables last copied to view_dev: an unchanged view
  // (the same layer every call) costs no copy; a changed one goes through a
  // pinned staging buffer, so the host never blocks on a pageable copy.
  std::vector<uint8_t> view_image;
  void* view_pinned = nullptr;
  size_t view_pinned_bytes = 0;
  cudaEvent_t view_copied = nullptr;
  bool view_pending = false;
  void* k2_scratch = nullptr;
  size_t k2_scratch_bytes = 0;
  // The last launch that reads `dev`: any rewrite of the list (upload, device
  // build) on another stream waits for it.
  cudaEvent_t last_use = nullptr;
  bool used = false;

  ~dbsp_schedule() {
    if (pending && uploaded) cudaEventSynchronize(uploaded);
    if (used && last_use) cudaEventSynchronize(last_use);
    if (last_use) cudaEventDestroy(last_use);
    if (dev) cudaFree(dev);
    if (pinned) cudaFreeHost(pinned);
    if (uploaded) cudaEventDestroy(uploaded);
    if (view_pending && view_copied) cudaEventSynchronize(view_copied);
    if (view_copied) cudaEventDestroy(view_copied);
    if (view_pinned) cudaFreeHost(view_pinned);
    if (view_dev) cudaFree(view_dev);
    if (k2_scratch) cudaFree(k2_scratch);
  }
};

namespace dbsp_k2 {
void build(const uint64_t* d_words, uint32_t nq_global, uint32_t nk_global,
           const dbsp_core::LocalView& v, uint32_t flags, const uint32_t* d_head_ids,
           const uint32_t* d_q_ids, const uint64_t* d_present, const int32_t* d_kv_local,
           dbsp_core::WorkItem* items_out, uint32_t* entries_out, void*& scratch, size_t& scratch_bytes,
           cudaStream_t stream);
}

using dbsp_capi::guard;

namespace {

// Copies items + entries to the device through a pinned staging buffer, on
// `stream`, only when the host schedule changed since the last upload.
// Orders a rewrite of sched->dev on `stream` after the last launch that read
// it (a caller may alternate streams between calls).
void wait_last_use(dbsp_schedule* sched, cudaStream_t stream) {
  if (sched->used) cuda_check(cudaStreamWaitEvent(stream, sched->last_use, 0), "wait last use");
}

void mark_use(dbsp_schedule* sched, cudaStream_t stream) {
  if (!sched->last_use)
    cuda_check(cudaEventCreateWithFlags(&sched->last_use, cudaEventDisableTiming), "event");
  cuda_check(cudaEventRecord(sched->last_use, stream), "event record");
  sched->used = true;
}

void upload_schedule(dbsp_schedule* sched, cudaStream_t stream) {
  if (!sched->dirty) return;
  wait_last_use(sched, stream);
  const Schedule& h = sched->host;
  const size_t item_bytes = h.items.size() * sizeof(WorkItem);
  const size_t bytes = item_bytes + h.entries.size() * sizeof(uint32_t);
  if (!sched->uploaded)
    cuda_check(cudaEventCreateWithFlags(&sched->uploaded, cudaEventDisableTiming), "event");
  if (sched->pending) {
    cuda_check(cudaEventSynchronize(sched->uploaded), "schedule upload sync");
    sched->pending = false;
  }
  if (sched->pinned_bytes < bytes) {
    if (sched->pinned) cudaFreeHost(sched->pinned);
    sched->pinned = nullptr;
    cuda_check(cudaMallocHost(&sched->pinned, bytes), "cudaMallocHost");
    sched->pinned_bytes = bytes;
  }
  if (sched->dev_bytes < bytes) {
    if (sched->dev) cudaFree(sched->dev);
    sched->dev = nullptr;
    cuda_check(cudaMalloc(&sched->dev, bytes), "cudaMalloc schedule");
    sched->dev_bytes = bytes;
  }
  std::memcpy(sched->pinned, h.items.data(), item_bytes);
  if (!h.entries.empty())
    std::memcpy(static_cast<uint8_t*>(sched->pinned) + item_bytes, h.entries.data(),
                h.entries.size() * sizeof(uint32_t));
  cuda_check(cudaMemcpyAsync(sched->dev, sched->pinned, bytes, cudaMemcpyHostToDevice, stream),
             "schedule upload");
  cuda_check(cudaEventRecord(sched->uploaded, stream), "event record");
  sched->pending = true;
  sched->item_bytes = item_bytes;
  sched->dirty = false;
}

}  // namespace

extern "C" {

int dbsp_schedule_create(dbsp_schedule** out) {
  return guard([&] {
    if (!out) fail(kContract, "null output");
    *out = new dbsp_schedule();
  });
}

void dbsp_schedule_destroy(dbsp_schedule* s) { delete s; }

int dbsp_schedule_build(dbsp_schedule* sched, const dbsp_mask_set* set,
                        const dbsp_local_view* view, int32_t flags) {
  return guard([&] {
    if (!sched || !set) fail(kContract, "null schedule or mask set");
    const MaskView m =
        make_view(set->heads, set->num_heads, set->num_q_blocks, set->num_kv_blocks, set->block_size);
    LocalView lv;
    if (view) {
      lv.heads = view->num_heads;
      lv.head_ids = view->head_ids;
      lv.q_blocks = view->num_q_blocks;
      lv.q_ids = view->q_block_ids;
      lv.kv_blocks = view->num_kv_blocks;
      lv.kv_ids = view->kv_block_ids;
      lv.kv_tokens_global = view->kv_tokens_global;
    } else {
      lv.heads = m.H;
      lv.q_blocks = m.nq;
      lv.kv_blocks = m.nk;
    }
    build_schedule(m, lv, uint32_t(flags), sched->host);
    sched->dirty = true;
    sched->on_device = false;
  });
}

int dbsp_schedule_build_device(dbsp_schedule* sched, const uint64_t* d_words, uint32_t heads,
                               uint32_t q_blocks, uint32_t kv_blocks, const dbsp_local_view* view,
                               int32_t flags_in, void* stream_ptr) {
  return guard([&] {
    if (!sched || !d_words) fail(kContract, "null schedule or mask words");
    if (heads == 0 || q_blocks == 0 || kv_blocks == 0) fail(kConfig, "mask dimensions must be positive");
    const uint32_t flags = normalize_sched_flags(uint32_t(flags_in));
    cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_ptr);
    LocalView lv;
    lv.heads = view ? view->num_heads : heads;
    lv.q_blocks = view ? view->num_q_blocks : q_blocks;
    lv.kv_blocks = view ? view->num_kv_blocks : kv_blocks;
    lv.kv_tokens_global = view ? view->kv_tokens_global : 0;
    if (lv.heads == 0 || lv.q_blocks == 0 || lv.kv_blocks == 0)
      fail(kConfig, "local view dimensions must be positive");
    if (lv.kv_blocks > kEntryKvMask) fail(kConfig, "too many local KV blocks");
    const uint32_t wpr = (kv_blocks + 63) / 64;
    // Host-side view tables (small), uploaded with the build.
    std::vector<uint32_t> hid(lv.heads), qid(lv.q_blocks);
    std::vector<uint64_t> present(wpr, 0);
    std::vector<int32_t> kvl(kv_blocks, -1);
    for (uint32_t i = 0; i < lv.heads; ++i) {
      hid[i] = view && view->head_ids ? view->head_ids[i] : i;
      if (hid[i] >= heads) fail(kContract, "local head maps past the mask set");
    }
    for (uint32_t i = 0; i < lv.q_blocks; ++i) {
      qid[i] = view && view->q_block_ids ? view->q_block_ids[i] : i;
      if (qid[i] >= q_blocks) fail(kContract, "local Q block maps past the mask grid");
    }
    for (uint32_t i = 0; i < lv.kv_blocks; ++i) {
      const uint32_t k = view && view->kv_block_ids ? view->kv_block_ids[i] : i;
      if (k >= kv_blocks) fail(kContract, "local KV block maps past the mask grid");
      if (kvl[k] >= 0) fail(kContract, "KV block listed twice in the local view");
      kvl[k] = int32_t(i);
      present[k / 64] |= 1ull << (k % 64);
    }
    // The previous launch from this schedule may still read the list and the
    // view tables (it may have run on another stream).
    wait_last_use(sched, stream);
    if (sched->pending) {
      cuda_check(cudaEventSynchronize(sched->uploaded), "schedule upload sync");
      sched->pending = false;
    }
    // view_dev: present | hid | qid | kvl
    const size_t off_hid = present.size() * 8;
    const size_t off_qid = off_hid + hid.size() * 4, off_kvl = off_qid + qid.size() * 4;
    const size_t vb = off_kvl + kvl.size() * 4;
    std::vector<uint8_t> image(vb, 0);
    std::memcpy(image.data(), present.data(), present.size() * 8);
    std::memcpy(image.data() + off_hid, hid.data(), hid.size() * 4);
    std::memcpy(image.data() + off_qid, qid.data(), qid.size() * 4);
    std::memcpy(image.data() + off_kvl, kvl.data(), kvl.size() * 4);
    if (sched->view_bytes < vb) {
      if (sched->view_dev) cudaFree(sched->view_dev);
      sched->view_dev = nullptr;
      cuda_check(cudaMalloc(&sched->view_dev, vb + 64), "cudaMalloc view");
      sched->view_bytes = vb + 64;
      sched->view_image.clear();
    }
    if (image != sched->view_image) {
      if (!sched->view_copied)
        cuda_check(cudaEventCreateWithFlags(&sched->view_copied, cudaEventDisableTiming), "event");
      if (sched->view_pending) cuda_check(cudaEventSynchronize(sched->view_copied), "view staging sync");
      if (sched->view_pinned_bytes < vb) {
        if (sched->view_pinned) cudaFreeHost(sched->view_pinned);
        sched->view_pinned = nullptr;
        cuda_check(cudaMallocHost(&sched->view_pinned, vb), "cudaMallocHost view");
        sched->view_pinned_bytes = vb;
      }
      std::memcpy(sched->view_pinned, image.data(), vb);
      cuda_check(cudaMemcpyAsync(sched->view_dev, sched->view_pinned, vb, cudaMemcpyHostToDevice, stream), "view");
      cuda_check(cudaEventRecord(sched->view_copied, stream), "event record");
      sched->view_pending = true;
      sched->view_image = std::move(image);
    }
    uint8_t* vd = static_cast<uint8_t*>(sched->view_dev);
    uint64_t* d_present = reinterpret_cast<uint64_t*>(vd);  // 8-byte aligned first
    uint32_t* d_hid = reinterpret_cast<uint32_t*>(vd + off_hid);
    uint32_t* d_qid = reinterpret_cast<uint32_t*>(vd + off_qid);
    int32_t* d_kvl = reinterpret_cast<int32_t*>(vd + off_kvl);

    // DBSP_SCHED_AUTO_D128 builds the pair layout (normalize_sched_flags).
    const bool quad = (flags & kSchedQuad) != 0;
    const uint32_t step = quad ? 4 : (flags & kSchedPairQ) ? 2 : 1;
    const uint32_t n_items = lv.heads * ((lv.q_blocks + step - 1) / step);
    const size_t item_bytes = size_t(n_items) * sizeof(WorkItem);
    const size_t bytes = item_bytes + size_t(n_items) * lv.kv_blocks * sizeof(uint32_t);
    if (sched->dev_bytes < bytes) {
      if (sched->dev) cudaFree(sched->dev);
      sched->dev = nullptr;
      cuda_check(cudaMalloc(&sched->dev, bytes), "cudaMalloc schedule");
      sched->dev_bytes = bytes;
    }
    uint8_t* base = static_cast<uint8_t*>(sched->dev);
    dbsp_k2::build(d_words, q_blocks, kv_blocks, lv, flags, d_hid, d_qid, d_present, d_kvl,
                   reinterpret_cast<WorkItem*>(base), reinterpret_cast<uint32_t*>(base + item_bytes),
                   sched->k2_scratch, sched->k2_scratch_bytes, stream);
    // Bounds for the launch-time checks; the host copy of the list is empty.
    sched->host.items.clear();
    sched->host.entries.clear();
    sched->host.tile_visits = sched->host.dense_tiles = 0;
    sched->host.flags = flags;
    sched->host.max_head = lv.heads - 1;
    sched->host.max_q_block = lv.q_blocks - 1;
    sched->host.max_kv_block = lv.kv_blocks - 1;
    sched->on_device = true;
    sched->dirty = false;
    sched->dev_quad = quad;
    sched->dev_items = n_items;
    sched->item_bytes = item_bytes;
  });
}

namespace {
// Device-built list read back to host; diagnostics only.
void download_device(const dbsp_schedule* s, std::vector<WorkItem>& items, std::vector<uint32_t>& entries,
                     bool& quad) {
  quad = s->dev_quad;
  cuda_check(cudaDeviceSynchronize(), "sync");
  const uint8_t* base = static_cast<const uint8_t*>(s->dev);
  const uint32_t n_items = s->dev_items;
  const size_t ib = s->item_bytes;
  items.resize(n_items);
  if (n_items) cuda_check(cudaMemcpy(items.data(), base, ib, cudaMemcpyDeviceToHost), "d2h");
  uint64_t n = 0;
  for (const WorkItem& w : items) n += w.count;
  entries.resize(n);
  if (n) cuda_check(cudaMemcpy(entries.data(), base + ib, n * 4, cudaMemcpyDeviceToHost), "d2h");
}
}  // namespace

int dbsp_schedule_stats(const dbsp_schedule* s, uint64_t* items, uint64_t* visits,
                        uint64_t* dense) {
  return guard([&] {
    if (!s) fail(kContract, "null schedule");
    if (!s->on_device) {
      if (items) *items = s->host.items.size();
      if (visits) *visits = s->host.tile_visits;
      if (dense) *dense = s->host.dense_tiles;
      return;
    }
    std::vector<WorkItem> it;
    std::vector<uint32_t> e;
    bool quad = false;
    download_device(s, it, e, quad);
    const uint32_t dmask = quad ? (0xFu << 22) : (kEntryDenseA | kEntryDenseB);
    uint64_t dn = 0;
    for (uint32_t x : e) dn += __builtin_popcount(x & dmask);
    if (items) *items = it.size();
    if (visits) *visits = e.size();
    if (dense) *dense = dn;
  });
}

int dbsp_schedule_layout(const dbsp_schedule* s, uint32_t* flags) {
  return guard([&] {
    if (!s || !flags) fail(kContract, "null argument");
    if (!s->on_device) {
      *flags = s->host.flags;
      return;
    }
    *flags = s->host.flags;
  });
}

int dbsp_schedule_download(const dbsp_schedule* s, void* items_out, uint32_t* entries_out,
                           uint64_t max_entries) {
  return guard([&] {
    if (!s || !items_out) fail(kContract, "null argument");
    if (!s->on_device) {
      std::memcpy(items_out, s->host.items.data(), s->host.items.size() * sizeof(WorkItem));
      if (s->host.entries.size() > max_entries) fail(kContract, "entries buffer too small");
      if (entries_out) std::memcpy(entries_out, s->host.entries.data(), s->host.entries.size() * 4);
      return;
    }
    std::vector<WorkItem> it;
    std::vector<uint32_t> e;
    bool quad = false;
    download_device(s, it, e, quad);
    std::memcpy(items_out, it.data(), it.size() * sizeof(WorkItem));
    if (e.size() > max_entries) fail(kContract, "entries buffer too small");
    if (entries_out && !e.empty()) std::memcpy(entries_out, e.data(), e.size() * 4);
  });
}

int dbsp_schedule_upload(dbsp_schedule* sched, void* stream) {
  return guard([&] {
    if (!sched) fail(kContract, "null schedule");
    upload_schedule(sched, reinterpret_cast<cudaStream_t>(stream));
  });
}

int dbsp_schedule_upload_bytes(const dbsp_schedule* s, uint64_t* bytes) {
  return guard([&] {
    if (!s || !bytes) fail(kContract, "null argument");
    *bytes = s->host.items.size() * sizeof(WorkItem) + s->host.entries.size() * sizeof(uint32_t);
  });
}

namespace {
void attention_launch(dbsp_schedule* sched, const dbsp_attn_args* a, const dbsp_out_scatter* sc,
                      void* stream_ptr) {
  {
    if (!sched || !a) fail(kContract, "null schedule or args");
    if (a->head_dim != 64 && a->head_dim != 128) fail(kConfig, "head_dim must be 64 or 128");
    if (!a->q || !a->k || !a->v) fail(kContract, "null q/k/v");
    if (a->q_tokens == 0 || a->kv_tokens == 0 || a->heads == 0)
      fail(kConfig, "attention dimensions must be positive");
    if (reinterpret_cast<uintptr_t>(a->q) % 16) fail(kContract, "q must be 16-byte aligned");
    const bool acc = a->accumulate != 0;
    if (acc && (!a->o_accum || !a->lse_accum)) fail(kContract, "accumulate needs o_accum/lse_accum");
    if ((!acc || a->finalize) && !a->o && !sc) fail(kContract, "null output");
    if (sc && (!sc->out_peers || !sc->q_block_map || !sc->head_map || sc->out_heads == 0))
      fail(kContract, "incomplete output scatter");
    cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_ptr);
    const Schedule& h = sched->host;
    const uint32_t n_items = sched->on_device ? sched->dev_items : uint32_t(h.items.size());
    if (n_items == 0) return;
    const uint32_t q_blocks = (a->q_tokens + 63) / 64, kv_blocks = (a->kv_tokens + 63) / 64;
    if (h.max_head >= a->heads || h.max_q_block >= q_blocks)
      fail(kContract, "schedule addresses past the Q buffer");
    if ((sched->on_device || !h.entries.empty()) && h.max_kv_block >= kv_blocks)
      fail(kContract, "schedule addresses past the K/V buffers");
    if (!sched->on_device) upload_schedule(sched, stream);

    dbsp_dev::AttnParams prm;
    prm.items = static_cast<const WorkItem*>(sched->dev);
    prm.entries =
        reinterpret_cast<const uint32_t*>(static_cast<uint8_t*>(sched->dev) + sched->item_bytes);
    prm.q = static_cast<const __nv_bfloat16*>(a->q);
    prm.out = static_cast<__nv_bfloat16*>(a->o);
    prm.lse = a->lse;
    prm.o_acc = a->o_accum;
    prm.lse_acc = a->lse_accum;
    prm.q_tokens = a->q_tokens;
    prm.heads = a->heads;
    prm.mode = (acc ? dbsp_dev::kModeAccumulate : 0u) | (a->finalize ? dbsp_dev::kModeFinalize : 0u);
    const float scale = a->softmax_scale > 0.f ? a->softmax_scale : 1.0f / std::sqrt(float(a->head_dim));
    prm.scale_log2 = scale * 1.4426950408889634f;
    prm.trace = g_trace;
    prm.clock_probe = g_clock_probe;
    prm.out_peers = sc ? reinterpret_cast<__nv_bfloat16* const*>(sc->out_peers) : nullptr;
    prm.scatter_rows = sc ? sc->q_block_map : nullptr;
    prm.scatter_heads = sc ? sc->head_map : nullptr;
    prm.out_heads = sc ? sc->out_heads : 0;
    const CUtensorMap tq = make_tmap(a->q, a->q_tokens, a->heads, a->head_dim);
    const CUtensorMap tk = make_tmap(a->k, a->kv_tokens, a->heads, a->head_dim);
    const CUtensorMap tv = make_tmap(a->v, a->kv_tokens, a->heads, a->head_dim);
    if (h.flags & kSchedQuad) {
      if (a->head_dim != 128) fail(kConfig, "the CTA-pair kernel (quad schedules) needs head_dim 128");
      launch_pd3(tq, tk, tv, prm, n_items, stream);
    } else if (a->head_dim == 128) {
      launch_kernel<128>(tq, tk, tv, prm, n_items, stream);
    } else {
      launch_kernel<64>(tq, tk, tv, prm, n_items, stream);
    }
    mark_use(sched, stream);
  }
}
}  // namespace

int dbsp_attention_launch(dbsp_schedule* sched, const dbsp_attn_args* a, void* stream) {
  return guard([&] { attention_launch(sched, a, nullptr, stream); });
}

int dbsp_attention_launch_scatter(dbsp_schedule* sched, const dbsp_attn_args* a,
                                  const dbsp_out_scatter* sc, void* stream) {
  return guard([&] {
    if (!sc) fail(kContract, "null output scatter");
    attention_launch(sched, a, sc, stream);
  });
}

int dbsp_sparse_attention(const dbsp_mask_set* set, const dbsp_attn_args* args, void* stream) {
  // One schedule and one device copy of the mask words per thread, reused by
  // every call.  The words go to the device (1.3 MB for the Wan layer) and K2
  // builds the list there, so a call with fresh masks costs no host pass over
  // the masks.
  struct OneShot {
    dbsp_schedule* sched = nullptr;
    uint64_t* words = nullptr;
    size_t cap = 0;
    ~OneShot() {
      if (sched) dbsp_schedule_destroy(sched);  // waits for the last launch
      if (words) cudaFree(words);
    }
  };
  static thread_local OneShot os;
  dbsp_local_view v;
  int32_t flags = 0;
  int rc = guard([&] {
    if (!set || !args) fail(kContract, "null mask set or args");
    if (!set->heads) fail(kContract, "null mask rows");
    if (set->num_heads == 0 || set->num_q_blocks == 0 || set->num_kv_blocks == 0)
      fail(kConfig, "mask dimensions must be positive");
    if (!os.sched) os.sched = new dbsp_schedule();
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const size_t wpr = (set->num_kv_blocks + 63) / 64;
    const size_t per_head = size_t(set->num_q_blocks) * wpr;
    const size_t bytes = per_head * set->num_heads * sizeof(uint64_t);
    wait_last_use(os.sched, st);  // the previous call's K2 read the words
    if (os.cap < bytes) {
      if (os.words) cudaFree(os.words);
      os.words = nullptr;
      cuda_check(cudaMalloc(&os.words, bytes), "cudaMalloc mask words");
      os.cap = bytes;
    }
    for (uint32_t h = 0; h < set->num_heads; ++h) {
      if (!set->heads[h]) fail(kContract, "null mask rows");
      cuda_check(cudaMemcpyAsync(os.words + h * per_head, set->heads[h], per_head * sizeof(uint64_t),
                                 cudaMemcpyHostToDevice, st), "mask words H2D");
    }
    std::memset(&v, 0, sizeof(v));
    v.num_heads = set->num_heads;
    v.num_q_blocks = set->num_q_blocks;
    v.num_kv_blocks = set->num_kv_blocks;
    v.kv_tokens_global = args->kv_tokens;
    flags = args->head_dim == 128 ? (DBSP_SCHED_PAIR_Q | DBSP_SCHED_AUTO_D128) : DBSP_SCHED_PAIR_Q;
  });
  if (rc) return rc;
  rc = dbsp_schedule_build_device(os.sched, os.words, set->num_heads, set->num_q_blocks, set->num_kv_blocks,
                                  &v, flags, stream);
  if (rc) return rc;
  return dbsp_attention_launch(os.sched, args, stream);
}

uint64_t dbsp_launch_count(void) { return dbsp_core::g_launches.load(std::memory_order_relaxed); }

// Debug hook (not in the public header): device buffer of 16 blocks x 256
// tiles x 8 events u64 clock64 stamps, used by DBSP_TRACE builds.
int dbsp_debug_set_trace(unsigned long long* dev) {
  g_trace = dev;
  return 0;
}

// Debug hook (not in the public header): 4 x u64 device buffer that CTA 0 of
// the default kernel fills with {clock64, globaltimer} at start and end.
int dbsp_debug_set_clock_probe(unsigned long long* dev) {
  g_clock_probe = dev;
  return 0;
}

int dbsp_copy_2d(void* dst, uint64_t dst_pitch, const void* src, uint64_t src_pitch,
                 uint64_t width, uint64_t rows, int32_t to_device, void* stream) {
  return guard([&] {
    if (!dst || !src) fail(kContract, "null pointer");
    cuda_check(cudaMemcpy2DAsync(dst, dst_pitch, src, src_pitch, width, rows,
                                 to_device ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost,
                                 reinterpret_cast<cudaStream_t>(stream)),
               "cudaMemcpy2DAsync");
  });
}

int dbsp_accum_init(float* o_accum, float* lse_accum, uint32_t q_tokens, uint32_t heads,
                    uint32_t head_dim, void* stream) {
  return guard([&] {
    if (!o_accum || !lse_accum) fail(kContract, "null accumulators");
    const size_t n_o = size_t(q_tokens) * heads * head_dim, n_l = size_t(q_tokens) * heads;
    dbsp_core::count_launch();
    dbsp_dev::accum_init_kernel<<<592, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        o_accum, lse_accum, n_o, n_l);
    cuda_check(cudaGetLastError(), "accum_init launch");
  });
}

int dbsp_mask_stats_device(const uint64_t* d_words, uint32_t heads, uint32_t nq, uint32_t nk,
                           uint64_t* d_head_counts, uint64_t* d_row_weights,
                           uint64_t* d_col_weights, void* stream_ptr) {
  return guard([&] {
    if (!d_words || !d_head_counts || !d_row_weights || !d_col_weights)
      fail(kContract, "null device pointer");
    if (heads == 0 || nq == 0 || nk == 0) fail(kConfig, "mask dimensions must be positive");
    cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_ptr);
    const uint32_t wpr = (nk + 63) / 64;
    cuda_check(cudaMemsetAsync(d_head_counts, 0, sizeof(uint64_t) * heads, stream), "memset");
    cuda_check(cudaMemsetAsync(d_row_weights, 0, sizeof(uint64_t) * nq, stream), "memset");
    cuda_check(cudaMemsetAsync(d_col_weights, 0, sizeof(uint64_t) * nk, stream), "memset");
    const uint32_t rows = heads * nq;
    dbsp_core::count_launch();
    dbsp_dev::mask_rows_kernel<<<(rows + 255) / 256, 256, 0, stream>>>(
        d_words, heads, nq, wpr, reinterpret_cast<unsigned long long*>(d_head_counts),
        reinterpret_cast<unsigned long long*>(d_row_weights));
    cuda_check(cudaGetLastError(), "mask_rows launch");
    const uint32_t rpb = 256;
    dim3 grid(wpr, (rows + rpb - 1) / rpb);
    dbsp_core::count_launch();
    dbsp_dev::mask_cols_kernel<<<grid, 64, 0, stream>>>(
        d_words, rows, nk, wpr, rpb, reinterpret_cast<unsigned long long*>(d_col_weights));
    cuda_check(cudaGetLastError(), "mask_cols launch");
  });
}

}  // extern "C"
