// K2 on the device: the attention work schedule built from device mask words
// (SURVEY.md §2.2 K2), so a call with live (e.g. SpargeAttn-style) masks
// needs no host pass over the masks and no schedule upload.  Produces exactly
// the items/entries of the host builder (schedule.cpp) -- same pairing, same
// entry encoding, same LPT order (ties by item index) -- which the tests
// check entry for entry.
//
//   k2_count  one thread per item: popcount of (row_a | row_b) & local-KV set
//   CUB radix sort of (head | ~count | index) keys -> LPT order
//   CUB exclusive scan of the sorted counts -> entry offsets
//   k2_write  one warp per item: WorkItem + entries (ballot-compacted bit walk)
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include "../../include/dbsp_b200.h"
#include "capi_util.hpp"
#include "core.hpp"
#include "schedule.hpp"

namespace dbsp_dev {

using dbsp_core::WorkItem;

struct K2Args {
  const uint64_t* words;      // [H_global][nq_global][wpr]
  uint32_t nq_global, wpr;
  const uint32_t* head_ids;   // local head -> global head
  const uint32_t* q_ids;      // local Q block -> global Q block
  uint32_t nq_local;
  const uint64_t* present;    // [wpr] local KV set as a global-block bitmap
  const int32_t* kv_local;    // [nk_global] global KV block -> local index or -1
  uint32_t kv_tokens_global;  // 0 = all blocks full
  uint32_t items_per_head;
  uint32_t step;              // 1, 2 (paired Q blocks) or 4 (quad items of the CTA-pair kernel)
  uint32_t head_group;        // heads per ordering group; 0 = global LPT (schedule.hpp)
};

// The Q rows of item i (schedule.cpp): local head, up to four local Q blocks
// (padded rows repeat the first block and set bit r of `pad`).
struct ItemRows {
  uint32_t hl, q[4], pad, n;
  const uint64_t* row[4];
};

__device__ __forceinline__ ItemRows item_rows(const K2Args& a, uint32_t i) {
  ItemRows r;
  r.hl = i / a.items_per_head;
  const uint32_t q0 = (i % a.items_per_head) * a.step;
  const uint32_t h = a.head_ids[r.hl];
  r.pad = 0;
  r.n = a.step;
#pragma unroll
  for (uint32_t j = 0; j < 4; ++j) {
    const bool in = j < a.step && q0 + j < a.nq_local;
    r.q[j] = in ? q0 + j : q0;
    r.row[j] = in ? a.words + (size_t(h) * a.nq_global + a.q_ids[q0 + j]) * a.wpr : nullptr;
    if (!in && j < a.step) r.pad |= 1u << j;
  }
  return r;
}

__device__ __forceinline__ uint64_t row_word(const ItemRows& r, uint32_t j, uint32_t w) {
  return r.row[j] ? r.row[j][w] : 0ull;
}

__global__ void k2_count(K2Args a, uint32_t n_items, uint32_t* counts, unsigned long long* keys) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_items) return;
  const ItemRows r = item_rows(a, i);
  uint32_t c = 0;
  for (uint32_t w = 0; w < a.wpr; ++w) {
    const uint64_t p = a.present[w];
    uint64_t uni = 0;
#pragma unroll
    for (uint32_t j = 0; j < 4; ++j) uni |= row_word(r, j, w) & p;
    c += __popcll(uni);
  }
  counts[i] = c;
  const unsigned long long head_key = a.head_group ? (unsigned long long)(r.hl / a.head_group) : 0ull;
  if (keys) keys[i] = (head_key << 44) | ((unsigned long long)(0xFFFFFu - min(c, 0xFFFFFu)) << 24) | i;
}

__global__ void k2_sorted_counts(const unsigned long long* sorted_keys, const uint32_t* counts,
                                 uint32_t n_items, uint32_t* sorted_counts) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n_items) sorted_counts[j] = counts[uint32_t(sorted_keys[j] & 0xFFFFFFull)];
}

__global__ void k2_write(K2Args a, uint32_t n_items, const unsigned long long* sorted_keys,
                         const uint32_t* sorted_counts, const uint32_t* begins, WorkItem* items,
                         uint32_t* entries) {
  const uint32_t j = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const uint32_t lane = threadIdx.x & 31;
  if (j >= n_items) return;
  const uint32_t i = uint32_t(sorted_keys[j] & 0xFFFFFFull);
  const ItemRows r = item_rows(a, i);
  const bool quad = a.step == 4;
  const uint32_t begin = begins[j];
  if (lane == 0) {
    if (quad)
      items[j] = WorkItem{r.hl, r.q[0], r.q[1], begin, sorted_counts[j], r.pad, r.q[2], r.q[3]};
    else
      items[j] = WorkItem{r.hl, r.q[0], a.step == 2 ? r.q[1] : r.q[0], begin, sorted_counts[j],
                          (a.step == 1 || r.pad) ? 1u : 0u, 0, 0};
  }
  const uint32_t valid_shift = quad ? dbsp_core::kQuadValidShift : dbsp_core::kEntryValidShift;
  uint32_t out = begin;
  for (uint32_t w = 0; w < a.wpr; ++w) {
    uint64_t rw[4];
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q) rw[q] = row_word(r, q, w);
    const uint64_t uni = (rw[0] | rw[1] | rw[2] | rw[3]) & a.present[w];
    // lanes take bits lane and lane+32 of the word, in ascending k order
    for (uint32_t half = 0; half < 2; ++half) {
      const uint32_t bit = half * 32 + lane;
      const bool on = (uni >> bit) & 1ull;
      const uint32_t mask = __ballot_sync(0xffffffffu, on);
      if (on) {
        const uint32_t k = w * 64 + bit;
        uint32_t valid = 64;
        if (a.kv_tokens_global) {
          const uint64_t start = uint64_t(k) * 64;
          const uint64_t rest = a.kv_tokens_global - start;
          valid = start >= a.kv_tokens_global ? 1u : uint32_t(rest < 64 ? rest : 64);
        }
        uint32_t e = uint32_t(a.kv_local[k]) | ((valid - 1) << valid_shift);
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q)
          if ((rw[q] >> bit) & 1ull) e |= 1u << (22 + q);  // pair: bits 22/23 = kEntryDenseA/B
        entries[out + __popc(mask & ((1u << lane) - 1u))] = e;
      }
      out += __popc(mask);
    }
  }
}

// Small lists (n <= kFusedItems, the common case: one rank's view, or a
// whole layer of <= 16K items): after k2_count (all SMs), the LPT sort, the
// scan and the item records run in ONE CTA.  Key = (head << 22) | (0x3FFFFF - count), sorted stably by a block
// radix sort over the blocked arrangement (item i in thread i / kK2Items), so
// ties keep ascending item order exactly as the host's stable_sort does.
constexpr int kK2Threads = 1024, kK2Items = 16, kFusedItems = kK2Threads * kK2Items;
using K2Sort = cub::BlockRadixSort<uint32_t, kK2Threads, kK2Items, uint32_t>;
using K2Scan = cub::BlockScan<uint32_t, kK2Threads>;
using K2Red = cub::BlockReduce<unsigned long long, kK2Threads>;
union K2Smem {
  typename K2Sort::TempStorage sort;
  typename K2Scan::TempStorage scan;
  typename K2Red::TempStorage red;
};

__global__ void __launch_bounds__(kK2Threads, 1)
    k2_plan_fused(K2Args a, uint32_t n_items, uint32_t key_bits, const uint32_t* __restrict__ counts,
                  WorkItem* items, uint32_t* sorted_idx, uint32_t* begins) {
  extern __shared__ __align__(16) uint8_t k2_smem[];
  K2Smem& sm = *reinterpret_cast<K2Smem*>(k2_smem);
  uint32_t keys[kK2Items], idx[kK2Items];
#pragma unroll
  for (int s = 0; s < kK2Items; ++s) {
    const uint32_t i = threadIdx.x * kK2Items + s;
    idx[s] = i;
    keys[s] = 0xFFFFFFFFu;  // padding sorts last
    if (i < n_items) {
      const uint32_t hl = i / a.items_per_head;
      keys[s] = ((a.head_group ? hl / a.head_group : 0u) << 22) | (0x3FFFFFu - counts[i]);  // counts < 2^22
    }
  }
  K2Sort(sm.sort).Sort(keys, idx, 0, int(key_bits));
  __syncthreads();
  uint32_t cnt[kK2Items], sum = 0;
#pragma unroll
  for (int s = 0; s < kK2Items; ++s) {
    cnt[s] = keys[s] == 0xFFFFFFFFu ? 0u : 0x3FFFFFu - (keys[s] & 0x3FFFFFu);
    sum += cnt[s];
  }
  uint32_t base = 0;
  K2Scan(sm.scan).ExclusiveSum(sum, base);
  const bool quad = a.step == 4;
#pragma unroll
  for (int s = 0; s < kK2Items; ++s) {
    const uint32_t j = threadIdx.x * kK2Items + s;
    if (j < n_items) {
      const ItemRows r = item_rows(a, idx[s]);
      items[j] = quad ? WorkItem{r.hl, r.q[0], r.q[1], base, cnt[s], r.pad, r.q[2], r.q[3]}
                      : WorkItem{r.hl, r.q[0], a.step == 2 ? r.q[1] : r.q[0], base, cnt[s],
                                 (a.step == 1 || r.pad) ? 1u : 0u, 0, 0};
      sorted_idx[j] = idx[s];
      begins[j] = base;
    }
    base += cnt[s];
  }
}

// Entries of a fused-planned list: one warp per sorted item.
__global__ void k2_write_fused(K2Args a, uint32_t n_items, const uint32_t* sorted_idx, const uint32_t* begins,
                               uint32_t* entries) {
  const uint32_t j = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const uint32_t lane = threadIdx.x & 31;
  if (j >= n_items) return;
  const ItemRows r = item_rows(a, sorted_idx[j]);
  const uint32_t valid_shift = a.step == 4 ? dbsp_core::kQuadValidShift : dbsp_core::kEntryValidShift;
  uint32_t out = begins[j];
  for (uint32_t w = 0; w < a.wpr; ++w) {
    uint64_t rw[4];
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q) rw[q] = row_word(r, q, w);
    const uint64_t uni = (rw[0] | rw[1] | rw[2] | rw[3]) & a.present[w];
    if (!uni) continue;
    for (uint32_t half = 0; half < 2; ++half) {
      const uint32_t bit = half * 32 + lane;
      const bool on = (uni >> bit) & 1ull;
      const uint32_t mask = __ballot_sync(0xffffffffu, on);
      if (on) {
        const uint32_t k = w * 64 + bit;
        uint32_t valid = 64;
        if (a.kv_tokens_global) {
          const uint64_t start = uint64_t(k) * 64;
          const uint64_t rest = a.kv_tokens_global - start;
          valid = start >= a.kv_tokens_global ? 1u : uint32_t(rest < 64 ? rest : 64);
        }
        uint32_t e = uint32_t(a.kv_local[k]) | ((valid - 1) << valid_shift);
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q)
          if ((rw[q] >> bit) & 1ull) e |= 1u << (22 + q);
        entries[out + __popc(mask & ((1u << lane) - 1u))] = e;
      }
      out += __popc(mask);
    }
  }
}

}  // namespace dbsp_dev

namespace {

using namespace dbsp_core;

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(kCuda, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

namespace dbsp_k2 {

// Builds one layout into `items_out` / `entries_out` (device, caller-sized:
// n_items and n_items * nk_local entries).  Stream-ordered.
void build(const uint64_t* d_words, uint32_t nq_global, uint32_t nk_global, const LocalView& v,
           uint32_t flags, const uint32_t* d_head_ids, const uint32_t* d_q_ids,
           const uint64_t* d_present, const int32_t* d_kv_local, dbsp_core::WorkItem* items_out,
           uint32_t* entries_out, void*& scratch, size_t& scratch_bytes, cudaStream_t stream) {
  const uint32_t head_group = lpt_head_group(flags, v.heads, v.kv_blocks);  // 0 = global LPT
  const uint32_t step = (flags & kSchedQuad) ? 4 : (flags & kSchedPairQ) ? 2 : 1;
  const uint32_t per_head = (v.q_blocks + step - 1) / step;
  const uint32_t n = v.heads * per_head;
  if (n >= (1u << 24)) fail(kConfig, "too many work items for the device schedule builder");
  dbsp_dev::K2Args a{d_words, nq_global, (nk_global + 63) / 64, d_head_ids, d_q_ids, v.q_blocks,
                     d_present, d_kv_local, v.kv_tokens_global, per_head, step,
                     head_group};
  const uint32_t n_groups = head_group ? (v.heads + head_group - 1) / head_group : 1u;
  const uint32_t head_bits = head_group ? uint32_t(32 - __builtin_clz(std::max(n_groups, 2u) - 1)) : 0u;
  if (n <= uint32_t(dbsp_dev::kFusedItems) && 22 + head_bits <= 32) {
    // one-CTA planner + the entry writer (3 launches)
    const size_t need = 3 * size_t(n) * 4 + 256;
    if (scratch_bytes < need) {
      if (scratch) {
        ck(cudaStreamSynchronize(stream), "k2 scratch regrow");
        cudaFree(scratch);
      }
      scratch = nullptr;
      ck(cudaMalloc(&scratch, std::max<size_t>(need, 1 << 16)), "cudaMalloc k2 scratch");
      scratch_bytes = std::max<size_t>(need, 1 << 16);
    }
    uint32_t* sidx = static_cast<uint32_t*>(scratch);
    uint32_t* begins = sidx + n;
    uint32_t* cnts = begins + n;
    static std::once_flag attr;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(attr, [] {
      attr_err = cudaFuncSetAttribute(dbsp_dev::k2_plan_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(sizeof(dbsp_dev::K2Smem)));
    });
    ck(attr_err, "k2_plan_fused attribute");
    dbsp_core::count_launch();
    dbsp_dev::k2_count<<<(n + 255) / 256, 256, 0, stream>>>(a, n, cnts, nullptr);
    ck(cudaGetLastError(), "k2_count");
    dbsp_core::count_launch();
    dbsp_dev::k2_plan_fused<<<1, dbsp_dev::kK2Threads, sizeof(dbsp_dev::K2Smem), stream>>>(
        a, n, 22 + head_bits, cnts, items_out, sidx, begins);
    ck(cudaGetLastError(), "k2_plan_fused");
    dbsp_core::count_launch();
    dbsp_dev::k2_write_fused<<<(n + 7) / 8, 256, 0, stream>>>(a, n, sidx, begins, entries_out);
    ck(cudaGetLastError(), "k2_write_fused");
    return;
  }
  // scratch: counts, keys, sorted keys, sorted counts, begins, cub temp
  size_t sort_tmp = 0, scan_tmp = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, sort_tmp, (unsigned long long*)nullptr,
                                 (unsigned long long*)nullptr, int(n), 0, 64, stream);
  cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp, (uint32_t*)nullptr, (uint32_t*)nullptr, int(n), stream);
  const size_t al = 256;
  auto up = [&](size_t x) { return (x + al - 1) / al * al; };
  const size_t need = up(n * 4) + 2 * up(n * 8) + 2 * up(n * 4) + up(std::max(sort_tmp, scan_tmp));
  if (scratch_bytes < need) {
    if (scratch) {
      ck(cudaStreamSynchronize(stream), "k2 scratch regrow");  // the previous build may still use it
      cudaFree(scratch);
    }
    scratch = nullptr;
    ck(cudaMalloc(&scratch, need), "cudaMalloc k2 scratch");
    scratch_bytes = need;
  }
  uint8_t* s = static_cast<uint8_t*>(scratch);
  uint32_t* counts = reinterpret_cast<uint32_t*>(s);
  s += up(n * 4);
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(s);
  s += up(n * 8);
  unsigned long long* sorted = reinterpret_cast<unsigned long long*>(s);
  s += up(n * 8);
  uint32_t* scounts = reinterpret_cast<uint32_t*>(s);
  s += up(n * 4);
  uint32_t* begins = reinterpret_cast<uint32_t*>(s);
  s += up(n * 4);
  void* tmp = s;
  dbsp_core::count_launch();
  dbsp_dev::k2_count<<<(n + 255) / 256, 256, 0, stream>>>(a, n, counts, keys);
  ck(cudaGetLastError(), "k2_count");
  size_t t1 = sort_tmp;
  ck(cub::DeviceRadixSort::SortKeys(tmp, t1, keys, sorted, int(n), 0, 64, stream), "k2 sort");
  dbsp_core::count_launch();
  dbsp_dev::k2_sorted_counts<<<(n + 255) / 256, 256, 0, stream>>>(sorted, counts, n, scounts);
  ck(cudaGetLastError(), "k2_sorted_counts");
  size_t t2 = scan_tmp;
  ck(cub::DeviceScan::ExclusiveSum(tmp, t2, scounts, begins, int(n), stream), "k2 scan");
  dbsp_core::count_launch();
  dbsp_dev::k2_write<<<(n + 7) / 8, 256, 0, stream>>>(a, n, sorted, scounts, begins, items_out,
                                                      entries_out);
  ck(cudaGetLastError(), "k2_write");
}

}  // namespace dbsp_k2
