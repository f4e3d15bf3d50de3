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
  uint32_t step;              // 2 = paired Q blocks
  uint32_t head_order;        // 1 = per-head LPT, 0 = global LPT
};

__device__ __forceinline__ void item_rows(const K2Args& a, uint32_t i, uint32_t& hl, uint32_t& qa,
                                          uint32_t& qb, bool& single) {
  hl = i / a.items_per_head;
  qa = (i % a.items_per_head) * a.step;
  single = a.step == 1 || qa + 1 >= a.nq_local;
  qb = single ? qa : qa + 1;
}

__global__ void k2_count(K2Args a, uint32_t n_items, uint32_t* counts, unsigned long long* keys) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_items) return;
  uint32_t hl, qa, qb;
  bool single;
  item_rows(a, i, hl, qa, qb, single);
  const uint32_t h = a.head_ids[hl];
  const uint64_t* ra = a.words + (size_t(h) * a.nq_global + a.q_ids[qa]) * a.wpr;
  const uint64_t* rb = a.words + (size_t(h) * a.nq_global + a.q_ids[qb]) * a.wpr;
  uint32_t c = 0;
  for (uint32_t w = 0; w < a.wpr; ++w) c += __popcll((ra[w] | (single ? 0ull : rb[w])) & a.present[w]);
  counts[i] = c;
  const unsigned long long head_key = a.head_order ? (unsigned long long)hl : 0ull;
  keys[i] = (head_key << 44) | ((unsigned long long)(0xFFFFFu - min(c, 0xFFFFFu)) << 24) | i;
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
  uint32_t hl, qa, qb;
  bool single;
  item_rows(a, i, hl, qa, qb, single);
  const uint32_t begin = begins[j];
  if (lane == 0) items[j] = WorkItem{hl, qa, qb, begin, sorted_counts[j], single ? 1u : 0u, 0, 0};
  const uint32_t h = a.head_ids[hl];
  const uint64_t* ra = a.words + (size_t(h) * a.nq_global + a.q_ids[qa]) * a.wpr;
  const uint64_t* rb = a.words + (size_t(h) * a.nq_global + a.q_ids[qb]) * a.wpr;
  uint32_t out = begin;
  for (uint32_t w = 0; w < a.wpr; ++w) {
    const uint64_t wa = ra[w], wb = single ? 0ull : rb[w];
    const uint64_t uni = (wa | wb) & a.present[w];
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
        const uint32_t e = uint32_t(a.kv_local[k]) | (((wa >> bit) & 1ull) ? dbsp_core::kEntryDenseA : 0u) |
                           (((wb >> bit) & 1ull) ? dbsp_core::kEntryDenseB : 0u) |
                           ((valid - 1) << dbsp_core::kEntryValidShift);
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

// Device-side state attached to a dbsp_schedule (see attention.cu).
struct dbsp_device_schedule {
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
};

namespace dbsp_k2 {

// Builds into `items_out` / `entries_out` (device, caller-sized: n_items and
// n_items * min(nk_local_present, nk) entries).  All work is stream-ordered.
void build(const uint64_t* d_words, uint32_t nq_global, uint32_t nk_global, const LocalView& v,
           uint32_t flags, const uint32_t* d_head_ids, const uint32_t* d_q_ids,
           const uint64_t* d_present, const int32_t* d_kv_local, dbsp_core::WorkItem* items_out,
           uint32_t* entries_out, void*& scratch, size_t& scratch_bytes, cudaStream_t stream) {
  const bool pair = (flags & kSchedPairQ) != 0;
  bool global_lpt = (flags & kSchedGlobalLpt) != 0;
  if (!(flags & (kSchedGlobalLpt | kSchedHeadOrder))) global_lpt = uint64_t(v.heads) * v.kv_blocks <= 4096;
  const uint32_t step = pair ? 2 : 1;
  const uint32_t per_head = (v.q_blocks + step - 1) / step;
  const uint32_t n = v.heads * per_head;
  if (n >= (1u << 24)) fail(kConfig, "too many work items for the device schedule builder");
  dbsp_dev::K2Args a{d_words, nq_global, (nk_global + 63) / 64, d_head_ids, d_q_ids, v.q_blocks,
                     d_present, d_kv_local, v.kv_tokens_global, per_head, step,
                     global_lpt ? 0u : 1u};
  // scratch: counts, keys, sorted keys, sorted counts, begins, cub temp
  size_t sort_tmp = 0, scan_tmp = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, sort_tmp, (unsigned long long*)nullptr,
                                 (unsigned long long*)nullptr, int(n), 0, 64, stream);
  cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp, (uint32_t*)nullptr, (uint32_t*)nullptr, int(n), stream);
  const size_t al = 256;
  auto up = [&](size_t x) { return (x + al - 1) / al * al; };
  const size_t need = up(n * 4) + 2 * up(n * 8) + 2 * up(n * 4) + up(std::max(sort_tmp, scan_tmp));
  if (scratch_bytes < need) {
    if (scratch) cudaFree(scratch);
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
  dbsp_dev::k2_count<<<(n + 255) / 256, 256, 0, stream>>>(a, n, counts, keys);
  ck(cudaGetLastError(), "k2_count");
  size_t t1 = sort_tmp;
  ck(cub::DeviceRadixSort::SortKeys(tmp, t1, keys, sorted, int(n), 0, 64, stream), "k2 sort");
  dbsp_dev::k2_sorted_counts<<<(n + 255) / 256, 256, 0, stream>>>(sorted, counts, n, scounts);
  ck(cudaGetLastError(), "k2_sorted_counts");
  size_t t2 = scan_tmp;
  ck(cub::DeviceScan::ExclusiveSum(tmp, t2, scounts, begins, int(n), stream), "k2 scan");
  dbsp_dev::k2_write<<<(n + 7) / 8, 256, 0, stream>>>(a, n, sorted, scounts, begins, items_out,
                                                      entries_out);
  ck(cudaGetLastError(), "k2_write");
}

}  // namespace dbsp_k2
