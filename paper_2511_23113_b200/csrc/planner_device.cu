// GPU inputs of the U x R selector; see planner_device.hpp.
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "planner_device.hpp"

namespace dbsp_dev {
// K1 (attention.cu).
__global__ void mask_rows_kernel(const uint64_t* __restrict__ words, uint32_t heads, uint32_t nq,
                                 uint32_t wpr, unsigned long long* head_counts,
                                 unsigned long long* row_w);
__global__ void mask_cols_kernel(const uint64_t* __restrict__ words, uint32_t rows, uint32_t nk,
                                 uint32_t wpr, uint32_t rows_per_block, unsigned long long* col_w);

struct TableJobDev {
  uint32_t y, gpus;        // ring degree, x*y
  uint32_t head_off;       // into assign[]: H head assignments
  uint32_t q_off;          // into assign[]: nq Q assignments
  uint32_t group_off;      // into groups[]: y * wpr words of KV-group bitsets
  uint32_t out_off;        // into counts[]: y * gpus counters
};

// metrics.hpp:133-168 for y > 1: every (head, Q row) adds, per KV group g,
// popcount(row & group_g) to period (g + y - r) mod y on GPU u*y + r.  One
// thread per mask row; counters accumulate in shared memory (y*gpus <= 64 at
// G=8) and are flushed with one atomic per counter per block.
__global__ void workload_tables_kernel(const uint64_t* __restrict__ words, uint32_t H, uint32_t nq,
                                       uint32_t wpr, const TableJobDev* __restrict__ jobs,
                                       const uint32_t* __restrict__ assign,
                                       const uint64_t* __restrict__ groups,
                                       unsigned long long* counts) {
  extern __shared__ unsigned long long s_cnt[];
  const TableJobDev jb = jobs[blockIdx.y];
  const uint32_t ncnt = jb.y * jb.gpus;
  for (uint32_t i = threadIdx.x; i < ncnt; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  const uint32_t row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row < H * nq) {
    const uint32_t h = row / nq, qb = row % nq;
    const uint32_t u = assign[jb.head_off + h], rr = assign[jb.q_off + qb];
    const uint32_t gpu = u * jb.y + rr;
    const uint64_t* w = words + size_t(row) * wpr;
    const uint64_t* gb = groups + jb.group_off;
    for (uint32_t g = 0; g < jb.y; ++g) {
      unsigned long long c = 0;
      for (uint32_t i = 0; i < wpr; ++i) c += __popcll(w[i] & gb[size_t(g) * wpr + i]);
      if (c) atomicAdd(&s_cnt[((g + jb.y - rr) % jb.y) * jb.gpus + gpu], c);
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < ncnt; i += blockDim.x)
    if (s_cnt[i]) atomicAdd(&counts[jb.out_off + i], s_cnt[i]);
}
}  // namespace dbsp_dev

namespace dbsp_device_planner {

using namespace dbsp_core;

namespace {

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(kCuda, std::string(what) + ": " + cudaGetErrorString(e));
}

// Per-thread device and pinned scratch, grown on demand.
struct Scratch {
  void* dev = nullptr;
  size_t dev_bytes = 0;
  void* host = nullptr;
  size_t host_bytes = 0;
  ~Scratch() {
    if (dev) cudaFree(dev);
    if (host) cudaFreeHost(host);
  }
  void* device(size_t n) {
    if (n > dev_bytes) {
      if (dev) cudaFree(dev);
      dev = nullptr;
      check(cudaMalloc(&dev, n), "cudaMalloc planner scratch");
      dev_bytes = n;
    }
    return dev;
  }
  void* pinned(size_t n) {
    if (n > host_bytes) {
      if (host) cudaFreeHost(host);
      host = nullptr;
      check(cudaMallocHost(&host, n), "cudaMallocHost planner scratch");
      host_bytes = n;
    }
    return host;
  }
};
thread_local Scratch g_stats, g_tables;

size_t align8(size_t n) { return (n + 7) & ~size_t(7); }

}  // namespace

MaskStats mask_stats(const uint64_t* d_words, uint32_t H, uint32_t nq, uint32_t nk, void* stream_ptr) {
  if (!d_words) fail(kContract, "null device mask words");
  if (H == 0 || nq == 0 || nk == 0) fail(kConfig, "mask dimensions must be positive");
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_ptr);
  const uint32_t wpr = (nk + 63) / 64;
  const size_t n = size_t(H) + nq + nk;
  unsigned long long* d = static_cast<unsigned long long*>(g_stats.device(n * 8));
  check(cudaMemsetAsync(d, 0, n * 8, stream), "memset");
  const uint32_t rows = H * nq;
  dbsp_core::count_launch();
  dbsp_dev::mask_rows_kernel<<<(rows + 255) / 256, 256, 0, stream>>>(d_words, H, nq, wpr, d, d + H);
  check(cudaGetLastError(), "mask_rows launch");
  const uint32_t rpb = 256;
  dbsp_core::count_launch();
  dbsp_dev::mask_cols_kernel<<<dim3(wpr, (rows + rpb - 1) / rpb), 64, 0, stream>>>(d_words, rows, nk, wpr, rpb,
                                                                                   d + H + nq);
  check(cudaGetLastError(), "mask_cols launch");
  uint64_t* h = static_cast<uint64_t*>(g_stats.pinned(n * 8));
  check(cudaMemcpyAsync(h, d, n * 8, cudaMemcpyDeviceToHost, stream), "stats d2h");
  check(cudaStreamSynchronize(stream), "stats sync");
  MaskStats st;
  st.head_counts.assign(h, h + H);
  st.row_weights.assign(h + H, h + H + nq);
  st.col_weights.assign(h + H + nq, h + n);
  st.total = 0;
  for (uint64_t c : st.head_counts) st.total += c;
  st.have_marginals = true;
  return st;
}

std::vector<Table> workload_tables(const uint64_t* d_words, const MaskView& m, const MaskStats& st,
                                   const std::vector<TableJob>& jobs, void* stream_ptr) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_ptr);
  const size_t wpr = m.wpr;
  std::vector<Table> out(jobs.size());
  std::vector<dbsp_dev::TableJobDev> dj;
  std::vector<size_t> job_of;  // device job -> jobs index
  size_t n_assign = 0, n_groups = 0, n_counts = 0;
  for (size_t i = 0; i < jobs.size(); ++i) {
    const Strategy s = jobs[i].s;
    const Plan& p = *jobs[i].plan;
    Table& t = out[i];
    t.gpus = s.x * s.y;
    if (s.y == 1) {  // per-u head sums: host, from K1's head counts
      t.periods = 1;
      t.counts.assign(t.gpus, 0);
      for (uint32_t h = 0; h < m.H; ++h) t.counts[p.head[h]] += st.head_counts[h];
      continue;
    }
    t.periods = s.y;
    dbsp_dev::TableJobDev j;
    j.y = s.y;
    j.gpus = t.gpus;
    j.head_off = uint32_t(n_assign);
    j.q_off = uint32_t(n_assign + m.H);
    j.group_off = uint32_t(n_groups);
    j.out_off = uint32_t(n_counts);
    n_assign += m.H + m.nq;
    n_groups += size_t(s.y) * wpr;
    n_counts += size_t(s.y) * t.gpus;
    if (size_t(s.y) * t.gpus > 1024) fail(kConfig, "workload table too large for the device path");
    dj.push_back(j);
    job_of.push_back(i);
  }
  if (dj.empty()) return out;
  // One pinned staging block: jobs | assignments | group bitsets | counts (back).
  const size_t b_jobs = align8(dj.size() * sizeof(dbsp_dev::TableJobDev));
  const size_t b_assign = align8(n_assign * 4);
  const size_t b_groups = n_groups * 8, b_counts = n_counts * 8;
  const size_t up = b_jobs + b_assign + b_groups;
  uint8_t* h = static_cast<uint8_t*>(g_tables.pinned(up + b_counts));
  std::memcpy(h, dj.data(), dj.size() * sizeof(dbsp_dev::TableJobDev));
  uint32_t* ha = reinterpret_cast<uint32_t*>(h + b_jobs);
  uint64_t* hg = reinterpret_cast<uint64_t*>(h + b_jobs + b_assign);
  std::memset(hg, 0, b_groups);
  for (size_t k = 0; k < dj.size(); ++k) {
    const Plan& p = *jobs[job_of[k]].plan;
    std::memcpy(ha + dj[k].head_off, p.head.data(), m.H * 4);
    std::memcpy(ha + dj[k].q_off, p.q.data(), m.nq * 4);
    uint64_t* g = hg + dj[k].group_off;
    for (uint32_t kb = 0; kb < m.nk; ++kb) g[size_t(p.kv[kb]) * wpr + kb / 64] |= 1ull << (kb % 64);
  }
  uint8_t* d = static_cast<uint8_t*>(g_tables.device(up + b_counts));
  check(cudaMemcpyAsync(d, h, up, cudaMemcpyHostToDevice, stream), "tables h2d");
  unsigned long long* dc = reinterpret_cast<unsigned long long*>(d + up);
  check(cudaMemsetAsync(dc, 0, b_counts, stream), "memset");
  const uint32_t rows = m.H * m.nq;
  uint32_t max_cnt = 0;
  for (const auto& j : dj) max_cnt = std::max(max_cnt, j.y * j.gpus);
  dbsp_core::count_launch();
  dbsp_dev::workload_tables_kernel<<<dim3((rows + 255) / 256, uint32_t(dj.size())), 256, max_cnt * 8, stream>>>(
      d_words, m.H, m.nq, uint32_t(wpr), reinterpret_cast<const dbsp_dev::TableJobDev*>(d),
      reinterpret_cast<const uint32_t*>(d + b_jobs), reinterpret_cast<const uint64_t*>(d + b_jobs + b_assign), dc);
  check(cudaGetLastError(), "workload_tables launch");
  uint64_t* hc = reinterpret_cast<uint64_t*>(h + up);
  check(cudaMemcpyAsync(hc, dc, b_counts, cudaMemcpyDeviceToHost, stream), "tables d2h");
  check(cudaStreamSynchronize(stream), "tables sync");
  for (size_t k = 0; k < dj.size(); ++k) {
    Table& t = out[job_of[k]];
    t.counts.assign(hc + dj[k].out_off, hc + dj[k].out_off + size_t(t.periods) * t.gpus);
  }
  return out;
}

}  // namespace dbsp_device_planner
