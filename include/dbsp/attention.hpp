// The attention call the reference only models: block-
// sparse softmax(QK^T/sqrt(d))V over the dense 64x64 tiles of a mask set, run
// by the sm_100a tcgen05 kernel in libdbsp_b200.so.  Device pointers, bf16,
// token-major [tokens, heads, d], d in {64, 128}; stream-ordered.
#pragma once

#include <cstdint>
#include <vector>

#include "../dbsp_b200.h"
#include "error.hpp"
#include "mask.hpp"
#include "metrics.hpp"

namespace dbsp {

struct AttentionArgs {
  const void* q = nullptr;  // bf16 [q_tokens, heads, d]
  const void* k = nullptr;  // bf16 [kv_tokens, heads, d]
  const void* v = nullptr;
  void* o = nullptr;        // bf16 [q_tokens, heads, d]
  float* lse = nullptr;     // optional fp32 [heads, q_tokens]
  uint32_t q_tokens = 0, kv_tokens = 0, heads = 0, head_dim = 0;
  float softmax_scale = 0.f;  // 0 -> 1/sqrt(d)
};

// Reusable work list: build once per (mask set, local view), launch many times.
class AttentionSchedule {
 public:
  AttentionSchedule() { detail::check(dbsp_schedule_create(&h_)); }
  ~AttentionSchedule() { dbsp_schedule_destroy(h_); }
  AttentionSchedule(const AttentionSchedule&) = delete;
  AttentionSchedule& operator=(const AttentionSchedule&) = delete;

  // Whole-problem schedule (identity local view).  head_dim 128 lets the builder
  // pick the CTA-pair kernel where it pays (DBSP_SCHED_AUTO_D128).
  void build(const AttentionMaskSet& set, uint32_t kv_tokens, uint32_t head_dim = 0) {
    detail::MaskView v(set);
    dbsp_local_view lv{set.num_heads(), nullptr, set.num_q_blocks(), nullptr,
                       set.num_kv_blocks(), nullptr, kv_tokens};
    detail::check(dbsp_schedule_build(h_, v.get(), &lv, flags_for(head_dim)));
  }
  // One rank's share: local head / Q-block / KV-block ids in buffer order.
  void build(const AttentionMaskSet& set, const std::vector<uint32_t>& heads,
             const std::vector<uint32_t>& q_blocks, const std::vector<uint32_t>& kv_blocks,
             uint32_t kv_tokens_global, uint32_t head_dim = 0) {
    detail::MaskView v(set);
    dbsp_local_view lv{uint32_t(heads.size()), heads.data(), uint32_t(q_blocks.size()),
                       q_blocks.data(), uint32_t(kv_blocks.size()), kv_blocks.data(),
                       kv_tokens_global};
    detail::check(dbsp_schedule_build(h_, v.get(), &lv, flags_for(head_dim)));
  }
  void launch(const AttentionArgs& a, void* stream) {
    const dbsp_attn_args c{a.q, a.k, a.v, a.o, a.lse, nullptr, nullptr, a.q_tokens, a.kv_tokens,
                           a.heads, a.head_dim, a.softmax_scale, 0, 0};
    detail::check(dbsp_attention_launch(h_, &c, stream));
  }
  dbsp_schedule* handle() const { return h_; }

 private:
  static int32_t flags_for(uint32_t head_dim) {
    return head_dim == 128 ? (DBSP_SCHED_PAIR_Q | DBSP_SCHED_AUTO_D128) : DBSP_SCHED_PAIR_Q;
  }
  dbsp_schedule* h_ = nullptr;
};

inline void sparse_attention(const AttentionMaskSet& set, const AttentionArgs& a, void* stream) {
  detail::MaskView v(set);
  const dbsp_attn_args c{a.q, a.k, a.v, a.o, a.lse, nullptr, nullptr, a.q_tokens, a.kv_tokens,
                         a.heads, a.head_dim, a.softmax_scale, 0, 0};
  detail::check(dbsp_sparse_attention(v.get(), &c, stream));
}

// The sequence-parallel call: one context per GPU process
// owns the NCCL communicator; rank 0 makes the id, every rank passes it in.
class SpContext {
 public:
  static std::vector<uint8_t> unique_id() {
    std::vector<uint8_t> id(128);
    detail::check(dbsp_nccl_unique_id(id.data(), uint32_t(id.size())));
    return id;
  }
  SpContext(uint32_t rank, uint32_t world, const std::vector<uint8_t>& nccl_id) {
    detail::check(dbsp_sp_context_create(rank, world, nccl_id.data(), &h_));
  }
  ~SpContext() { dbsp_sp_context_destroy(h_); }
  SpContext(const SpContext&) = delete;
  SpContext& operator=(const SpContext&) = delete;
  dbsp_sp_context* handle() const { return h_; }

 private:
  dbsp_sp_context* h_ = nullptr;
};

// q/k/v/o: this rank's home shards, bf16 [home tokens, H, d] (rank g holds
// blocks [g*nb/G, (g+1)*nb/G)); stream-ordered.
inline void sparse_attention(SpContext& ctx, const AttentionMaskSet& set, ParallelStrategy strategy,
                             const PartitionPlan& plan, const void* q, const void* k, const void* v, void* o,
                             uint32_t head_dim, void* stream) {
  detail::MaskView mv(set);
  std::vector<uint32_t> h = plan.head_assignment, qa = plan.q_assignment, kv = plan.kv_assignment;
  const dbsp_plan cp{h.data(), qa.data(), kv.data()};
  detail::check(dbsp_sp_attention(ctx.handle(), mv.get(), dbsp_strategy{strategy.ulysses, strategy.ring}, &cp,
                                  q, k, v, o, set.num_q_blocks() * set.block_size(), head_dim, stream));
}

// K6: the layer's QKV projection (nn.Linear weight [3*H*d, hidden]); with
// `scatter` non-null the Q/K/V rows go straight into the consuming ranks'
// local buffers (the fused all-to-all(v) send of the SP call).
inline void qkv_project(const void* x, const void* w, const void* bias, void* out, uint32_t tokens,
                        uint32_t hidden, uint32_t heads, uint32_t head_dim, const dbsp_qkv_scatter* scatter,
                        void* stream) {
  const dbsp_qkv_args a{x, w, bias, out, tokens, hidden, heads, head_dim};
  detail::check(dbsp_qkv_project(&a, scatter, stream));
}

}  // namespace dbsp
