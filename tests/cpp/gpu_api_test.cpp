// The C++ faces on a GPU, as a C++ DiT engine would call them: the selector
// from device mask words (dbsp::select_device) against the host selector, and
// single-GPU block-sparse attention (dbsp::sparse_attention) on random bf16
// data against a CPU fp32 reference on sampled rows.  Built and run by
// tests/test_cpp_api.py::test_cpp_gpu_faces (GPU box).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "dbsp/attention.hpp"
#include "dbsp/latency.hpp"
#include "dbsp/mask.hpp"
#include "dbsp/selector.hpp"

static int failures = 0;
#define EXPECT(c, what)                                       \
  do {                                                        \
    if (!(c)) {                                               \
      std::printf("[FAIL] %s (%s:%d)\n", what, __FILE__, __LINE__); \
      ++failures;                                             \
    } else {                                                  \
      std::printf("[PASS] %s\n", what);                       \
    }                                                         \
  } while (0)

int main() {
  // ---- selector: device words vs host
  dbsp::GeneratorSpec spec;
  spec.num_heads = 40;
  spec.num_q_blocks = spec.num_kv_blocks = 512;
  spec.pattern = dbsp::MaskPattern::clustered;
  spec.min_density = 0.15;
  spec.max_density = 0.45;
  spec.seed = 1;
  const dbsp::AttentionMaskSet masks = dbsp::generate_mask_set(spec);
  const size_t wpr = (spec.num_kv_blocks + 63) / 64;
  std::vector<uint64_t> words;
  for (const dbsp::BlockMask& m : masks.masks()) words.insert(words.end(), m.data(), m.data() + spec.num_q_blocks * wpr);
  uint64_t* d_words = nullptr;
  cudaMalloc(&d_words, words.size() * 8);
  cudaMemcpy(d_words, words.data(), words.size() * 8, cudaMemcpyHostToDevice);
  dbsp::MachineProfile prof = dbsp::load_profile(DBSP_PROFILE_JSON);
  dbsp::SelectorState host_state(8), dev_state(8);
  bool same = true;
  for (int layer = 0; layer < 3; ++layer) {
    const dbsp::Selection a = dbsp::select(layer, masks, prof, dbsp::PlannerConfig{}, host_state);
    const dbsp::Selection b = dbsp::select_device(layer, d_words, spec.num_heads, spec.num_q_blocks,
                                                  spec.num_kv_blocks, 64, prof, dbsp::PlannerConfig{}, dev_state);
    same = same && a.strategy == b.strategy && a.outcome.plan == b.outcome.plan &&
           a.outcome.rho_post == b.outcome.rho_post && a.latency.total_s == b.latency.total_s;
  }
  EXPECT(same, "select_device equals select (strategy, plan, rho, latency) over 3 calls");
  cudaFree(d_words);

  // ---- single-GPU attention through the C++ face
  const uint32_t H = 4, S = 1024, d = 128, nb = S / 64;
  dbsp::GeneratorSpec s2 = spec;
  s2.num_heads = H;
  s2.num_q_blocks = s2.num_kv_blocks = nb;
  const dbsp::AttentionMaskSet m2 = dbsp::generate_mask_set(s2);
  std::mt19937 rng(7);
  std::normal_distribution<float> nd;
  const size_t n = size_t(S) * H * d;
  std::vector<__nv_bfloat16> hq(n), hk(n), hv(n), ho(n);
  std::vector<float> fq(n), fk(n), fv(n);
  for (size_t i = 0; i < n; ++i) {
    hq[i] = __float2bfloat16(nd(rng));
    hk[i] = __float2bfloat16(nd(rng));
    hv[i] = __float2bfloat16(nd(rng));
    fq[i] = __bfloat162float(hq[i]);
    fk[i] = __bfloat162float(hk[i]);
    fv[i] = __bfloat162float(hv[i]);
  }
  void *dq, *dk, *dv, *dout;
  cudaMalloc(&dq, n * 2);
  cudaMalloc(&dk, n * 2);
  cudaMalloc(&dv, n * 2);
  cudaMalloc(&dout, n * 2);
  cudaMemcpy(dq, hq.data(), n * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dk, hk.data(), n * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, hv.data(), n * 2, cudaMemcpyHostToDevice);
  dbsp::AttentionArgs args;
  args.q = dq;
  args.k = dk;
  args.v = dv;
  args.o = dout;
  args.q_tokens = args.kv_tokens = S;
  args.heads = H;
  args.head_dim = d;
  dbsp::sparse_attention(m2, args, nullptr);
  cudaMemcpy(ho.data(), dout, n * 2, cudaMemcpyDeviceToHost);
  // CPU reference on sampled rows: softmax over the dense tiles of the row's Q block
  auto sampled_error = [&](const std::vector<__nv_bfloat16>& ho) {
  double max_err = 0.0;
  const float scale = 1.0f / std::sqrt(float(d));
  for (uint32_t h = 0; h < H; ++h)
    for (uint32_t t = 5; t < S; t += 97) {
      const uint32_t qb = t / 64;
      std::vector<double> sc;
      std::vector<uint32_t> keys;
      for (uint32_t kb = 0; kb < nb; ++kb)
        if (m2.masks()[h].get(qb, kb))
          for (uint32_t kk = kb * 64; kk < kb * 64 + 64; ++kk) {
            double dot = 0;
            for (uint32_t c = 0; c < d; ++c) dot += double(fq[(size_t(t) * H + h) * d + c]) * fk[(size_t(kk) * H + h) * d + c];
            sc.push_back(dot * scale);
            keys.push_back(kk);
          }
      double mx = -1e300, sum = 0;
      for (double x : sc) mx = std::max(mx, x);
      for (double& x : sc) sum += (x = std::exp(x - mx));
      for (uint32_t c = 0; c < d; ++c) {
        double o = 0;
        for (size_t i = 0; i < keys.size(); ++i) o += sc[i] / sum * fv[(size_t(keys[i]) * H + h) * d + c];
        if (keys.empty()) o = 0;
        max_err = std::max(max_err, std::fabs(o - double(__bfloat162float(ho[(size_t(t) * H + h) * d + c]))));
      }
    }
  return max_err;
  };
  const double max_err = sampled_error(ho);
  std::printf("attention max-abs error on sampled rows: %.3e\n", max_err);
  EXPECT(max_err <= 2e-2, "dbsp::sparse_attention matches the CPU reference within 2e-2");

  // ---- the CTA-pair kernel (cta_group::2, attn_kernel_pd3.cuh) through the C ABI
  {
    dbsp::detail::MaskView mv(m2);
    dbsp_schedule* sch = nullptr;
    EXPECT(dbsp_schedule_create(&sch) == 0, "schedule create");
    dbsp_local_view lv{H, nullptr, nb, nullptr, nb, nullptr, S};
    const int32_t fl = DBSP_SCHED_PAIR_Q | DBSP_SCHED_QUAD | DBSP_SCHED_KEY128 | DBSP_SCHED_CTA_PAIR;
    EXPECT(dbsp_schedule_build(sch, mv.get(), &lv, fl) == 0, "CTA-pair schedule build");
    uint32_t got_flags = 0;
    EXPECT(dbsp_schedule_layout(sch, &got_flags) == 0 && got_flags == uint32_t(fl), "schedule layout reports the CTA-pair build");
    cudaMemset(dout, 0, n * 2);
    const dbsp_attn_args ca{dq, dk, dv, dout, nullptr, nullptr, nullptr, S, S, H, d, 0.f, 0, 0};
    EXPECT(dbsp_attention_launch(sch, &ca, nullptr) == 0, "CTA-pair launch");
    cudaMemcpy(ho.data(), dout, n * 2, cudaMemcpyDeviceToHost);
    const double e2 = sampled_error(ho);
    std::printf("CTA-pair kernel max-abs error on sampled rows: %.3e\n", e2);
    EXPECT(e2 <= 2e-2, "the CTA-pair kernel matches the CPU reference within 2e-2");
    dbsp_schedule_destroy(sch);
  }
  cudaFree(dq);
  cudaFree(dk);
  cudaFree(dv);
  cudaFree(dout);
  std::printf("%d failure(s)\n", failures);
  return failures ? 1 : 0;
}
