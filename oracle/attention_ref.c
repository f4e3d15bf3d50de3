/*
 * ORACLE — test infrastructure only.  Never linked into or called by the
 * product path; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs load it, as the checker or as the
 * timed CPU baseline.
 *
 * CPU restatement of block-sparse DiT attention (no reference code exists for
 * the numerics: SPEC.md:13,109 put kernels out of the reference's scope).
 * Semantics, fixed here and in DESIGN.md:
 *   - per head, O = softmax(Q K^T * scale) V
 *   - only tiles whose mask bit (q_block, kv_block) is set are computed; a
 *     masked tile contributes nothing (score -inf)     (
 *     reference BlockMask bit meaning, proj/include/dbsp/mask.hpp:18-20)
 *   - KV tokens past kv_tokens (partial last block) are excluded
 *   - a query row with no dense tile has O = 0, LSE = -inf
 * Inputs are fp32 [tokens, heads, d]; accumulation is in double, so this is
 * at least as accurate as the "fp32 CPU oracle" the tolerance is stated
 * against.  Parity was cross-checked against torch's SDPA with the block mask
 * expanded to tokens (tests/test_oracle.py).
 *
 * The optional `kv_allow` bitmap (ceil(nk/64) words, NULL = all) restricts the
 * KV blocks considered, which replays one ring period; merging periods with
 * their LSEs reproduces the full result (the ring merge of PAPER.md:93).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

static inline int bit_of(const uint64_t* row, uint32_t k) { return (int)((row[k >> 6] >> (k & 63)) & 1u); }

/* rows: optional list of (head, q_block) pairs (2*nrows ints); NULL = all. */
int oracle_sparse_attention(const float* q, const float* k, const float* v, uint32_t Sq,
                            uint32_t Sk, uint32_t H, uint32_t d, const uint64_t* words,
                            uint32_t nq, uint32_t nk, uint32_t block, float scale,
                            const uint64_t* kv_allow, const int32_t* rows, int64_t nrows,
                            float* out, float* lse) {
  const uint32_t wpr = (nk + 63) / 64;
  if (nq * block < Sq || nk * block < Sk) return 1;
  const int64_t total = rows ? nrows : (int64_t)H * nq;
#pragma omp parallel
  {
    double* sc = (double*)malloc(sizeof(double) * (size_t)nk * block);
    double* acc = (double*)malloc(sizeof(double) * d);
    uint32_t* keys = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)nk * block);
#pragma omp for schedule(dynamic, 1)
    for (int64_t it = 0; it < total; ++it) {
      const uint32_t h = rows ? (uint32_t)rows[2 * it] : (uint32_t)(it / nq);
      const uint32_t qb = rows ? (uint32_t)rows[2 * it + 1] : (uint32_t)(it % nq);
      const uint64_t* mrow = words + ((size_t)h * nq + qb) * wpr;
      uint32_t nkeys = 0;
      for (uint32_t kb = 0; kb < nk; ++kb) {
        if (!bit_of(mrow, kb)) continue;
        if (kv_allow && !bit_of(kv_allow, kb)) continue;
        for (uint32_t j = 0; j < block; ++j) {
          const uint32_t t = kb * block + j;
          if (t < Sk) keys[nkeys++] = t;
        }
      }
      for (uint32_t r = 0; r < block; ++r) {
        const uint32_t tq = qb * block + r;
        if (tq >= Sq) break;
        const float* qv = q + ((size_t)tq * H + h) * d;
        float* o = out + ((size_t)tq * H + h) * d;
        if (nkeys == 0) {
          memset(o, 0, sizeof(float) * d);
          if (lse) lse[(size_t)h * Sq + tq] = -INFINITY;
          continue;
        }
        double mx = -INFINITY;
        for (uint32_t i = 0; i < nkeys; ++i) {
          const float* kv = k + ((size_t)keys[i] * H + h) * d;
          double s = 0.0;
          for (uint32_t c = 0; c < d; ++c) s += (double)qv[c] * (double)kv[c];
          s *= (double)scale;
          sc[i] = s;
          if (s > mx) mx = s;
        }
        double den = 0.0;
        for (uint32_t c = 0; c < d; ++c) acc[c] = 0.0;
        for (uint32_t i = 0; i < nkeys; ++i) {
          const double p = exp(sc[i] - mx);
          den += p;
          const float* vv = v + ((size_t)keys[i] * H + h) * d;
          for (uint32_t c = 0; c < d; ++c) acc[c] += p * (double)vv[c];
        }
        for (uint32_t c = 0; c < d; ++c) o[c] = (float)(acc[c] / den);
        if (lse) lse[(size_t)h * Sq + tq] = (float)(mx + log(den));
      }
    }
    free(sc);
    free(acc);
    free(keys);
  }
  return 0;
}

/* FNV-1a 64 over raw bytes (mask-set fingerprints in the golden file). */
uint64_t oracle_fnv1a(const uint8_t* data, uint64_t n) {
  uint64_t h = 1469598103934665603ull;
  for (uint64_t i = 0; i < n; ++i) {
    h ^= data[i];
    h *= 1099511628211ull;
  }
  return h;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
