/*
 * dbsp_b200.h — C ABI of the B200-native db-SP hot path.
 *
 * This is the drop-in boundary.  The reference (arxiv 2511.23113, `proj/`) is a
 * header-only C++20 library with no FFI of its own; every entry point below
 * replaces one reference function (cited as path:line under the reference
 * `proj/include/dbsp/`) or one of the new execution-layer components the
 * reference only models.  The C++ API in `include/dbsp/*.hpp`
 * (same names and signatures as the reference) is a thin layer over these
 * functions, and so is the Python package (ctypes).
 *
 * Conventions
 *  - Plain pointers and sizes only; no torch / STL types cross this boundary.
 *  - Caller owns every buffer.  Output arrays are sized by the caller from the
 *    dimensions it passed in (H heads, Nq Q blocks, Nk KV blocks).
 *  - Every function returns a status; on failure `dbsp_last_error()` returns
 *    a thread-local message.  Status codes mirror the reference CLI exit codes
 *    (tools/dbsp.cpp:437-456): 2 configuration, 3 I/O, 4 contract; the
 *    subclasses parse_error / search_space_error get their own codes so the
 *    C++ layer can rethrow the exact reference exception class (error.hpp:10-44).
 *  - Masks use the reference BlockMask layout (mask.hpp:18-28): per head, Q-major
 *    rows of ceil(Nk/64) little-endian u64 words, bit k of a row at word k/64,
 *    position k%64, padding bits zero.  A mask set is passed as an array of H
 *    per-head word pointers so both contiguous buffers and per-head vectors
 *    (the reference's std::vector<BlockMask>) can be passed without copying.
 *  - Device entry points take device pointers and a cudaStream_t passed as
 *    void*; they are stream-ordered and never synchronise the device unless
 *    documented.
 */
#ifndef DBSP_B200_H_
#define DBSP_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------------ */
/* Status codes (reference error.hpp:10-44, CLI mapping tools/dbsp.cpp:440-455) */
enum {
  DBSP_OK = 0,
  DBSP_ERR_INTERNAL = 1,     /* unexpected failure (bad_alloc, ...)            */
  DBSP_ERR_CONFIG = 2,       /* dbsp::config_error                             */
  DBSP_ERR_IO = 3,           /* dbsp::io_error                                 */
  DBSP_ERR_CONTRACT = 4,     /* dbsp::contract_error                           */
  DBSP_ERR_PARSE = 5,        /* dbsp::parse_error (an io_error)                */
  DBSP_ERR_SEARCH_SPACE = 6, /* dbsp::search_space_error (a config_error)      */
  DBSP_ERR_CUDA = 7          /* CUDA runtime / driver failure (new; no ref)    */
};

/* Thread-local message of the last failing call on this thread. */
const char* dbsp_last_error(void);
/* Library build string (arch, version). */
const char* dbsp_version(void);

/* ------------------------------------------------------------------------ */
/* Value types                                                               */

/* Per-head block masks of one attention call (mask.hpp:83-113). */
typedef struct dbsp_mask_set {
  const uint64_t* const* heads; /* H pointers, each Nq*ceil(Nk/64) words     */
  uint32_t num_heads;
  uint32_t num_q_blocks;
  uint32_t num_kv_blocks;
  uint32_t block_size; /* tokens per block; payload metadata only           */
} dbsp_mask_set;

/* UxRy hybrid strategy (metrics.hpp:20-26). */
typedef struct dbsp_strategy {
  uint32_t ulysses; /* x */
  uint32_t ring;    /* y */
} dbsp_strategy;

/* Partition plan (metrics.hpp:70-76); caller-allocated arrays H / Nq / Nk. */
typedef struct dbsp_plan {
  uint32_t* head_assignment;
  uint32_t* q_assignment;
  uint32_t* kv_assignment;
} dbsp_plan;

/* PlannerConfig (planner.hpp:21-35); defaults P_s = 1.10, R_b = 0. */
typedef struct dbsp_planner_config {
  double reuse_threshold; /* P_s */
  double exchange_reward; /* R_b; +inf keeps every block home */
} dbsp_planner_config;

/* PlanOutcome scalars (planner.hpp:37-42). */
typedef struct dbsp_plan_outcome {
  int32_t head_replanned;
  double rho_pre;
  double rho_post;
} dbsp_plan_outcome;

/* GeneratorSpec (mask.hpp:137-162); pattern 0 random, 1 banded, 2 clustered. */
typedef struct dbsp_generator_spec {
  uint32_t num_heads, num_q_blocks, num_kv_blocks, block_size;
  uint32_t pattern;
  double min_density, max_density, skew;
  uint64_t seed;
} dbsp_generator_spec;

/* ExchangeVolume (metrics.hpp:190-196). */
typedef struct dbsp_exchange {
  uint64_t q_blocks_moved, kv_blocks_moved, token_payload;
} dbsp_exchange;

/* MachineProfile (latency.hpp:45-67) flattened: piecewise-linear knots for
 * each all2all / p2p degree, concatenated; curve i owns knots
 * [offsets[i], offsets[i+1]). */
typedef struct dbsp_profile {
  uint32_t num_all2all;
  const uint32_t* all2all_degrees;  /* num_all2all            */
  const uint32_t* all2all_offsets;  /* num_all2all + 1        */
  const double* all2all_x;          /* payload bytes           */
  const double* all2all_y;          /* seconds                 */
  uint32_t num_p2p;
  const uint32_t* p2p_degrees;
  const uint32_t* p2p_offsets;
  const double* p2p_x;
  const double* p2p_y;
  double dense_attn_seconds;
  double launch_seconds;
  double exchange_overlap;
  double replan_seconds;
  double bytes_per_token_per_head;
} dbsp_profile;

/* LatencyBreakdown (latency.hpp:172-184). */
typedef struct dbsp_latency {
  double all2all_s, attn_compute_s, ring_p2p_exposed_s, imbalance_penalty_s;
  double exchange_s, replan_s, total_s;
} dbsp_latency;

/* CallInputs (latency.hpp:199-206). */
typedef struct dbsp_call_inputs {
  uint32_t heads, q_blocks, kv_blocks, block_size;
  dbsp_strategy strategy;
  double density;
  double rho;
  dbsp_exchange exchange;
  int32_t charge_replan;
} dbsp_call_inputs;

/* ------------------------------------------------------------------------ */
/* Mask model (mask.hpp)                                                     */

/* generate_mask_set (mask.hpp:233-256): writes H*Nq*ceil(Nk/64) words. */
int dbsp_generate_mask_set(const dbsp_generator_spec* spec, uint64_t* words_out);
/* perturb_mask_set (mask.hpp:260-273): in = out allowed (same layout). */
int dbsp_perturb_mask_set(const dbsp_mask_set* set, double flip_rate, uint64_t seed,
                          uint64_t* words_out);
/* total_blocks / blocks_per_head / density (mask.hpp:275-292). */
int dbsp_total_blocks(const dbsp_mask_set* set, uint64_t* out);
int dbsp_blocks_per_head(const dbsp_mask_set* set, uint64_t* out /* H */);
int dbsp_density(const dbsp_mask_set* set, double* out);
/* mix_seed (rng.hpp:37-40). */
uint64_t dbsp_mix_seed(uint64_t base, uint64_t a, uint64_t b);

/* DBSPMSK1 mask files (mask_io.hpp:131-207): atomic save; load in two calls
 * (header for the dimensions, then words sized H*Nq*ceil(Nk/64)).  Errors:
 * DBSP_ERR_IO for filesystem failures, DBSP_ERR_PARSE with the byte offset. */
int dbsp_save_mask_set(const dbsp_mask_set* set, const char* path);
int dbsp_load_mask_set_header(const char* path, uint32_t* heads, uint32_t* q_blocks,
                              uint32_t* kv_blocks, uint32_t* block_size);
int dbsp_load_mask_set(const char* path, uint64_t* words_out);

/* ------------------------------------------------------------------------ */
/* Strategy / plan / rho_s (metrics.hpp)                                     */

/* enumerate_strategies (metrics.hpp:56-66); out has room for 33 entries. */
int dbsp_enumerate_strategies(uint32_t total_gpus, dbsp_strategy* out, uint32_t* count);
/* validate_plan (metrics.hpp:78-90). */
int dbsp_validate_plan(const dbsp_mask_set* set, dbsp_strategy s, const dbsp_plan* plan);
/* default_plan (metrics.hpp:94-113). */
int dbsp_default_plan(const dbsp_mask_set* set, dbsp_strategy s, dbsp_plan* out);
/* workload_table (metrics.hpp:133-168): counts is periods x gpus, row-major,
 * room for max(1, y) * x * y entries; *periods receives 1 (y==1) or y. */
int dbsp_workload_table(const dbsp_mask_set* set, dbsp_strategy s, const dbsp_plan* plan,
                        uint64_t* counts, uint32_t* periods);
/* imbalance_ratio (metrics.hpp:173-186). */
int dbsp_imbalance_ratio(const uint64_t* counts, uint32_t periods, uint32_t gpus,
                         double* out);
/* exchange_volume (metrics.hpp:198-211). */
int dbsp_exchange_volume(const dbsp_mask_set* set, dbsp_strategy s, const dbsp_plan* plan,
                         dbsp_exchange* out);

/* ------------------------------------------------------------------------ */
/* Dual-balanced partitioner (planner.hpp)                                   */

/* summed_grid (planner.hpp:47-61): Nq*Nk counts. */
int dbsp_summed_grid(const dbsp_mask_set* set, uint64_t* grid_out);
/* head_level_imbalance (planner.hpp:65-76). */
int dbsp_head_level_imbalance(const uint64_t* weights, const uint32_t* assignment,
                              uint32_t n, uint32_t x, double* out);
/* partition_heads (planner.hpp:96-112). */
int dbsp_partition_heads(const dbsp_mask_set* set, uint32_t x, uint32_t* out /* H */);
/* partition_blocks (planner.hpp:151-170). */
int dbsp_partition_blocks(const dbsp_mask_set* set, uint32_t y, double reward,
                          uint32_t* q_out /* Nq */, uint32_t* kv_out /* Nk */);
/* detail::biased_greedy (planner.hpp:119-145), exposed for tests. */
int dbsp_biased_greedy(const uint64_t* weights, uint32_t n, uint32_t y, double reward,
                       uint32_t* out);
/* plan_dual (planner.hpp:175-217); prev may be NULL. */
int dbsp_plan_dual(const dbsp_mask_set* set, dbsp_strategy s, const dbsp_planner_config* cfg,
                   const dbsp_plan* prev, dbsp_plan* out, dbsp_plan_outcome* outcome);
/* brute_force_heads (planner.hpp:249-273). */
int dbsp_brute_force_heads(const dbsp_mask_set* set, uint32_t x, uint32_t* out);
/* brute_force_blocks (planner.hpp:282-338). */
int dbsp_brute_force_blocks(const uint64_t* grid, uint32_t nq, uint32_t nk, uint32_t y,
                            uint32_t* q_out, uint32_t* kv_out, double* rho_out);

/* ------------------------------------------------------------------------ */
/* Latency model (latency.hpp)                                               */

/* fit_profile (latency.hpp:114-169).  Samples: primitive 0 all2all, 1 p2p,
 * 2 dense.  The fitted curves are written into caller buffers sized for
 * n_samples knots; *_count receive the number of distinct degrees. */
typedef struct dbsp_profile_sample {
  uint32_t primitive;
  uint32_t degree;
  double x;
  double seconds;
} dbsp_profile_sample;
typedef struct dbsp_fit_options {
  double exchange_overlap, replan_seconds, bytes_per_token_per_head;
} dbsp_fit_options;
typedef struct dbsp_profile_storage {
  uint32_t* all2all_degrees; uint32_t* all2all_offsets; double* all2all_x; double* all2all_y;
  uint32_t* p2p_degrees; uint32_t* p2p_offsets; double* p2p_x; double* p2p_y;
} dbsp_profile_storage;
int dbsp_fit_profile(const dbsp_profile_sample* samples, uint32_t n_samples,
                     const dbsp_fit_options* options, dbsp_profile_storage* storage,
                     dbsp_profile* out);
/* PiecewiseLinear::eval (latency.hpp:27-40). */
int dbsp_pwl_eval(const double* xs, const double* ys, uint32_t n, double x, double* out);
/* predict_from_inputs (latency.hpp:225-268). */
int dbsp_predict_from_inputs(const dbsp_call_inputs* in, const dbsp_profile* profile,
                             dbsp_latency* out);
/* predict_latency (latency.hpp:270-283). */
int dbsp_predict_latency(const dbsp_mask_set* set, dbsp_strategy s, const dbsp_plan* plan,
                         const dbsp_profile* profile, int32_t charge_replan,
                         dbsp_latency* out);

/* ------------------------------------------------------------------------ */
/* Strategy selector (selector.hpp)                                          */

/* SelectorState (selector.hpp:18-43): opaque, internally locked. */
typedef struct dbsp_selector dbsp_selector;
int dbsp_selector_create(uint32_t total_gpus, dbsp_selector** out);
void dbsp_selector_destroy(dbsp_selector* state);
/* SelectorState::stored (selector.hpp:26-31): *found = 0 when absent;
 * plan arrays sized H/Nq/Nk of the stored plan (query sizes with plan=NULL). */
int dbsp_selector_stored(const dbsp_selector* state, int64_t layer, int32_t* found,
                         dbsp_strategy* strategy, uint32_t* sizes /* 3 */, dbsp_plan* plan);
/* SelectorState::store (selector.hpp:33-36). */
int dbsp_selector_store(dbsp_selector* state, int64_t layer, dbsp_strategy s,
                        const dbsp_plan* plan, const uint32_t* sizes /* 3 */);

/* One row per feasible strategy, in enumeration order (latency.hpp:295-315). */
typedef struct dbsp_prediction {
  dbsp_strategy strategy;
  dbsp_plan_outcome outcome;
  dbsp_latency latency;
} dbsp_prediction;

/* predict_all (latency.hpp:295-315).  prev_plans: n_prev strategies with plans
 * (may be 0).  plans_out: room for 33 plans, each with H/Nq/Nk arrays
 * (may be NULL to skip plan output). */
int dbsp_predict_all(const dbsp_mask_set* set, const dbsp_profile* profile,
                     uint32_t total_gpus, const dbsp_planner_config* cfg,
                     const dbsp_strategy* prev_strategies, const dbsp_plan* prev_plans,
                     uint32_t n_prev, dbsp_prediction* out, dbsp_plan* plans_out,
                     uint32_t* count);

/* select (selector.hpp:55-75): argmin, ties to larger x; stores the choice. */
int dbsp_select(dbsp_selector* state, int64_t layer, const dbsp_mask_set* set,
                const dbsp_profile* profile, const dbsp_planner_config* cfg,
                dbsp_strategy* strategy_out, dbsp_plan* plan_out,
                dbsp_plan_outcome* outcome_out, dbsp_latency* latency_out);

/* select() with every mask-dependent integer computed on the GPU from
 * device-resident mask words (u64 [heads][q_blocks][ceil(kv_blocks/64)], the
 * BlockMask row layout): K1 head counts and grid marginals, then one kernel
 * for the workload tables of all (strategy, plan) pairs.  The LPT/greedy
 * assignments and every double run on the host in the reference's order, so
 * the result equals dbsp_select bit for bit.
 * Synchronous on `stream`.  Replaces selector.hpp:55-75 for GPU callers.   */
int dbsp_select_device(dbsp_selector* state, int64_t layer, const uint64_t* d_words, uint32_t heads,
                       uint32_t q_blocks, uint32_t kv_blocks, uint32_t block_size,
                       const dbsp_profile* profile, const dbsp_planner_config* cfg,
                       dbsp_strategy* strategy_out, dbsp_plan* plan_out,
                       dbsp_plan_outcome* outcome_out, dbsp_latency* latency_out, void* stream);
/* The same two-phase selection (assignments first, then one batch of
 * workload tables) with host tables: CPU check of dbsp_select_device's
 * planning code.  Results equal dbsp_select.                               */
int dbsp_select_two_phase(dbsp_selector* state, int64_t layer, const dbsp_mask_set* set,
                          const dbsp_profile* profile, const dbsp_planner_config* cfg,
                          dbsp_strategy* strategy_out, dbsp_plan* plan_out,
                          dbsp_plan_outcome* outcome_out, dbsp_latency* latency_out);

/* ------------------------------------------------------------------------ */
/* Block-sparse attention on sm_100a (new)          */
/*
 * Tensors are bf16, token-major [tokens, heads, head_dim] with head_dim in
 * {64, 128}.  Bit (q, k) of head h's mask means the 64x64 tile between Q
 * block q and KV block k is computed (mask.hpp:18-20); masked tiles are
 * excluded (score -inf), KV tokens past kv_tokens are excluded, and a query
 * row with no dense tile gets O = 0, LSE = -inf.
 */

/* Work schedule for one launch: a list of (head, Q tile) items, each with
 * the dense KV blocks it visits.  Built on the host from the masks
 * (dbsp_schedule_build) and uploaded with the launch. */
typedef struct dbsp_schedule dbsp_schedule;

/* Mapping of one rank's local buffers onto the global mask grid.  NULL
 * arrays mean identity (single GPU / whole problem). */
typedef struct dbsp_local_view {
  uint32_t num_heads;          /* local heads in the Q/K/V buffers              */
  const uint32_t* head_ids;    /* local head -> global head (mask index)        */
  uint32_t num_q_blocks;       /* local Q blocks in the Q/O buffers             */
  const uint32_t* q_block_ids; /* local Q block -> global Q block               */
  uint32_t num_kv_blocks;      /* local KV blocks in the K/V buffers            */
  const uint32_t* kv_block_ids;/* local KV block -> global KV block             */
  uint32_t kv_tokens_global;   /* global KV length; tail block is partial       */
} dbsp_local_view;

int dbsp_schedule_create(dbsp_schedule** out);
void dbsp_schedule_destroy(dbsp_schedule* sched);
/* Schedule flags.  PAIR_Q packs two Q blocks per 128-row tile (the tcgen05
 * M=128 path).  Launch order is heaviest-first; GLOBAL_LPT orders across
 * heads, HEAD_ORDER within each head (K/V of concurrently running CTAs stays
 * L2-resident); with neither, heaviest-first within groups of
 * max(1, 2048 / local KV blocks) heads (a group's K/V fits the L2), one group
 * for views of <= 4096 head x KV blocks. */
enum { DBSP_SCHED_PAIR_Q = 1, DBSP_SCHED_GLOBAL_LPT = 2, DBSP_SCHED_HEAD_ORDER = 4,
       DBSP_SCHED_QUAD = 8 /* layout bit: 4 Q blocks per item (set by CTA_PAIR) */,
       DBSP_SCHED_KEY128 = 16 /* layout bit: 128-key steps (set by CTA_PAIR) */,
       DBSP_SCHED_CTA_PAIR = 128 /* head_dim 128: quad items for the CTA-pair kernel (cta_group::2, two
                                    split-KV stages); implies PAIR_Q | QUAD | KEY128 */,
       DBSP_SCHED_AUTO_D128 = 256 /* head_dim 128: the measured-fastest layout; since round 2 that is the
                                     pair schedule on every measured mask family (schedule.hpp) */ };
/* QUAD or KEY128 without CTA_PAIR, and any other bit, are DBSP_CONFIG_ERROR. */
/* Builds the work list for `view` against `set` (host). */
int dbsp_schedule_build(dbsp_schedule* sched, const dbsp_mask_set* set,
                        const dbsp_local_view* view, int32_t flags);
/* K2 on the device: the same work list built from DEVICE mask words
 * [heads][q_blocks][ceil(kv_blocks/64)] on `stream` (no host pass over the
 * masks, no upload).  `view` holds host arrays (small); NULL = identity. */
int dbsp_schedule_build_device(dbsp_schedule* sched, const uint64_t* d_words, uint32_t heads,
                               uint32_t q_blocks, uint32_t kv_blocks,
                               const dbsp_local_view* view, int32_t flags, void* stream);
/* Copies the built list to host (32-byte items, u32 entries); diagnostics. */
int dbsp_schedule_download(const dbsp_schedule* sched, void* items_out, uint32_t* entries_out,
                           uint64_t max_entries);
/* Stats of the last build: items, entries (tile visits), dense tiles. */
int dbsp_schedule_stats(const dbsp_schedule* sched, uint64_t* items, uint64_t* tile_visits,
                        uint64_t* dense_tiles);
/* Layout of the last build: DBSP_SCHED_* bits actually used (an AUTO_D128 build
 * reports the layout it resolved to; the 64-row Q blocks per item are 4 with
 * DBSP_SCHED_QUAD, else 2 with DBSP_SCHED_PAIR_Q, else 1). */
int dbsp_schedule_layout(const dbsp_schedule* sched, uint32_t* flags);

/* Uploads the built schedule to the device (async on `stream`); a no-op when
 * it is already resident.  dbsp_attention_launch uploads implicitly. */
int dbsp_schedule_upload(dbsp_schedule* sched, void* stream);
/* Bytes one upload moves host -> device. */
int dbsp_schedule_upload_bytes(const dbsp_schedule* sched, uint64_t* bytes);

typedef struct dbsp_attn_args {
  const void* q;     /* bf16 [q_tokens, heads, d]                             */
  const void* k;     /* bf16 [kv_tokens, heads, d]                            */
  const void* v;     /* bf16 [kv_tokens, heads, d]                            */
  void* o;           /* bf16 [q_tokens, heads, d]                             */
  float* lse;        /* fp32 [heads, q_tokens] natural-log LSE, may be NULL   */
  float* o_accum;    /* fp32 [q_tokens, heads, d] ring accumulator or NULL    */
  float* lse_accum;  /* fp32 [heads, q_tokens] ring accumulator or NULL       */
  uint32_t q_tokens; /* rows in Q/O buffers (local)                           */
  uint32_t kv_tokens;/* rows in K/V buffers (local)                           */
  uint32_t heads;    /* local heads                                           */
  uint32_t head_dim; /* 64 or 128                                             */
  float softmax_scale; /* 0 -> 1/sqrt(head_dim)                               */
  uint32_t accumulate; /* 0: write o/lse; 1: merge into o_accum/lse_accum      */
  uint32_t finalize;   /* with accumulate: also write bf16 o from the merge     */
} dbsp_attn_args;

/* Launches K4 (tcgen05/TMEM/TMA block-sparse FlashAttention forward) for a
 * built schedule on `stream`.  Uploads the schedule asynchronously. */
int dbsp_attention_launch(dbsp_schedule* sched, const dbsp_attn_args* args, void* stream);

/* Fused O return for sequence parallelism: the reverse all-to-all(v) done
 * in K4's epilogue.  Each bf16 output row (local token t, local head h) is
 * stored straight into its home rank's output buffer (a peer pointer over
 * NVLink / NVSwitch, e.g. from CUDA IPC or torch symmetric memory) instead of
 * the local `o`.  Replaces the separate O exchange of the SP path
 * (sp.py step 3); SURVEY.md §8(e) "reverse all-to-allv".  All arrays are
 * device-resident.                                                          */
typedef struct dbsp_out_scatter {
  void* const* out_peers;       /* [ranks] bf16 [home_tokens_r, out_heads, d] */
  const uint32_t* q_block_map;  /* [3 * local Q blocks]: home rank, first home
                                   row, valid rows of that block              */
  const uint32_t* head_map;     /* [local heads] -> global head               */
  uint32_t out_heads;           /* heads of the home buffers (global H)       */
} dbsp_out_scatter;

/* dbsp_attention_launch with the fused O return: writes go to the home
 * buffers (`args->o` is not written; it may be NULL).  The default (pair)
 * schedule and the quad schedules support it. */
int dbsp_attention_launch_scatter(dbsp_schedule* sched, const dbsp_attn_args* args,
                                  const dbsp_out_scatter* scatter, void* stream);

/* Convenience: build + launch for a whole single-GPU problem (identity view). */
int dbsp_sparse_attention(const dbsp_mask_set* set, const dbsp_attn_args* args, void* stream);

/* Kernel launches this library has issued so far in the process (every
 * launch site of its own kernels; CUB's kernels inside K2 are not counted). */
uint64_t dbsp_launch_count(void);

/* Strided host<->device copy (cudaMemcpy2DAsync): moves a head slice of a
 * token-major [tokens, heads, d] tensor, so host-resident layers can stream
 * to the GPU in head chunks that overlap with K4 (see e2e.py). */
int dbsp_copy_2d(void* dst, uint64_t dst_pitch, const void* src, uint64_t src_pitch,
                 uint64_t width, uint64_t rows, int32_t to_device, void* stream);

/* Accumulator init for a ring: o_accum = 0, lse_accum = -inf. */
int dbsp_accum_init(float* o_accum, float* lse_accum, uint32_t q_tokens, uint32_t heads,
                    uint32_t head_dim, void* stream);

/* ------------------------------------------------------------------------ */
/* Sequence-parallel attention call (SpContext +
 * sparse_attention).  One process per GPU; the context owns the NCCL
 * communicator (ncclCommInitRank over `nccl_id`, the ncclUniqueId bytes rank 0
 * obtained from dbsp_nccl_unique_id) and a communication stream.  Home layout:
 * rank g holds token blocks [floor(g*nb/G), floor((g+1)*nb/G)) of Q, K, V, O
 * with all heads, bf16 [home tokens, H, d].  One call = fused all-to-all(v)
 * (Ulysses head scatter + db-SP balancing moves), y ring periods of K4 with the
 * KV exchange on the communication stream, reverse all-to-all(v) of O.       */
typedef struct dbsp_sp_context dbsp_sp_context;
int dbsp_nccl_unique_id(uint8_t* out, uint32_t size /* >= 128 */);
int dbsp_sp_context_create(uint32_t rank, uint32_t world, const uint8_t* nccl_id, dbsp_sp_context** out);
void dbsp_sp_context_destroy(dbsp_sp_context* ctx);
int dbsp_sp_attention(dbsp_sp_context* ctx, const dbsp_mask_set* set, dbsp_strategy strategy,
                      const dbsp_plan* plan, const void* q_home, const void* k_home, const void* v_home,
                      void* o_home, uint32_t tokens, uint32_t head_dim, void* stream);
/* Empty ring groups are allowed: that period exchanges and computes nothing
 * (the accumulator is finalised if it was a rank's last period).
 * Per-period K4 timing of the next calls (CUDA events on the compute stream),
 * read back with dbsp_sp_period_ms (ms[p] for ring period p of the last call;
 * synchronises on those events).                                            */
int dbsp_sp_set_timing(dbsp_sp_context* ctx, int32_t on);
int dbsp_sp_period_ms(dbsp_sp_context* ctx, float* ms, uint32_t cap, uint32_t* n_periods);
/* Waits until the call's work on `stream` and on the context's communication
 * stream has finished, polling ncclCommGetAsyncError.  An asynchronous NCCL
 * error, or no completion within timeout_ms (0 = no limit), aborts the
 * communicator (ncclCommAbort) and returns DBSP_ERR_CUDA; every later call on
 * the context then fails with DBSP_ERR_CUDA.  dbsp_sp_attention also checks
 * the communicator's asynchronous error state on entry.                     */
int dbsp_sp_synchronize(dbsp_sp_context* ctx, void* stream, uint32_t timeout_ms);
/* The same call for all G = x*y ranks on this one GPU, device copies as the
 * transport: *_homes[g] are rank g's home shards.  Tests the multi-rank
 * layouts, packing and ring rotation without a second GPU.                  */
int dbsp_sp_attention_simulated(const dbsp_mask_set* set, dbsp_strategy strategy, const dbsp_plan* plan,
                                const void* const* q_homes, const void* const* k_homes,
                                const void* const* v_homes, void* const* o_homes, uint32_t tokens,
                                uint32_t head_dim, void* stream);

/* ------------------------------------------------------------------------ */
/* K6: QKV projection with the sequence-parallel all-to-all(v) fused into its
 * epilogue.  Y = X W^T (+ bias) on one rank's home
 * tokens, tcgen05 bf16 GEMM with fp32 accumulation; without `scatter` Y is
 * written to `out` [tokens, 3*H*d]; with it every 32-column row segment of Q
 * (K, V) goes straight into the local Q (K, V) buffer of the rank that
 * consumes it under the plan -- the buffers of dbsp_sp_attention's step 1. */
typedef struct dbsp_qkv_args {
  const void* x;     /* bf16 [tokens, hidden] (home tokens)                   */
  const void* w;     /* bf16 [3*heads*head_dim, hidden] (nn.Linear weight)    */
  const void* bias;  /* bf16 [3*heads*head_dim] or NULL                      */
  void* out;         /* bf16 [tokens, 3*heads*head_dim] when not scattering  */
  uint32_t tokens, hidden, heads, head_dim;
} dbsp_qkv_args;
typedef struct dbsp_qkv_scatter {
  void* const* q_peers;       /* [G] device array: rank -> local Q buffer [nq_loc*64, Hu, d]   */
  void* const* k_peers;       /* [G] rank -> local K buffer of its period-0 group              */
  void* const* v_peers;       /* [G]                                                           */
  const uint32_t* block_map;  /* [4 * home blocks]: Q ring rank, Q local block, KV group, KV local block */
  const uint32_t* head_map;   /* [2 * heads]: Ulysses rank u, local head index                 */
  const uint32_t* heads_of;   /* [G]: local head count of each rank                            */
  uint32_t ring;              /* y                                                              */
} dbsp_qkv_scatter;
int dbsp_qkv_project(const dbsp_qkv_args* args, const dbsp_qkv_scatter* scatter /* or NULL */, void* stream);

/* ------------------------------------------------------------------------ */
/* Mask statistics on device (K1).  Masks are device u64
 * words [H][Nq][ceil(Nk/64)].  Outputs are exact integers.                  */
int dbsp_mask_stats_device(const uint64_t* d_words, uint32_t heads, uint32_t nq, uint32_t nk,
                           uint64_t* d_head_counts /* H */, uint64_t* d_row_weights /* Nq */,
                           uint64_t* d_col_weights /* Nk */, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DBSP_B200_H_ */
