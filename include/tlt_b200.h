/*
 * tlt_b200.h — C-ABI of the B200-native adaptive speculative-decoding rollout
 * step (TLT, arXiv 2511.16665). Drop-in for the reference `specsim` hot path:
 * drafter propose -> target verify -> accept -> KV commit -> strategy select.
 *
 * Every entry point replaces a reference C++ symbol; the citation on each
 * declaration names it (paths relative to /root/reference/proj/include/specsim).
 * The reference is header-only C++20 with no ABI, so this header is the first
 * stable boundary: plain pointers and sizes, caller-owned host buffers, an int
 * status code per call (0 = OK) and tlt_last_error() for the message.
 *
 * Error mapping (reference errors.hpp:9-34):
 *   TLT_ERR_CONFIG  <-> specsim::ConfigError   (field path in the message)
 *   TLT_ERR_ROUTING <-> specsim::RoutingError  (beg_mab.hpp:141-143)
 *   TLT_ERR_CUDA    <-> device/runtime failure (no reference analogue)
 *
 * Threading: one engine per GPU, driven by exactly one host thread; calls are
 * not re-entrant on a handle (reference SPEC.md:312 "single-owner" MAB).
 */
#ifndef TLT_B200_H
#define TLT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TLT_API __attribute__((visibility("default")))

enum {
    TLT_OK = 0,
    TLT_ERR_INTERNAL = 1,
    TLT_ERR_CONFIG = 2,
    TLT_ERR_ROUTING = 3,
    TLT_ERR_CUDA = 4,
    TLT_ERR_STATE = 5
};

/* Reference TokenId is int32 (token_model.hpp:18); EOS = 0, BEGIN = 1 (:22-23). */
#define TLT_EOS_TOKEN 0
#define TLT_BEGIN_TOKEN 1

/* Decode modes, reference DecodeMode (spec_decode.hpp:315). */
enum { TLT_MODE_GREEDY_TREE = 0, TLT_MODE_STOCHASTIC_LINEAR = 1 };

/* Reference SpecStrategy (spec_decode.hpp:19-45). */
typedef struct {
    int32_t draft_depth;
    int32_t top_k;
    int32_t tokens_to_verify;
} tlt_strategy;

/* Llama/Qwen-style target + one-layer EAGLE drafter sharing embedding, final
 * norm and LM head. Replaces the Markov target (token_model.hpp:100-156) and
 * the count drafter (drafter.hpp:20-67) as the leaf oracles of the path. */
typedef struct {
    int32_t vocab;
    int32_t hidden;
    int32_t layers;
    int32_t heads;
    int32_t kv_heads;
    int32_t head_dim;
    int32_t ffn;
    int32_t qkv_bias;   /* Qwen2-style q/k/v bias */
    float rope_theta;
    float rms_eps;
    int32_t max_slots;  /* concurrent requests (KV slots) */
    int32_t max_ctx;    /* positions per slot (prompt + response + tree) */
} tlt_model_cfg;

/* Seeded synthetic random-init weights (no checkpoints offline). All values are
 * a counter-based hash of (seed, tensor, index), identical on CPU and GPU. */
typedef struct {
    uint64_t seed;
    float layer_scale; /* std of attention/MLP weights ("structure" knob) */
    float lm_gain;     /* bigram structure of the LM head */
    float lm_alt;      /* relative gain of the second (alternative) successor */
    float lm_noise;    /* unstructured part of the LM head */
    float fc_noise;    /* drafter fc deviation from the embedding passthrough */
    int32_t drafter_lm_fp8; /* 1: the drafter's LM head runs in e4m3 (per-row scales, kind::f8f6f4);
                               the target's stays bf16. 0 = bf16 everywhere (struct padding slot) */
} tlt_init_cfg;

typedef struct tlt_engine tlt_engine;

/* ---- lifecycle ---------------------------------------------------------- */
TLT_API int tlt_engine_create(const tlt_model_cfg* cfg, const tlt_init_cfg* init, int device, tlt_engine** out);
TLT_API void tlt_engine_destroy(tlt_engine* e);
/* Last error message for the engine (or the calling thread when e == NULL). */
TLT_API const char* tlt_last_error(const tlt_engine* e);
TLT_API void tlt_set_last_error(const char* msg);
/* Library build/version string. */
TLT_API const char* tlt_version(void);

/* ---- request state ------------------------------------------------------ */
/* Prefill b requests into KV slots. tokens holds the prompts back to back
 * (lens[i] tokens each, every len >= 1). The last prompt token becomes the
 * step root (its KV is written by the first verify), exactly as the reference
 * context `prompt ++ generated` feeds target_next_dist (token_model.hpp:161). */
TLT_API int tlt_prefill(tlt_engine* e, int b, const int32_t* slot_ids, const int32_t* lens, const int32_t* tokens);
TLT_API int tlt_release(tlt_engine* e, int slot_id);
/* Committed target KV length of a slot (positions 0..len-1 hold KV). */
TLT_API int tlt_slot_len(tlt_engine* e, int slot_id, int32_t* len);
/* C2 (drafter training samples; the reference hands finished
 * sequences to DataBuffer, data_buffer.hpp:48-68): copies a live slot's
 * committed tokens [0, len] (len = tlt_slot_len; token len is the pending
 * root) and its target features [0, len) as bf16 [len][hidden] into caller
 * memory, host or device (cudaMemcpyDefault). Either pointer may be NULL.
 * Call before tlt_release. */
TLT_API int tlt_export_sequence(tlt_engine* e, int slot_id, int32_t* tokens, int max_tokens, void* features,
                                size_t features_bytes, int32_t* len);

/* ---- drafter weights (spot drafter training) ---------- */
/* Device view of one weight tensor: bf16 [rows][cols] row-major. */
typedef struct {
    const char* name;  /* fc, attn_norm, qkv, qkv_bias, o, mlp_norm, gate_up (rows interleaved gate/up), down,
                          embed, final_norm, lm_head */
    void* ptr;         /* device pointer (engine-owned) */
    int64_t rows;
    int64_t cols;
    int32_t trainable; /* 1: the drafter's own (fc + its decoder layer); 0: shared with the target, frozen */
} tlt_tensor_view;
/* Lists the drafter's tensors (the trainer updates trainable ones in place,
 * on any stream, then calls tlt_drafter_published). *n = count. */
TLT_API int tlt_drafter_tensors(tlt_engine* e, tlt_tensor_view* out, int cap, int32_t* n);
/* New drafter weights are in place (reference DrafterSnapshot publish,
 * rollout.hpp:61-64): the drafter KV of live slots is recomputed on their next
 * EAGLE step; `version` is the snapshot's drafter version. */
TLT_API int tlt_drafter_published(tlt_engine* e, int64_t version);
TLT_API int tlt_drafter_version(tlt_engine* e, int64_t* version);
/* FNV-1a-64 (reference checkpoint.hpp:26-33), the drafter checkpoints' trailer. */
TLT_API uint64_t tlt_fnv1a64(const void* data, size_t len);

/* ---- one engine step ---------------------------------------------------- */
/* Tree produced by the drafter, reference DraftTree (spec_decode.hpp:50-70),
 * rank order, parent -1 = root. Caller-owned, sized [b][tokens_to_verify]. */
typedef struct {
    int32_t* tokens;
    int32_t* parents;
    int32_t* depths;
    double* probs;
    double* path_probs;
    int32_t* n_nodes; /* [b] */
} tlt_tree_out;

/* Verify outcome, reference AcceptResult (spec_decode.hpp:74-80) plus the
 * accepted tree indices and the committed KV slot map (new). Sized
 * [b][draft_depth] for accepted / nodes / kv_src, [b] otherwise. */
typedef struct {
    int32_t* accepted;     /* accepted tokens (root-to-node path) */
    int32_t* nodes;        /* accepted tree node indices */
    int32_t* accept_len;   /* reference accept_length */
    int32_t* bonus;        /* reference bonus */
    int32_t* kv_src;       /* committed KV: slot L+1+j <- L+1+kv_src[j] (tree slot) */
    int32_t* kv_len;       /* committed target KV length after the step */
    float* elapsed_ms;     /* [1] device time of the step (CUDA events) */
} tlt_accept_out;

/* Greedy tree SD step: build_draft_tree (spec_decode.hpp:111-197) with the
 * EAGLE drafter, one tree-masked target verify forward, verify_greedy
 * (:245-268), KV compaction. The whole step replays one CUDA graph keyed on
 * (batch bucket, strategy) when a pool is built. `tree` may be NULL. */
TLT_API int tlt_sd_step(tlt_engine* e, const tlt_strategy* s, int b, const int32_t* slot_ids, tlt_tree_out* tree,
                        tlt_accept_out* out);
/* ---- split boundary: propose and verify as separate calls ---------------- */
/* The reference's drafter seam is DraftPlanner (spec_decode.hpp:319-341),
 * a (ctx, strategy, rng) -> DraftTree function consumed by spec_generate,
 * and its target side is verify_greedy(target, ctx, tree) (:245-268). These
 * two calls back that seam; tlt_sd_step is their fused, graph-replayed form.
 *
 * tlt_draft: build_draft_tree (spec_decode.hpp:111-197) with the EAGLE
 * drafter for each request; writes the tree (rank order, parent -1 = root)
 * and commits nothing to the target (the drafter's own KV of the committed
 * positions is written; drafting twice is idempotent). */
TLT_API int tlt_draft(tlt_engine* e, const tlt_strategy* s, int b, const int32_t* slot_ids, tlt_tree_out* tree);
/* A caller-supplied tree (reference DraftTree, spec_decode.hpp:50-70) per
 * request: nodes in rank order, each parent index < its own (-1 = root).
 * Arrays are [b][stride]; probs / path_probs may be NULL (reported as 1). */
typedef struct {
    const int32_t* tokens;
    const int32_t* parents;
    const double* probs;
    const double* path_probs;
    const int32_t* n_nodes; /* [b], 0 <= n <= stride */
    int32_t stride;         /* <= 128 nodes per request, depth <= 15 */
} tlt_tree_in;
/* verify_greedy (spec_decode.hpp:245-268) of one tree per request in one
 * tree-masked target forward, then the KV commit of the accepted branch.
 * tree == NULL verifies the engine's own last tlt_draft of exactly these
 * slots (device-resident, no upload); otherwise the host tree is uploaded.
 * `out` arrays are [b][stride] (stride = tree->stride, or the drafted
 * strategy's draft_depth when tree == NULL). */
TLT_API int tlt_verify_accept_commit(tlt_engine* e, int b, const int32_t* slot_ids, const tlt_tree_in* tree,
                                     tlt_accept_out* out);

/* Stochastic linear-chain SD step: build_sampled_chain (:202-223) +
 * verify_stochastic (:275-313), temperature t > 0. Uniforms are the
 * reference RngStream draws (rng.hpp:54-56), host-generated per request in
 * consumption order (draft_depth chain draws, then accept draws, then one
 * residual/bonus draw); `uniforms` is [b][2*draft_depth+1]. */
TLT_API int tlt_sd_step_stochastic(tlt_engine* e, int draft_depth, float temperature, int b,
                                   const int32_t* slot_ids, const double* uniforms, tlt_accept_out* out);
/* Greedy verify of host-proposed linear chains (the model-free n-gram
 * branch of run_rollout, rollout.hpp:212-216): chain_from_tokens
 * (spec_decode.hpp:228-240) of chains[i*draft_depth .. +chain_lens[i]]
 * (0 <= len <= draft_depth; an empty chain is a plain step emitting the
 * bonus), then the same tree-masked target verify, verify_greedy and KV
 * compaction as tlt_sd_step. The drafter does not run. */
TLT_API int tlt_sd_step_chain(tlt_engine* e, int draft_depth, int b, const int32_t* slot_ids, const int32_t* chains,
                              const int32_t* chain_lens, tlt_accept_out* out);
/* Stochastic mode of the same branch: verify_stochastic (spec_decode.hpp:
 * 275-313) of host chains with an empty draft_dist (q one-hot at the drafted
 * token), temperature t > 0. uniforms: [b][draft_depth+1] RngStream draws in
 * consumption order (one per tested node, then one residual/bonus draw);
 * tlt_debug_chain reports how many each request consumed. */
TLT_API int tlt_sd_step_chain_stochastic(tlt_engine* e, int draft_depth, float temperature, int b,
                                         const int32_t* slot_ids, const int32_t* chains, const int32_t* chain_lens,
                                         const double* uniforms, tlt_accept_out* out);
/* Plain autoregressive step (the 2x denominator): reference plain branch
 * (rollout.hpp:247-261) / generate_autoregressive (token_model.hpp:190-203). */
TLT_API int tlt_ar_step(tlt_engine* e, int b, const int32_t* slot_ids, int32_t* out_tokens, float* elapsed_ms);

/* ---- CUDA-graph pool ---------------------------------------------------- */
/* One entry per reference CaptureEntry (capture_plan.hpp:25-33): side 0 =
 * TARGET(bucket, tokens_to_verify), 1 = DRAFT(bucket, top_k, draft_depth). */
typedef struct {
    int32_t side;
    int32_t bucket_lo;
    int32_t bucket_hi;
    int32_t tokens_to_verify;
    int32_t top_k;
    int32_t draft_depth;
    double memory_units;
} tlt_capture_entry;
/* Pre-captures the pool (replaces any existing graphs): for every bucket
 * [lo, hi] of the entries, one fused step graph per TARGET(T) x DRAFT(k, D)
 * pair whose strategy is valid, captured at batch hi and replayed for any
 * batch in the bucket (padding requests inert, their GEMM token tiles
 * skipped on the device); plus plain-decode graphs at padded batch sizes
 * 1, 2, 4, 8, 16, 24, ... max_slots. An SD step whose (batch, strategy) is
 * outside the pool falls back to an exact-batch graph captured on first use.
 * graph_bytes = device memory the pool took (cudaMemGetInfo delta; all
 * graphs share the engine's activation buffers). */
TLT_API int tlt_graph_pool_build(tlt_engine* e, const tlt_capture_entry* entries, int n, size_t* graph_bytes);
/* Granularity of the next tlt_graph_pool_build: sub_bucket_width 0 = one
 * graph per plan bucket (the paper's plan: a step at batch b replays the
 * graph of its bucket's largest batch); w > 0 = every plan bucket cut into
 * sub-buckets of <= w batch sizes, same strategies (less padding, more
 * graphs; w = 1 is one graph per batch size). ar_width: plain-decode graph
 * sizes, 0 = 1, 2, 4, 8, 16, 24, ..., w > 0 = every w-th size. */
TLT_API int tlt_graph_pool_configure(tlt_engine* e, int sub_bucket_width, int ar_width);
/* Last pool build: graphs captured, plan pairs skipped (draft rows beyond
 * the engine buffers at that bucket size), bytes, host build time, and the
 * number of executable graphs the engine holds now (pool + on-demand). */
TLT_API int tlt_graph_pool_stats(tlt_engine* e, int32_t* n_graphs, int32_t* n_skipped, size_t* graph_bytes,
                                 double* build_ms, int32_t* n_live);
/* Destroys every graph and forgets the pool's buckets (exact-batch graphs
 * are captured on demand again). */
TLT_API int tlt_graph_pool_clear(tlt_engine* e);

/* ---- strategy selection (host, reference semantics) ---------------------- */
/* BEG-MAB, reference beg_mab.hpp:28-170. Opaque single-owner state. */
typedef struct tlt_mab tlt_mab;
TLT_API int tlt_mab_create(const tlt_strategy* strategies, int n, const int32_t* thresholds, int n_thr,
                           double epsilon, int window, tlt_mab** out);
TLT_API void tlt_mab_destroy(tlt_mab* m);
/* beg_select (beg_mab.hpp:140-170). rng_state is the caller's RngStream
 * (mt19937_64 state handle, see tlt_rng_*). Writes the picked arm index. */
typedef struct tlt_rng tlt_rng;
TLT_API int tlt_mab_select(tlt_mab* m, int batch, tlt_rng* rng, int32_t* arm, tlt_strategy* out);
/* beg_record (beg_mab.hpp:111-134). */
TLT_API int tlt_mab_record(tlt_mab* m, const tlt_strategy* s, double elapsed, const int32_t* accept_lens, int batch);
/* Window medians/selection counts per arm (beg_state_to_json, :174-193). */
TLT_API int tlt_mab_arm_stats(tlt_mab* m, int arm, double* median_reward, int64_t* selections, int32_t* n_rewards);
/* Reward / accept-length window of one arm, oldest first (the arrays of
 * beg_state_to_json, beg_mab.hpp:174-193); *n = window fill. */
TLT_API int tlt_mab_arm_window(tlt_mab* m, int arm, double* rewards, double* accept_lens, int cap, int32_t* n);
/* Multi-GPU merge (C1): apply one foreign rank's record to this replica. */
TLT_API int tlt_mab_apply_record(tlt_mab* m, int arm, double reward, double a_bar);
/* C1 (cross-rank bandit statistics): return and clear the records this
 * replica's beg_record logged since the last call (records applied through
 * tlt_mab_apply_record are not logged). */
TLT_API int tlt_mab_take_log(tlt_mab* m, int32_t* arm, double* reward, double* a_bar, int cap, int32_t* n);
/* C1 inside the library: after a rollout every rank's new beg_record
 * records (tlt_mab_take_log) go into a fixed-size block (count + max_records
 * x {arm, reward, a_bar}), the blocks are all-gathered and applied to
 * `shared` in rank order (bit-identical on every rank; with one rank exactly
 * the local beg_record sequence), and `local` restarts from `shared`.
 * Transport: NCCL (an engine-device communicator on its own side stream;
 * rank 0 makes the id with tlt_c1_nccl_unique_id, the host distributes it),
 * or a host all-gather callback: gather `bytes` from every rank into
 * recv[world][bytes] in rank order, return 0 on success. */
typedef struct tlt_c1 tlt_c1;
typedef int (*tlt_allgather_fn)(void* user, const void* send, void* recv, size_t bytes);
TLT_API int tlt_c1_nccl_unique_id(void* id128);
TLT_API int tlt_c1_create_nccl(tlt_engine* e, const void* id128, int world, int rank, int max_records, tlt_c1** out);
TLT_API int tlt_c1_create_callback(int world, int rank, tlt_allgather_fn fn, void* user, int max_records,
                                   tlt_c1** out);
TLT_API int tlt_c1_merge(tlt_c1* c, tlt_mab* local, tlt_mab* shared, int32_t* n_merged);
TLT_API void tlt_c1_destroy(tlt_c1* c);
/* Copy the full bandit state (windows, selection counts) of src into dst. */
TLT_API int tlt_mab_copy(tlt_mab* dst, const tlt_mab* src);
/* Deterministic streams, reference RngStream (rng.hpp:34-86). */
TLT_API int tlt_rng_create(uint64_t seed, uint64_t stream_id, tlt_rng** out);
TLT_API int tlt_rng_fork(const tlt_rng* r, uint64_t label, tlt_rng** out);
TLT_API void tlt_rng_destroy(tlt_rng* r);
/* RngStream::seed() / stream_id() (rng.hpp:43-44): a forked stream is the
 * pair (seed, stream_id), e.g. to hand it to tlt_rollout_cfg. */
TLT_API int tlt_rng_ids(const tlt_rng* r, uint64_t* seed, uint64_t* stream_id);
TLT_API uint64_t tlt_rng_next_u64(tlt_rng* r);
TLT_API double tlt_rng_uniform01(tlt_rng* r);

/* Model-free n-gram drafter, reference NgramIndex / ngram_insert /
 * ngram_draft (ngram.hpp:13-103) and the per-request NgramTracker cursor
 * (rollout.hpp:103-120). Opaque single-owner state. */
typedef struct tlt_ngram tlt_ngram;
TLT_API int tlt_ngram_create(int n, int continuation_len, tlt_ngram** out);
TLT_API void tlt_ngram_destroy(tlt_ngram* g);
/* ngram_insert (ngram.hpp:62-78): every n-gram of the response. */
TLT_API int tlt_ngram_insert(tlt_ngram* g, const int32_t* response, int len, int64_t step_id);
/* NgramTracker::extend (rollout.hpp:107-118): complete windows of the stream
 * from the tracker cursor on. */
TLT_API int tlt_ngram_extend(tlt_ngram* g, const int32_t* stream, int len, int64_t step_id);
/* ngram_draft (ngram.hpp:83-101): writes up to depth tokens, *out_len = count. */
TLT_API int tlt_ngram_draft(const tlt_ngram* g, const int32_t* ctx, int len, int depth, int32_t* out, int32_t* out_len);
/* Number of stored (key, continuation) entries (NgramIndex::size, :34-38). */
TLT_API int tlt_ngram_size(const tlt_ngram* g, int64_t* size);

/* plan_captures (capture_plan.hpp:87-126) with BucketSpec (:42-45). Writes up
 * to max_entries entries; *n_entries = number produced. vanilla != 0 gives
 * plan_captures_vanilla (:130-155). */
TLT_API int tlt_plan_captures(const tlt_strategy* strategies, int n, const int32_t* thresholds, int n_thr,
                              int max_batch, int vanilla, tlt_capture_entry* out, int max_entries, int* n_entries,
                              double* total_memory_units);

/* ---- rollout (the step loop's caller, reference run_rollout) ------------- */
/* Reference CostModelParams (cost_model.hpp:16-33), abstract time units. */
typedef struct {
    double t_launch;
    double model_bytes;
    double mem_bw;
    double flops_per_token;
    double peak_flops;
    double drafter_step_cost;
} tlt_cost_model;
/* step_latency (cost_model.hpp:38-48); sd == NULL is a plain decode step. */
TLT_API int tlt_step_latency(const tlt_cost_model* cost, int batch, int tokens_per_request, const tlt_strategy* sd,
                             double* out);

/* Reference StepMetrics (rollout.hpp:31-38), one per engine step. The step's
 * accept_lens are trace_accept_lens[accept_off .. accept_off + n_accept). */
typedef struct {
    int32_t step_index;
    int32_t batch_size;
    int32_t sd_active;
    int32_t has_strategy;
    tlt_strategy strategy;
    double elapsed;    /* what beg_record saw: device ms, or step_latency units (parity_elapsed) */
    double device_ms;  /* measured device time of the step (CUDA events) */
    int64_t accept_off;
    int32_t n_accept;
    int32_t via_ngram; /* the step drafted with the model-free n-gram tracker */
} tlt_step_metrics;
/* Reference RolloutConfig (rollout.hpp:66-77) subset on the GPU path. */
typedef struct {
    int32_t enable_sd;
    int32_t elastic_threshold; /* should_enable_sd (rollout.hpp:54-57) */
    int32_t mode;              /* TLT_MODE_* */
    float temperature;         /* stochastic mode only */
    tlt_strategy fixed_strategy;
    int32_t use_mab;           /* 1: BEG-MAB select/record with measured elapsed */
    uint64_t seed;             /* RngStream seed of the rollout (fork labels as rollout.hpp:151,153) */
    int32_t use_graphs;        /* replay the CUDA-graph pool */
    /* Drafter freshness (rollout.hpp:142-144, 209-216): 0 = the EAGLE snapshot
     * is fresh (target step - snapshot step <= drafter_staleness_bound); 1 =
     * stale or absent, SD steps draft with the per-request model-free n-gram
     * tracker instead (greedy mode). Zero-initialised callers keep EAGLE. */
    int32_t drafter_stale;
    int32_t ngram_n;                /* reference default 2 */
    int32_t ngram_continuation_len; /* reference default 8 */
    int64_t target_step_id;         /* recency stamp of n-gram records (target.step_id()) */
    /* Deterministic elapsed (reference step_latency, cost_model.hpp:38-48):
     * 0 = each step's elapsed is its measured device time in ms (CUDA
     * events; the product setting), 1 = elapsed = step_latency(cost, batch,
     * T or 1, strategy or none) in cost-model units, exactly as the
     * reference run_rollout computes it (rollout.hpp:242,258), so a BEG-MAB
     * rollout replays the reference's arm sequence bit for bit. */
    int32_t parity_elapsed;
    /* 1: finished requests keep their KV slot live (slot i) after the call,
     * so the caller can tlt_export_sequence (C2) them before tlt_release;
     * 0: slots are released as requests finish. */
    int32_t keep_finished;
    tlt_cost_model cost;            /* all zero = reference defaults (cost_model.hpp:16-22) */
    /* The rollout's RngStream is (seed, rng_stream) (rng.hpp:37-41): 0 = the
     * root stream of `seed`; a caller passing rng.fork(label) hands over that
     * fork's stream_id (tlt_rng_ids). Request / select forks as rollout.hpp:151,153. */
    uint64_t rng_stream;
} tlt_rollout_cfg;

/* Reference RolloutResult (rollout.hpp:79-97) flattened. generated: [n][max_len]. */
typedef struct {
    int32_t* generated;     /* [n][max_len_stride] */
    int32_t* gen_len;       /* [n] */
    int64_t sd_steps;
    int64_t plain_steps;
    int64_t verify_events;
    int64_t accepted_total; /* sum of accept_len over verify events (mean_accept_len numerator) */
    int64_t emitted_total;  /* tokens appended (accepted + bonus, truncated) */
    double device_ms;       /* sum of per-step device time */
    double wall_ms;         /* host wall time of the whole rollout */
    int64_t gpu_launches;   /* kernel launches issued (graph nodes counted) */
    /* --- the rest of reference RolloutResult (rollout.hpp:79-97); every
     * pointer below is caller-owned and may be NULL --- */
    double total_time;            /* sum of step elapsed (rollout.hpp:263) */
    int64_t ngram_verify_events;  /* verify events drafted by the n-gram tracker (:226) */
    int64_t* accept_at_least;     /* [accept_at_least_cap]: [i] = events with accept_len > i (:227-229) */
    int32_t accept_at_least_cap;
    int32_t accept_at_least_len;  /* out: max draft depth (reference vector size) */
    double* finish_time;          /* [n]: total_time when request i finished (:264-268) */
    tlt_step_metrics* trace;      /* [trace_cap] (:270) */
    int64_t trace_cap;
    int64_t trace_len;            /* out: engine steps (entries beyond trace_cap are counted, not stored) */
    int32_t* trace_accept_lens;   /* [trace_accept_cap] concatenated per-step accept_lens */
    int64_t trace_accept_cap;
} tlt_rollout_result;

/* Runs n requests (prompts back to back, max_len per request) to completion
 * through prefill + the SD/AR step loop (rollout.hpp:130-276). mab may be NULL
 * when cfg->use_mab == 0. */
TLT_API int tlt_run_rollout(tlt_engine* e, const tlt_rollout_cfg* cfg, tlt_mab* mab, int n, const int32_t* request_ids,
                            const int32_t* prompt_lens, const int32_t* prompts, const int32_t* max_lens,
                            int max_len_stride, tlt_rollout_result* out);

/* ---- parity / debug exports (tests only) -------------------------------- */
/* After the last tlt_sd_step: per-request drafter expansion rows. For request
 * i, expansion e: the path from the root (tokens, up to draft_depth) and the
 * full fp64 drafter distribution used by the tree (vocab entries).
 * Enabled by tlt_set_debug(e, 1) before the step (graphs bypassed). */
TLT_API int tlt_set_debug(tlt_engine* e, int on);
TLT_API int tlt_debug_expansions(tlt_engine* e, int i, int max_exp, int32_t* n_exp, int32_t* path_len,
                                 int32_t* paths /* [max_exp][depth] */, double* rows /* [max_exp][V] */);
/* Target logits (fp32) of the verify rows of request i: [T+1][V], row 0 = root. */
TLT_API int tlt_debug_verify_logits(tlt_engine* e, int i, float* logits, int max_rows, int32_t* n_rows);
/* Drafted chain of request i in the last tlt_sd_step_stochastic and the
 * number of uniforms it consumed (draft_depth + examined positions + 1). */
TLT_API int tlt_debug_chain(tlt_engine* e, int i, int32_t* chain, int32_t* n, int32_t* consumed);
/* Raw (untempered) target rows, fp64, of the root + chain of request i in the
 * last stochastic step: [D+1][V], computed by the accept kernel's code. */
TLT_API int tlt_debug_target_rows(tlt_engine* e, int i, double* rows, int max_rows, int32_t* n_rows);
/* Target logits of the last tlt_ar_step: [b][V]. */
TLT_API int tlt_debug_ar_logits(tlt_engine* e, float* logits, int b);

/* Live timing of one of the engine's own GEMM sites on its stream with its
 * own weights (successive layers, so every launch streams fresh weights):
 * kind 0 gate_up+SwiGLU, 1 qkv (+RoPE, KV write), 2 down (+residual),
 * 3 LM head fp32 logits, 4 LM head + fused top-1, 5 o-proj (+residual),
 * 6 drafter LM head. Reports the average launch duration (best of 5 timed
 * passes of `iters` launches) and the algorithmic bytes / flops of one launch. */
TLT_API int tlt_probe_kernel(tlt_engine* e, int kind, int m_tok, int iters, float* avg_ms, double* bytes,
                             double* flops);

/* Live timing of the engine's attention (flash-decode + split combine) on
 * its stream over successive layers' caches: b requests x ctx committed keys
 * x rows_per_req query rows (1 = plain decode, T+1 = tree verify). Reports
 * the average per-layer duration (graph replay, best of 5) and the
 * algorithmic bytes (K/V read + q/out). */
TLT_API int tlt_probe_attention(tlt_engine* e, int b, int ctx, int rows_per_req, int iters, float* avg_ms,
                                double* bytes);

/* ---- kernel-level entry points for unit tests ---------------------------- */
/* Y = X W^T through the tcgen05 GEMM. kind: 0 f32 store, 1 bf16 store,
 * 3 SwiGLU (W rows interleaved gate/up). Returns the split-K factor used. */
TLT_API int tlt_dev_gemm(const void* x, int m, int k, const void* w, int n, int kind, float* y_f32, void* y_bf16,
                         float* ws, long long ws_elems, int max_splits);
/* tlt_dev_gemm with a device-resident live-row count (the graph pool's
 * padding-tile skip, EpiParams::dyn_n): rows >= *live_rows may stay unwritten. */
TLT_API int tlt_dev_gemm_live(const void* x, int m, int k, const void* w, int n, int kind, float* y_f32,
                              void* y_bf16, float* ws, long long ws_elems, const int* live_rows);
/* Average device ms of one GEMM launch over `iters` back-to-back launches
 * (CUDA events on a private stream). Returns the split-K factor. */
TLT_API int tlt_dev_time_gemm(const void* x, int m, int k, const void* w, int n, int kind, float* y_f32,
                              void* y_bf16, float* ws, long long ws_elems, int iters, float* avg_ms);
/* LM head with the fused top-k epilogue: per row the top-k of x W^T by
 * (logit desc, id asc), M = max and S = sum exp(l - M), without materialising
 * the logits (part: [ceil(n/128)][m][2+2k] floats of scratch; thr: null or m
 * zeroed uints for the per-row k-th-value bounds, zeroed again on return).
 * Returns >= 1. */
TLT_API int tlt_dev_lm_topk(const void* x, int m, int k, const void* w, int n, int topk, float* part, int* out_tok,
                            float* out_logit, float* out_M, float* out_S, unsigned* thr);
/* Row top-k by (logit desc, id asc) + row max M and S = sum exp(l - M) over
 * fp32 logits [R][V] (the drafter child selection); `part` is scratch of
 * [ceil(V/128)][R][2+2k] floats. Average ms over `iters` launches. Returns the
 * number of chunks per row. */
TLT_API int tlt_dev_row_topk(const float* logits, int R, int V, int k, float* part, int* out_tok, float* out_logit,
                             float* out_M, float* out_S, int iters, float* avg_ms);
/* e4m3 GEMM (kind::f8f6f4) through the production path: x [m][k] and w [n][k]
 * bf16 quantised per row (scale = amax/448), y = (qx qw^T) * sx[t] * sw[n]
 * fp32; the quantised operands / scales are returned for the reference. */
TLT_API int tlt_dev_gemm_e4m3(const void* x, int m, int k, const void* w, int n, float* y, void* qx, float* sx,
                              void* qw, float* sw);
/* Tree-masked attention over explicit device buffers (q [R][H*hd], K/V
 * caches [slots][KV][cap][hd] bf16, row slots / 1024-bit tail masks, group
 * slot / committed length / tail start / tail length): kernel 0 = mma.sync
 * kernels, 1 = tcgen05 + TMEM kernel. Writes out [R][H*hd] bf16. */
TLT_API int tlt_dev_attention(const void* q, const void* kc, const void* vc, void* out, int n_groups,
                              int rows_per_req, int H, int KV, int hd, int cap, const int* row_slot,
                              const unsigned* row_mask, const int* g_slot, const int* g_lc, const int* g_tail0,
                              const int* g_ntail, int max_keys, int kernel);

#ifdef __cplusplus
}
#endif
#endif /* TLT_B200_H */
