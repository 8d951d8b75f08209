/*
 * tlt_oracle.h — CPU restatement of the reference hot path (TEST INFRASTRUCTURE).
 *
 * This library is the checker, never the product: only tests/, the smoke()
 * entry and bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Two halves:
 *  1. Discrete semantics restated in plain C from the reference specsim
 *     headers (/root/reference/proj/include/specsim): RngStream, argmax /
 *     inverse-CDF / tempering, build_draft_tree, build_sampled_chain,
 *     verify_greedy, verify_stochastic, spec_generate, BEG-MAB, capture plan,
 *     elastic gate. Each function cites the reference file:line it follows and
 *     is PINNED against the reference itself (oracle/_ref, compiled in place
 *     from /root/reference by oracle/Makefile) in tests/test_oracle_pinning.py,
 *     and against golden vectors in tests/golden/.
 *  2. The neural leaf oracles the reference does not contain:
 *     a Llama/Qwen-style target and a one-layer EAGLE drafter with the same
 *     weights (counter-hash init), bf16 rounding points and RoPE table as the
 *     GPU engine, fp32 accumulation. Logit parity with the GPU is a stated
 *     tolerance; that half is "parity unpinned" by any reference test.
 */
#ifndef TLT_ORACLE_H
#define TLT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- RNG ---- */
/* rng.hpp:34-86: std::mt19937_64 seeded through SplitMix64. */
typedef struct {
    uint64_t mt[312];
    int mti;
    uint64_t seed;
    uint64_t stream_id;
} orc_rng;

void orc_rng_init(orc_rng* r, uint64_t seed, uint64_t stream_id);
void orc_rng_fork(const orc_rng* r, uint64_t label, orc_rng* out);
uint64_t orc_rng_next_u64(orc_rng* r);
double orc_rng_uniform01(orc_rng* r);
uint64_t orc_rng_uniform_int(orc_rng* r, uint64_t n);
double orc_rng_normal(orc_rng* r);
size_t orc_rng_sizeof(void);

/* Uniform source: the RngStream itself, or a pre-drawn buffer with a cursor
 * (the GPU path consumes host-uploaded draws in the same order). */
typedef struct {
    orc_rng* rng;
    const double* buf;
    int n;
    int cursor;
} orc_usrc;
double orc_usrc_next(orc_usrc* s);

/* --------------------------------------------------- distributions ---- */
int32_t orc_argmax(const double* p, int v);                      /* token_model.hpp:44-50 */
int32_t orc_inverse_cdf_pick(const double* p, int v, double u);  /* token_model.hpp:83-91 */
/* target_next_dist tempering (token_model.hpp:161-173) of a raw row. */
void orc_temper(const double* raw, int v, double t, double* out);

/* ---------------------------------------------------------- strategy ---- */
typedef struct {
    int32_t draft_depth;
    int32_t top_k;
    int32_t tokens_to_verify;
} orc_strategy;
int64_t orc_max_tree_nodes(const orc_strategy* s); /* spec_decode.hpp:25-34 */
/* spec_decode.hpp:36-42. Returns 0 ok, else writes the failing field. */
int orc_strategy_validate(const orc_strategy* s, const char** field);

/* ------------------------------------------------------------- tree ---- */
typedef struct {
    int32_t token;
    int32_t parent;
    int32_t depth;
    double prob;
    double path_prob;
} orc_node;

/* Drafter / target seam (reference NextDist, spec_decode.hpp:111-113): fill
 * out[V] with the distribution after ctx ++ path. Return 0 on success. */
typedef int (*orc_row_fn)(void* user, const int32_t* path, int path_len, double* out);

/* build_draft_tree (spec_decode.hpp:111-197). Writes <= T nodes in rank
 * order; returns the node count (or -1 on invalid strategy / callback error).
 * Optional trace: the path of every expanded node in expansion order. */
int orc_build_draft_tree(orc_row_fn f, void* user, int vocab, const orc_strategy* s, orc_node* out);

/* verify_greedy (spec_decode.hpp:245-268) with the target's raw-row argmax
 * supplied per path (argmax_fn returns the token or < 0 on error). */
typedef int32_t (*orc_argmax_fn)(void* user, const int32_t* path, int path_len);
typedef struct {
    int32_t accepted[256];
    int32_t nodes[256];
    int32_t accept_length;
    int32_t bonus;
} orc_accept;
int orc_verify_greedy(orc_argmax_fn f, void* user, const orc_node* tree, int n_nodes, orc_accept* out);

/* build_sampled_chain (spec_decode.hpp:202-223): draft_dists [depth][V]. */
int orc_build_sampled_chain(orc_row_fn f, void* user, int vocab, int depth, orc_usrc* u, orc_node* out,
                            double* draft_dists);
/* verify_stochastic (spec_decode.hpp:275-313). target_fn returns the raw
 * (untempered) row, tempered here with temperature t (target_next_dist).
 * draft_dists may be NULL (one-hot proposals, chain_from_tokens). */
int orc_verify_stochastic(orc_row_fn target_fn, void* user, int vocab, double t, const orc_node* chain,
                          int n, const double* draft_dists, orc_usrc* u, orc_accept* out);

/* ------------------------------------------------------------ BEG-MAB ---- */
#define ORC_MAB_MAX_ARMS 64
#define ORC_MAB_MAX_WIN 256
typedef struct {
    orc_strategy strategy;
    double rewards[ORC_MAB_MAX_WIN];
    double accept_lens[ORC_MAB_MAX_WIN];
    int n; /* window fill (rewards and accept_lens move together) */
    int64_t selections;
} orc_arm;
typedef struct {
    orc_arm arms[ORC_MAB_MAX_ARMS];
    int n_arms;
    int thresholds[32];
    int n_thr;
    int groups[32][ORC_MAB_MAX_ARMS];
    int group_size[32];
    double epsilon;
    int window;
} orc_mab;
size_t orc_mab_sizeof(void);
/* beg_initialize (beg_mab.hpp:74-106). 0 ok, -1 config error. */
int orc_mab_init(orc_mab* m, const orc_strategy* s, int n, const int* thr, int n_thr, double eps, int window);
/* beg_record (beg_mab.hpp:111-134). */
int orc_mab_record(orc_mab* m, const orc_strategy* s, double elapsed, const int32_t* accept_lens, int batch);
/* beg_select (beg_mab.hpp:140-170). Returns the arm index, -2 routing error. */
int orc_mab_select(orc_mab* m, int batch, orc_rng* rng);
double orc_median(const double* v, int n); /* beg_mab.hpp:47-54 */
int orc_mab_arm_stats(const orc_mab* m, int arm, double* median_reward, int64_t* selections, int* n,
                      double* last_reward, double* last_accept);

/* ------------------------------------------------------- capture plan ---- */
typedef struct {
    int32_t side; /* 0 TARGET, 1 DRAFT */
    int32_t bucket_lo, bucket_hi, tokens_to_verify, top_k, draft_depth;
    double memory_units;
} orc_capture;
/* plan_captures (capture_plan.hpp:87-126) / plan_captures_vanilla (:130-155). */
int orc_plan_captures(const orc_strategy* s, int n, const int* thr, int n_thr, int max_batch, int vanilla,
                      orc_capture* out, int max_out, double* total_units);

/* ------------------------------------------------------- rollout bits ---- */
int orc_should_enable_sd(int active, int threshold); /* rollout.hpp:54-57; -1 on bad threshold */
/* step_latency (cost_model.hpp:38-48), default CostModelParams (:16-33). */
double orc_step_latency(int batch, int tokens_per_request, const orc_strategy* sd_or_null);

/* spec_generate (spec_decode.hpp:351-380) over callback seams. planner builds
 * a tree for ctx ++ generated (mode 0 greedy tree, 1 stochastic chain). */
typedef struct {
    orc_row_fn draft_fn;   /* drafter NextDist over (prompt ++ generated ++ path) */
    orc_row_fn target_fn;  /* raw target row over (prompt ++ generated ++ path) */
    void* user;            /* receives the full context through orc_ctx_* below */
} orc_seams;

/* ========================================================= neural oracle ==
 * Model + weight initialization (identical to the GPU engine). */
typedef struct {
    int vocab, hidden, layers, heads, kv_heads, head_dim, ffn, qkv_bias;
    float rope_theta, rms_eps;
    int max_ctx;
} orc_model_cfg;
typedef struct {
    uint64_t seed;
    float layer_scale, lm_gain, lm_alt, lm_noise, fc_noise;
    /* 1: the drafter's LM head in e4m3 as the engine runs it (tlt_init_cfg.
     * drafter_lm_fp8): per-row scale amax/448, RNE saturating e4m3 of the
     * weight rows and of the normed drafter row, fp32 dot product, logits x
     * (row scale x token scale). The target's LM head stays bf16. */
    int32_t drafter_lm_fp8;
} orc_init_cfg;

typedef struct orc_model orc_model;
orc_model* orc_model_create(const orc_model_cfg* cfg, const orc_init_cfg* init, int n_threads);
void orc_model_set_threads(orc_model* m, int n_threads);
void orc_model_destroy(orc_model* m);
/* Raw bf16 bits of a named weight (test access): tensor ids as in DESIGN.md. */
int orc_model_weight(orc_model* m, int tensor_id, int layer, const uint16_t** ptr, int64_t* n);
/* The counter-hash init value of element idx of tensor (tensor_id, layer). */
uint16_t orc_init_value(const orc_init_cfg* init, const orc_model_cfg* cfg, int tensor_id, int layer, int64_t idx);
/* e4m3 quantisation of one row as the engine's k_quant_rows_e4m3: scale =
 * amax / 448 (1 for an all-zero row), q[i] = the e4m3 value (RNE,
 * saturating) of x[i] / scale, returned as a float. Returns the scale. */
float orc_e4m3_quant_row(const float* x, int n, float* q);

/* Per-request decoding state: target KV (all layers), drafter KV, feature
 * history. */
typedef struct orc_seq orc_seq;
orc_seq* orc_seq_create(orc_model* m);
void orc_seq_destroy(orc_seq* s);
/* Feed committed tokens through the target (positions len..len+n-1); writes
 * fp32 logits of the last row when logits != NULL. Features are recorded. */
int orc_target_extend(orc_seq* s, const int32_t* toks, int n, float* logits_last);
int orc_seq_len(orc_seq* s);
int orc_seq_append(orc_seq* s, const int32_t* toks, int n);
/* Logits after (committed ++ path) without committing (path may be empty:
 * then the committed last row). Used for tree verify rows. */
int orc_target_logits_path(orc_seq* s, const int32_t* path, int n, float* logits);
/* Drafter: commit drafter KV for committed positions not yet processed (uses
 * target features), then the distribution of the next token after
 * committed ++ path, with EAGLE self-feeding along path. fp64 softmax. */
int orc_drafter_row(orc_seq* s, const int32_t* path, int n, double* probs, float* logits);
/* Target hidden states (final residual stream, bf16 bits) of committed
 * positions [from, from + n): the drafter's input features. */
int orc_seq_features(orc_seq* s, int from, int n, uint16_t* out);
/* Truncate the committed state (target and drafter) to len tokens. */
int orc_seq_truncate(orc_seq* s, int len);

/* Greedy tree SD generate on the neural model: reference spec_generate
 * (spec_decode.hpp:351-380) with build_draft_tree over the EAGLE drafter and
 * verify_greedy over the target. Outputs generated tokens, per-step accept
 * lengths and (optionally) the trees [steps][T] nodes. Returns #steps. */
int orc_neural_spec_generate(orc_model* m, const int32_t* prompt, int prompt_len, int max_len,
                             const orc_strategy* s, int32_t* out_tokens, int* out_len, int32_t* accept_lens,
                             orc_node* trees, int32_t* tree_sizes, int max_steps);
/* Rejection-sampling SD generate (StochasticLinear), uniforms from
 * RngStream(seed, stream) in reference consumption order. */
int orc_neural_spec_generate_stochastic(orc_model* m, const int32_t* prompt, int prompt_len, int max_len, int depth,
                                        double temperature, uint64_t seed, uint64_t stream, int32_t* out_tokens,
                                        int* out_len, int32_t* accept_lens, int max_steps);
/* Greedy AR decode (generate_autoregressive at temperature 0). */
int orc_neural_generate_ar(orc_model* m, const int32_t* prompt, int prompt_len, int max_len, int32_t* out_tokens);

/* Timing helper for the CPU baseline: returns seconds. */
double orc_now(void);

/* Deterministic test rows for pinning: a quantized random distribution keyed
 * by (seed, path); quantization creates exact probability ties. */
typedef struct {
    uint64_t seed;
    int vocab;
    int levels;   /* quantization levels (0 = none) */
    int zero_pct; /* percent of entries forced to 0 */
} orc_test_rows;
int orc_test_row(void* user /* orc_test_rows* */, const int32_t* path, int path_len, double* out);
int32_t orc_test_argmax(void* user, const int32_t* path, int path_len);

#ifdef __cplusplus
}
#endif
#endif
