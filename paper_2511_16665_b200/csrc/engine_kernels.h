// Launch wrappers + parameter blocks of the engine kernels (kernels.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../../include/tlt_init.h"
#include "kernels.cuh"

namespace tlt {

struct AttnParams {
    const __nv_bfloat16* q;  // [R][H*hd]
    __nv_bfloat16* out;      // [R][H*hd]
    const __nv_bfloat16* kc; // layer base [slots][KV][cap][hd]
    const __nv_bfloat16* vc;
    Rows rows;
    Groups g;
    int rows_per_req, n_groups;
    int H, KV, hd, cap;
    float scale_log2;
    int chunk, max_splits, qv_cap;
    float *ws_m, *ws_l, *ws_o;
    int impl;  // 0: CUDA-core reference kernel, 1: tensor-core flash-decode (attn_mma.cu)
    int* counters;  // non-null: fused split combine (last CTA per tile), zeroed buffer
    int dec;        // 1: decode kernel (<= 16 query vectors per request/head), chunk = multiple of 256
    int dyn_splits; // > 0: split size chosen per request from its ACTUAL key count (split_chunk
                    // below) for this many target splits; 0 = fixed p.chunk
    int gran;       // dyn_splits > 0: split granularity in keys (a multiple of the 64-key tile)
    int min_chunk;  // dyn_splits > 0: shortest split (keys); the host sizes max_splits with it
    int direct1;    // 1: a request whose keys fit one split gets its output written by the attention
                    // kernel itself (the combine skips it)
    // optional L2 warm-up of the NEXT kernel's weights (the o-proj): the
    // attention kernels are latency-bound and leave HBM idle, so each CTA
    // issues a bulk L2 prefetch of its slice of [pf, pf + pf_bytes)
    const void* pf;
    long long pf_bytes;
};

// Keys per split for a request with `total` keys. Fixed p.chunk unless
// dyn_splits > 0 (flash-decode inside CUDA graphs, whose grid is sized for the
// cache capacity): then the request's own key count is cut into <= dyn_splits
// splits of whole 64-key tiles, never shorter than 256 keys (the per-CTA tile
// count is the critical path: 5 x 64-key tiles in one CTA is slower than
// 4 + 1 in two plus the combine). Number of active splits <= min(dyn_splits,
// ceil(total / 256)), which is what the host sizes max_splits for.
__host__ __device__ __forceinline__ int split_chunk(const AttnParams& p, int total) {
    if (p.dyn_splits <= 0) return p.chunk;
    const int tiles = (total + p.gran - 1) / p.gran;
    const int per = (tiles + p.dyn_splits - 1) / p.dyn_splits;
    return per * p.gran < p.min_chunk ? p.min_chunk : per * p.gran;
}
// Active splits of a request (<= max_splits, which the host sizes as
// min(dyn_splits, ceil(max_keys / min_chunk))).
__host__ __device__ __forceinline__ int split_count(const AttnParams& p, int total) {
    const int ch = split_chunk(p, total);
    const int n = (total + ch - 1) / ch;
    return n < p.max_splits ? n : p.max_splits;
}
void launch_attention_mma(const AttnParams& p, cudaStream_t st, bool allow_tc = true);
// test hooks: the mma.sync kernels + combine, and the combine alone
void launch_attention_legacy(const AttnParams& p, cudaStream_t st);
void launch_attn_combine_only(const AttnParams& p, cudaStream_t st);
// e4m3 quantisation, one fp32 scale per row (q: [rows][cols] bytes)
void launch_quant_rows_e4m3(const __nv_bfloat16* x, int rows, int cols, long long ld, void* q, float* scale,
                            cudaStream_t st);
bool attention_tc_eligible(const AttnParams& p);
bool attention_tc_shape_ok(const AttnParams& p);
void launch_attention_tc(const AttnParams& p, cudaStream_t st);
int attention_mma_split();
int attention_dec_chunk(int n_groups, int kv, int max_keys);
int attention_dec_target_splits(int n_groups, int kv);
// split sizing shared by the engine and the test entry: fills p.chunk / dec /
// dyn_splits / gran / min_chunk / max_splits for max_keys keys per request
void attention_plan_splits(AttnParams& p, int max_keys);

struct TreeParams {
    const StepIn* step;
    int b, b_hi;
    int level, D, k, T;
    Cand* arena;
    int arena_cap;
    int *arena_n, *kept, *kept_n, *exp_n, *done;
    // rows of this level
    int lvl_base, lm_F;
    int* row_node;     // [R_draft]
    const int* root_row;
    const int* tk_tok;
    const float* tk_logit;
    const float* tk_M;
    const float* tk_S;
    // next level
    int nxt_base, nxt_F;
    Rows rows;         // drafter rows (all levels)
    Groups g_next;
    // final tree + verify rows
    int* tree_tok;
    int* tree_par;
    int* tree_dep;
    double* tree_prob;
    double* tree_pp;
    int* tree_n;
    Rows vrows;
    Groups vg;
    const int* tok_hist;
    int cap;
};

struct AcceptParams {
    const StepIn* step;
    int b, b_hi, T, maxD;
    const int* tree_tok;
    const int* tree_par;
    const int* tree_n;
    const int* argmax;  // [b_hi*(T+1)]
    int* acc_nodes;     // [b_hi][maxD]
    int* acc_tok;
    int* acc_len;
    int* bonus;
};

struct CommitParams {
    const StepIn* step;
    int b, b_hi, maxD, layers, KV, hd, cap, d, row_stride;
    __nv_bfloat16** kc;  // device array of per-layer bases
    __nv_bfloat16** vc;
    const int* acc_nodes;
    const int* acc_tok;
    const int* acc_len;
    const int* bonus;
    int* tok_hist;
    __nv_bfloat16* feat_hist;
    const __nv_bfloat16* vfeat;
    int* kv_len;
};

void launch_init(uint16_t* dst, long long n, const tlt_init_params& p, int tensor, int layer, cudaStream_t st);
void launch_embed(const Rows& rows, int R, const __nv_bfloat16* E, int d, float* x, cudaStream_t st);
void launch_draft_in(const Rows& rows, int R, const __nv_bfloat16* E, int d, const __nv_bfloat16* hist,
                     const __nv_bfloat16* dfeat, __nv_bfloat16* X2, cudaStream_t st);
void launch_gather_rows(const float* x, const int* src, int n, int d, float* out, cudaStream_t st);
void launch_to_bf16(const float* x, long long n, __nv_bfloat16* out, cudaStream_t st);
void launch_rmsnorm(const float* x, int R, int d, const __nv_bfloat16* g, float eps, __nv_bfloat16* out,
                    cudaStream_t st);
void launch_raw_rows(const float* logits, int R, int V, double* out, cudaStream_t st);
void launch_sample_rows(const float* logits, int R, int V, const int* live, double temperature, const double* uni,
                        double* pbuf, int* out_tok, cudaStream_t st);
void launch_chain_sample(const float* logits, int R, int V, const int* live, double* q, int level, int D,
                         const double* uni, int uni_stride, int* out_tok, float* out_logit, float* out_M, float* out_S,
                         cudaStream_t st);
void launch_accept_stochastic(const StepIn* step, int b, int D, int V, double temperature, const float* vlogits,
                              const double* q, const int* chain, const int* chain_n, const double* uni,
                              int uni_stride, double* pbuf, int* acc_nodes, int* acc_tok, int* acc_len, int* bonus,
                              int* consumed, int maxD, int chain_stride, int cur0, cudaStream_t st);
void launch_reduce_resid_norm(const float* ws, long long plane, int splits, int R, int d, float* x,
                              const __nv_bfloat16* g, float eps, __nv_bfloat16* out, cudaStream_t st);
void launch_attention(const AttnParams& p, cudaStream_t st);
// TMA-fed variant (attn_tma.cu): tk / tv = 2D maps of the layer's K / V cache
// ([slots * KV * cap][hd], 64 x 64 boxes, 128B swizzle, make_tmap_kv)
CUtensorMap make_tmap_kv(const void* base, long long rows, int hd);
bool attention_tma_enabled(const AttnParams& p);
void launch_attention_tma(const CUtensorMap& tk, const CUtensorMap& tv, const AttnParams& p, cudaStream_t st);
// tcgen05 / TMEM tree attention (attn_tc5.cu), same maps and split plan, hd = 128
bool attention_tree_tc_eligible(const AttnParams& p);
void launch_attention_tree_tc(const CUtensorMap& tk, const CUtensorMap& tv, const AttnParams& p, cudaStream_t st);

int launch_row_topk_chunked(const float* logits, int R, int V, const int* live, int k, float* part, cudaStream_t st);
// thr_reset: the fused LM head's per-row bound array (EpiParams::topk_thr), cleared per row
void launch_topk_merge(const float* part, int n_tiles, int R, int k, const int* live, int* out_tok, float* out_logit,
                       float* out_M, float* out_S, cudaStream_t st, unsigned* thr_reset = nullptr);
void launch_row_probs(const float* logits, int R, int V, const float* M, const float* S, double* out,
                      cudaStream_t st);
void launch_rows_level1(const StepIn* st, int b, int b_hi, int D1, const Rows& rows, const Groups& g, int* root_row,
                        const int* tok_hist, int cap, cudaStream_t s);
void launch_rows_ar(const StepIn* st, int b, int b_hi, const Rows& rows, const Groups& g, const int* tok_hist,
                    int cap, cudaStream_t s);
void launch_tree_level(const TreeParams& p, cudaStream_t st);
void launch_tree_final(const TreeParams& p, cudaStream_t st);
void launch_accept_greedy(const AcceptParams& p, cudaStream_t st);
void launch_commit(const CommitParams& p, cudaStream_t st);
void launch_commit_ar(const StepIn* st, int b, const int* argmax, const __nv_bfloat16* feat, int d, int* tok_hist,
                      __nv_bfloat16* feat_hist, int cap, int* out_tok, cudaStream_t s);

}  // namespace tlt
