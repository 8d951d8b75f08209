// Host-side engine: owns weights, KV caches, histories, activation buffers and
// the CUDA-graph pool; runs prefill, the greedy tree SD step and the AR step.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "../../include/tlt_b200.h"
#include "../../include/tlt_init.h"
#include "engine_kernels.h"
#include "tlt_internal.h"

namespace tlt {

using bf16 = __nv_bfloat16;

struct LayerW {
    bf16 *attn_norm = nullptr, *qkv = nullptr, *qkv_b = nullptr, *o = nullptr, *mlp_norm = nullptr, *gu = nullptr,
         *down = nullptr;
    CUtensorMap tm_qkv, tm_o, tm_gu, tm_down;
};

struct StepOutHost {  // pinned staging of one step's results
    int32_t* acc_len;
    int32_t* bonus;
    int32_t* acc_tok;    // [b_hi][maxD]
    int32_t* acc_nodes;  // [b_hi][maxD]
    int32_t* tree_tok;   // [b_hi][T]
    int32_t* tree_par;
    int32_t* tree_dep;
    double* tree_prob;
    double* tree_pp;
    int32_t* tree_n;
    int32_t* ar_tok;     // [b_hi]
};

struct DebugExp {  // one drafter expansion of one request (parity export)
    std::vector<int32_t> path;
    std::vector<double> row;
};

class Engine {
public:
    Engine(const tlt_model_cfg& cfg, const tlt_init_cfg& init, int device);
    ~Engine();

    void prefill(int b, const int32_t* slots, const int32_t* lens, const int32_t* tokens);
    void release(int slot);
    void truncate(int slot, int len);
    std::vector<tlt_tensor_view> drafter_tensors();
    void drafter_published(int64_t version);
    int64_t drafter_version_ = 0;
    // C2 (drafter training samples): committed tokens [0, lt] and target
    // features [0, lt) of a live slot into caller memory (host or device)
    int export_sequence(int slot, int32_t* tokens, int max_tokens, void* features, size_t features_bytes);
    // greedy tree SD step; returns device ms
    float sd_step(const tlt_strategy& s, int b, const int32_t* slots, tlt_tree_out* tree, tlt_accept_out* out);
    float ar_step(int b, const int32_t* slots, int32_t* out_tokens);
    // split boundary (reference DraftPlanner seam, spec_decode.hpp:319-341):
    // propose only (build_draft_tree with the EAGLE drafter, no commit) ...
    float draft(const tlt_strategy& s, int b, const int32_t* slots, tlt_tree_out* tree);
    // ... and verify_greedy + KV commit of a tree: the engine's own last draft
    // (tree == nullptr, device-resident) or an arbitrary host tree
    float verify_tree(int b, const int32_t* slots, const tlt_tree_in* tree, tlt_accept_out* out);
    // greedy verify of host-proposed chains (n-gram fallback drafter)
    // temperature > 0: verify_stochastic with one-hot q and uniforms [b][D+1]
    float sd_step_chain(int D, int b, const int32_t* slots, const int32_t* chains, const int32_t* lens,
                        tlt_accept_out* out, float temperature = 0.f, const double* uniforms = nullptr);
    // rejection-sampling SD over a drafter-sampled chain (stochastic.cu);
    // uniforms [b][2D+1] in RngStream consumption order
    float sd_step_stochastic(int D, float temperature, int b, const int32_t* slots, const double* uniforms,
                             tlt_accept_out* out);
    std::vector<std::vector<double>> dbg_praw;   // [request i] [(D+1)*V] raw target rows examined (stochastic)
    std::vector<int> last_consumed;              // uniforms consumed per request by the last stochastic step
    std::vector<std::vector<int>> last_chain;    // drafted chain per request of the last stochastic step

    int slot_len(int slot) const { return lt_.at(slot); }
    int device() const { return dev_; }
    void set_debug(bool on) { debug_ = on; }
    bool use_graphs = true;
    size_t graph_pool_build(const std::vector<tlt_capture_entry>& entries, bool with_ar = true);
    size_t pool_bytes_ = 0;       // device memory taken by the last pool build
    double pool_capture_ms_ = 0;  // host time of the last pool build
    int pool_graphs_ = 0;         // graphs captured by the last pool build
    int pool_skipped_ = 0;        // plan pairs not capturable (draft rows beyond the engine buffers)
    int pool_sub_width_ = 0;      // 0: one graph per plan bucket; w: sub-buckets of <= w batch sizes
    int pool_ar_width_ = 0;       // 0: plain-decode sizes 1,2,4,8,16,24,..; w: every w-th size (1 = exact)
    int graph_count() const {  // production graphs (debug-export variants excluded)
        int n = 0;
        for (const auto& kv : graphs_) n += std::get<4>(kv.first) != 4;
        return n;
    }
    void graph_pool_clear();
    int bucket_hi_for(int b, int T) const;
    float probe_kernel(int kind, int M, int iters, double* bytes, double* flops);
    float probe_attention(int b, int ctx, int rpr, int iters, double* bytes);

    // parity exports
    std::vector<std::vector<DebugExp>> dbg_exp;  // [request i] expansions of the last stochastic step
    std::vector<float> dbg_ar_logits;            // [b*V]
    // greedy tree step: expansions / verify logits of request i of the last
    // debug sd_step, extracted after the step from the device copies the
    // step's own (graph-captured) sequence made
    const std::vector<DebugExp>& debug_expansions(int i);
    std::vector<float> debug_verify_logits(int i);

    const tlt_model_cfg cfg;
    long long launches = 0;
    float last_prefill_ms = 0.f;  // device time of the last prefill (CUDA events)  // kernel launches issued (graph replays count their nodes)

private:
    void alloc_weights(const tlt_init_cfg& init);
    void alloc_state();
    const CUtensorMap& tmap_act(const void* p, int rows, int cols, long long ld, int box);
    const CUtensorMap& tmap_kv(const bf16* base, int cache_cap);
    void gemm(const bf16* X, int M, int K, long long ldx, const CUtensorMap& tmW, int N, const EpiParams& ep);
    GemmPlan make_plan(int M, int N, int K, int kind, int variant) const;
    int tuned_variant(const bf16* X, int M, int K, long long ldx, const CUtensorMap& tmW, int N, const EpiParams& ep);
    std::map<std::tuple<int, int, int, int>, int> gemm_variant_;  // autotuned plan variant per (M, N, K, epilogue)
    cudaEvent_t tune_ev0_ = nullptr, tune_ev1_ = nullptr;
    bool tune_cache_loaded_ = false;
    void layer_forward(const LayerW& w, bf16* kc, bf16* vc, int cache_cap, const Rows& rw, const Groups& gp, int R,
                       int rpr, int ngroups, int max_keys, bool h_ready, const bf16* next_norm);
    void gemm_resid_norm(const bf16* X, int M, int K, long long ldx, const CUtensorMap& tmW, const bf16* norm_w);
    void attention(const bf16* kc, const bf16* vc, int cache_cap, const Rows& rw, const Groups& gp, int rpr,
                   int ngroups, int max_keys, const void* pf = nullptr, long long pf_bytes = 0);
    void lm_head(const float* x, int n, float* logits, bool h_ready = false);
    void target_forward(const Rows& rw, const Groups& gp, int R, int rpr, int ngroups, int max_keys,
                        float* logits, bf16* feat);
    void drafter_forward(const Rows& rw, const Groups& gp, int R, int rpr, int ngroups, int max_keys,
                         const int* gather, int n_lm, int k, const int* live, bool want_logits, bf16* dfeat_out);
    void lm_topk(const float* x, int n, int k, const int* live, bool want_logits, bool h_ready = false,
                 bool drafter = false);
    void drafter_logits(int n);  // h_ -> logits_ through the drafter's LM head (bf16 or e4m3)
    void drafter_lm_head(const float* x, int n);  // final norm + drafter_logits
    bool drafter_fp8_ = false;
    uint8_t *lm8_ = nullptr, *h8_ = nullptr;
    float *lm8_s_ = nullptr, *h8_s_ = nullptr;
    CUtensorMap tm_lm8_;
    float* topk_part_ = nullptr;  // EPI_TOPK partials [vocab tiles][R][2 + 2k]
    unsigned* topk_thr_ = nullptr;  // EPI_TOPK k > 1 per-row k-th-value bounds [R] (0 = none)
    void scatter_features(const Rows& rw, int R, const bf16* feat);
    float catchup_drafter(int b, const int32_t* slots);
    void sd_device_sequence(int b_hi, int D, int k, int T, bool dbg, int b_real, bool verify = true);
    void tree_to_host(int b_hi, int T);
    int prepare_tree_step(const tlt_strategy& s, int b, const int32_t* slots, float* catchup_ms);
    void copy_step_out(int b, const int32_t* slots, int T, int stride, tlt_tree_out* tree, tlt_accept_out* out);
    // split boundary state: the last tlt_draft (slots, strategy, lt at draft time)
    std::vector<int32_t> draft_slots_;
    std::vector<int> draft_lt_;
    int draft_T_ = 0, draft_D_ = 0;
    void verify_accept_commit(int b_hi, int T, bool dbg, int b_real);
    void stoch_verify_commit(int b_hi, int D, double temperature, bool dbg, int b_real, const double* q, int cur0);
    void ar_device_sequence(int b_hi);
    void stoch_device_sequence(int b_hi, int D, double temperature, bool dbg, int b_real);
    void ar_sample_sequence(int b_hi, double temperature);
    void ensure_stoch_buffers();

public:
    float ar_step_sampled(int b, const int32_t* slots, float temperature, const double* uniforms,
                          int32_t* out_tokens);

private:
    // stochastic-path buffers
    double* qrows_ = nullptr;   // drafter chain rows [S][kMaxDepth][V]
    double* pbuf_ = nullptr;    // target row scratch [S][V]
    double* d_uni_ = nullptr;   // uploaded uniforms [S][2*kMaxDepth+1]
    double* h_uni_ = nullptr;   // pinned staging
    int* consumed_ = nullptr;
    int* h_consumed_ = nullptr;
    void upload_rows_host(const std::vector<int>& tok, const std::vector<int>& pos, const std::vector<int>& slot,
                          const std::vector<int>& cidx, const std::vector<int>& fkind,
                          const std::vector<long long>& fidx, const std::vector<uint32_t>& mask,
                          const std::vector<int>& gslot, const std::vector<int>& glc, const std::vector<int>& gt0,
                          const std::vector<int>& gnt);

    int dev_;
    cudaStream_t st_;
    tlt_init_params ip_;
    // weights
    bf16 *embed_ = nullptr, *lm_head_ = nullptr, *final_norm_ = nullptr, *fc_ = nullptr;
    std::vector<LayerW> layers_;
    LayerW drafter_;
    CUtensorMap tm_lm_, tm_fc_;
    float *rope_cos_ = nullptr, *rope_sin_ = nullptr;
    // caches / histories
    int cap_ = 0, dcap_ = 0;
    std::vector<bf16*> kc_, vc_;
    bf16 *dkc_ = nullptr, *dvc_ = nullptr;
    bf16** d_kc_arr_ = nullptr;
    bf16** d_vc_arr_ = nullptr;
    int32_t* tok_hist_ = nullptr;
    bf16* feat_hist_ = nullptr;
    // activations (capacity R_)
    int R_ = 0, Rmeta_ = 0;
    float* x_ = nullptr;
    float* xg_ = nullptr;  // gathered rows for LM head
    bf16 *h_ = nullptr, *q_ = nullptr, *attn_ = nullptr, *act_ = nullptr, *feat_ = nullptr, *x2_ = nullptr;
    bf16* dfeat_ = nullptr;  // drafter output features per drafter row [Rmeta][d]
    float* logits_ = nullptr;
    float* ws_ = nullptr;
    size_t ws_elems_ = 0;
    float *aws_m_ = nullptr, *aws_l_ = nullptr, *aws_o_ = nullptr;
    size_t aws_elems_ = 0;
    int* attn_counters_ = nullptr;  // fused attention split-combine election
    // row metadata
    Rows drows_, vrows_, prows_;
    Groups dg_[kMaxDepth + 2], vg_, pg_;
    int *root_row_ = nullptr, *row_node_ = nullptr;
    int* tk_tok_ = nullptr;
    float *tk_logit_ = nullptr, *tk_M_ = nullptr, *tk_S_ = nullptr;
    int* argmax_ = nullptr;
    double* dbg_probs_ = nullptr;
    // Debug export of the greedy tree step. The sequence itself enqueues
    // device-to-device copies (per drafter level: fp32 logits rows, M, S,
    // row liveness; at the end: arena, row->node map, verify logits), so a
    // debug step replays a CUDA graph exactly like a production step (same
    // kernels, plus copy nodes). Host extraction is lazy, per request.
    struct DbgStep {
        bool valid = false, greedy = false;
        int b_hi = 0, b_real = 0, D = 0, T = 0;
        std::vector<int> Fd, base, lmoff;  // per level: rows/request, drafter row base, logits row offset
        int meta_rows = 0;                 // drafter rows of the step (row_node / slot copies)
    } dbgs_;
    std::map<int, std::vector<DebugExp>> dbg_cache_;
    float *dbg_lg_ = nullptr, *dbg_M_ = nullptr, *dbg_S_ = nullptr, *dbg_vlg_ = nullptr;
    int *dbg_live_ = nullptr, *dbg_node_ = nullptr;
    Cand* dbg_arena_ = nullptr;
    size_t dbg_lg_rows_ = 0, dbg_vlg_rows_ = 0, dbg_meta_rows_ = 0, dbg_arena_reqs_ = 0;
    void ensure_debug_buffers(int b_hi, int D, int k, int T);
    void free_debug_buffers();
    // tree + accept
    Cand* arena_ = nullptr;
    int arena_cap_ = 16384;
    int *arena_n_ = nullptr, *kept_ = nullptr, *kept_n_ = nullptr, *exp_n_ = nullptr, *done_ = nullptr;
    int *tree_tok_ = nullptr, *tree_par_ = nullptr, *tree_dep_ = nullptr, *tree_n_ = nullptr;
    double *tree_prob_ = nullptr, *tree_pp_ = nullptr;
    int *acc_nodes_ = nullptr, *acc_tok_ = nullptr, *acc_len_ = nullptr, *bonus_ = nullptr, *kv_len_ = nullptr;
    int* ar_tok_ = nullptr;
    static constexpr int kMaxD = kMaxDepth;
    StepIn *d_step_ = nullptr, *h_step_ = nullptr;
    // live request count of the current step (bucketed graphs: the step is
    // padded to the bucket's b_hi; GEMMs skip the padding rows' tiles)
    int *d_nreal_ = nullptr, *h_nreal_ = nullptr;
    int dyn_b_hi_ = 0;
    void set_dyn(EpiParams& e, int M) const;
    struct DynScope {
        Engine* e;
        int prev;
        DynScope(Engine* en, int b_hi) : e(en), prev(en->dyn_b_hi_) { en->dyn_b_hi_ = b_hi; }
        ~DynScope() { e->dyn_b_hi_ = prev; }
    };
    // CUDA-graph pool built from plan_captures (tlt_graph_pool_build)
    struct PoolBucket {
        int lo, hi;
        std::vector<int> Ts;                     // TARGET entries: tokens_to_verify
        std::vector<std::pair<int, int>> kd;     // DRAFT entries: (top_k, draft_depth)
    };
    std::vector<PoolBucket> pool_;
    std::vector<int> ar_sizes_;                  // padded plain-decode batch sizes
    int ar_bucket_for(int b) const;
    void capture_graph(const std::tuple<int, int, int, int, int>& key, bool ar);
    StepOutHost ho_{};
    int max_b_ = 0;
    // host mirrors
    std::vector<int> lt_, ld_, live_;
    bool debug_ = false;
    int attn_impl_ = 1;  // TLT_ATTN=0 selects the CUDA-core attention (cross-check)
    // caches
    std::unordered_map<std::string, CUtensorMap> tmaps_;
    std::map<std::tuple<int, int, int, int, int>, std::pair<cudaGraphExec_t, long long>> graphs_;
    cudaEvent_t ev0_, ev1_;
    long long launches_in_seq_ = 0;
    bool counting_ = false;
    void count_launch(int n = 1) { launches_in_seq_ += n; }
    friend struct Counter;
};

}  // namespace tlt
