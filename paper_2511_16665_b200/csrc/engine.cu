// Engine: weights, caches, forwards, the greedy tree SD step, the AR step and
// the CUDA-graph pool keyed on the reference CaptureEntry keys
// (capture_plan.hpp:25-33): one graph per (bucket, top_k, draft_depth,
// tokens_to_verify) replaying draft -> verify -> accept -> commit.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "engine.h"
#include "host_select.h"
#include "pdl.cuh"

namespace tlt {

namespace {
template <typename T>
T* dmalloc(size_t n) {
    void* p = nullptr;
    if (n == 0) n = 1;
    CUDA_CHECK(cudaMalloc(&p, n * sizeof(T)));
    return static_cast<T*>(p);
}
template <typename T>
T* hmalloc(size_t n) {
    void* p = nullptr;
    if (n == 0) n = 1;
    CUDA_CHECK(cudaMallocHost(&p, n * sizeof(T)));
    return static_cast<T*>(p);
}
Rows alloc_rows(int n) {
    Rows r;
    r.tok = dmalloc<int>(n);
    r.pos = dmalloc<int>(n);
    r.slot = dmalloc<int>(n);
    r.cidx = dmalloc<int>(n);
    r.fkind = dmalloc<int>(n);
    r.fidx = dmalloc<long long>(n);
    r.mask = dmalloc<uint32_t>((size_t)n * kMaskWords);
    CUDA_CHECK(cudaMemset(r.slot, 0xff, sizeof(int) * n));
    CUDA_CHECK(cudaMemset(r.mask, 0, sizeof(uint32_t) * (size_t)n * kMaskWords));
    return r;
}
void free_rows(Rows& r) {
    cudaFree(r.tok);
    cudaFree(r.pos);
    cudaFree(r.slot);
    cudaFree(r.cidx);
    cudaFree(r.fkind);
    cudaFree(r.fidx);
    cudaFree(r.mask);
}
Groups alloc_groups(int n) {
    Groups g;
    g.slot = dmalloc<int>(n);
    g.lc = dmalloc<int>(n);
    g.tail0 = dmalloc<int>(n);
    g.ntail = dmalloc<int>(n);
    CUDA_CHECK(cudaMemset(g.slot, 0xff, sizeof(int) * n));
    CUDA_CHECK(cudaMemset(g.ntail, 0, sizeof(int) * n));
    return g;
}
void free_groups(Groups& g) {
    cudaFree(g.slot);
    cudaFree(g.lc);
    cudaFree(g.tail0);
    cudaFree(g.ntail);
}
Rows sub(const Rows& r, int base) {
    Rows s = r;
    s.tok += base;
    s.pos += base;
    s.slot += base;
    s.cidx += base;
    s.fkind += base;
    s.fidx += base;
    s.mask += (size_t)base * kMaskWords;
    return s;
}
int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v ? std::atoi(v) : dflt;
}
// Drafter levels of a (b_hi, D, k, T) tree step: rows per request Fd[lv]
// (level 1: pending + root; level lv >= 2: min(T, k^(lv-1)) frontier rows),
// drafter row base[lv], and lmoff[lv] = LM-head row offset of the level in a
// level-concatenated array (level 1 has one LM row per request).
void level_plan(int b_hi, int D, int k, int T, std::vector<int>& base, std::vector<int>& Fd,
                std::vector<int>& lmoff) {
    base.assign(D + 2, 0);
    Fd.assign(D + 2, 0);
    lmoff.assign(D + 2, 0);
    Fd[1] = D + 1;
    long long kp = 1;
    for (int lv = 2; lv <= D; ++lv) {
        kp = std::min<long long>(kp * k, 1 << 20);
        Fd[lv] = (int)std::min<long long>(T, kp);
        base[lv] = base[lv - 1] + b_hi * Fd[lv - 1];
    }
    for (int lv = 1; lv <= D; ++lv) lmoff[lv + 1] = lmoff[lv] + (lv == 1 ? b_hi : b_hi * Fd[lv]);
}
}  // namespace

Engine::Engine(const tlt_model_cfg& c, const tlt_init_cfg& init, int device) : cfg(c), dev_(device) {
    if (c.vocab < 2) throw ConfigErr("vocab", "must be >= 2");
    if (c.hidden % 64 != 0) throw ConfigErr("hidden", "must be a multiple of 64");
    if (c.head_dim != 64 && c.head_dim != 128) throw ConfigErr("head_dim", "must be 64 or 128");
    if (c.heads < 1 || c.kv_heads < 1 || c.heads % c.kv_heads) throw ConfigErr("kv_heads", "must divide heads");
    if (c.ffn % 8 != 0) throw ConfigErr("ffn", "must be a multiple of 8");
    if (c.layers < 1) throw ConfigErr("layers", "must be >= 1");
    if (c.max_slots < 1 || c.max_ctx < 2) throw ConfigErr("max_ctx", "must be >= 2");
    CUDA_CHECK(cudaSetDevice(device));
    CUDA_CHECK(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    CUDA_CHECK(cudaEventCreate(&ev0_));
    CUDA_CHECK(cudaEventCreate(&ev1_));
    ip_ = tlt_init_params{init.seed, init.layer_scale, init.lm_gain, init.lm_alt, init.lm_noise, init.fc_noise,
                          c.vocab,   c.hidden,         c.heads,      c.kv_heads,    c.head_dim, c.ffn};
    alloc_weights(init);
    alloc_state();
    attn_impl_ = env_int("TLT_ATTN", 1);
    CUDA_CHECK(cudaStreamSynchronize(st_));
}

Engine::~Engine() {
    cudaSetDevice(dev_);
    graph_pool_clear();
    cudaStreamSynchronize(st_);
    auto f = [](void* p) {
        if (p) cudaFree(p);
    };
    f(embed_), f(lm_head_), f(final_norm_), f(fc_), f(rope_cos_), f(rope_sin_);
    f(lm8_), f(lm8_s_), f(h8_), f(h8_s_);
    for (auto& L : layers_) f(L.attn_norm), f(L.qkv), f(L.qkv_b), f(L.o), f(L.mlp_norm), f(L.gu), f(L.down);
    f(drafter_.attn_norm), f(drafter_.qkv), f(drafter_.qkv_b), f(drafter_.o), f(drafter_.mlp_norm), f(drafter_.gu),
        f(drafter_.down);
    for (auto p : kc_) f(p);
    for (auto p : vc_) f(p);
    f(dkc_), f(dvc_), f(d_kc_arr_), f(d_vc_arr_), f(tok_hist_), f(feat_hist_);
    f(x_), f(xg_), f(h_), f(q_), f(attn_), f(act_), f(feat_), f(x2_), f(dfeat_), f(logits_), f(ws_);
    f(aws_m_), f(aws_l_), f(aws_o_);
    if (attn_counters_) cudaFree(attn_counters_);
    free_rows(drows_), free_rows(vrows_), free_rows(prows_);
    for (auto& g : dg_) free_groups(g);
    free_groups(vg_), free_groups(pg_);
    f(root_row_), f(row_node_), f(tk_tok_), f(tk_logit_), f(tk_M_), f(tk_S_), f(argmax_), f(dbg_probs_);
    free_debug_buffers();
    f(arena_), f(arena_n_), f(kept_), f(kept_n_), f(exp_n_), f(done_);
    f(tree_tok_), f(tree_par_), f(tree_dep_), f(tree_n_), f(tree_prob_), f(tree_pp_);
    f(acc_nodes_), f(acc_tok_), f(acc_len_), f(bonus_), f(kv_len_), f(ar_tok_), f(d_step_);
    f(topk_part_), f(topk_thr_), f(d_nreal_);
    if (h_step_) cudaFreeHost(h_step_);
    if (h_nreal_) cudaFreeHost(h_nreal_);
    void* hp[] = {ho_.acc_len, ho_.bonus, ho_.acc_tok, ho_.acc_nodes, ho_.tree_tok, ho_.tree_par,
                  ho_.tree_dep, ho_.tree_prob, ho_.tree_pp, ho_.tree_n, ho_.ar_tok};
    for (void* p : hp)
        if (p) cudaFreeHost(p);
    cudaEventDestroy(ev0_);
    if (tune_ev0_) cudaEventDestroy(tune_ev0_);
    if (tune_ev1_) cudaEventDestroy(tune_ev1_);
    cudaEventDestroy(ev1_);
    cudaStreamDestroy(st_);
}

void Engine::alloc_weights(const tlt_init_cfg& init) {
    const long long V = cfg.vocab, d = cfg.hidden, F = cfg.ffn;
    const long long nqkv = (long long)(cfg.heads + 2 * cfg.kv_heads) * cfg.head_dim;
    const long long nq = (long long)cfg.heads * cfg.head_dim;
    auto W = [&](long long n, int tensor, int layer) {
        bf16* p = dmalloc<bf16>(n);
        launch_init(reinterpret_cast<uint16_t*>(p), n, ip_, tensor, layer, st_);
        CUDA_CHECK(cudaGetLastError());
        return p;
    };
    embed_ = W(V * d, TLT_W_EMBED, 0);
    lm_head_ = W(V * d, TLT_W_LM_HEAD, 0);
    final_norm_ = W(d, TLT_W_FINAL_NORM, 0);
    fc_ = W(d * 2 * d, TLT_W_FC, TLT_DRAFTER_LAYER);
    auto mk_layer = [&](int l) {
        LayerW L;
        L.attn_norm = W(d, TLT_W_ATTN_NORM, l);
        L.qkv = W(nqkv * d, TLT_W_QKV, l);
        L.qkv_b = cfg.qkv_bias ? W(nqkv, TLT_W_QKV_BIAS, l) : nullptr;
        L.o = W(d * nq, TLT_W_O, l);
        L.mlp_norm = W(d, TLT_W_MLP_NORM, l);
        L.gu = W(2 * F * d, TLT_W_GATE_UP, l);
        L.down = W(d * F, TLT_W_DOWN, l);
        L.tm_qkv = make_tmap_bf16(L.qkv, (int)nqkv, (int)d, d, 128);
        L.tm_o = make_tmap_bf16(L.o, (int)d, (int)nq, nq, 128);
        L.tm_gu = make_tmap_bf16(L.gu, (int)(2 * F), (int)d, d, 128);
        L.tm_down = make_tmap_bf16(L.down, (int)d, (int)F, F, 128);
        return L;
    };
    for (int l = 0; l < cfg.layers; ++l) layers_.push_back(mk_layer(l));
    drafter_ = mk_layer(TLT_DRAFTER_LAYER);
    tm_lm_ = make_tmap_bf16(lm_head_, (int)V, (int)d, d, 128);
    drafter_fp8_ = init.drafter_lm_fp8 != 0 || env_int("TLT_DRAFTER_FP8", 0) != 0;
    if (drafter_fp8_) {  // e4m3 copy of the LM head for the drafter, one scale per vocab row
        lm8_ = dmalloc<uint8_t>((size_t)V * d);
        lm8_s_ = dmalloc<float>((size_t)V);
        launch_quant_rows_e4m3(lm_head_, (int)V, (int)d, d, lm8_, lm8_s_, st_);
        // weight operands are prefetched by the GEMMs before griddepcontrol.wait
        // (they are static): the e4m3 copy must be complete before any GEMM
        CUDA_CHECK(cudaStreamSynchronize(st_));
        tm_lm8_ = make_tmap_e4m3(lm8_, (int)V, (int)d, d, 128);
    }
    tm_fc_ = make_tmap_bf16(fc_, (int)d, (int)(2 * d), 2 * d, 128);
    // RoPE table, computed in double exactly as the oracle does, stored fp32
    cap_ = cfg.max_ctx + kMaxT + 2;
    const int half = cfg.head_dim / 2;
    const int rope_rows = cap_ + kMaxDepth + 2;
    std::vector<float> cs((size_t)rope_rows * half), sn((size_t)rope_rows * half);
    for (int pos = 0; pos < rope_rows; ++pos)
        for (int i = 0; i < half; ++i) {
            double inv = std::pow((double)cfg.rope_theta, -2.0 * (double)i / (double)cfg.head_dim);
            double ang = (double)pos * inv;
            cs[(size_t)pos * half + i] = (float)std::cos(ang);
            sn[(size_t)pos * half + i] = (float)std::sin(ang);
        }
    rope_cos_ = dmalloc<float>(cs.size());
    rope_sin_ = dmalloc<float>(sn.size());
    CUDA_CHECK(cudaMemcpy(rope_cos_, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice));
    CUDA_CHECK(cudaMemcpy(rope_sin_, sn.data(), sn.size() * 4, cudaMemcpyHostToDevice));
}

void Engine::alloc_state() {
    const int S = cfg.max_slots, KV = cfg.kv_heads, hd = cfg.head_dim, d = cfg.hidden, V = cfg.vocab;
    dcap_ = cap_ + 1024 + 8;
    const size_t kv_elems = (size_t)S * KV * cap_ * hd;
    for (int l = 0; l < cfg.layers; ++l) {
        kc_.push_back(dmalloc<bf16>(kv_elems));
        vc_.push_back(dmalloc<bf16>(kv_elems));
    }
    dkc_ = dmalloc<bf16>((size_t)S * KV * dcap_ * hd);
    dvc_ = dmalloc<bf16>((size_t)S * KV * dcap_ * hd);
    d_kc_arr_ = dmalloc<bf16*>(cfg.layers);
    d_vc_arr_ = dmalloc<bf16*>(cfg.layers);
    CUDA_CHECK(cudaMemcpy(d_kc_arr_, kc_.data(), sizeof(bf16*) * cfg.layers, cudaMemcpyHostToDevice));
    CUDA_CHECK(cudaMemcpy(d_vc_arr_, vc_.data(), sizeof(bf16*) * cfg.layers, cudaMemcpyHostToDevice));
    tok_hist_ = dmalloc<int32_t>((size_t)S * cap_);
    CUDA_CHECK(cudaMemset(tok_hist_, 0, sizeof(int32_t) * (size_t)S * cap_));
    feat_hist_ = dmalloc<bf16>((size_t)S * cap_ * d);

    R_ = env_int("TLT_MAX_ROWS", 2048);
    Rmeta_ = env_int("TLT_MAX_DRAFT_ROWS", 32768);
    const int nq = cfg.heads * hd, nqkv = (cfg.heads + 2 * KV) * hd;
    x_ = dmalloc<float>((size_t)R_ * 2 * d);
    xg_ = dmalloc<float>((size_t)R_ * d);
    h_ = dmalloc<bf16>((size_t)R_ * 2 * d);
    q_ = dmalloc<bf16>((size_t)R_ * std::max(nq, nqkv));
    attn_ = dmalloc<bf16>((size_t)R_ * nq);
    act_ = dmalloc<bf16>((size_t)R_ * cfg.ffn);
    feat_ = dmalloc<bf16>((size_t)R_ * d);
    x2_ = dmalloc<bf16>((size_t)R_ * 2 * d);
    dfeat_ = dmalloc<bf16>((size_t)Rmeta_ * d);
    logits_ = dmalloc<float>((size_t)R_ * V);
    ws_elems_ = (size_t)env_int("TLT_GEMM_WS_MFLOATS", 1) << 20;
    ws_ = dmalloc<float>(ws_elems_);
    aws_elems_ = (size_t)env_int("TLT_ATTN_WS_MFLOATS", 192) << 20;
    aws_m_ = dmalloc<float>(aws_elems_ / 32);
    aws_l_ = dmalloc<float>(aws_elems_ / 32);
    aws_o_ = dmalloc<float>(aws_elems_);
    drows_ = alloc_rows(Rmeta_);
    vrows_ = alloc_rows(R_);
    prows_ = alloc_rows(R_);
    max_b_ = S;
    for (auto& g : dg_) g = alloc_groups(S);
    vg_ = alloc_groups(S);
    pg_ = alloc_groups(std::max(S, R_));
    root_row_ = dmalloc<int>(S);
    row_node_ = dmalloc<int>(Rmeta_);
    tk_tok_ = dmalloc<int>((size_t)R_ * kMaxTopK);
    tk_logit_ = dmalloc<float>((size_t)R_ * kMaxTopK);
    tk_M_ = dmalloc<float>(R_);
    tk_S_ = dmalloc<float>(R_);
    argmax_ = dmalloc<int>(R_);
    topk_part_ = dmalloc<float>((size_t)((V + 127) / 128) * R_ * (2 + 2 * kEpiTopkMax));
    topk_thr_ = dmalloc<unsigned>(R_);
    CUDA_CHECK(cudaMemset(topk_thr_, 0, sizeof(unsigned) * R_));
    arena_ = dmalloc<Cand>((size_t)S * arena_cap_);
    arena_n_ = dmalloc<int>(S);
    kept_ = dmalloc<int>((size_t)S * kMaxT);
    kept_n_ = dmalloc<int>(S);
    exp_n_ = dmalloc<int>(S);
    done_ = dmalloc<int>(S);
    tree_tok_ = dmalloc<int>((size_t)S * kMaxT);
    tree_par_ = dmalloc<int>((size_t)S * kMaxT);
    tree_dep_ = dmalloc<int>((size_t)S * kMaxT);
    tree_n_ = dmalloc<int>(S);
    tree_prob_ = dmalloc<double>((size_t)S * kMaxT);
    tree_pp_ = dmalloc<double>((size_t)S * kMaxT);
    acc_nodes_ = dmalloc<int>((size_t)S * kMaxD);
    acc_tok_ = dmalloc<int>((size_t)S * kMaxD);
    acc_len_ = dmalloc<int>(S);
    bonus_ = dmalloc<int>(S);
    kv_len_ = dmalloc<int>(S);
    ar_tok_ = dmalloc<int>(S);
    d_step_ = dmalloc<StepIn>(S);
    h_step_ = hmalloc<StepIn>(S);
    d_nreal_ = dmalloc<int>(1);
    h_nreal_ = hmalloc<int>(1);
    *h_nreal_ = 0;
    ho_.acc_len = hmalloc<int32_t>(S);
    ho_.bonus = hmalloc<int32_t>(S);
    ho_.acc_tok = hmalloc<int32_t>((size_t)S * kMaxD);
    ho_.acc_nodes = hmalloc<int32_t>((size_t)S * kMaxD);
    ho_.tree_tok = hmalloc<int32_t>((size_t)S * kMaxT);
    ho_.tree_par = hmalloc<int32_t>((size_t)S * kMaxT);
    ho_.tree_dep = hmalloc<int32_t>((size_t)S * kMaxT);
    ho_.tree_prob = hmalloc<double>((size_t)S * kMaxT);
    ho_.tree_pp = hmalloc<double>((size_t)S * kMaxT);
    ho_.tree_n = hmalloc<int32_t>(S);
    ho_.ar_tok = hmalloc<int32_t>(S);
    lt_.assign(S, 0);
    ld_.assign(S, 0);
    live_.assign(S, 0);
}

// ------------------------------------------------------------------ helpers
const CUtensorMap& Engine::tmap_act(const void* p, int rows, int cols, long long ld, int box) {
    char key[96];
    std::snprintf(key, sizeof key, "%p/%d/%d/%lld/%d", p, rows, cols, ld, box);
    auto it = tmaps_.find(key);
    if (it != tmaps_.end()) return it->second;
    return tmaps_.emplace(key, make_tmap_bf16(p, rows, cols, ld, box)).first->second;
}

// GEMM plan of one site: the planner's variant plus the epilogue fix-ups.
GemmPlan Engine::make_plan(int M, int N, int K, int kind, int variant) const {
    GemmPlan g = plan_gemm(M, N, K, variant);
    if (kind == EPI_TOPK) {  // the fused top-k epilogue needs whole-K accumulators
        g.kb_per_split = g.kb_total;
        g.splits = 1;
    }
    static const int qkv_max_splits = [] {
        const char* v = std::getenv("TLT_QKV_MAX_SPLITS");
        return v ? std::atoi(v) : 4;
    }();
    if (kind == EPI_QKV && g.pair == 1 && g.splits > qkv_max_splits) {
        // measured (tools/probe.py): the QKV epilogue (bias, RoPE, KV-cache
        // scatter) after the in-cluster reduction prefers <= 4 splits
        g.kb_per_split = (g.kb_total + qkv_max_splits - 1) / qkv_max_splits;
        g.splits = (g.kb_total + g.kb_per_split - 1) / g.kb_per_split;
        gemm_one_wave(g);
    }
    return g;
}

// Per-shape plan autotuning (mid M, where the tensor-bound plans differ by up
// to ~20% between shapes: CTA pairs at 2 CTAs/SM, pairs with a deep 1-CTA/SM
// ring, the persistent pair kernel, single-CTA tiles, pairs with <= 128-token
// tiles; opt-in: pairs with up to 512-token tiles as two MMA sub-tiles, the
// pair split-K plan with 4 splits, weight multicast). The first eager
// encounter of (M, N, K, epilogue) times every distinct candidate plan on
// the engine stream (3 launches each, same inputs; a residual-add epilogue is
// timed as an fp32 store into scratch, every other epilogue is idempotent)
// and caches the fastest; the heuristic plan is kept unless a candidate
// beats it by > 2%. Never during graph capture (the cached choice is used
// there), never below TLT_GEMM_AUTOTUNE_MIN_M rows.
int Engine::tuned_variant(const bf16* X, int M, int K, long long ldx, const CUtensorMap& tmW, int N,
                          const EpiParams& ep_in) {
    static const int on = env_int("TLT_GEMM_AUTOTUNE", 1);
    static const int min_m = env_int("TLT_GEMM_AUTOTUNE_MIN_M", 128);
    if (!on || M < min_m || ep_in.norm_w || ep_in.row_scale) return 0;
    const auto key = std::make_tuple(M, N, K, (int)ep_in.kind);
    // TLT_GEMM_AUTOTUNE_CACHE=path: decisions persisted across processes
    // (lines "M N K epilogue variant"); a profiler run (ncu replays every
    // launch, so in-process timings are meaningless there) reuses the plans
    // an unprofiled run chose
    static const char* cache_path = std::getenv("TLT_GEMM_AUTOTUNE_CACHE");
    if (cache_path && !tune_cache_loaded_) {
        tune_cache_loaded_ = true;
        if (FILE* f = std::fopen(cache_path, "r")) {
            int m, n, k, kind, v;
            while (std::fscanf(f, "%d %d %d %d %d", &m, &n, &k, &kind, &v) == 5)
                gemm_variant_[std::make_tuple(m, n, k, kind)] = v;
            std::fclose(f);
        }
    }
    auto it = gemm_variant_.find(key);
    if (it != gemm_variant_.end()) return it->second;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CUDA_CHECK(cudaStreamIsCapturing(st_, &cs));
    if (cs != cudaStreamCaptureStatusNone) return 0;
    EpiParams e = ep_in;
    e.n_out = N;
    e.m_tok = M;
    e.dyn_n = nullptr;
    if (e.kind == EPI_RESID_ADD) {
        if ((size_t)M * N > (size_t)R_ * cfg.vocab) return 0;
        e.kind = EPI_F32;
        e.out_f32 = logits_;
        e.ld_f32 = N;
    }
    std::vector<GemmPlan> plans;
    std::vector<int> vars;
    // variants 6 (pair split-K x4), 7 (weight multicast) and 8 (512-token
    // tiles as two MMA sub-tiles) are kept for experiments
    // (TLT_GEMM_FORCE_VARIANT / tests) but not autotuned: they win on too few
    // shapes in isolation (profiles/r2_gemm_variants.txt, r2_gemm_multicast.txt,
    // r2_gemm_variant8.txt) and 8 (1 CTA/SM, all 512 TMEM columns) lost
    // ~2% of rollout throughput where the tuner took it (down-proj, M = 288)
    static const bool all_variants = env_int("TLT_GEMM_AUTOTUNE_ALL", 0) != 0;
    for (int v : {0, 1, 2, 3, 4, 8, 6, 7}) {
        if (!all_variants && (v == 6 || v == 7 || v == 8)) continue;
        const GemmPlan g = make_plan(M, N, K, (int)ep_in.kind, v);
        bool dup = false;
        for (const auto& q : plans) dup = dup || q.same_as(g);
        if (!dup) {
            plans.push_back(g);
            vars.push_back(v);
        }
    }
    int best = 0;
    if (plans.size() > 1) {
        if (!tune_ev0_) {  // own events: ev0_/ev1_ may be bracketing the step being run
            CUDA_CHECK(cudaEventCreate(&tune_ev0_));
            CUDA_CHECK(cudaEventCreate(&tune_ev1_));
        }
        std::vector<float> t(plans.size());
        for (size_t i = 0; i < plans.size(); ++i) {
            const CUtensorMap& tx = tmap_act(X, M, K, ldx, plans[i].box_rows);
            launch_gemm(plans[i], tmW, tx, e, ws_, ws_elems_, st_);  // warm
            CUDA_CHECK(cudaEventRecord(tune_ev0_, st_));
            for (int r = 0; r < 3; ++r) launch_gemm(plans[i], tmW, tx, e, ws_, ws_elems_, st_);
            CUDA_CHECK(cudaEventRecord(tune_ev1_, st_));
            CUDA_CHECK(cudaEventSynchronize(tune_ev1_));
            CUDA_CHECK(cudaEventElapsedTime(&t[i], tune_ev0_, tune_ev1_));
        }
        size_t bi = 0;
        for (size_t i = 1; i < plans.size(); ++i)
            if (t[i] < t[bi]) bi = i;
        if (bi != 0 && t[0] <= 1.02f * t[bi]) bi = 0;
        best = vars[bi];
        if (std::getenv("TLT_GEMM_AUTOTUNE_LOG")) {
            std::fprintf(stderr, "[tlt] autotune M=%d N=%d K=%d kind=%d:", M, N, K, (int)ep_in.kind);
            for (size_t i = 0; i < plans.size(); ++i) std::fprintf(stderr, " v%d=%.1fus", vars[i], t[i] * 1e3f / 3);
            std::fprintf(stderr, " -> v%d\n", best);
        }
    }
    gemm_variant_[key] = best;
    if (cache_path)
        if (FILE* f = std::fopen(cache_path, "a")) {
            std::fprintf(f, "%d %d %d %d %d\n", M, N, K, (int)ep_in.kind, best);
            std::fclose(f);
        }
    return best;
}

void Engine::gemm(const bf16* X, int M, int K, long long ldx, const CUtensorMap& tmW, int N, const EpiParams& ep_in) {
    const GemmPlan g = make_plan(M, N, K, (int)ep_in.kind, tuned_variant(X, M, K, ldx, tmW, N, ep_in));
    const CUtensorMap& tx = tmap_act(X, M, K, ldx, g.box_rows);
    EpiParams ep = ep_in;
    ep.n_out = N;
    ep.m_tok = M;
    set_dyn(ep, M);
    launch_gemm(g, tmW, tx, ep, ws_, ws_elems_, st_);
    count_launch(1);  // split-K reduction happens inside the same launch (cluster DSMEM)
}

// Bucketed graphs: inside a step sequence padded to b_hi requests, every
// GEMM over b_hi x rpr request-major rows skips the token tiles of the
// padding requests (the live count is uploaded with the step inputs).
void Engine::set_dyn(EpiParams& e, int M) const {
    if (dyn_b_hi_ > 0 && M % dyn_b_hi_ == 0) {
        e.dyn_n = d_nreal_;
        e.dyn_rpr = M / dyn_b_hi_;
    }
}

// x_ += X W^T, then h_ = bf16(rmsnorm(x_) * norm_w) when norm_w != null. The
// residual add is the GEMM epilogue (after the in-cluster split-K reduction at
// long-tail M); the norm of few rows spreads each row over an 8-CTA cluster.
void Engine::gemm_resid_norm(const bf16* X, int M, int K, long long ldx, const CUtensorMap& tmW, const bf16* norm_w) {
    const int d = cfg.hidden;
    EpiParams e{};
    e.n_out = d;
    e.m_tok = M;
    e.kind = EPI_RESID_ADD;
    e.out_f32 = x_;
    e.ld_f32 = d;
    const GemmPlan g = make_plan(M, d, K, EPI_RESID_ADD, tuned_variant(X, M, K, ldx, tmW, d, e));
    const CUtensorMap& tx = tmap_act(X, M, K, ldx, g.box_rows);
    set_dyn(e, M);
    static const int fuse_max_m = [] {
        // off by default: the serial tail of the electing CTA measured slower
        // than the 8-CTA cluster norm kernel under PDL (profiles/r1_*)
        const char* v = std::getenv("TLT_FUSED_NORM_MAX_M");
        return v ? std::atoi(v) : 0;
    }();
    if (norm_w && M <= fuse_max_m && g.pair == 1 && !g.persist) {
        // long-tail M: the GEMM's last CTA normalises the updated rows
        e.norm_w = norm_w;
        e.norm_out = h_;
        e.norm_eps = cfg.rms_eps;
        launch_gemm(g, tmW, tx, e, ws_, ws_elems_, st_);
        count_launch();
        return;
    }
    launch_gemm(g, tmW, tx, e, ws_, ws_elems_, st_);
    count_launch();
    if (norm_w) {
        static const int cluster_norm_max_m = [] {
            const char* v = std::getenv("TLT_CLUSTER_NORM_MAX_M");
            return v ? std::atoi(v) : 256;
        }();
        if (M <= cluster_norm_max_m)
            launch_reduce_resid_norm(nullptr, 0, 0, M, d, x_, norm_w, cfg.rms_eps, h_, st_);
        else
            launch_rmsnorm(x_, M, d, norm_w, cfg.rms_eps, h_, st_);
        count_launch();
    }
}

void Engine::attention(const bf16* kc, const bf16* vc, int cache_cap, const Rows& rw, const Groups& gp, int rpr,
                       int ngroups, int max_keys, const void* pf, long long pf_bytes) {
    AttnParams p{};
    p.pf = pf;
    p.pf_bytes = pf_bytes;
    p.q = q_;
    p.out = attn_;
    p.kc = kc;
    p.vc = vc;
    p.rows = rw;
    p.g = gp;
    p.rows_per_req = rpr;
    p.n_groups = ngroups;
    p.H = cfg.heads;
    p.KV = cfg.kv_heads;
    p.hd = cfg.head_dim;
    p.cap = cache_cap;
    p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)cfg.head_dim));
    p.impl = attn_impl_;
    attention_plan_splits(p, max_keys);  // per-request split sizing; grid covers the max_keys bound
    p.qv_cap = rpr * (cfg.heads / cfg.kv_heads);
    const size_t need = (size_t)ngroups * p.max_splits * p.qv_cap * cfg.kv_heads;
    if (need * cfg.head_dim > aws_elems_ || need > aws_elems_ / 32)
        throw CudaError("attention workspace too small (set TLT_ATTN_WS_MFLOATS)");
    p.ws_m = aws_m_;
    p.ws_l = aws_l_;
    p.ws_o = aws_o_;
    static const int fused_combine = [] {
        // -1 (auto): only for flash-decode with >= 128 (request, KV head)
        // pairs — there the last CTA's merge beats the separate combine
        // launch (b=32: 28.7 -> 27.1 us per layer), while at b <= 8 and on the
        // tree kernels the serial merge is slower (b=1: 16.7 -> 18.5 us;
        // rollout 5072 vs 5604 tok/s with it on everywhere;
        // profiles/r1_attn_dec_fused_combine_sweep.txt). 1 = always, 0 = never.
        const char* v = std::getenv("TLT_ATTN_FUSED_COMBINE");
        return v ? std::atoi(v) : -1;
    }();
    const bool use_fc = fused_combine > 0 || (fused_combine < 0 && p.dec && ngroups * cfg.kv_heads >= 128);
    if (use_fc && p.impl == 1) {
        if (!attn_counters_) {
            attn_counters_ = dmalloc<int>(1 << 16);
            CUDA_CHECK(cudaMemset(attn_counters_, 0, sizeof(int) << 16));
        }
        const long long n_qt = (p.rows_per_req * (cfg.heads / cfg.kv_heads) + 15) / 16;
        if ((long long)ngroups * cfg.kv_heads * n_qt <= (1 << 16)) p.counters = attn_counters_;
    }
    if (attention_tma_enabled(p)) {
        if (attention_tree_tc_eligible(p))
            launch_attention_tree_tc(tmap_kv(kc, cache_cap), tmap_kv(vc, cache_cap), p, st_);
        else
            launch_attention_tma(tmap_kv(kc, cache_cap), tmap_kv(vc, cache_cap), p, st_);
        count_launch(p.counters || p.max_splits == 1 ? 1 : 2);
        return;
    }
    launch_attention(p, st_);
    count_launch(p.counters || (p.dec && p.max_splits == 1) ? 1 : 2);
}

// TMA map of one KV cache ([max_slots][KV][cap][hd] bf16), cached per base pointer
const CUtensorMap& Engine::tmap_kv(const bf16* base, int cache_cap) {
    char key[64];
    std::snprintf(key, sizeof key, "kv/%p/%d", (const void*)base, cache_cap);
    auto it = tmaps_.find(key);
    if (it == tmaps_.end())
        it = tmaps_.emplace(key, make_tmap_kv(base, (long long)cfg.max_slots * cfg.kv_heads * cache_cap, cfg.head_dim))
                 .first;
    return it->second;
}

// One decoder layer over R rows (residual x_ in place).
void Engine::layer_forward(const LayerW& w, bf16* kc, bf16* vc, int cache_cap, const Rows& rw, const Groups& gp,
                           int R, int rpr, int ngroups, int max_keys, bool h_ready, const bf16* next_norm) {
    const int d = cfg.hidden, hd = cfg.head_dim;
    const int nq = cfg.heads * hd, nkv = cfg.kv_heads * hd;
    if (!h_ready) {
        launch_rmsnorm(x_, R, d, w.attn_norm, cfg.rms_eps, h_, st_);
        count_launch();
    }
    EpiParams e{};
    e.kind = EPI_QKV;
    e.out_bf16 = q_;
    e.ld_bf16 = nq;
    e.bias = w.qkv_b;
    e.rope_cos = rope_cos_;
    e.rope_sin = rope_sin_;
    e.tok_pos = rw.pos;
    e.tok_slot = rw.slot;
    e.tok_cidx = rw.cidx;
    e.kcache = kc;
    e.vcache = vc;
    e.n_q = nq;
    e.n_kvr = nkv;
    e.head_dim = hd;
    e.n_kv = cfg.kv_heads;
    e.max_ctx = cache_cap;
    gemm(h_, R, d, d, w.tm_qkv, nq + 2 * nkv, e);
    // TLT_L2PF_O=1: the attention kernel warms L2 with W_o (HBM is mostly
    // idle during the latency-bound attention). Off: measured -0.5% on the
    // rollout (contends with the KV stream at b >= 32, no gain at small b)
    static const int l2pf_o = [] {
        const char* v = std::getenv("TLT_L2PF_O");
        return v ? std::atoi(v) : 0;
    }();
    attention(kc, vc, cache_cap, rw, gp, rpr, ngroups, max_keys, l2pf_o ? w.o : nullptr, (long long)d * nq * 2);
    gemm_resid_norm(attn_, R, nq, nq, w.tm_o, w.mlp_norm);  // x += o W_o^T; h = norm(x)
    EpiParams s{};
    s.kind = EPI_SWIGLU;
    s.out_bf16 = act_;
    s.ld_bf16 = cfg.ffn;
    gemm(h_, R, d, d, w.tm_gu, 2 * cfg.ffn, s);
    gemm_resid_norm(act_, R, cfg.ffn, cfg.ffn, w.tm_down, next_norm);  // x += a W_down^T; h = next norm
}

void Engine::lm_head(const float* x, int n, float* logits, bool h_ready) {
    if (!h_ready) {
        launch_rmsnorm(x, n, cfg.hidden, final_norm_, cfg.rms_eps, h_, st_);
        count_launch();
    }
    EpiParams e{};
    e.kind = EPI_F32;
    e.out_f32 = logits;
    e.ld_f32 = cfg.vocab;
    gemm(h_, n, cfg.hidden, cfg.hidden, tm_lm_, cfg.vocab, e);
}

// Final norm + LM head with the fused top-k epilogue (EPI_TOPK) and the
// per-row merge: writes tk_tok_/tk_logit_ [n][k], tk_M_, tk_S_. The fp32
// logits are only materialized for the parity exports (want_logits).
// Drafter LM head over h_ (normalised rows) -> logits_ [n][V] fp32: bf16
// tcgen05 GEMM, or e4m3 (kind::f8f6f4) with per-token / per-vocab-row scales
// when the drafter runs its LM head in FP8.
void Engine::drafter_logits(int n) {
    EpiParams f{};
    f.kind = EPI_F32;
    f.out_f32 = logits_;
    f.ld_f32 = cfg.vocab;
    if (!drafter_fp8_) {
        gemm(h_, n, cfg.hidden, cfg.hidden, tm_lm_, cfg.vocab, f);
        return;
    }
    const int d = cfg.hidden;
    if (!h8_) {
        h8_ = dmalloc<uint8_t>((size_t)std::max(R_, Rmeta_) * d);
        h8_s_ = dmalloc<float>((size_t)std::max(R_, Rmeta_));
    }
    launch_quant_rows_e4m3(h_, n, d, d, h8_, h8_s_, st_);
    count_launch();
    GemmPlan g = plan_gemm_e4m3(n, cfg.vocab, d);
    char key[96];
    std::snprintf(key, sizeof key, "e4m3/%p/%d/%d", (void*)h8_, n, g.box_rows);
    auto it = tmaps_.find(key);
    if (it == tmaps_.end()) it = tmaps_.emplace(key, make_tmap_e4m3(h8_, n, d, d, g.box_rows)).first;
    f.n_out = cfg.vocab;
    f.m_tok = n;
    f.row_scale = lm8_s_;
    f.tok_scale = h8_s_;
    set_dyn(f, n);
    launch_gemm(g, tm_lm8_, it->second, f, ws_, ws_elems_, st_);
    count_launch();
}

void Engine::drafter_lm_head(const float* x, int n) {
    launch_rmsnorm(x, n, cfg.hidden, final_norm_, cfg.rms_eps, h_, st_);
    count_launch();
    drafter_logits(n);
}

void Engine::lm_topk(const float* x, int n, int k, const int* live, bool want_logits, bool h_ready, bool drafter) {
    if (!h_ready) {
        launch_rmsnorm(x, n, cfg.hidden, final_norm_, cfg.rms_eps, h_, st_);
        count_launch();
    }
    if (drafter && drafter_fp8_) {
        drafter_logits(n);
        const int nch = launch_row_topk_chunked(logits_, n, cfg.vocab, live, k, topk_part_, st_);
        launch_topk_merge(topk_part_, nch, n, k, live, tk_tok_, tk_logit_, tk_M_, tk_S_, st_);
        count_launch(2);
        return;
    }
    static const int fused_k = [] {
        const char* v = std::getenv("TLT_FUSED_TOPK_K");
        return v ? std::atoi(v) : 1;
    }();
    if (k > 1 && (k > fused_k || want_logits)) {
        // top-k > 1 (drafter children): fp32 logits + multi-CTA chunked top-k
        EpiParams f{};
        f.kind = EPI_F32;
        f.out_f32 = logits_;
        f.ld_f32 = cfg.vocab;
        gemm(h_, n, cfg.hidden, cfg.hidden, tm_lm_, cfg.vocab, f);
        const int nch = launch_row_topk_chunked(logits_, n, cfg.vocab, live, k, topk_part_, st_);
        launch_topk_merge(topk_part_, nch, n, k, live, tk_tok_, tk_logit_, tk_M_, tk_S_, st_);
        count_launch(2);
        return;  // logits_ already materialized for the parity exports
    }
    EpiParams e{};
    e.kind = EPI_TOPK;
    e.out_f32 = topk_part_;
    e.topk_k = k;
    e.topk_thr = k > 1 ? topk_thr_ : nullptr;
    gemm(h_, n, cfg.hidden, cfg.hidden, tm_lm_, cfg.vocab, e);
    const int n_tiles = (cfg.vocab + 127) / 128;
    launch_topk_merge(topk_part_, n_tiles, n, k, live, tk_tok_, tk_logit_, tk_M_, tk_S_, st_, e.topk_thr);
    count_launch();
    if (want_logits) {
        EpiParams f{};
        f.kind = EPI_F32;
        f.out_f32 = logits_;
        f.ld_f32 = cfg.vocab;
        gemm(h_, n, cfg.hidden, cfg.hidden, tm_lm_, cfg.vocab, f);
    }
}

void Engine::target_forward(const Rows& rw, const Groups& gp, int R, int rpr, int ngroups, int max_keys,
                            float* logits, bf16* feat) {
    if (R > R_) throw ConfigErr("rows", "forward exceeds TLT_MAX_ROWS");
    launch_embed(rw, R, embed_, cfg.hidden, x_, st_);
    count_launch();
    // each layer's down-proj epilogue normalizes for the next layer (the last
    // one with the final norm, leaving h_ ready for the LM head)
    for (int l = 0; l < cfg.layers; ++l)
        layer_forward(layers_[l], kc_[l], vc_[l], cap_, rw, gp, R, rpr, ngroups, max_keys, l > 0,
                      l + 1 < cfg.layers ? layers_[l + 1].attn_norm : final_norm_);
    if (feat) {
        launch_to_bf16(x_, (long long)R * cfg.hidden, feat, st_);
        count_launch();
    }
    if (logits) lm_head(x_, R, logits, true);
}

void Engine::drafter_forward(const Rows& rw, const Groups& gp, int R, int rpr, int ngroups, int max_keys,
                             const int* gather, int n_lm, int k, const int* live, bool want_logits, bf16* dfeat_out) {
    if (R > R_) throw ConfigErr("rows", "drafter forward exceeds TLT_MAX_ROWS");
    const int d = cfg.hidden;
    launch_draft_in(rw, R, embed_, d, feat_hist_, dfeat_, x2_, st_);
    count_launch();
    EpiParams e{};
    e.kind = EPI_F32;
    e.out_f32 = x_;
    e.ld_f32 = d;
    gemm(x2_, R, 2 * d, 2 * d, tm_fc_, d, e);
    layer_forward(drafter_, dkc_, dvc_, dcap_, rw, gp, R, rpr, ngroups, max_keys, false,
                  (k > 0 && !gather) ? final_norm_ : nullptr);
    if (dfeat_out) {
        launch_to_bf16(x_, (long long)R * d, dfeat_out, st_);
        count_launch();
    }
    if (k > 0) {
        if (gather) {
            launch_gather_rows(x_, gather, n_lm, d, xg_, st_);
            count_launch();
            lm_topk(xg_, n_lm, k, live, want_logits, false, true);
        } else {
            lm_topk(x_, n_lm, k, live, want_logits, true, true);
        }
    }
}

__global__ void k_scatter_feat(Rows rows, int d, const __nv_bfloat16* __restrict__ feat, __nv_bfloat16* hist, int cap) {
    pdl_wait();
    const int r = blockIdx.x;
    const int slot = rows.slot[r];
    if (slot < 0) return;
    const long long dst = ((long long)slot * cap + rows.pos[r]) * d;
    for (int e = threadIdx.x; e < d; e += blockDim.x) hist[dst + e] = feat[(long long)r * d + e];
}

void Engine::scatter_features(const Rows& rw, int R, const bf16* feat) {
    launch_pdl(k_scatter_feat, R, 256, 0, st_, rw, cfg.hidden, feat, feat_hist_, cap_);
    CUDA_CHECK(cudaGetLastError());
    count_launch();
}

void Engine::upload_rows_host(const std::vector<int>& tok, const std::vector<int>& pos, const std::vector<int>& slot,
                              const std::vector<int>& cidx, const std::vector<int>& fkind,
                              const std::vector<long long>& fidx, const std::vector<uint32_t>& mask,
                              const std::vector<int>& gslot, const std::vector<int>& glc, const std::vector<int>& gt0,
                              const std::vector<int>& gnt) {
    const size_t n = tok.size(), g = gslot.size();
    auto up = [&](void* dst, const void* src, size_t bytes) {
        CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st_));
    };
    up(prows_.tok, tok.data(), n * 4);
    up(prows_.pos, pos.data(), n * 4);
    up(prows_.slot, slot.data(), n * 4);
    up(prows_.cidx, cidx.data(), n * 4);
    up(prows_.fkind, fkind.data(), n * 4);
    up(prows_.fidx, fidx.data(), n * 8);
    up(prows_.mask, mask.data(), n * kMaskWords * 4);
    up(pg_.slot, gslot.data(), g * 4);
    up(pg_.lc, glc.data(), g * 4);
    up(pg_.tail0, gt0.data(), g * 4);
    up(pg_.ntail, gnt.data(), g * 4);
    CUDA_CHECK(cudaStreamSynchronize(st_));  // host vectors are freed on return
}

// ------------------------------------------------------------------ prefill
// Positions 0..len-2 of each prompt through the target (KV + features), then
// the drafter over the same positions with inputs (f_{p-1}, e(x_p)). The last
// prompt token is the first step's root.
void Engine::prefill(int b, const int32_t* slots, const int32_t* lens, const int32_t* tokens) {
    draft_slots_.clear();
    std::vector<int> off(b + 1, 0);
    for (int i = 0; i < b; ++i) {
        if (slots[i] < 0 || slots[i] >= cfg.max_slots) throw ConfigErr("slot_ids", "slot out of range");
        if (lens[i] < 1) throw ConfigErr("lens", "prompt must hold >= 1 token");
        if (lens[i] + 1 > cfg.max_ctx) throw ConfigErr("lens", "prompt exceeds max_ctx");
        off[i + 1] = off[i] + lens[i];
    }
    CUDA_CHECK(cudaEventRecord(ev0_, st_));
    // token histories
    for (int i = 0; i < b; ++i)
        CUDA_CHECK(cudaMemcpyAsync(tok_hist_ + (size_t)slots[i] * cap_, tokens + off[i], sizeof(int32_t) * lens[i],
                                   cudaMemcpyHostToDevice, st_));
    // rows per request per forward: the longest prompt (no padding rows for
    // short prompts), at most 512 so several requests share each GEMM
    int longest = 1;
    for (int i = 0; i < b; ++i) longest = std::max(longest, lens[i] - 1);
    const int chunk = std::max(16, std::min({512, std::max(1, R_ / 2), (longest + 15) / 16 * 16}));
    // process requests in groups; each group forward has stride = chunk rows per request
    for (int i0 = 0; i0 < b;) {
        int nreq = std::max(1, std::min(b - i0, R_ / chunk));
        const int i1 = i0 + nreq;
        int max_rows = 0;
        for (int i = i0; i < i1; ++i) max_rows = std::max(max_rows, lens[i] - 1);
        for (int c0 = 0; c0 < max_rows; c0 += chunk) {
            const int R = nreq * chunk;
            std::vector<int> tok(R, 0), pos(R, 0), slot(R, -1), cidx(R, 0), fk(R, 0), gs(nreq, -1), glc(nreq, 0),
                gt0(nreq, 0), gnt(nreq, 0);
            std::vector<long long> fidx(R, 0);
            std::vector<uint32_t> mask((size_t)R * kMaskWords, 0u);
            for (int q = 0; q < nreq; ++q) {
                const int i = i0 + q, s = slots[i], n = lens[i] - 1;
                const int cn = std::max(0, std::min(chunk, n - c0));
                gs[q] = cn > 0 ? s : -1;
                glc[q] = c0;
                gt0[q] = c0;
                gnt[q] = cn;
                for (int j = 0; j < cn; ++j) {
                    const int r = q * chunk + j, p = c0 + j;
                    tok[r] = tokens[off[i] + p];
                    pos[r] = p;
                    slot[r] = s;
                    cidx[r] = p;
                    fk[r] = p > 0 ? 1 : 0;
                    fidx[r] = (long long)s * cap_ + p - 1;
                    for (int t = 0; t <= j; ++t) mask[(size_t)r * kMaskWords + (t >> 5)] |= 1u << (t & 31);
                }
            }
            upload_rows_host(tok, pos, slot, cidx, fk, fidx, mask, gs, glc, gt0, gnt);
            target_forward(prows_, pg_, R, chunk, nreq, c0 + chunk, nullptr, feat_);
            scatter_features(prows_, R, feat_);
            drafter_forward(prows_, pg_, R, chunk, nreq, c0 + chunk, nullptr, 0, 0, nullptr, false, nullptr);
        }
        i0 = i1;
    }
    CUDA_CHECK(cudaEventRecord(ev1_, st_));
    CUDA_CHECK(cudaEventSynchronize(ev1_));
    CUDA_CHECK(cudaEventElapsedTime(&last_prefill_ms, ev0_, ev1_));
    for (int i = 0; i < b; ++i) {
        lt_[slots[i]] = lens[i] - 1;
        ld_[slots[i]] = lens[i] - 1;
        live_[slots[i]] = 1;
    }
}

void Engine::release(int slot) {
    if (slot < 0 || slot >= cfg.max_slots) throw ConfigErr("slot_id", "out of range");
    live_[slot] = 0;
    lt_[slot] = ld_[slot] = 0;
}

// Drafter weights (spot training): the trainable tensors of
// the EAGLE drafter (fc + its decoder layer) and the shared frozen ones, as
// device views the trainer updates in place. Every captured graph and tensor
// map keeps pointing at the same buffers, so a publish needs no re-capture.
std::vector<tlt_tensor_view> Engine::drafter_tensors() {
    const int64_t d = cfg.hidden, nq = (int64_t)cfg.heads * cfg.head_dim, nkv = (int64_t)cfg.kv_heads * cfg.head_dim,
                  F = cfg.ffn, V = cfg.vocab;
    std::vector<tlt_tensor_view> v = {
        {"fc", fc_, d, 2 * d, 1},
        {"attn_norm", drafter_.attn_norm, 1, d, 1},
        {"qkv", drafter_.qkv, nq + 2 * nkv, d, 1},
        {"o", drafter_.o, d, nq, 1},
        {"mlp_norm", drafter_.mlp_norm, 1, d, 1},
        {"gate_up", drafter_.gu, 2 * F, d, 1},
        {"down", drafter_.down, d, F, 1},
        {"embed", embed_, V, d, 0},
        {"final_norm", final_norm_, 1, d, 0},
        {"lm_head", lm_head_, V, d, 0},
    };
    if (drafter_.qkv_b) v.insert(v.begin() + 3, tlt_tensor_view{"qkv_bias", drafter_.qkv_b, 1, nq + 2 * nkv, 1});
    return v;
}

// After new drafter weights were published: drop the drafter KV of every live
// slot (it was computed with the old weights; the next EAGLE step's catch-up
// recomputes it from the committed target features) and bump the version.
void Engine::drafter_published(int64_t version) {
    CUDA_CHECK(cudaStreamSynchronize(st_));
    for (int s = 0; s < cfg.max_slots; ++s)
        if (live_[s]) ld_[s] = 0;
    drafter_version_ = version;
}

// Shorten a live slot's committed state to `len` positions (token len becomes
// the pending root): the rollout trims requests whose last step committed KV
// past the emission cut (EOS / max_len) before the sequence is exported.
void Engine::truncate(int slot, int len) {
    if (slot < 0 || slot >= cfg.max_slots || !live_[slot]) throw ConfigErr("slot_id", "slot not live");
    if (len < 0 || len > lt_[slot]) throw ConfigErr("len", "beyond the committed length");
    lt_[slot] = len;
    ld_[slot] = std::min(ld_[slot], len);
}

int Engine::export_sequence(int slot, int32_t* tokens, int max_tokens, void* features, size_t features_bytes) {
    if (slot < 0 || slot >= cfg.max_slots || !live_[slot]) throw ConfigErr("slot_id", "slot not live");
    const int n = lt_[slot];  // positions with committed KV / target features; token n is the pending root
    if (tokens) {
        if (max_tokens < n + 1) throw ConfigErr("max_tokens", "buffer smaller than slot_len + 1");
        CUDA_CHECK(cudaMemcpyAsync(tokens, tok_hist_ + (size_t)slot * cap_, sizeof(int32_t) * (n + 1),
                                   cudaMemcpyDefault, st_));
    }
    if (features) {
        const size_t bytes = sizeof(bf16) * (size_t)n * cfg.hidden;
        if (features_bytes < bytes) throw ConfigErr("features_bytes", "buffer smaller than slot_len x hidden x 2");
        CUDA_CHECK(cudaMemcpyAsync(features, feat_hist_ + (size_t)slot * cap_ * cfg.hidden, bytes, cudaMemcpyDefault,
                                   st_));
    }
    CUDA_CHECK(cudaStreamSynchronize(st_));
    return n;
}

// Drafter catch-up (after plain-decode steps): committed positions [ld, lt)
// with target features, chunked. The SD graph then sees exactly 1 + accepted
// pending rows per request.
float Engine::catchup_drafter(int b, const int32_t* slots) {
    // Batched like prefill: several requests per drafter forward, each with a
    // static stride of `chunk` rows; committed prefix [0, ld) + causal block.
    // Returns the device time (CUDA events), counted in the step's elapsed.
    std::vector<int> pend(b), from(b);
    int longest = 1;
    for (int i = 0; i < b; ++i) {
        from[i] = ld_[slots[i]];
        pend[i] = lt_[slots[i]] - ld_[slots[i]];
        longest = std::max(longest, pend[i]);
    }
    const int chunk = std::max(16, std::min({512, std::max(1, R_ / 2), (longest + 15) / 16 * 16}));
    // all pending tokens in one D2H pass
    std::vector<std::vector<int32_t>> htok(b);
    for (int i = 0; i < b; ++i) {
        htok[i].resize(std::max(1, pend[i]));
        if (pend[i] > 0)
            CUDA_CHECK(cudaMemcpyAsync(htok[i].data(), tok_hist_ + (size_t)slots[i] * cap_ + from[i],
                                       sizeof(int32_t) * pend[i], cudaMemcpyDeviceToHost, st_));
    }
    CUDA_CHECK(cudaStreamSynchronize(st_));
    CUDA_CHECK(cudaEventRecord(ev0_, st_));
    const int per_fwd = std::max(1, R_ / chunk);
    for (int i0 = 0; i0 < b; i0 += per_fwd) {
        const int nreq = std::min(per_fwd, b - i0);
        int rows_max = 0;
        for (int q = 0; q < nreq; ++q) rows_max = std::max(rows_max, pend[i0 + q]);
        for (int c0 = 0; c0 < rows_max; c0 += chunk) {
            const int R = nreq * chunk;
            std::vector<int> tok(R, 0), pos(R, 0), slot(R, -1), cidx(R, 0), fk(R, 0), gs(nreq, -1), glc(nreq, 0),
                gt0(nreq, 0), gnt(nreq, 0);
            std::vector<long long> fidx(R, 0);
            std::vector<uint32_t> mask((size_t)R * kMaskWords, 0u);
            int max_keys = 1;
            for (int q = 0; q < nreq; ++q) {
                const int i = i0 + q, s = slots[i];
                const int cn = std::max(0, std::min(chunk, pend[i] - c0));
                const int base = from[i] + c0;
                gs[q] = cn > 0 ? s : -1;
                glc[q] = base;
                gt0[q] = base;
                gnt[q] = cn;
                max_keys = std::max(max_keys, base + chunk);
                for (int j = 0; j < cn; ++j) {
                    const int r = q * chunk + j, p = base + j;
                    tok[r] = htok[i][c0 + j];
                    pos[r] = cidx[r] = p;
                    slot[r] = s;
                    fk[r] = p > 0 ? 1 : 0;
                    fidx[r] = (long long)s * cap_ + p - 1;
                    for (int t = 0; t <= j; ++t) mask[(size_t)r * kMaskWords + (t >> 5)] |= 1u << (t & 31);
                }
            }
            upload_rows_host(tok, pos, slot, cidx, fk, fidx, mask, gs, glc, gt0, gnt);
            drafter_forward(prows_, pg_, R, chunk, nreq, max_keys, nullptr, 0, 0, nullptr, false, nullptr);
        }
    }
    CUDA_CHECK(cudaEventRecord(ev1_, st_));
    CUDA_CHECK(cudaEventSynchronize(ev1_));
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, ev0_, ev1_));
    for (int i = 0; i < b; ++i) ld_[slots[i]] += pend[i];
    return ms;
}

// Batch bucket of an SD step (capture_plan.hpp:64-70,103-122): the step is
// padded to the hi end of the pool bucket holding b whose captured graphs
// verify T tokens; outside the pool (or without one) the exact batch.
int Engine::bucket_hi_for(int b, int T) const {
    for (const auto& pb : pool_)
        if (b >= pb.lo && b <= pb.hi && std::find(pb.Ts.begin(), pb.Ts.end(), T) != pb.Ts.end())
            return std::min(pb.hi, max_b_);
    return b;
}

// Plain-decode batch bucket: the smallest pooled size >= b (sizes 1, 2, 4, 8,
// then multiples of 8, as serving engines pad decode graphs), else exact b.
int Engine::ar_bucket_for(int b) const {
    for (int s : ar_sizes_)
        if (s >= b) return s;
    return b;
}


// ------------------------------------------------------------ kernel probe
// kernel probes (bench rooflines): best of this many timed passes
constexpr int kProbePasses = 5;

// Live per-kernel timing on the engine stream with the engine's own weights:
// `iters` launches of one GEMM site over successive layers (every launch
// streams a different weight matrix from HBM, as in a real forward), CUDA
// events around the whole sequence. Activations are whatever the buffers
// hold (values do not change the timing). kind: 0 gate_up (+SwiGLU), 1 qkv
// (+bias/RoPE/KV write into slot 0), 2 down (+residual), 3 bf16 LM head fp32
// logits, 4 LM head + fused top-1 (verify / decode), 5 o-proj (+residual),
// 6 the drafter's LM head as configured (e4m3 when drafter_lm_fp8).
float Engine::probe_kernel(int kind, int M, int iters, double* bytes, double* flops) {
    if (M < 1 || M > R_) throw ConfigErr("M", "out of range for the activation buffers");
    const int d = cfg.hidden, L = cfg.layers;
    const int nq = cfg.heads * cfg.head_dim, nkv = cfg.kv_heads * cfg.head_dim;
    long long N = 0, K = 0;
    // The engine replays its GEMMs inside CUDA graphs (PDL edges between
    // kernels): the probe does the same -- one eager pass (plans, autotuner,
    // tensor maps, first touch), the `iters` launches captured once, and the
    // best of kProbePasses timed replays (power-capped clocks move single
    // replays). Eager timing would add the host launch rate to small kernels.
    auto seq = [&] {
        for (int it = 0; it < iters; ++it) {
            const LayerW& w = layers_[it % L];
            EpiParams ep{};
            switch (kind) {
                case 0:
                    ep.kind = EPI_SWIGLU;
                    ep.out_bf16 = act_;
                    ep.ld_bf16 = cfg.ffn;
                    gemm(h_, M, d, d, w.tm_gu, 2 * cfg.ffn, ep);
                    N = 2LL * cfg.ffn;
                    K = d;
                    break;
                case 1:
                    ep.kind = EPI_QKV;
                    ep.out_bf16 = q_;
                    ep.ld_bf16 = nq;
                    ep.bias = w.qkv_b;
                    ep.rope_cos = rope_cos_;
                    ep.rope_sin = rope_sin_;
                    ep.tok_pos = prows_.pos;
                    ep.tok_slot = prows_.slot;
                    ep.tok_cidx = prows_.cidx;
                    ep.kcache = kc_[it % L];
                    ep.vcache = vc_[it % L];
                    ep.n_q = nq;
                    ep.n_kvr = nkv;
                    ep.head_dim = cfg.head_dim;
                    ep.n_kv = cfg.kv_heads;
                    ep.max_ctx = cap_;
                    gemm(h_, M, d, d, w.tm_qkv, nq + 2 * nkv, ep);
                    N = nq + 2LL * nkv;
                    K = d;
                    break;
                case 2: {
                    GemmPlan g = plan_gemm(M, d, cfg.ffn);
                    const CUtensorMap& tx = tmap_act(act_, M, cfg.ffn, cfg.ffn, g.box_rows);
                    ep.kind = EPI_RESID_ADD;
                    ep.n_out = d;
                    ep.m_tok = M;
                    ep.out_f32 = x_;
                    ep.ld_f32 = d;
                    launch_gemm(g, w.tm_down, tx, ep, ws_, ws_elems_, st_);
                    N = d;
                    K = cfg.ffn;
                } break;
                case 5: {  // o-proj + residual
                    GemmPlan g = plan_gemm(M, d, nq);
                    const CUtensorMap& tx = tmap_act(attn_, M, nq, nq, g.box_rows);
                    ep.kind = EPI_RESID_ADD;
                    ep.n_out = d;
                    ep.m_tok = M;
                    ep.out_f32 = x_;
                    ep.ld_f32 = d;
                    launch_gemm(g, w.tm_o, tx, ep, ws_, ws_elems_, st_);
                    N = d;
                    K = nq;
                } break;
                case 3:
                    ep.kind = EPI_F32;
                    ep.out_f32 = logits_;
                    ep.ld_f32 = cfg.vocab;
                    gemm(h_, M, d, d, tm_lm_, cfg.vocab, ep);
                    N = cfg.vocab;
                    K = d;
                    break;
                case 6:  // the drafter's LM head as configured (bf16 or e4m3 incl. activation quantisation)
                    drafter_logits(M);
                    N = cfg.vocab;
                    K = d;
                    break;
                default:
                    ep.kind = EPI_TOPK;
                    ep.out_f32 = topk_part_;
                    ep.topk_k = 1;
                    gemm(h_, M, d, d, tm_lm_, cfg.vocab, ep);
                    N = cfg.vocab;
                    K = d;
                    break;
            }
        }
    };
    seq();
    CUDA_CHECK(cudaStreamSynchronize(st_));
    cudaGraph_t gr;
    CUDA_CHECK(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
    seq();
    CUDA_CHECK(cudaStreamEndCapture(st_, &gr));
    cudaGraphExec_t ex;
    CUDA_CHECK(cudaGraphInstantiate(&ex, gr, 0));
    CUDA_CHECK(cudaGraphDestroy(gr));
    float ms = 3.4e38f;
    for (int rep = 0; rep <= kProbePasses; ++rep) {  // warm replay, then the best of kProbePasses timed
        CUDA_CHECK(cudaEventRecord(ev0_, st_));
        CUDA_CHECK(cudaGraphLaunch(ex, st_));
        CUDA_CHECK(cudaEventRecord(ev1_, st_));
        CUDA_CHECK(cudaEventSynchronize(ev1_));
        float t = 0.f;
        CUDA_CHECK(cudaEventElapsedTime(&t, ev0_, ev1_));
        if (rep > 0) ms = std::min(ms, t);
    }
    CUDA_CHECK(cudaGraphExecDestroy(ex));
    const double out_b = kind == 0 ? (double)M * N / 2 * 2 : kind == 1 ? (double)M * N * 2
                         : (kind == 2 || kind == 5) ? (double)M * N * 8 : kind == 6 ? (double)M * N * 4 : kind == 3 ? (double)M * N * 4 : (double)M * 16;
    // the e4m3 drafter LM head streams one byte per weight + one fp32 scale per row
    const double w_b = (kind == 6 && drafter_fp8_) ? (double)N * K + (double)N * 4 : (double)N * K * 2;
    if (bytes) *bytes = w_b + (double)M * K * 2 + out_b;
    if (flops) *flops = 2.0 * M * N * K;
    return ms / iters;
}


// Live timing of the engine's attention (tree-masked flash-decode + split
// combine) over successive layers' caches: b requests with ctx committed keys
// and rpr query rows each (rpr = 1: plain decode; T + 1: tree verify with a
// chain mask). Cache contents are whatever the buffers hold.
float Engine::probe_attention(int b, int ctx, int rpr, int iters, double* bytes) {
    if (b < 1 || b > cfg.max_slots || rpr < 1 || b * rpr > R_ || ctx + rpr + 1 > cap_ || rpr > 32 * kMaskWords)
        throw ConfigErr("probe", "attention probe shape out of range");
    const int R = b * rpr;
    std::vector<int> tok(R, 1), pos(R), slot(R), cidx(R), fk(R, 0), gs(b), glc(b), gt0(b), gnt(b);
    std::vector<long long> fidx(R, 0);
    std::vector<uint32_t> mask((size_t)R * kMaskWords, 0u);
    for (int i = 0; i < b; ++i) {
        gs[i] = i;
        glc[i] = ctx;
        gt0[i] = ctx;
        gnt[i] = rpr;
        for (int j = 0; j < rpr; ++j) {
            const int r = i * rpr + j;
            pos[r] = cidx[r] = ctx + j;
            slot[r] = i;
            for (int t = 0; t <= j; ++t) mask[(size_t)r * kMaskWords + (t >> 5)] |= 1u << (t & 31);
        }
    }
    upload_rows_host(tok, pos, slot, cidx, fk, fidx, mask, gs, glc, gt0, gnt);
    // the engine replays its attention launches inside CUDA graphs (PDL
    // edges between kernels): the probe does the same — eager warm-up, then
    // the `iters` launches captured once and the graph replay timed
    auto seq = [&] {
        for (int it = 0; it < iters; ++it) {
            const int l = it % cfg.layers;
            attention(kc_[l], vc_[l], cap_, prows_, pg_, rpr, b, cap_);  // grid sized as in the engine
        }
    };
    seq();
    CUDA_CHECK(cudaStreamSynchronize(st_));
    cudaGraph_t g;
    CUDA_CHECK(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
    seq();
    CUDA_CHECK(cudaStreamEndCapture(st_, &g));
    cudaGraphExec_t ex;
    CUDA_CHECK(cudaGraphInstantiate(&ex, g, 0));
    CUDA_CHECK(cudaGraphDestroy(g));
    float ms = 3.4e38f;
    for (int rep = 0; rep <= kProbePasses; ++rep) {  // warm replay, then the best of kProbePasses timed
        CUDA_CHECK(cudaEventRecord(ev0_, st_));
        CUDA_CHECK(cudaGraphLaunch(ex, st_));
        CUDA_CHECK(cudaEventRecord(ev1_, st_));
        CUDA_CHECK(cudaEventSynchronize(ev1_));
        float t = 0.f;
        CUDA_CHECK(cudaEventElapsedTime(&t, ev0_, ev1_));
        if (rep > 0) ms = std::min(ms, t);
    }
    CUDA_CHECK(cudaGraphExecDestroy(ex));
    const double kv = (double)b * (ctx + rpr) * cfg.kv_heads * cfg.head_dim * 2 * 2;
    const double qo = (double)R * cfg.heads * cfg.head_dim * 2 * 2;
    if (bytes) *bytes = kv + qo;
    return ms / iters;
}

// ----------------------------------------------------------- SD device seq
// draft (D levels) -> tree final -> verify forward -> argmax -> accept ->
// commit. All shapes static in (b_hi, D, k, T); per-step data lives on the
// device (StepIn uploaded first), so the sequence is graph-capturable.
void Engine::sd_device_sequence(int b_hi, int D, int k, int T, bool dbg, int b_real, bool verify) {
    (void)b_real;
    const int d = cfg.hidden, V = cfg.vocab, D1 = D + 1;
    CUDA_CHECK(cudaMemcpyAsync(d_step_, h_step_, sizeof(StepIn) * b_hi, cudaMemcpyHostToDevice, st_));
    CUDA_CHECK(cudaMemcpyAsync(d_nreal_, h_nreal_, sizeof(int), cudaMemcpyHostToDevice, st_));
    DynScope dyn(this, b_hi);
    std::vector<int> base, Fd, lmoff;
    level_plan(b_hi, D, k, T, base, Fd, lmoff);
    if (D >= 2 && base[D] + b_hi * Fd[D] > Rmeta_) throw ConfigErr("strategy", "draft rows exceed TLT_MAX_DRAFT_ROWS");
    const int max_keys_d = dcap_;
    launch_rows_level1(d_step_, b_hi, b_hi, D1, drows_, dg_[1], root_row_, tok_hist_, cap_, st_);
    count_launch();
    TreeParams tp{};
    tp.step = d_step_;
    tp.b = b_hi;
    tp.b_hi = b_hi;
    tp.D = D;
    tp.k = k;
    tp.T = T;
    tp.arena = arena_;
    tp.arena_cap = arena_cap_;
    tp.arena_n = arena_n_;
    tp.kept = kept_;
    tp.kept_n = kept_n_;
    tp.exp_n = exp_n_;
    tp.done = done_;
    tp.row_node = row_node_;
    tp.root_row = root_row_;
    tp.tk_tok = tk_tok_;
    tp.tk_logit = tk_logit_;
    tp.tk_M = tk_M_;
    tp.tk_S = tk_S_;
    tp.rows = drows_;
    tp.tree_tok = tree_tok_;
    tp.tree_par = tree_par_;
    tp.tree_dep = tree_dep_;
    tp.tree_prob = tree_prob_;
    tp.tree_pp = tree_pp_;
    tp.tree_n = tree_n_;
    tp.vrows = vrows_;
    tp.vg = vg_;
    tp.tok_hist = tok_hist_;
    tp.cap = cap_;
    auto d2d = [&](void* dst, const void* src, size_t bytes) {
        CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st_));
    };
    for (int lv = 1; lv <= D; ++lv) {
        const int R = b_hi * Fd[lv];
        const Rows rw = sub(drows_, base[lv]);
        const int n_lm = lv == 1 ? b_hi : R;
        drafter_forward(rw, dg_[lv], R, Fd[lv], b_hi, max_keys_d, lv == 1 ? root_row_ : nullptr, n_lm, k,
                        lv == 1 ? dg_[1].slot : rw.slot, dbg, dfeat_ + (size_t)base[lv] * d);
        if (dbg) {
            // parity export: this level's fp32 logits, row max / normaliser and
            // liveness, copied on the stream (graph-capturable, no host sync)
            d2d(dbg_lg_ + (size_t)lmoff[lv] * V, logits_, sizeof(float) * (size_t)n_lm * V);
            d2d(dbg_M_ + lmoff[lv], tk_M_, sizeof(float) * n_lm);
            d2d(dbg_S_ + lmoff[lv], tk_S_, sizeof(float) * n_lm);
            d2d(dbg_live_ + lmoff[lv], lv == 1 ? dg_[1].slot : rw.slot, sizeof(int) * n_lm);
        }
        tp.level = lv;
        tp.lvl_base = base[lv];
        tp.lm_F = lv == 1 ? 1 : Fd[lv];
        tp.nxt_base = lv < D ? base[lv + 1] : 0;
        tp.nxt_F = lv < D ? Fd[lv + 1] : 0;
        tp.g_next = dg_[std::min(lv + 1, kMaxDepth + 1)];
        launch_tree_level(tp, st_);
        count_launch();
    }
    launch_tree_final(tp, st_);
    count_launch();
    if (dbg) {
        d2d(dbg_arena_, arena_, sizeof(Cand) * (size_t)b_hi * arena_cap_);
        d2d(dbg_node_, row_node_, sizeof(int) * (size_t)(base[D] + b_hi * Fd[D]));
    }
    if (verify) verify_accept_commit(b_hi, T, dbg, b_real);
    else tree_to_host(b_hi, T);
}

// Target verify over root + the final tree (rows written by k_tree_final),
// argmax, verify_greedy, KV compaction, results into pinned host memory.
void Engine::verify_accept_commit(int b_hi, int T, bool dbg, int b_real) {
    const int d = cfg.hidden, V = cfg.vocab;
    const int max_keys_t = cap_;
    const int T1 = T + 1, RV = b_hi * T1;
    target_forward(vrows_, vg_, RV, T1, b_hi, max_keys_t, nullptr, feat_);
    lm_topk(x_, RV, 1, vrows_.slot, dbg, true);  // argmax per verify row (fused epilogue + merge)
    if (dbg)  // verify logits (fp32, from the same LM-head GEMM) for the parity export
        CUDA_CHECK(cudaMemcpyAsync(dbg_vlg_, logits_, sizeof(float) * (size_t)RV * V, cudaMemcpyDeviceToDevice, st_));
    (void)b_real;
    AcceptParams ap{};
    ap.step = d_step_;
    ap.b = b_hi;
    ap.b_hi = b_hi;
    ap.T = T;
    ap.maxD = kMaxD;
    ap.tree_tok = tree_tok_;
    ap.tree_par = tree_par_;
    ap.tree_n = tree_n_;
    ap.argmax = tk_tok_;  // top-1 of each verify row
    ap.acc_nodes = acc_nodes_;
    ap.acc_tok = acc_tok_;
    ap.acc_len = acc_len_;
    ap.bonus = bonus_;
    launch_accept_greedy(ap, st_);
    count_launch();
    CommitParams cp{};
    cp.step = d_step_;
    cp.b = b_hi;
    cp.b_hi = b_hi;
    cp.maxD = kMaxD;
    cp.layers = cfg.layers;
    cp.KV = cfg.kv_heads;
    cp.hd = cfg.head_dim;
    cp.cap = cap_;
    cp.d = d;
    cp.row_stride = T1;
    cp.kc = d_kc_arr_;
    cp.vc = d_vc_arr_;
    cp.acc_nodes = acc_nodes_;
    cp.acc_tok = acc_tok_;
    cp.acc_len = acc_len_;
    cp.bonus = bonus_;
    cp.tok_hist = tok_hist_;
    cp.feat_hist = feat_hist_;
    cp.vfeat = feat_;
    cp.kv_len = kv_len_;
    launch_commit(cp, st_);
    count_launch();
    // results -> pinned host
    auto d2h = [&](void* dst, const void* src, size_t bytes) {
        CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st_));
    };
    d2h(ho_.acc_len, acc_len_, sizeof(int) * b_hi);
    d2h(ho_.bonus, bonus_, sizeof(int) * b_hi);
    d2h(ho_.acc_tok, acc_tok_, sizeof(int) * b_hi * kMaxD);
    d2h(ho_.acc_nodes, acc_nodes_, sizeof(int) * b_hi * kMaxD);
    tree_to_host(b_hi, T);
}

void Engine::tree_to_host(int b_hi, int T) {
    auto d2h = [&](void* dst, const void* src, size_t bytes) {
        CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st_));
    };
    d2h(ho_.tree_tok, tree_tok_, sizeof(int) * b_hi * T);
    d2h(ho_.tree_par, tree_par_, sizeof(int) * b_hi * T);
    d2h(ho_.tree_dep, tree_dep_, sizeof(int) * b_hi * T);
    d2h(ho_.tree_prob, tree_prob_, sizeof(double) * b_hi * T);
    d2h(ho_.tree_pp, tree_pp_, sizeof(double) * b_hi * T);
    d2h(ho_.tree_n, tree_n_, sizeof(int) * b_hi);
}

int Engine::prepare_tree_step(const tlt_strategy& s, int b, const int32_t* slots, float* catchup_ms) {
    const int D = s.draft_depth, k = s.top_k, T = s.tokens_to_verify;
    if (D < 1) throw ConfigErr("draft_depth", "must be >= 1");
    if (k < 1) throw ConfigErr("top_k", "must be >= 1");
    if (T < 1) throw ConfigErr("tokens_to_verify", "must be >= 1");
    {  // capacity (spec_decode.hpp:25-42)
        long long total = 0, level = 1;
        for (int i = 0; i < D && total < (1LL << 40); ++i) {
            level = std::min(level * k, 1LL << 40);
            total += level;
        }
        if (T > total) throw ConfigErr("tokens_to_verify", "exceeds tree capacity for (top_k, draft_depth)");
    }
    if (D > kMaxD - 1 || k > kMaxTopK || T > kMaxT) throw ConfigErr("strategy", "exceeds engine limits (D<=15,k<=8,T<=128)");
    if ((long long)(D - 1) * T + 1 > kMaskWords * 32) throw ConfigErr("strategy", "too many drafter expansions");
    if ((long long)k * std::min(T, (int)std::min<long long>(1LL << 20, (long long)std::pow(k, D - 1))) > 1024 ||
        T + (long long)k * T > 2048)
        throw ConfigErr("strategy", "frontier too large");
    if (b < 1 || b > max_b_) throw ConfigErr("batch", "out of range");
    for (int i = 0; i < b; ++i) {
        const int sl = slots[i];
        if (sl < 0 || sl >= cfg.max_slots || !live_[sl]) throw ConfigErr("slot_ids", "slot not prefilled");
        if (lt_[sl] + T + 2 > cap_ - 1 || lt_[sl] + 1 + (D - 1) * T + 2 > dcap_) throw ConfigErr("max_ctx", "context full");
    }
    // drafter catch-up for requests whose pending rows exceed the graph stride
    // (after plain-decode steps); its device time is part of the step's
    *catchup_ms = 0.f;
    {
        std::vector<int32_t> need;
        for (int i = 0; i < b; ++i)
            if (lt_[slots[i]] - ld_[slots[i]] + 1 > D + 1) need.push_back(slots[i]);
        if (!need.empty()) *catchup_ms = catchup_drafter((int)need.size(), need.data());
    }
    const int b_hi = bucket_hi_for(b, T);
    *h_nreal_ = b;
    for (int i = 0; i < b_hi; ++i) {
        if (i < b) {
            const int sl = slots[i];
            if (lt_[sl] - ld_[sl] + 1 > D + 1) {  // only reachable when catch-up was skipped
                throw ConfigErr("drafter", "pending rows exceed draft_depth + 1");
            }
            h_step_[i] = StepIn{sl, lt_[sl], ld_[sl], 0};
        } else {
            h_step_[i] = StepIn{-1, 0, 0, 0};
        }
    }
    return b_hi;
}

// Step results (pinned staging) -> caller arrays ([b][stride] accept arrays,
// [b][T] tree arrays); host mirrors are updated by the caller.
void Engine::copy_step_out(int b, const int32_t* slots, int T, int stride, tlt_tree_out* tree, tlt_accept_out* out) {
    for (int i = 0; i < b; ++i) {
        const int sl = slots[i];
        if (out) {
            const int a = ho_.acc_len[i];
            if (out->accept_len) out->accept_len[i] = a;
            if (out->bonus) out->bonus[i] = ho_.bonus[i];
            for (int j = 0; j < a && j < stride; ++j) {
                if (out->accepted) out->accepted[(size_t)i * stride + j] = ho_.acc_tok[(size_t)i * kMaxD + j];
                if (out->nodes) out->nodes[(size_t)i * stride + j] = ho_.acc_nodes[(size_t)i * kMaxD + j];
                if (out->kv_src) out->kv_src[(size_t)i * stride + j] = ho_.acc_nodes[(size_t)i * kMaxD + j];
            }
            if (out->kv_len) out->kv_len[i] = lt_[sl] + 1 + a;
        }
        if (tree) {
            const int n = ho_.tree_n[i];
            if (tree->n_nodes) tree->n_nodes[i] = n;
            for (int t = 0; t < n; ++t) {
                const size_t o = (size_t)i * T + t;
                if (tree->tokens) tree->tokens[o] = ho_.tree_tok[o];
                if (tree->parents) tree->parents[o] = ho_.tree_par[o];
                if (tree->depths) tree->depths[o] = ho_.tree_dep[o];
                if (tree->probs) tree->probs[o] = ho_.tree_prob[o];
                if (tree->path_probs) tree->path_probs[o] = ho_.tree_pp[o];
            }
        }
    }
}

float Engine::sd_step(const tlt_strategy& s, int b, const int32_t* slots, tlt_tree_out* tree, tlt_accept_out* out) {
    const int D = s.draft_depth, k = s.top_k, T = s.tokens_to_verify;
    draft_slots_.clear();
    float catchup_ms = 0.f;
    const int b_hi = prepare_tree_step(s, b, slots, &catchup_ms);
    const bool dbg = debug_;
    if (dbg) ensure_debug_buffers(b_hi, D, k, T);  // may drop debug graphs: before the lookup
    CUDA_CHECK(cudaEventRecord(ev0_, st_));
    // debug steps replay their own graphs (the production sequence plus the
    // parity-export copy nodes), keyed apart from the production ones
    auto key = std::make_tuple(b_hi, D, k, T, dbg ? 4 : 0);
    auto it = graphs_.find(key);
    if (use_graphs && it != graphs_.end()) {
        CUDA_CHECK(cudaGraphLaunch(it->second.first, st_));
        launches += it->second.second;
    } else {
        launches_in_seq_ = 0;
        sd_device_sequence(b_hi, D, k, T, dbg, b);
        launches += launches_in_seq_;
    }
    CUDA_CHECK(cudaEventRecord(ev1_, st_));
    CUDA_CHECK(cudaEventSynchronize(ev1_));
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, ev0_, ev1_));
    ms += catchup_ms;
    if (dbg) {
        level_plan(b_hi, D, k, T, dbgs_.base, dbgs_.Fd, dbgs_.lmoff);
        dbgs_.valid = dbgs_.greedy = true;
        dbgs_.b_hi = b_hi;
        dbgs_.b_real = b;
        dbgs_.D = D;
        dbgs_.T = T;
        dbgs_.meta_rows = dbgs_.base[D] + b_hi * dbgs_.Fd[D];
        dbg_cache_.clear();
    }
    // capture for the next replay (after a successful eager run)
    if (use_graphs && it == graphs_.end()) capture_graph(key, false);
    copy_step_out(b, slots, T, D, tree, out);
    for (int i = 0; i < b; ++i) {  // host mirrors
        const int sl = slots[i];
        ld_[sl] = lt_[sl] + 1;
        lt_[sl] = lt_[sl] + 1 + ho_.acc_len[i];
    }
    if (out && out->elapsed_ms) out->elapsed_ms[0] = ms;
    return ms;
}

// Split boundary, propose half: the drafter levels + tree selection of the
// fused step (sd_device_sequence without the verify tail), eager. Nothing is
// committed to the target; the drafter's KV of the pending committed rows is
// (idempotently) rewritten. The device tree stays resident for
// verify_tree(tree == nullptr).
float Engine::draft(const tlt_strategy& s, int b, const int32_t* slots, tlt_tree_out* tree) {
    const int D = s.draft_depth, k = s.top_k, T = s.tokens_to_verify;
    draft_slots_.clear();
    float catchup_ms = 0.f;
    const int b_hi = prepare_tree_step(s, b, slots, &catchup_ms);
    CUDA_CHECK(cudaEventRecord(ev0_, st_));
    launches_in_seq_ = 0;
    sd_device_sequence(b_hi, D, k, T, false, b, /*verify=*/false);
    launches += launches_in_seq_;
    CUDA_CHECK(cudaEventRecord(ev1_, st_));
    CUDA_CHECK(cudaEventSynchronize(ev1_));
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, ev0_, ev1_));
    copy_step_out(b, slots, T, 0, tree, nullptr);
    draft_slots_.assign(slots, slots + b);
    draft_lt_.resize(b);
    for (int i = 0; i < b; ++i) draft_lt_[i] = lt_[slots[i]];
    draft_T_ = T;
    draft_D_ = D;
    return ms + catchup_ms;
}

// Split boundary, verify half: verify_greedy + KV commit of the engine's
// own last draft (tree == nullptr) or of caller trees, uploaded into the
// tree arena as each request's kept list (arena index = rank) so k_tree_final
// builds the verify rows / ancestor masks exactly as for a drafted tree.
float Engine::verify_tree(int b, const int32_t* slots, const tlt_tree_in* tree, tlt_accept_out* out) {
    if (b < 1 || b > max_b_) throw ConfigErr("batch", "out of range");
    // did the drafter (tlt_draft) process these slots at their current length?
    bool drafted = (int)draft_slots_.size() == b;
    for (int i = 0; drafted && i < b; ++i) drafted = draft_slots_[i] == slots[i] && draft_lt_[i] == lt_[slots[i]];
    if (!tree && !drafted) throw ConfigErr("tree", "no tlt_draft of these slots at their current length");
    const int T = tree ? tree->stride : draft_T_;
    const int stride = tree ? tree->stride : draft_D_;
    if (T < 1 || T > kMaxT) throw ConfigErr("tree.stride", "must be in [1, 128]");
    for (int i = 0; i < b; ++i) {
        const int sl = slots[i];
        if (sl < 0 || sl >= cfg.max_slots || !live_[sl]) throw ConfigErr("slot_ids", "slot not prefilled");
        if (lt_[sl] + T + 2 > cap_ - 1) throw ConfigErr("max_ctx", "context full");
        h_step_[i] = StepIn{sl, lt_[sl], ld_[sl], 0};
    }
    std::vector<Cand> cand;
    std::vector<int> kept, kept_n;
    if (tree) {
        if (!tree->tokens || !tree->parents || !tree->n_nodes) throw ConfigErr("tree", "null node arrays");
        cand.resize((size_t)b * T);
        kept.resize((size_t)b * T);
        kept_n.resize(b);
        for (int i = 0; i < b; ++i) {
            const int n = tree->n_nodes[i];
            if (n < 0 || n > T) throw ConfigErr("tree.n_nodes", "must be in [0, stride]");
            kept_n[i] = n;
            for (int j = 0; j < T; ++j) {
                const size_t o = (size_t)i * T + j;
                Cand c{};
                c.row = c.eslot = -1;
                c.birth = j;
                kept[o] = j;
                if (j < n) {
                    c.token = tree->tokens[o];
                    c.parent = tree->parents[o];
                    if (c.token < 0 || c.token >= cfg.vocab) throw ConfigErr("tree.tokens", "token out of range");
                    if (c.parent < -1 || c.parent >= j)
                        throw ConfigErr("tree.parents", "parent must precede its child (rank order)");
                    c.depth = c.parent < 0 ? 1 : cand[(size_t)i * T + c.parent].depth + 1;
                    if (c.depth > kMaxD - 1) throw ConfigErr("tree", "depth exceeds 15");
                    c.prob = tree->probs ? tree->probs[o] : 1.0;
                    c.pp = tree->path_probs ? tree->path_probs[o] : 1.0;
                }
                cand[o] = c;
            }
        }
    }
    draft_slots_.clear();
    CUDA_CHECK(cudaEventRecord(ev0_, st_));
    launches_in_seq_ = 0;
    CUDA_CHECK(cudaMemcpyAsync(d_step_, h_step_, sizeof(StepIn) * b, cudaMemcpyHostToDevice, st_));
    if (tree) {
        CUDA_CHECK(cudaMemcpy2DAsync(arena_, sizeof(Cand) * arena_cap_, cand.data(), sizeof(Cand) * T,
                                     sizeof(Cand) * T, b, cudaMemcpyHostToDevice, st_));
        CUDA_CHECK(cudaMemcpyAsync(kept_, kept.data(), sizeof(int) * kept.size(), cudaMemcpyHostToDevice, st_));
        CUDA_CHECK(cudaMemcpyAsync(kept_n_, kept_n.data(), sizeof(int) * b, cudaMemcpyHostToDevice, st_));
        TreeParams tp{};
        tp.step = d_step_;
        tp.b = b;
        tp.b_hi = b;
        tp.D = kMaxD - 1;
        tp.k = 1;
        tp.T = T;
        tp.arena = arena_;
        tp.arena_cap = arena_cap_;
        tp.arena_n = arena_n_;
        tp.kept = kept_;
        tp.kept_n = kept_n_;
        tp.exp_n = exp_n_;
        tp.done = done_;
        tp.row_node = row_node_;
        tp.root_row = root_row_;
        tp.rows = drows_;
        tp.tree_tok = tree_tok_;
        tp.tree_par = tree_par_;
        tp.tree_dep = tree_dep_;
        tp.tree_prob = tree_prob_;
        tp.tree_pp = tree_pp_;
        tp.tree_n = tree_n_;
        tp.vrows = vrows_;
        tp.vg = vg_;
        tp.tok_hist = tok_hist_;
        tp.cap = cap_;
        launch_tree_final(tp, st_);
        count_launch();
    }
    verify_accept_commit(b, T, false, b);
    launches += launches_in_seq_;
    CUDA_CHECK(cudaEventRecord(ev1_, st_));
    CUDA_CHECK(cudaEventSynchronize(ev1_));
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, ev0_, ev1_));
    copy_step_out(b, slots, T, stride, nullptr, out);
    for (int i = 0; i < b; ++i) {
        const int sl = slots[i];
        if (drafted) ld_[sl] = lt_[sl] + 1;  // the drafter's KV covers the committed root
        lt_[sl] = lt_[sl] + 1 + ho_.acc_len[i];
    }
    if (out && out->elapsed_ms) out->elapsed_ms[0] = ms;
    return ms;
}

// n-gram fallback branch of run_rollout (rollout.hpp:212-216): the host
// proposes a linear chain per request (chain_from_tokens, spec_decode.hpp:
// 228-240: parent i-1, depth i+1, prob = path_prob = 1); it is written into
// the tree arena as the kept list, and k_tree_final + the common verify tail
// do the rest. Eager (chains are data-dependent host input; one H2D of
// b*D candidates per step).
float Engine::sd_step_chain(int D, int b, const int32_t* slots, const int32_t* chains, const int32_t* lens,
                            tlt_accept_out* out, float temperature, const double* uniforms) {
    if (D < 1 || D > kMaxD - 1 || D > kMaxT) throw ConfigErr("draft_depth", "out of range (1..15)");
    draft_slots_.clear();
    const bool stoch = temperature != 0.f;
    if (stoch && !(temperature > 0.f)) throw ConfigErr("temperature", "must be > 0");
    if (stoch && !uniforms) throw ConfigErr("uniforms", "required");
    if (b < 1 || b > max_b_) throw ConfigErr("batch", "out of range");
    for (int i = 0; i < b; ++i) {
        const int sl = slots[i];
        if (sl < 0 || sl >= cfg.max_slots || !live_[sl]) throw ConfigErr("slot_ids", "slot not prefilled");
        if (lens[i] < 0 || lens[i] > D) throw ConfigErr("chain_lens", "must be in [0, draft_depth]");
        if (lt_[sl] + D + 2 > cap_ - 1) throw ConfigErr("max_ctx", "context full");
        for (int j = 0; j < lens[i]; ++j)
            if (chains[(size_t)i * D + j] < 0 || chains[(size_t)i * D + j] >= cfg.vocab)
                throw ConfigErr("chains", "token out of range");
    }
    const int b_hi = b, T = D;
    for (int i = 0; i < b_hi; ++i) h_step_[i] = StepIn{slots[i], lt_[slots[i]], ld_[slots[i]], 0};
    const int US = 2 * kMaxDepth + 1;
    if (stoch) {
        ensure_stoch_buffers();
        for (int i = 0; i < b_hi; ++i)
            for (int j = 0; j < US; ++j) h_uni_[(size_t)i * US + j] = j < D + 1 ? uniforms[(size_t)i * (D + 1) + j] : 2.0;
    }
    std::vector<Cand> cand((size_t)b_hi * D);
    std::vector<int> kept((size_t)b_hi * D), kept_n(b_hi);
    for (int i = 0; i < b_hi; ++i) {
        kept_n[i] = lens[i];
        for (int j = 0; j < D; ++j) {
            Cand c{};
            c.pp = 1.0;
            c.prob = 1.0;
            c.token = j < lens[i] ? chains[(size_t)i * D + j] : 0;
            c.parent = j - 1;
            c.depth = j + 1;
            c.birth = j;
            c.row = -1;
            c.eslot = -1;
            cand[(size_t)i * D + j] = c;
            kept[(size_t)i * D + j] = j;
        }
    }
    CUDA_CHECK(cudaEventRecord(ev0_, st_));
    launches_in_seq_ = 0;
    CUDA_CHECK(cudaMemcpyAsync(d_step_, h_step_, sizeof(StepIn) * b_hi, cudaMemcpyHostToDevice, st_));
    CUDA_CHECK(cudaMemcpy2DAsync(arena_, sizeof(Cand) * arena_cap_, cand.data(), sizeof(Cand) * D, sizeof(Cand) * D,
                                 b_hi, cudaMemcpyHostToDevice, st_));
    CUDA_CHECK(cudaMemcpyAsync(kept_, kept.data(), sizeof(int) * kept.size(), cudaMemcpyHostToDevice, st_));
    CUDA_CHECK(cudaMemcpyAsync(kept_n_, kept_n.data(), sizeof(int) * b_hi, cudaMemcpyHostToDevice, st_));
    if (stoch)
        CUDA_CHECK(cudaMemcpyAsync(d_uni_, h_uni_, sizeof(double) * b_hi * US, cudaMemcpyHostToDevice, st_));
    TreeParams tp{};
    tp.step = d_step_;
    tp.b = b_hi;
    tp.b_hi = b_hi;
    tp.D = D;
    tp.k = 1;
    tp.T = T;
    tp.arena = arena_;
    tp.arena_cap = arena_cap_;
    tp.arena_n = arena_n_;
    tp.kept = kept_;
    tp.kept_n = kept_n_;
    tp.exp_n = exp_n_;
    tp.done = done_;
    tp.row_node = row_node_;
    tp.root_row = root_row_;
    tp.rows = drows_;
    tp.tree_tok = tree_tok_;
    tp.tree_par = tree_par_;
    tp.tree_dep = tree_dep_;
    tp.tree_prob = tree_prob_;
    tp.tree_pp = tree_pp_;
    tp.tree_n = tree_n_;
    tp.vrows = vrows_;
    tp.vg = vg_;
    tp.tok_hist = tok_hist_;
    tp.cap = cap_;
    launch_tree_final(tp, st_);
    count_launch();
    if (stoch)
        stoch_verify_commit(b_hi, D, (double)temperature, debug_, b, nullptr, 0);
    else
        verify_accept_commit(b_hi, T, false, b);
    launches += launches_in_seq_;
    CUDA_CHECK(cudaEventRecord(ev1_, st_));
    CUDA_CHECK(cudaEventSynchronize(ev1_));
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, ev0_, ev1_));
    for (int i = 0; i < b; ++i) {
        const int sl = slots[i];
        const int a = ho_.acc_len[i];
        if (out) {
            if (out->accept_len) out->accept_len[i] = a;
            if (out->bonus) out->bonus[i] = ho_.bonus[i];
            for (int j = 0; j < a; ++j) {
                if (out->accepted) out->accepted[(size_t)i * D + j] = ho_.acc_tok[(size_t)i * kMaxD + j];
                if (out->nodes) out->nodes[(size_t)i * D + j] = ho_.acc_nodes[(size_t)i * kMaxD + j];
                if (out->kv_src) out->kv_src[(size_t)i * D + j] = ho_.acc_nodes[(size_t)i * kMaxD + j];
            }
            if (out->kv_len) out->kv_len[i] = lt_[sl] + 1 + a;
        }
        if (stoch) {
            last_consumed.resize(b);
            last_chain.resize(b);
            last_consumed[i] = h_consumed_[i];
            last_chain[i].assign(chains + (size_t)i * D, chains + (size_t)i * D + lens[i]);
        }
        lt_[sl] = lt_[sl] + 1 + a;  // the drafter did not run: ld_ stays (catch-up on the next EAGLE step)
    }
    if (out && out->elapsed_ms) out->elapsed_ms[0] = ms;
    return ms;
}

void Engine::ar_device_sequence(int b_hi) {
    CUDA_CHECK(cudaMemcpyAsync(d_step_, h_step_, sizeof(StepIn) * b_hi, cudaMemcpyHostToDevice, st_));
    CUDA_CHECK(cudaMemcpyAsync(d_nreal_, h_nreal_, sizeof(int), cudaMemcpyHostToDevice, st_));
    DynScope dyn(this, b_hi);
    launch_rows_ar(d_step_, b_hi, b_hi, prows_, pg_, tok_hist_, cap_, st_);
    count_launch();
    target_forward(prows_, pg_, b_hi, 1, b_hi, cap_, nullptr, feat_);
    lm_topk(x_, b_hi, 1, prows_.slot, debug_, true);
    launch_commit_ar(d_step_, b_hi, tk_tok_, feat_, cfg.hidden, tok_hist_, feat_hist_, cap_, ar_tok_, st_);
    count_launch();
    CUDA_CHECK(cudaMemcpyAsync(ho_.ar_tok, ar_tok_, sizeof(int) * b_hi, cudaMemcpyDeviceToHost, st_));
}

float Engine::ar_step(int b, const int32_t* slots, int32_t* out_tokens) {
    draft_slots_.clear();
    if (b < 1 || b > max_b_) throw ConfigErr("batch", "out of range");
    for (int i = 0; i < b; ++i) {
        const int sl = slots[i];
        if (sl < 0 || sl >= cfg.max_slots || !live_[sl]) throw ConfigErr("slot_ids", "slot not prefilled");
        if (lt_[sl] + 2 > cap_ - 1) throw ConfigErr("max_ctx", "context full");
    }
    const int b_hi = use_graphs && !debug_ ? std::min(ar_bucket_for(b), max_b_) : b;
    for (int i = 0; i < b_hi; ++i) h_step_[i] = i < b ? StepIn{slots[i], lt_[slots[i]], ld_[slots[i]], 0} : StepIn{-1, 0, 0, 0};
    *h_nreal_ = b;
    CUDA_CHECK(cudaEventRecord(ev0_, st_));
    auto key = std::make_tuple(b_hi, 0, 0, 0, 1);
    auto it = graphs_.find(key);
    if (use_graphs && !debug_ && it != graphs_.end()) {
        CUDA_CHECK(cudaGraphLaunch(it->second.first, st_));
        launches += it->second.second;
    } else {
        launches_in_seq_ = 0;
        ar_device_sequence(b_hi);
        launches += launches_in_seq_;
    }
    CUDA_CHECK(cudaEventRecord(ev1_, st_));
    CUDA_CHECK(cudaEventSynchronize(ev1_));
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, ev0_, ev1_));
    if (debug_) {
        dbg_ar_logits.resize((size_t)b * cfg.vocab);
        CUDA_CHECK(cudaMemcpy(dbg_ar_logits.data(), logits_, sizeof(float) * dbg_ar_logits.size(),
                              cudaMemcpyDeviceToHost));
    }
    if (use_graphs && !debug_ && it == graphs_.end()) capture_graph(key, true);
    for (int i = 0; i < b; ++i) {
        if (out_tokens) out_tokens[i] = ho_.ar_tok[i];
        lt_[slots[i]] += 1;
    }
    return ms;
}

// ------------------------------------------------------------ debug export
void Engine::free_debug_buffers() {
    auto f = [](void* p) {
        if (p) cudaFree(p);
    };
    f(dbg_lg_), f(dbg_M_), f(dbg_S_), f(dbg_vlg_), f(dbg_live_), f(dbg_node_), f(dbg_arena_);
    dbg_lg_ = dbg_M_ = dbg_S_ = dbg_vlg_ = nullptr;
    dbg_live_ = dbg_node_ = nullptr;
    dbg_arena_ = nullptr;
    dbg_lg_rows_ = dbg_vlg_rows_ = dbg_meta_rows_ = dbg_arena_reqs_ = 0;
}

void Engine::ensure_debug_buffers(int b_hi, int D, int k, int T) {
    std::vector<int> base, Fd, lmoff;
    level_plan(b_hi, D, k, T, base, Fd, lmoff);
    const size_t lg = lmoff[D + 1], vlg = (size_t)b_hi * (T + 1), meta = base[D] + b_hi * Fd[D];
    if (lg <= dbg_lg_rows_ && vlg <= dbg_vlg_rows_ && meta <= dbg_meta_rows_ && (size_t)b_hi <= dbg_arena_reqs_) return;
    // growing: debug graphs hold the old addresses
    CUDA_CHECK(cudaStreamSynchronize(st_));
    for (auto it = graphs_.begin(); it != graphs_.end();) {
        if (std::get<4>(it->first) == 4) {
            cudaGraphExecDestroy(it->second.first);
            it = graphs_.erase(it);
        } else {
            ++it;
        }
    }
    const size_t nlg = std::max(lg, dbg_lg_rows_), nv = std::max(vlg, dbg_vlg_rows_),
                 nm = std::max(meta, dbg_meta_rows_), na = std::max((size_t)b_hi, dbg_arena_reqs_);
    free_debug_buffers();
    const size_t V = cfg.vocab;
    dbg_lg_ = dmalloc<float>(nlg * V);
    dbg_M_ = dmalloc<float>(nlg);
    dbg_S_ = dmalloc<float>(nlg);
    dbg_live_ = dmalloc<int>(nlg);
    dbg_vlg_ = dmalloc<float>(nv * V);
    dbg_node_ = dmalloc<int>(nm);
    dbg_arena_ = dmalloc<Cand>(na * arena_cap_);
    dbg_lg_rows_ = nlg;
    dbg_vlg_rows_ = nv;
    dbg_meta_rows_ = nm;
    dbg_arena_reqs_ = na;
}

// Expansions of request i in the last debug sd_step, in the order the
// eager export used (level by level, row order): the path from the root
// (arena parents) and the full fp64 drafter row p = exp((double)(l - M)) / S
// computed by k_row_probs from the copied fp32 logits.
const std::vector<DebugExp>& Engine::debug_expansions(int i) {
    if (!dbgs_.valid || !dbgs_.greedy) {
        if (i < 0 || i >= (int)dbg_exp.size()) throw ConfigErr("i", "no debug data for request");
        return dbg_exp[i];
    }
    if (i < 0 || i >= dbgs_.b_real) throw ConfigErr("i", "no debug data for request");
    auto hit = dbg_cache_.find(i);
    if (hit != dbg_cache_.end()) return hit->second;
    const int V = cfg.vocab, D = dbgs_.D;
    std::vector<Cand> ar(arena_cap_);
    CUDA_CHECK(cudaMemcpy(ar.data(), dbg_arena_ + (size_t)i * arena_cap_, sizeof(Cand) * arena_cap_,
                          cudaMemcpyDeviceToHost));
    const int maxF = *std::max_element(dbgs_.Fd.begin() + 1, dbgs_.Fd.begin() + D + 1);
    if (!dbg_probs_) dbg_probs_ = dmalloc<double>((size_t)std::max(R_, 256) * V);
    std::vector<double> rows((size_t)maxF * V);
    std::vector<DebugExp> out;
    for (int lv = 1; lv <= D; ++lv) {
        const int F = lv == 1 ? 1 : dbgs_.Fd[lv];
        const int r0 = lv == 1 ? i : i * F;  // LM rows of request i within the level
        std::vector<int> live(F), node(F, -1);
        CUDA_CHECK(cudaMemcpy(live.data(), dbg_live_ + dbgs_.lmoff[lv] + r0, sizeof(int) * F, cudaMemcpyDeviceToHost));
        if (lv > 1)
            CUDA_CHECK(cudaMemcpy(node.data(), dbg_node_ + dbgs_.base[lv] + r0, sizeof(int) * F,
                                  cudaMemcpyDeviceToHost));
        const size_t lr = dbgs_.lmoff[lv] + r0;
        launch_row_probs(dbg_lg_ + lr * V, F, V, dbg_M_ + lr, dbg_S_ + lr, dbg_probs_, st_);
        CUDA_CHECK(cudaGetLastError());
        CUDA_CHECK(cudaMemcpyAsync(rows.data(), dbg_probs_, sizeof(double) * (size_t)F * V, cudaMemcpyDeviceToHost,
                                   st_));
        CUDA_CHECK(cudaStreamSynchronize(st_));
        for (int r = 0; r < F; ++r) {
            if (live[r] < 0) continue;
            DebugExp ex;
            if (lv > 1) {
                for (int a = node[r]; a >= 0; a = ar[a].parent) ex.path.push_back(ar[a].token);
                std::reverse(ex.path.begin(), ex.path.end());
            }
            ex.row.assign(rows.begin() + (size_t)r * V, rows.begin() + (size_t)(r + 1) * V);
            out.push_back(std::move(ex));
        }
    }
    return dbg_cache_.emplace(i, std::move(out)).first->second;
}

std::vector<float> Engine::debug_verify_logits(int i) {
    if (!dbgs_.valid || !dbgs_.greedy || i < 0 || i >= dbgs_.b_real)
        throw ConfigErr("i", "no debug data for request");
    const size_t V = cfg.vocab, T1 = dbgs_.T + 1;
    std::vector<float> v(T1 * V);
    CUDA_CHECK(cudaMemcpy(v.data(), dbg_vlg_ + (size_t)i * T1 * V, sizeof(float) * v.size(), cudaMemcpyDeviceToHost));
    return v;
}

// Capture one step sequence into an executable graph (the sequence is only
// recorded, not run: device state is unchanged). key = (b_hi, D, k, T, kind):
// kind 0 greedy tree SD step, 4 its debug-export variant, 1 plain decode.
void Engine::capture_graph(const std::tuple<int, int, int, int, int>& key, bool ar) {
    const int b_hi = std::get<0>(key), D = std::get<1>(key), k = std::get<2>(key), T = std::get<3>(key);
    const bool dbg = std::get<4>(key) == 4;
    cudaGraph_t g;
    launches_in_seq_ = 0;
    CUDA_CHECK(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
    try {
        if (ar)
            ar_device_sequence(b_hi);
        else
            sd_device_sequence(b_hi, D, k, T, dbg, b_hi);
    } catch (...) {
        cudaStreamEndCapture(st_, &g);
        throw;
    }
    CUDA_CHECK(cudaStreamEndCapture(st_, &g));
    cudaGraphExec_t ex;
    CUDA_CHECK(cudaGraphInstantiate(&ex, g, 0));
    CUDA_CHECK(cudaGraphDestroy(g));
    auto old = graphs_.find(key);
    if (old != graphs_.end()) cudaGraphExecDestroy(old->second.first);
    graphs_[key] = {ex, launches_in_seq_};
}

// Pre-capture the pool of plan_captures (capture_plan.hpp:87-126): every
// TARGET(bucket, T) x DRAFT(bucket, k, D) pair of a bucket becomes one fused
// step graph keyed (bucket_hi, D, k, T) (within a bucket BEG-MAB routes only
// that bucket's arms, beg_mab.hpp:95-105), captured for the bucket's largest
// batch and replayed for every batch in it (padding requests inert, their
// GEMM tiles skipped). Plain decode gets graphs for padded batch sizes 1, 2,
// 4, 8, 16, 24, ... up to max_slots. Each sequence runs once eagerly with
// every request padding (touches lazily created host state, changes no
// device state) before it is captured. Returns the device memory the pool
// took (cudaMemGetInfo delta; every graph shares the engine's activation
// buffers, so this is the executable graphs' own footprint).
size_t Engine::graph_pool_build(const std::vector<tlt_capture_entry>& entries, bool with_ar) {
    graph_pool_clear();
    for (const auto& e : entries) {
        if (e.bucket_lo < 1 || e.bucket_hi < e.bucket_lo) throw ConfigErr("entries", "bad bucket range");
        PoolBucket* pb = nullptr;
        for (auto& q : pool_)
            if (q.lo == e.bucket_lo && q.hi == e.bucket_hi) pb = &q;
        if (!pb) {
            pool_.push_back(PoolBucket{e.bucket_lo, e.bucket_hi, {}, {}});
            pb = &pool_.back();
        }
        if (e.side == 0) {
            if (std::find(pb->Ts.begin(), pb->Ts.end(), e.tokens_to_verify) == pb->Ts.end())
                pb->Ts.push_back(e.tokens_to_verify);
        } else if (e.side == 1) {
            auto kd = std::make_pair((int)e.top_k, (int)e.draft_depth);
            if (std::find(pb->kd.begin(), pb->kd.end(), kd) == pb->kd.end()) pb->kd.push_back(kd);
        } else {
            throw ConfigErr("entries", "side must be 0 (TARGET) or 1 (DRAFT)");
        }
    }
    if (pool_sub_width_ > 0) {  // sub-buckets of at most pool_sub_width_ batch sizes (same strategies)
        std::vector<PoolBucket> fine;
        for (const auto& pb : pool_)
            for (int lo = pb.lo; lo <= pb.hi; lo += pool_sub_width_)
                fine.push_back(PoolBucket{lo, std::min(pb.hi, lo + pool_sub_width_ - 1), pb.Ts, pb.kd});
        pool_.swap(fine);
    }
    if (with_ar) {
        if (pool_ar_width_ > 0)
            for (int s = pool_ar_width_; s < max_b_ + pool_ar_width_; s += pool_ar_width_) ar_sizes_.push_back(std::min(s, max_b_));
        else
            for (int s = 1; s <= max_b_; s = s < 8 ? 2 * s : s + 8) ar_sizes_.push_back(s);
        if (pool_ar_width_ == 1 || pool_ar_width_ > 1) ar_sizes_.insert(ar_sizes_.begin(), 1);
        std::sort(ar_sizes_.begin(), ar_sizes_.end());
        ar_sizes_.erase(std::unique(ar_sizes_.begin(), ar_sizes_.end()), ar_sizes_.end());
        if (ar_sizes_.empty() || ar_sizes_.back() != max_b_) ar_sizes_.push_back(max_b_);
    }
    CUDA_CHECK(cudaStreamSynchronize(st_));
    size_t free0 = 0, total = 0;
    CUDA_CHECK(cudaMemGetInfo(&free0, &total));
    const auto t0 = std::chrono::steady_clock::now();
    pool_graphs_ = pool_skipped_ = 0;
    auto warm_and_capture = [&](int b_hi, int D, int k, int T, bool ar) {
        for (int i = 0; i < b_hi; ++i) h_step_[i] = StepIn{-1, 0, 0, 0};
        *h_nreal_ = 0;
        launches_in_seq_ = 0;
        if (ar)
            ar_device_sequence(b_hi);
        else
            sd_device_sequence(b_hi, D, k, T, false, 0);
        CUDA_CHECK(cudaStreamSynchronize(st_));
        capture_graph(std::make_tuple(b_hi, ar ? 0 : D, ar ? 0 : k, ar ? 0 : T, ar ? 1 : 0), ar);
        ++pool_graphs_;
    };
    for (const auto& pb : pool_) {
        const int b_hi = std::min(pb.hi, max_b_);
        if (pb.lo > max_b_) continue;
        for (int T : pb.Ts)
            for (const auto& kd : pb.kd) {
                tlt_strategy s{kd.second, kd.first, T};
                try {
                    validate(s);
                } catch (const ConfigErr&) {
                    continue;  // T beyond this (k, D)'s tree capacity: never selected together
                }
                try {
                    warm_and_capture(b_hi, s.draft_depth, s.top_k, T, false);
                } catch (const ConfigErr&) {
                    ++pool_skipped_;  // exceeds the engine's draft-row buffers at this bucket size
                }
            }
    }
    for (int s : ar_sizes_) warm_and_capture(s, 0, 0, 0, true);
    CUDA_CHECK(cudaDeviceSynchronize());
    size_t free1 = 0;
    CUDA_CHECK(cudaMemGetInfo(&free1, &total));
    pool_capture_ms_ = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    pool_bytes_ = free0 > free1 ? free0 - free1 : 0;
    return pool_bytes_;
}

void Engine::graph_pool_clear() {
    cudaStreamSynchronize(st_);
    for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second.first);
    graphs_.clear();
    pool_.clear();
    ar_sizes_.clear();
}

}  // namespace tlt
