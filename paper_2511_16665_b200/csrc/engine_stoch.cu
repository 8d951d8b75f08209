// Engine: rejection-sampling SD step (stochastic linear chains, config 4).
// Reference: build_sampled_chain (spec_decode.hpp:202-223) + verify_stochastic
// (spec_decode.hpp:275-313); uniforms from the request RngStream
// (rollout.hpp:151) uploaded in consumption order: draft_depth chain draws,
// one draw per examined position, one residual/bonus draw.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "engine.h"
#include "pdl.cuh"

namespace tlt {

namespace {
Rows sub_rows(const Rows& r, int base) {
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
template <typename T>
T* dalloc(size_t n) {
    void* p = nullptr;
    CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    return static_cast<T*>(p);
}
}  // namespace

void Engine::stoch_device_sequence(int b_hi, int D, double temperature, bool dbg, int b_real) {
    const int d = cfg.hidden, V = cfg.vocab, D1 = D + 1, US = 2 * kMaxDepth + 1;
    CUDA_CHECK(cudaMemcpyAsync(d_step_, h_step_, sizeof(StepIn) * b_hi, cudaMemcpyHostToDevice, st_));
    CUDA_CHECK(cudaMemcpyAsync(d_uni_, h_uni_, sizeof(double) * b_hi * US, cudaMemcpyHostToDevice, st_));
    launch_rows_level1(d_step_, b_hi, b_hi, D1, drows_, dg_[1], root_row_, tok_hist_, cap_, st_);
    count_launch();
    TreeParams tp{};
    tp.step = d_step_;
    tp.b = b_hi;
    tp.b_hi = b_hi;
    tp.D = D;
    tp.k = 1;
    tp.T = D;
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
    if (dbg) {
        dbg_exp.assign(b_real, {});
        dbgs_.valid = true;
        dbgs_.greedy = false;  // tlt_debug_expansions reads dbg_exp (q rows of the chain)
    }
    // chain levels: one drafter row per request per level (k = 1)
    for (int lv = 1; lv <= D; ++lv) {
        const int base = lv == 1 ? 0 : b_hi * D1 + (lv - 2) * b_hi;
        const int rpr = lv == 1 ? D1 : 1;
        const int R = b_hi * rpr;
        const Rows rw = sub_rows(drows_, base);
        drafter_forward(rw, dg_[lv], R, rpr, b_hi, dcap_, nullptr, 0, 0, nullptr, false, dfeat_ + (size_t)base * d);
        if (lv == 1) {
            launch_gather_rows(x_, root_row_, b_hi, d, xg_, st_);
            count_launch();
            drafter_lm_head(xg_, b_hi);
        } else {
            drafter_lm_head(x_, b_hi);
        }
        launch_chain_sample(logits_, b_hi, V, lv == 1 ? dg_[1].slot : rw.slot, qrows_, lv, kMaxDepth, d_uni_, US,
                            tk_tok_, tk_logit_, tk_M_, tk_S_, st_);
        count_launch();
        if (dbg) {
            std::vector<int> live(b_hi);
            std::vector<double> rows((size_t)b_hi * V);
            CUDA_CHECK(cudaMemcpyAsync(live.data(), lv == 1 ? dg_[1].slot : rw.slot, sizeof(int) * b_hi,
                                       cudaMemcpyDeviceToHost, st_));
            for (int i = 0; i < b_hi; ++i)
                CUDA_CHECK(cudaMemcpyAsync(rows.data() + (size_t)i * V, qrows_ + ((size_t)i * kMaxDepth + lv - 1) * V,
                                           sizeof(double) * V, cudaMemcpyDeviceToHost, st_));
            std::vector<int> tok(b_hi);
            CUDA_CHECK(cudaStreamSynchronize(st_));
            for (int i = 0; i < b_real; ++i) {
                if (live[i] < 0) continue;
                DebugExp ex;  // path filled by the caller from the returned chain
                ex.path.assign(lv - 1, -1);
                ex.row.assign(rows.begin() + (size_t)i * V, rows.begin() + (size_t)(i + 1) * V);
                dbg_exp[i].push_back(std::move(ex));
            }
        }
        tp.level = lv;
        tp.lvl_base = base;
        tp.lm_F = 1;
        tp.nxt_base = lv < D ? b_hi * D1 + (lv - 1) * b_hi : 0;
        tp.nxt_F = lv < D ? 1 : 0;
        tp.g_next = dg_[std::min(lv + 1, kMaxDepth + 1)];
        launch_tree_level(tp, st_);
        count_launch();
    }
    launch_tree_final(tp, st_);
    count_launch();
    stoch_verify_commit(b_hi, D, temperature, dbg, b_real, qrows_, D);
}

// Target verify over root + chain (rows from k_tree_final), verify_stochastic
// with draft rows q (nullptr = one-hot, host n-gram chains) starting at
// uniform cur0, KV commit, results into pinned host memory.
void Engine::stoch_verify_commit(int b_hi, int D, double temperature, bool dbg, int b_real, const double* q,
                                 int cur0) {
    const int d = cfg.hidden, V = cfg.vocab, D1 = D + 1, US = 2 * kMaxDepth + 1;
    // target verify over root + chain: full fp32 logits of every row
    const int RV = b_hi * D1;
    target_forward(vrows_, vg_, RV, D1, b_hi, cap_, nullptr, feat_);
    lm_head(x_, RV, logits_, true);
    launch_accept_stochastic(d_step_, b_hi, D, V, temperature, logits_, q, tree_tok_, tree_n_, d_uni_, US, pbuf_,
                             acc_nodes_, acc_tok_, acc_len_, bonus_, consumed_, kMaxD, D, cur0, st_);
    count_launch();
    if (dbg) {
        // raw target rows along the chain, computed by the accept kernel's own
        // device code (what it tempers), for the oracle-in-the-loop check
        dbg_praw.assign(b_real, {});
        double* raw = nullptr;
        CUDA_CHECK(cudaMalloc(&raw, sizeof(double) * (size_t)RV * V));
        launch_raw_rows(logits_, RV, V, raw, st_);
        std::vector<double> hr((size_t)RV * V);
        CUDA_CHECK(cudaMemcpyAsync(hr.data(), raw, sizeof(double) * hr.size(), cudaMemcpyDeviceToHost, st_));
        CUDA_CHECK(cudaStreamSynchronize(st_));
        CUDA_CHECK(cudaFree(raw));
        for (int i = 0; i < b_real; ++i)
            dbg_praw[i].assign(hr.begin() + (size_t)i * D1 * V, hr.begin() + (size_t)(i + 1) * D1 * V);
    }
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
    cp.row_stride = D1;
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
    auto d2h = [&](void* dst, const void* src, size_t bytes) {
        CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st_));
    };
    d2h(ho_.acc_len, acc_len_, sizeof(int) * b_hi);
    d2h(ho_.bonus, bonus_, sizeof(int) * b_hi);
    d2h(ho_.acc_tok, acc_tok_, sizeof(int) * b_hi * kMaxD);
    d2h(ho_.acc_nodes, acc_nodes_, sizeof(int) * b_hi * kMaxD);
    d2h(ho_.tree_tok, tree_tok_, sizeof(int) * b_hi * D);
    d2h(ho_.tree_n, tree_n_, sizeof(int) * b_hi);
    d2h(h_consumed_, consumed_, sizeof(int) * b_hi);
}

void Engine::ensure_stoch_buffers() {
    if (qrows_) return;
    const int V = cfg.vocab, US = 2 * kMaxDepth + 1;
    qrows_ = dalloc<double>((size_t)cfg.max_slots * kMaxDepth * V);
    pbuf_ = dalloc<double>((size_t)cfg.max_slots * V);
    d_uni_ = dalloc<double>((size_t)cfg.max_slots * US);
    consumed_ = dalloc<int>(cfg.max_slots);
    CUDA_CHECK(cudaMallocHost(&h_uni_, sizeof(double) * cfg.max_slots * US));
    CUDA_CHECK(cudaMallocHost(&h_consumed_, sizeof(int) * cfg.max_slots));
}

void Engine::ar_sample_sequence(int b_hi, double temperature) {
    CUDA_CHECK(cudaMemcpyAsync(d_step_, h_step_, sizeof(StepIn) * b_hi, cudaMemcpyHostToDevice, st_));
    CUDA_CHECK(cudaMemcpyAsync(d_uni_, h_uni_, sizeof(double) * b_hi, cudaMemcpyHostToDevice, st_));
    launch_rows_ar(d_step_, b_hi, b_hi, prows_, pg_, tok_hist_, cap_, st_);
    count_launch();
    target_forward(prows_, pg_, b_hi, 1, b_hi, cap_, nullptr, feat_);
    lm_head(x_, b_hi, logits_, true);
    launch_sample_rows(logits_, b_hi, cfg.vocab, prows_.slot, temperature, d_uni_, pbuf_, argmax_, st_);
    count_launch();
    launch_commit_ar(d_step_, b_hi, argmax_, feat_, cfg.hidden, tok_hist_, feat_hist_, cap_, ar_tok_, st_);
    count_launch();
    CUDA_CHECK(cudaMemcpyAsync(ho_.ar_tok, ar_tok_, sizeof(int) * b_hi, cudaMemcpyDeviceToHost, st_));
}

// Plain decode with sampling (rollout.hpp:247-261 at temperature > 0): one
// uniform per request (sample_token over target_next_dist).
float Engine::ar_step_sampled(int b, const int32_t* slots, float temperature, const double* uniforms,
                              int32_t* out_tokens) {
    draft_slots_.clear();
    if (b < 1 || b > max_b_) throw ConfigErr("batch", "out of range");
    if (!(temperature >= 0.0f)) throw ConfigErr("temperature", "must be >= 0");
    for (int i = 0; i < b; ++i) {
        const int sl = slots[i];
        if (sl < 0 || sl >= cfg.max_slots || !live_[sl]) throw ConfigErr("slot_ids", "slot not prefilled");
        if (lt_[sl] + 2 > cap_ - 1) throw ConfigErr("max_ctx", "context full");
    }
    ensure_stoch_buffers();
    for (int i = 0; i < b; ++i) {
        h_step_[i] = StepIn{slots[i], lt_[slots[i]], ld_[slots[i]], 0};
        h_uni_[i] = uniforms[i];
    }
    CUDA_CHECK(cudaEventRecord(ev0_, st_));
    auto key = std::make_tuple(b, 0, (int)(temperature * 1e6f), 0, 3);
    auto it = graphs_.find(key);
    if (use_graphs && !debug_ && it != graphs_.end()) {
        CUDA_CHECK(cudaGraphLaunch(it->second.first, st_));
        launches += it->second.second;
    } else {
        launches_in_seq_ = 0;
        ar_sample_sequence(b, (double)temperature);
        launches += launches_in_seq_;
    }
    CUDA_CHECK(cudaEventRecord(ev1_, st_));
    CUDA_CHECK(cudaEventSynchronize(ev1_));
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, ev0_, ev1_));
    if (use_graphs && !debug_ && it == graphs_.end()) {
        cudaGraph_t g;
        launches_in_seq_ = 0;
        CUDA_CHECK(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
        try {
            ar_sample_sequence(b, (double)temperature);
        } catch (...) {
            cudaStreamEndCapture(st_, &g);
            throw;
        }
        CUDA_CHECK(cudaStreamEndCapture(st_, &g));
        cudaGraphExec_t ex;
        CUDA_CHECK(cudaGraphInstantiate(&ex, g, 0));
        CUDA_CHECK(cudaGraphDestroy(g));
        graphs_[key] = {ex, launches_in_seq_};
    }
    for (int i = 0; i < b; ++i) {
        if (out_tokens) out_tokens[i] = ho_.ar_tok[i];
        lt_[slots[i]] += 1;
    }
    return ms;
}

float Engine::sd_step_stochastic(int D, float temperature, int b, const int32_t* slots, const double* uniforms,
                                 tlt_accept_out* out) {
    draft_slots_.clear();
    if (D < 1 || D > kMaxD - 1) throw ConfigErr("draft_depth", "must be in [1, 15]");
    if (!(temperature > 0.0f)) throw ConfigErr("temperature", "stochastic_linear requires temperature > 0");
    if (b < 1 || b > max_b_) throw ConfigErr("batch", "out of range");
    if (!uniforms) throw ConfigErr("uniforms", "required");
    for (int i = 0; i < b; ++i) {
        const int sl = slots[i];
        if (sl < 0 || sl >= cfg.max_slots || !live_[sl]) throw ConfigErr("slot_ids", "slot not prefilled");
        if (lt_[sl] + D + 2 > cap_ - 1) throw ConfigErr("max_ctx", "context full");
    }
    const int US = 2 * kMaxDepth + 1;
    ensure_stoch_buffers();
    float catchup_ms = 0.f;  // drafter catch-up after plain decode: part of the step's device time
    {
        std::vector<int32_t> need;
        for (int i = 0; i < b; ++i)
            if (lt_[slots[i]] - ld_[slots[i]] + 1 > D + 1) need.push_back(slots[i]);
        if (!need.empty()) catchup_ms = catchup_drafter((int)need.size(), need.data());
    }
    const int b_hi = b;
    for (int i = 0; i < b_hi; ++i) {
        h_step_[i] = StepIn{slots[i], lt_[slots[i]], ld_[slots[i]], 0};
        for (int j = 0; j < US; ++j) h_uni_[(size_t)i * US + j] = j < 2 * D + 1 ? uniforms[(size_t)i * (2 * D + 1) + j] : 2.0;
    }
    CUDA_CHECK(cudaEventRecord(ev0_, st_));
    auto key = std::make_tuple(b_hi, D, (int)(temperature * 1e6f), 0, 2);
    auto it = graphs_.find(key);
    const bool dbg = debug_;
    if (use_graphs && !dbg && it != graphs_.end()) {
        CUDA_CHECK(cudaGraphLaunch(it->second.first, st_));
        launches += it->second.second;
    } else {
        launches_in_seq_ = 0;
        stoch_device_sequence(b_hi, D, (double)temperature, dbg, b);
        launches += launches_in_seq_;
    }
    CUDA_CHECK(cudaEventRecord(ev1_, st_));
    CUDA_CHECK(cudaEventSynchronize(ev1_));
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, ev0_, ev1_));
    ms += catchup_ms;
    if (use_graphs && !dbg && it == graphs_.end()) {
        cudaGraph_t g;
        launches_in_seq_ = 0;
        CUDA_CHECK(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
        try {
            stoch_device_sequence(b_hi, D, (double)temperature, false, b);
        } catch (...) {
            cudaStreamEndCapture(st_, &g);
            throw;
        }
        CUDA_CHECK(cudaStreamEndCapture(st_, &g));
        cudaGraphExec_t ex;
        CUDA_CHECK(cudaGraphInstantiate(&ex, g, 0));
        CUDA_CHECK(cudaGraphDestroy(g));
        graphs_[key] = {ex, launches_in_seq_};
    }
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
        last_consumed.resize(b);
        last_chain.resize(b);
        last_consumed[i] = h_consumed_[i];
        last_chain[i].assign(ho_.tree_tok + (size_t)i * D, ho_.tree_tok + (size_t)i * D + ho_.tree_n[i]);
        ld_[sl] = lt_[sl] + 1;
        lt_[sl] = lt_[sl] + 1 + a;
    }
    if (out && out->elapsed_ms) out->elapsed_ms[0] = ms;
    return ms;
}

}  // namespace tlt
