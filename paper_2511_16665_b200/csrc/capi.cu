// C-ABI of libtlt_b200.so (include/tlt_b200.h): status codes + last error,
// engine lifecycle, steps, graph pool, BEG-MAB / RNG / capture plan, and the
// rollout loop (reference run_rollout, rollout.hpp:130-276).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <deque>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/tlt_b200.h"
#include "capi_types.h"

namespace {
int fail(int code, const char* msg) {
    tlt_set_last_error(msg);
    return code;
}
template <typename F>
int guard(F&& f) {
    try {
        f();
        return TLT_OK;
    } catch (const tlt::ConfigErr& e) {
        return fail(TLT_ERR_CONFIG, e.what());
    } catch (const tlt::RoutingErr& e) {
        return fail(TLT_ERR_ROUTING, e.what());
    } catch (const tlt::CudaError& e) {
        return fail(TLT_ERR_CUDA, e.what());
    } catch (const std::exception& e) {
        return fail(TLT_ERR_INTERNAL, e.what());
    }
}
}  // namespace

extern "C" {

TLT_API int tlt_engine_create(const tlt_model_cfg* cfg, const tlt_init_cfg* init, int device, tlt_engine** out) {
    if (!cfg || !init || !out) return fail(TLT_ERR_CONFIG, "null argument");
    return guard([&] {
        auto* h = new tlt_engine;
        try {
            h->e = std::make_unique<tlt::Engine>(*cfg, *init, device);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

TLT_API void tlt_engine_destroy(tlt_engine* e) { delete e; }

TLT_API int tlt_prefill(tlt_engine* e, int b, const int32_t* slot_ids, const int32_t* lens, const int32_t* tokens) {
    if (!e) return fail(TLT_ERR_STATE, "null engine");
    return guard([&] { e->e->prefill(b, slot_ids, lens, tokens); });
}

TLT_API int tlt_release(tlt_engine* e, int slot_id) {
    if (!e) return fail(TLT_ERR_STATE, "null engine");
    return guard([&] { e->e->release(slot_id); });
}

TLT_API int tlt_export_sequence(tlt_engine* e, int slot_id, int32_t* tokens, int max_tokens, void* features,
                                size_t features_bytes, int32_t* len) {
    if (!e || !len) return fail(TLT_ERR_STATE, "null argument");
    return guard([&] { *len = e->e->export_sequence(slot_id, tokens, max_tokens, features, features_bytes); });
}

// FNV-1a-64 (reference checkpoint.hpp:26-33), for the drafter checkpoints
TLT_API uint64_t tlt_fnv1a64(const void* data, size_t len) {
    const uint8_t* b = static_cast<const uint8_t*>(data);
    uint64_t h = 0xcbf29ce484222325ULL;
    for (size_t i = 0; i < len; ++i) {
        h ^= b[i];
        h *= 0x100000001b3ULL;
    }
    return h;
}

TLT_API int tlt_drafter_tensors(tlt_engine* e, tlt_tensor_view* out, int cap, int32_t* n) {
    if (!e || !n) return fail(TLT_ERR_STATE, "null argument");
    return guard([&] {
        const auto v = e->e->drafter_tensors();
        *n = (int32_t)v.size();
        if (out)
            for (int i = 0; i < (int)v.size() && i < cap; ++i) out[i] = v[i];
    });
}
TLT_API int tlt_drafter_published(tlt_engine* e, int64_t version) {
    if (!e) return fail(TLT_ERR_STATE, "null engine");
    return guard([&] { e->e->drafter_published(version); });
}
TLT_API int tlt_drafter_version(tlt_engine* e, int64_t* version) {
    if (!e || !version) return fail(TLT_ERR_STATE, "null argument");
    *version = e->e->drafter_version_;
    return TLT_OK;
}

TLT_API int tlt_slot_len(tlt_engine* e, int slot_id, int32_t* len) {
    if (!e || !len) return fail(TLT_ERR_STATE, "null argument");
    return guard([&] {
        if (slot_id < 0 || slot_id >= e->e->cfg.max_slots) throw tlt::ConfigErr("slot_id", "out of range");
        *len = e->e->slot_len(slot_id);
    });
}

TLT_API int tlt_sd_step(tlt_engine* e, const tlt_strategy* s, int b, const int32_t* slot_ids, tlt_tree_out* tree,
                        tlt_accept_out* out) {
    if (!e || !s || !slot_ids) return fail(TLT_ERR_STATE, "null argument");
    return guard([&] { e->e->sd_step(*s, b, slot_ids, tree, out); });
}

TLT_API int tlt_draft(tlt_engine* e, const tlt_strategy* s, int b, const int32_t* slot_ids, tlt_tree_out* tree) {
    if (!e || !s || !slot_ids) return fail(TLT_ERR_STATE, "null argument");
    return guard([&] { e->e->draft(*s, b, slot_ids, tree); });
}

TLT_API int tlt_verify_accept_commit(tlt_engine* e, int b, const int32_t* slot_ids, const tlt_tree_in* tree,
                                     tlt_accept_out* out) {
    if (!e || !slot_ids) return fail(TLT_ERR_STATE, "null argument");
    return guard([&] { e->e->verify_tree(b, slot_ids, tree, out); });
}

TLT_API int tlt_sd_step_chain(tlt_engine* e, int draft_depth, int b, const int32_t* slot_ids, const int32_t* chains,
                              const int32_t* chain_lens, tlt_accept_out* out) {
    if (!e || !slot_ids || !chains || !chain_lens) return fail(TLT_ERR_STATE, "null argument");
    return guard([&] { e->e->sd_step_chain(draft_depth, b, slot_ids, chains, chain_lens, out); });
}

TLT_API int tlt_sd_step_chain_stochastic(tlt_engine* e, int draft_depth, float temperature, int b,
                                         const int32_t* slot_ids, const int32_t* chains, const int32_t* chain_lens,
                                         const double* uniforms, tlt_accept_out* out) {
    if (!e || !slot_ids || !chains || !chain_lens || !uniforms) return fail(TLT_ERR_STATE, "null argument");
    if (!(temperature > 0.f)) return fail(TLT_ERR_CONFIG, "temperature: stochastic mode requires t > 0");
    return guard([&] { e->e->sd_step_chain(draft_depth, b, slot_ids, chains, chain_lens, out, temperature, uniforms); });
}

TLT_API int tlt_ngram_create(int n, int continuation_len, tlt_ngram** out) {
    if (!out) return fail(TLT_ERR_CONFIG, "null argument");
    return guard([&] { *out = new tlt_ngram{tlt::Ngram(n, continuation_len)}; });
}
TLT_API void tlt_ngram_destroy(tlt_ngram* g) { delete g; }
TLT_API int tlt_ngram_insert(tlt_ngram* g, const int32_t* response, int len, int64_t step_id) {
    if (!g || (len > 0 && !response) || len < 0) return fail(TLT_ERR_CONFIG, "bad argument");
    return guard([&] { g->g.insert(response, (size_t)len, step_id); });
}
TLT_API int tlt_ngram_extend(tlt_ngram* g, const int32_t* stream, int len, int64_t step_id) {
    if (!g || (len > 0 && !stream) || len < 0) return fail(TLT_ERR_CONFIG, "bad argument");
    return guard([&] { g->g.extend(stream, (size_t)len, step_id); });
}
TLT_API int tlt_ngram_draft(const tlt_ngram* g, const int32_t* ctx, int len, int depth, int32_t* out,
                            int32_t* out_len) {
    if (!g || !out || !out_len || (len > 0 && !ctx) || len < 0) return fail(TLT_ERR_CONFIG, "bad argument");
    return guard([&] {
        auto v = g->g.draft(ctx, (size_t)len, depth);
        std::copy(v.begin(), v.end(), out);
        *out_len = (int32_t)v.size();
    });
}
TLT_API int tlt_ngram_size(const tlt_ngram* g, int64_t* size) {
    if (!g || !size) return fail(TLT_ERR_CONFIG, "null argument");
    *size = (int64_t)g->g.size();
    return 0;
}

TLT_API int tlt_sd_step_stochastic(tlt_engine* e, int draft_depth, float temperature, int b, const int32_t* slot_ids,
                                   const double* uniforms, tlt_accept_out* out) {
    if (!e || !slot_ids) return fail(TLT_ERR_STATE, "null argument");
    return guard([&] { e->e->sd_step_stochastic(draft_depth, temperature, b, slot_ids, uniforms, out); });
}

TLT_API int tlt_debug_target_rows(tlt_engine* e, int i, double* rows, int max_rows, int32_t* n_rows) {
    if (!e) return fail(TLT_ERR_STATE, "null engine");
    return guard([&] {
        auto& E = *e->e;
        if (i < 0 || i >= (int)E.dbg_praw.size()) throw tlt::ConfigErr("i", "no debug data for request");
        const auto& v = E.dbg_praw[i];
        const int V = E.cfg.vocab;
        const int n = (int)(v.size() / V);
        *n_rows = n;
        std::memcpy(rows, v.data(), sizeof(double) * (size_t)std::min(n, max_rows) * V);
    });
}

TLT_API int tlt_debug_chain(tlt_engine* e, int i, int32_t* chain, int32_t* n, int32_t* consumed) {
    if (!e) return fail(TLT_ERR_STATE, "null engine");
    return guard([&] {
        auto& E = *e->e;
        if (i < 0 || i >= (int)E.last_chain.size()) throw tlt::ConfigErr("i", "no stochastic step recorded");
        *n = (int32_t)E.last_chain[i].size();
        for (size_t j = 0; j < E.last_chain[i].size(); ++j) chain[j] = E.last_chain[i][j];
        *consumed = E.last_consumed[i];
    });
}

TLT_API int tlt_ar_step(tlt_engine* e, int b, const int32_t* slot_ids, int32_t* out_tokens, float* elapsed_ms) {
    if (!e || !slot_ids) return fail(TLT_ERR_STATE, "null argument");
    return guard([&] {
        const float ms = e->e->ar_step(b, slot_ids, out_tokens);
        if (elapsed_ms) *elapsed_ms = ms;
    });
}

TLT_API int tlt_graph_pool_build(tlt_engine* e, const tlt_capture_entry* entries, int n, size_t* graph_bytes) {
    if (!e) return fail(TLT_ERR_STATE, "null engine");
    return guard([&] {
        std::vector<tlt_capture_entry> v(entries, entries + n);
        const size_t g = e->e->graph_pool_build(v);
        if (graph_bytes) *graph_bytes = g;
    });
}

TLT_API int tlt_graph_pool_configure(tlt_engine* e, int sub_bucket_width, int ar_width) {
    if (!e) return fail(TLT_ERR_STATE, "null engine");
    return guard([&] {
        if (sub_bucket_width < 0 || ar_width < 0) throw tlt::ConfigErr("width", "must be >= 0");
        e->e->pool_sub_width_ = sub_bucket_width;
        e->e->pool_ar_width_ = ar_width;
    });
}

TLT_API int tlt_graph_pool_stats(tlt_engine* e, int32_t* n_graphs, int32_t* n_skipped, size_t* graph_bytes,
                                 double* build_ms, int32_t* n_live) {
    if (!e) return fail(TLT_ERR_STATE, "null engine");
    return guard([&] {
        if (n_graphs) *n_graphs = e->e->pool_graphs_;
        if (n_skipped) *n_skipped = e->e->pool_skipped_;
        if (graph_bytes) *graph_bytes = e->e->pool_bytes_;
        if (build_ms) *build_ms = e->e->pool_capture_ms_;
        if (n_live) *n_live = e->e->graph_count();
    });
}

TLT_API int tlt_graph_pool_clear(tlt_engine* e) {
    if (!e) return fail(TLT_ERR_STATE, "null engine");
    return guard([&] { e->e->graph_pool_clear(); });
}

TLT_API int tlt_probe_kernel(tlt_engine* e, int kind, int m_tok, int iters, float* avg_ms, double* bytes,
                             double* flops) {
    if (!e || !avg_ms) return fail(TLT_ERR_STATE, "null argument");
    return guard([&] { *avg_ms = e->e->probe_kernel(kind, m_tok, iters < 1 ? 1 : iters, bytes, flops); });
}

TLT_API int tlt_probe_attention(tlt_engine* e, int b, int ctx, int rows_per_req, int iters, float* avg_ms,
                                double* bytes) {
    if (!e || !avg_ms) return fail(TLT_ERR_STATE, "null argument");
    return guard([&] { *avg_ms = e->e->probe_attention(b, ctx, rows_per_req, iters < 1 ? 1 : iters, bytes); });
}

TLT_API int tlt_set_debug(tlt_engine* e, int on) {
    if (!e) return fail(TLT_ERR_STATE, "null engine");
    e->e->set_debug(on != 0);
    return TLT_OK;
}

TLT_API int tlt_debug_expansions(tlt_engine* e, int i, int max_exp, int32_t* n_exp, int32_t* path_len, int32_t* paths,
                                 double* rows) {
    if (!e) return fail(TLT_ERR_STATE, "null engine");
    return guard([&] {
        auto& E = *e->e;
        const auto& ex = E.debug_expansions(i);
        const int n = std::min<int>(max_exp, (int)ex.size());
        *n_exp = (int32_t)ex.size();
        const int V = E.cfg.vocab;
        for (int j = 0; j < n; ++j) {
            path_len[j] = (int32_t)ex[j].path.size();
            for (size_t t = 0; t < ex[j].path.size(); ++t) paths[(size_t)j * tlt::kMaxDepth + t] = ex[j].path[t];
            if (rows) std::memcpy(rows + (size_t)j * V, ex[j].row.data(), sizeof(double) * V);
        }
    });
}

TLT_API int tlt_debug_verify_logits(tlt_engine* e, int i, float* logits, int max_rows, int32_t* n_rows) {
    if (!e) return fail(TLT_ERR_STATE, "null engine");
    return guard([&] {
        auto& E = *e->e;
        const auto v = E.debug_verify_logits(i);
        const int V = E.cfg.vocab;
        const int rows = (int)(v.size() / V);
        *n_rows = rows;
        std::memcpy(logits, v.data(), sizeof(float) * (size_t)std::min(rows, max_rows) * V);
    });
}

TLT_API int tlt_debug_ar_logits(tlt_engine* e, float* logits, int b) {
    if (!e) return fail(TLT_ERR_STATE, "null engine");
    return guard([&] {
        auto& E = *e->e;
        const size_t n = std::min(E.dbg_ar_logits.size(), (size_t)b * E.cfg.vocab);
        std::memcpy(logits, E.dbg_ar_logits.data(), sizeof(float) * n);
    });
}

// ---------------------------------------------------------------- BEG-MAB
TLT_API int tlt_mab_create(const tlt_strategy* strategies, int n, const int32_t* thresholds, int n_thr, double epsilon,
                           int window, tlt_mab** out) {
    if (!strategies || !thresholds || !out) return fail(TLT_ERR_CONFIG, "null argument");
    return guard([&] {
        std::vector<tlt_strategy> s(strategies, strategies + n);
        std::vector<int> t(thresholds, thresholds + n_thr);
        auto* h = new tlt_mab;
        try {
            h->m = std::make_unique<tlt::Mab>(s, t, epsilon, window);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}
TLT_API void tlt_mab_destroy(tlt_mab* m) { delete m; }
TLT_API int tlt_mab_select(tlt_mab* m, int batch, tlt_rng* rng, int32_t* arm, tlt_strategy* out) {
    if (!m || !rng) return fail(TLT_ERR_STATE, "null argument");
    return guard([&] {
        const size_t a = m->m->select(batch, rng->r);
        if (arm) *arm = (int32_t)a;
        if (out) *out = m->m->arms[a].strategy;
    });
}
TLT_API int tlt_mab_record(tlt_mab* m, const tlt_strategy* s, double elapsed, const int32_t* accept_lens, int batch) {
    if (!m || !s) return fail(TLT_ERR_STATE, "null argument");
    return guard([&] { m->m->record(*s, elapsed, accept_lens, batch); });
}
TLT_API int tlt_mab_arm_stats(tlt_mab* m, int arm, double* median_reward, int64_t* selections, int32_t* n_rewards) {
    if (!m) return fail(TLT_ERR_STATE, "null argument");
    return guard([&] {
        if (arm < 0 || arm >= (int)m->m->arms.size()) throw tlt::ConfigErr("arm", "out of range");
        const auto& a = m->m->arms[arm];
        if (median_reward) *median_reward = tlt::Mab::median(a.rewards);
        if (selections) *selections = a.selections;
        if (n_rewards) *n_rewards = (int32_t)a.rewards.size();
    });
}
TLT_API int tlt_mab_arm_window(tlt_mab* m, int arm, double* rewards, double* accept_lens, int cap, int32_t* n) {
    if (!m || !n) return fail(TLT_ERR_STATE, "null argument");
    return guard([&] {
        if (arm < 0 || arm >= (int)m->m->arms.size()) throw tlt::ConfigErr("arm", "out of range");
        const auto& a = m->m->arms[arm];
        *n = (int32_t)a.rewards.size();
        for (int i = 0; i < (int)a.rewards.size() && i < cap; ++i) {
            if (rewards) rewards[i] = a.rewards[i];
            if (accept_lens) accept_lens[i] = a.accept_lens[i];
        }
    });
}
TLT_API int tlt_mab_apply_record(tlt_mab* m, int arm, double reward, double a_bar) {
    if (!m) return fail(TLT_ERR_STATE, "null argument");
    return guard([&] {
        if (arm < 0 || arm >= (int)m->m->arms.size()) throw tlt::ConfigErr("arm", "out of range");
        m->m->push(m->m->arms[arm], reward, a_bar, false);  // merged records are not re-logged
    });
}

TLT_API int tlt_mab_take_log(tlt_mab* m, int32_t* arm, double* reward, double* a_bar, int cap, int32_t* n) {
    if (!m || !n) return fail(TLT_ERR_STATE, "null argument");
    return guard([&] {
        auto& lg = m->m->log;
        if ((int)lg.size() > cap) throw tlt::ConfigErr("cap", "record log larger than the output arrays");
        for (size_t i = 0; i < lg.size(); ++i) {
            arm[i] = lg[i].arm;
            reward[i] = lg[i].reward;
            a_bar[i] = lg[i].a_bar;
        }
        *n = (int32_t)lg.size();
        lg.clear();
    });
}

TLT_API int tlt_mab_copy(tlt_mab* dst, const tlt_mab* src) {
    if (!dst || !src) return fail(TLT_ERR_STATE, "null argument");
    return guard([&] {
        *dst->m = *src->m;
        dst->m->log.clear();
    });
}

// ---------------------------------------------------------------- RNG
TLT_API int tlt_rng_create(uint64_t seed, uint64_t stream_id, tlt_rng** out) {
    if (!out) return fail(TLT_ERR_CONFIG, "null argument");
    *out = new tlt_rng{tlt::Rng(seed, stream_id)};
    return TLT_OK;
}
TLT_API int tlt_rng_fork(const tlt_rng* r, uint64_t label, tlt_rng** out) {
    if (!r || !out) return fail(TLT_ERR_CONFIG, "null argument");
    *out = new tlt_rng{r->r.fork(label)};
    return TLT_OK;
}
TLT_API void tlt_rng_destroy(tlt_rng* r) { delete r; }
TLT_API int tlt_rng_ids(const tlt_rng* r, uint64_t* seed, uint64_t* stream_id) {
    if (!r) return fail(TLT_ERR_CONFIG, "null argument");
    if (seed) *seed = r->r.seed();
    if (stream_id) *stream_id = r->r.stream_id();
    return TLT_OK;
}
TLT_API uint64_t tlt_rng_next_u64(tlt_rng* r) { return r->r.next_u64(); }
TLT_API double tlt_rng_uniform01(tlt_rng* r) { return r->r.uniform01(); }

// ---------------------------------------------------------------- capture plan
TLT_API int tlt_plan_captures(const tlt_strategy* strategies, int n, const int32_t* thresholds, int n_thr, int max_batch,
                              int vanilla, tlt_capture_entry* out, int max_entries, int* n_entries,
                              double* total_memory_units) {
    if (!strategies || !thresholds) return fail(TLT_ERR_CONFIG, "null argument");
    return guard([&] {
        std::vector<tlt_strategy> s(strategies, strategies + n);
        std::vector<int> t(thresholds, thresholds + n_thr);
        auto plan = tlt::plan_captures(s, t, max_batch, vanilla != 0, total_memory_units);
        if (n_entries) *n_entries = (int)plan.size();
        if ((int)plan.size() > max_entries) throw tlt::ConfigErr("max_entries", "output buffer too small");
        for (size_t i = 0; i < plan.size(); ++i) out[i] = plan[i];
    });
}

// ---------------------------------------------------------------- rollout
TLT_API int tlt_step_latency(const tlt_cost_model* cost, int batch, int tokens_per_request, const tlt_strategy* sd,
                             double* out) {
    if (!out) return fail(TLT_ERR_CONFIG, "null argument");
    return guard([&] {
        const tlt_cost_model c = tlt::cost_or_default(cost ? *cost : tlt_cost_model{});
        *out = tlt::step_latency(c, batch, tokens_per_request, sd);
    });
}

// Reference run_rollout (rollout.hpp:130-276) on the GPU engine: elastic gate,
// BEG-MAB select/record (measured elapsed), greedy tree SD or plain decode per
// engine step, emission truncated at EOS / max_len (:231-240), requests
// finish independently. Each request occupies KV slot i.
TLT_API int tlt_run_rollout(tlt_engine* e, const tlt_rollout_cfg* cfg, tlt_mab* mab, int n, const int32_t* request_ids,
                            const int32_t* prompt_lens, const int32_t* prompts, const int32_t* max_lens,
                            int max_len_stride, tlt_rollout_result* out) {
    if (!e || !cfg || !out) return fail(TLT_ERR_STATE, "null argument");
    return guard([&] {
        auto& E = *e->e;
        const auto t0 = std::chrono::steady_clock::now();
        if (n < 1 || n > E.cfg.max_slots) throw tlt::ConfigErr("requests", "count exceeds max_slots");
        if (cfg->elastic_threshold < 1) throw tlt::ConfigErr("threshold", "must be >= 1");
        const bool stoch = cfg->mode == TLT_MODE_STOCHASTIC_LINEAR;
        if (cfg->mode != TLT_MODE_GREEDY_TREE && !stoch) throw tlt::ConfigErr("mode", "unknown decode mode");
        // experiment.hpp:136-137: stochastic_linear requires temperature > 0
        if (stoch && !(cfg->temperature > 0.0f)) throw tlt::ConfigErr("temperature", "stochastic_linear requires t > 0");
        if (cfg->temperature < 0.0f) throw tlt::ConfigErr("temperature", "must be >= 0");
        if (cfg->use_mab && !mab) throw tlt::ConfigErr("mab", "use_mab requires a bandit state");
        if (!cfg->use_mab && cfg->enable_sd) tlt::validate(cfg->fixed_strategy);
        const tlt_cost_model cost = tlt::cost_or_default(cfg->cost);  // run_rollout: cost.validate() (:135)
        E.use_graphs = cfg->use_graphs != 0;
        std::vector<int32_t> slots(n);
        for (int i = 0; i < n; ++i) {
            slots[i] = i;
            if (max_lens[i] < 1) throw tlt::ConfigErr("requests", "max_len must be >= 1");
            if (max_lens[i] > max_len_stride) throw tlt::ConfigErr("max_len_stride", "smaller than max_len");
        }
        tlt::Rng root(cfg->seed, cfg->rng_stream);  // the caller's RngStream (seed, stream_id)
        std::vector<tlt::Rng> req_rng;
        for (int i = 0; i < n; ++i) req_rng.push_back(root.fork(0x52515254ULL + (uint64_t)request_ids[i]));
        tlt::Rng select_rng = root.fork(0x53454CULL);
        const bool via_ngram = cfg->drafter_stale != 0;  // rollout.hpp:209 `via_ngram = !adaptive_fresh`
        std::vector<tlt::Ngram> trackers;
        if (via_ngram)
            for (int i = 0; i < n; ++i) trackers.emplace_back(cfg->ngram_n, cfg->ngram_continuation_len);
        std::vector<std::vector<int32_t>> ctxs;  // prompt ++ generated, for the trackers
        if (via_ngram)
            for (int i = 0, off = 0; i < n; off += prompt_lens[i], ++i)
                ctxs.emplace_back(prompts + off, prompts + off + prompt_lens[i]);
        std::vector<int32_t> chains, chain_lens;
        E.prefill(n, slots.data(), prompt_lens, prompts);
        if (std::getenv("TLT_TRACE")) std::fprintf(stderr, "[tlt] prefill_ms %.3f n=%d\n", E.last_prefill_ms, n);
        std::vector<int> running(n, 1), glen(n, 0);
        out->sd_steps = out->plain_steps = out->verify_events = out->accepted_total = out->emitted_total = 0;
        out->ngram_verify_events = 0;
        out->total_time = 0.0;
        out->trace_len = 0;
        int64_t trace_acc_n = 0;
        std::vector<double> finish(n, 0.0);
        out->device_ms = E.last_prefill_ms;
        const long long launches0 = E.launches;
        // accept_at_least sized by the largest arm depth (rollout.hpp:157-163)
        int maxD = 1;
        if (cfg->use_mab)
            for (auto& a : mab->m->arms) maxD = std::max(maxD, a.strategy.draft_depth);
        else
            maxD = cfg->fixed_strategy.draft_depth > 0 ? cfg->fixed_strategy.draft_depth : 1;  // nullopt -> 1
        std::vector<int64_t> at_least(std::max(maxD, 0), 0);
        int step_index = 0;
        std::vector<int32_t> act, acc_len, bonus, accepted, tok;
        // per-request queue of RngStream draws: the device consumes them in
        // reference order, the host pops exactly what was consumed
        std::vector<std::deque<double>> uq(n);
        std::vector<double> ubuf;
        auto take = [&](int i, int cnt, double* dst) {
            while ((int)uq[i].size() < cnt) uq[i].push_back(req_rng[i].uniform01());
            for (int c = 0; c < cnt; ++c) dst[c] = uq[i][c];
        };
        auto pop = [&](int i, int cnt) {
            for (int c = 0; c < cnt; ++c) uq[i].pop_front();
        };
        for (;;) {
            act.clear();
            for (int i = 0; i < n; ++i)
                if (running[i]) act.push_back(i);
            if (act.empty()) break;
            const int batch = (int)act.size();
            const bool sd = cfg->enable_sd && batch < cfg->elastic_threshold;  // rollout.hpp:174
            static const bool trace = std::getenv("TLT_TRACE") != nullptr;
            tlt_step_metrics sm{};  // StepMetrics (rollout.hpp:31-38, :175-178)
            sm.step_index = step_index;
            sm.batch_size = batch;
            sm.sd_active = sd ? 1 : 0;
            sm.accept_off = trace_acc_n;
            sm.via_ngram = sd && via_ngram ? 1 : 0;
            auto emit = [&](int i, int32_t t) {
                out->generated[(size_t)i * max_len_stride + glen[i]] = t;
                glen[i] += 1;
                if (via_ngram) ctxs[i].push_back(t);
                out->emitted_total += 1;
                if (t == TLT_EOS_TOKEN || glen[i] >= max_lens[i]) {
                    running[i] = 0;
                    return true;
                }
                return false;
            };
            if (sd) {
                tlt_strategy s = cfg->fixed_strategy;
                if (cfg->use_mab) s = mab->m->arms[mab->m->select(batch, select_rng)].strategy;
                const int D = s.draft_depth;
                if (trace) std::fprintf(stderr, "[tlt] sd_begin b=%d (%d,%d,%d)\n", batch, D, s.top_k, s.tokens_to_verify);
                acc_len.assign(batch, 0);
                bonus.assign(batch, 0);
                accepted.assign((size_t)batch * D, 0);
                float ms = 0.f;
                tlt_accept_out ao{accepted.data(), nullptr, acc_len.data(), bonus.data(), nullptr, nullptr, &ms};
                if (via_ngram) {
                    // rollout.hpp:214-216: tracker.extend(ctx), chain_from_tokens(ngram_draft(ctx, D))
                    chains.assign((size_t)batch * D, 0);
                    chain_lens.assign(batch, 0);
                    for (int j = 0; j < batch; ++j) {
                        const int i = act[j];
                        trackers[i].extend(ctxs[i].data(), ctxs[i].size(), cfg->target_step_id);
                        auto c = trackers[i].draft(ctxs[i].data(), ctxs[i].size(), D);
                        std::copy(c.begin(), c.end(), chains.begin() + (size_t)j * D);
                        chain_lens[j] = (int32_t)c.size();
                    }
                    if (stoch) {
                        ubuf.assign((size_t)batch * (D + 1), 0.0);
                        for (int j = 0; j < batch; ++j) take(act[j], D + 1, ubuf.data() + (size_t)j * (D + 1));
                        E.sd_step_chain(D, batch, act.data(), chains.data(), chain_lens.data(), &ao, cfg->temperature,
                                        ubuf.data());
                        for (int j = 0; j < batch; ++j) pop(act[j], E.last_consumed[j]);
                    } else {
                        E.sd_step_chain(D, batch, act.data(), chains.data(), chain_lens.data(), &ao);
                    }
                } else if (stoch) {
                    const int U = 2 * D + 1;
                    ubuf.assign((size_t)batch * U, 0.0);
                    for (int j = 0; j < batch; ++j) take(act[j], U, ubuf.data() + (size_t)j * U);
                    E.sd_step_stochastic(D, cfg->temperature, batch, act.data(), ubuf.data(), &ao);
                    for (int j = 0; j < batch; ++j) pop(act[j], E.last_consumed[j]);
                } else {
                    E.sd_step(s, batch, act.data(), nullptr, &ao);
                }
                for (int j = 0; j < batch; ++j) {
                    const int i = act[j];
                    out->verify_events += 1;
                    out->ngram_verify_events += via_ngram ? 1 : 0;
                    out->accepted_total += acc_len[j];
                    for (int d = 0; d < acc_len[j] && d < maxD; ++d) at_least[d] += 1;  // rollout.hpp:227-229
                    if (out->trace_accept_lens && trace_acc_n < out->trace_accept_cap)
                        out->trace_accept_lens[trace_acc_n] = acc_len[j];
                    ++trace_acc_n;
                    bool done = false;
                    for (int t = 0; t < acc_len[j] && !done; ++t) done = emit(i, accepted[(size_t)j * D + t]);
                    if (!done) emit(i, bonus[j]);
                }
                out->device_ms += ms;
                if (trace) {
                    int acc = 0;
                    for (int j = 0; j < batch; ++j) acc += acc_len[j];
                    std::fprintf(stderr, "[tlt] sd_ms %.3f b=%d D=%d k=%d T=%d acc=%d\n", ms, batch, D, s.top_k,
                                 s.tokens_to_verify, acc);
                }
                // rollout.hpp:242-245: elapsed -> beg_record
                const double elapsed = cfg->parity_elapsed ? tlt::step_latency(cost, batch, s.tokens_to_verify, &s)
                                                           : (double)ms;
                if (cfg->use_mab) mab->m->record(s, elapsed, acc_len.data(), batch);
                sm.has_strategy = 1;
                sm.strategy = s;
                sm.elapsed = elapsed;
                sm.device_ms = ms;
                sm.n_accept = batch;
                out->sd_steps += 1;
            } else {
                tok.assign(batch, 0);
                ubuf.assign(batch, 0.0);
                // sample_token consumes one draw per request (rollout.hpp:252-253)
                for (int j = 0; j < batch; ++j) take(act[j], 1, ubuf.data() + j);
                const float ms = cfg->temperature > 0.0f
                                     ? E.ar_step_sampled(batch, act.data(), cfg->temperature, ubuf.data(), tok.data())
                                     : E.ar_step(batch, act.data(), tok.data());
                for (int j = 0; j < batch; ++j) {
                    pop(act[j], 1);
                    emit(act[j], tok[j]);
                }
                out->device_ms += ms;
                if (trace) std::fprintf(stderr, "[tlt] ar_ms %.3f b=%d\n", ms, batch);
                sm.elapsed = cfg->parity_elapsed ? tlt::step_latency(cost, batch, 1, nullptr) : (double)ms;  // :258
                sm.device_ms = ms;
                out->plain_steps += 1;
            }
            out->total_time += sm.elapsed;  // rollout.hpp:263-268
            for (int j = 0; j < batch; ++j)
                if (!running[act[j]] && finish[act[j]] == 0.0) finish[act[j]] = out->total_time;
            if (out->trace && out->trace_len < out->trace_cap) out->trace[out->trace_len] = sm;
            out->trace_len += 1;
            ++step_index;
            for (int j = 0; j < batch; ++j) {
                const int i = act[j];
                if (running[i]) continue;
                if (cfg->keep_finished)  // committed = prompt ++ generated, last emitted token = pending root
                    E.truncate(i, prompt_lens[i] + glen[i] - 1);
                else
                    E.release(i);
            }
        }
        out->accept_at_least_len = (int32_t)at_least.size();
        if (out->accept_at_least)
            for (int d = 0; d < (int)at_least.size() && d < out->accept_at_least_cap; ++d)
                out->accept_at_least[d] = at_least[d];
        if (out->finish_time)
            for (int i = 0; i < n; ++i) out->finish_time[i] = finish[i];
        for (int i = 0; i < n; ++i) out->gen_len[i] = glen[i];
        out->gpu_launches = E.launches - launches0;
        out->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    });
}

}  // extern "C"
