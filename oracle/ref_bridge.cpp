// extern "C" bridge onto the UNMODIFIED reference headers
// (/root/reference/proj/include/specsim), compiled in place by oracle/Makefile
// into oracle/_ref/libspecsim_ref.so. TEST INFRASTRUCTURE: it lets the pytest
// suite pin the C restatement (oracle/orc_discrete.c) and the GPU outputs
// against the reference's own code on identical inputs. No reference source is
// copied; this file only calls reference functions.
#include <cstdint>
#include <cstring>
#include <exception>
#include <vector>

#include "specsim/beg_mab.hpp"
#include "specsim/capture_plan.hpp"
#include "specsim/checkpoint.hpp"
#include "specsim/cost_model.hpp"
#include "specsim/data_buffer.hpp"
#include "specsim/model_gen.hpp"
#include "specsim/packing.hpp"
#include "specsim/rollout.hpp"
#include "specsim/spec_decode.hpp"

using namespace specsim;

namespace {
using row_fn = int (*)(void*, const int32_t*, int, double*);

int code_of(const std::exception_ptr& ep) {
    try {
        std::rethrow_exception(ep);
    } catch (const ConfigError&) {
        return -1;
    } catch (const RoutingError&) {
        return -2;
    } catch (...) {
        return -3;
    }
}

DraftTree tree_from(int n, const int32_t* tok, const int32_t* par, const int32_t* dep, const double* prob,
                    const double* pp) {
    DraftTree t;
    for (int i = 0; i < n; ++i) {
        DraftNode d;
        d.token = tok[i];
        d.parent = par[i];
        d.depth = dep ? dep[i] : 1;
        d.prob = prob ? prob[i] : 1.0;
        d.path_prob = pp ? pp[i] : 1.0;
        t.nodes.push_back(std::move(d));
    }
    return t;
}

TokenSeq path_to(const DraftTree& t, int idx) {
    TokenSeq p;
    for (int i = idx; i != -1; i = t.nodes[static_cast<size_t>(i)].parent) p.push_back(t.nodes[static_cast<size_t>(i)].token);
    return TokenSeq(p.rbegin(), p.rend());
}

// Markov table whose order covers every queried context, so that raw_row()
// returns exactly the row the caller supplied for (ctx ++ path).
MarkovTargetModel table_target(int vocab, const TokenSeq& ctx, const std::vector<TokenSeq>& paths,
                               const std::vector<std::vector<double>>& rows, double temperature) {
    size_t maxp = 0;
    for (auto& p : paths) maxp = std::max(maxp, p.size());
    const int order = static_cast<int>(ctx.size() + maxp + 1);
    MarkovTargetModel probe(vocab, order, 1.0, {});
    MarkovTargetModel::Table table;
    for (size_t i = 0; i < paths.size(); ++i) {
        TokenSeq full = ctx;
        full.insert(full.end(), paths[i].begin(), paths[i].end());
        table.emplace(probe.context_key(full), Distribution{rows[i]});
    }
    return MarkovTargetModel(vocab, order, temperature, std::move(table));
}
}  // namespace

extern "C" {

// ------------------------------------------------------------------ RNG
void* ref_rng_create(uint64_t seed, uint64_t stream) { return new RngStream(seed, stream); }
void* ref_rng_fork(void* r, uint64_t label) { return new RngStream(static_cast<RngStream*>(r)->fork(label)); }
void ref_rng_destroy(void* r) { delete static_cast<RngStream*>(r); }
uint64_t ref_rng_next_u64(void* r) { return static_cast<RngStream*>(r)->next_u64(); }
double ref_rng_uniform01(void* r) { return static_cast<RngStream*>(r)->uniform01(); }
uint64_t ref_rng_uniform_int(void* r, uint64_t n) { return static_cast<RngStream*>(r)->uniform_int(n); }
double ref_rng_normal(void* r) { return static_cast<RngStream*>(r)->normal(); }
int ref_sample_response_length(double mu, double sigma, int max_len, void* r) {
    try {
        return sample_response_length(mu, sigma, max_len, *static_cast<RngStream*>(r));
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// --------------------------------------------------------- distributions
int ref_argmax(const double* p, int v) { return Distribution{std::vector<double>(p, p + v)}.argmax(); }
int ref_inverse_cdf_pick(const double* p, int v, double u) {
    return inverse_cdf_pick(Distribution{std::vector<double>(p, p + v)}, u);
}
int ref_target_next_dist(const double* raw, int v, double t, double* out) {
    try {
        MarkovTargetModel::Table table;
        table.emplace(TokenSeq{}, Distribution{std::vector<double>(raw, raw + v)});
        MarkovTargetModel m(v, 0, t, std::move(table));
        Distribution d = target_next_dist(m, std::span<const TokenId>());
        std::memcpy(out, d.probs.data(), sizeof(double) * static_cast<size_t>(v));
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// ------------------------------------------------------------- strategy
long long ref_max_tree_nodes(int d, int k, int t) { return SpecStrategy{d, k, t}.max_tree_nodes(); }
int ref_strategy_validate(int d, int k, int t) {
    try {
        SpecStrategy{d, k, t}.validate();
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// ---------------------------------------------------------------- tree
int ref_build_draft_tree(row_fn f, void* user, int vocab, const int32_t* ctx, int ctx_len, int D, int k, int T,
                         int32_t* tok, int32_t* par, int32_t* dep, double* prob, double* pp) {
    try {
        const size_t base = static_cast<size_t>(ctx_len);
        int failed = 0;
        auto next = [&](const TokenSeq& c) {
            Distribution d{std::vector<double>(static_cast<size_t>(vocab))};
            const int32_t* path = c.data() + base;
            if (f(user, path, static_cast<int>(c.size() - base), d.probs.data()) != 0) failed = 1;
            return d;
        };
        DraftTree t = build_draft_tree(next, std::span<const TokenId>(ctx, static_cast<size_t>(ctx_len)),
                                       SpecStrategy{D, k, T});
        if (failed) return -3;
        for (size_t i = 0; i < t.nodes.size(); ++i) {
            tok[i] = t.nodes[i].token;
            par[i] = t.nodes[i].parent;
            dep[i] = t.nodes[i].depth;
            prob[i] = t.nodes[i].prob;
            pp[i] = t.nodes[i].path_prob;
        }
        return static_cast<int>(t.nodes.size());
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// verify_greedy with target rows supplied by f for the root (path = {}) and
// every tree node path. Writes accepted tokens, accept_length and bonus.
int ref_verify_greedy(row_fn f, void* user, int vocab, const int32_t* ctx, int ctx_len, int n, const int32_t* tok,
                      const int32_t* par, int32_t* accepted, int32_t* accept_len, int32_t* bonus) {
    try {
        DraftTree tree = tree_from(n, tok, par, nullptr, nullptr, nullptr);
        std::vector<TokenSeq> paths{TokenSeq{}};
        for (int i = 0; i < n; ++i) paths.push_back(path_to(tree, i));
        std::vector<std::vector<double>> rows;
        for (auto& p : paths) {
            std::vector<double> r(static_cast<size_t>(vocab));
            if (f(user, p.data(), static_cast<int>(p.size()), r.data()) != 0) return -3;
            rows.push_back(std::move(r));
        }
        TokenSeq c(ctx, ctx + ctx_len);
        MarkovTargetModel target = table_target(vocab, c, paths, rows, 0.0);
        AcceptResult res = verify_greedy(target, c, tree);
        for (int i = 0; i < res.accept_length; ++i) accepted[i] = res.accepted[static_cast<size_t>(i)];
        *accept_len = res.accept_length;
        *bonus = res.bonus;
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// build_sampled_chain over f with RngStream(seed, stream); draft_dists [depth][V].
int ref_build_sampled_chain(row_fn f, void* user, int vocab, const int32_t* ctx, int ctx_len, int depth, void* rng,
                            int32_t* tok, double* prob, double* pp, double* draft_dists) {
    try {
        const size_t base = static_cast<size_t>(ctx_len);
        auto next = [&](const TokenSeq& c) {
            Distribution d{std::vector<double>(static_cast<size_t>(vocab))};
            f(user, c.data() + base, static_cast<int>(c.size() - base), d.probs.data());
            return d;
        };
        DraftTree t = build_sampled_chain(next, std::span<const TokenId>(ctx, base), depth, *static_cast<RngStream*>(rng));
        for (size_t i = 0; i < t.nodes.size(); ++i) {
            tok[i] = t.nodes[i].token;
            prob[i] = t.nodes[i].prob;
            pp[i] = t.nodes[i].path_prob;
            std::memcpy(draft_dists + i * static_cast<size_t>(vocab), t.nodes[i].draft_dist.data(),
                        sizeof(double) * static_cast<size_t>(vocab));
        }
        return static_cast<int>(t.nodes.size());
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// verify_stochastic over a linear chain; target raw rows from f for every
// chain prefix (0..n); draft_dists may be NULL (one-hot proposals).
int ref_verify_stochastic(row_fn f, void* user, int vocab, double temperature, const int32_t* ctx, int ctx_len, int n,
                          const int32_t* tok, const double* draft_dists, void* rng, int32_t* accepted,
                          int32_t* accept_len, int32_t* bonus) {
    try {
        DraftTree chain;
        for (int i = 0; i < n; ++i) {
            DraftNode d;
            d.token = tok[i];
            d.parent = i - 1;
            d.depth = i + 1;
            if (draft_dists)
                d.draft_dist.assign(draft_dists + static_cast<size_t>(i) * static_cast<size_t>(vocab),
                                    draft_dists + static_cast<size_t>(i + 1) * static_cast<size_t>(vocab));
            chain.nodes.push_back(std::move(d));
        }
        std::vector<TokenSeq> paths;
        std::vector<std::vector<double>> rows;
        for (int i = 0; i <= n; ++i) {
            TokenSeq p(tok, tok + i);
            std::vector<double> r(static_cast<size_t>(vocab));
            if (f(user, p.data(), i, r.data()) != 0) return -3;
            paths.push_back(std::move(p));
            rows.push_back(std::move(r));
        }
        TokenSeq c(ctx, ctx + ctx_len);
        MarkovTargetModel target = table_target(vocab, c, paths, rows, temperature);
        AcceptResult res = verify_stochastic(target, c, chain, *static_cast<RngStream*>(rng));
        for (int i = 0; i < res.accept_length; ++i) accepted[i] = res.accepted[static_cast<size_t>(i)];
        *accept_len = res.accept_length;
        *bonus = res.bonus;
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// ------------------------------------------------------------- BEG-MAB
void* ref_mab_create(const int32_t* dkt, int n, const int32_t* thr, int n_thr, double eps, int window, int* rc) {
    try {
        std::vector<SpecStrategy> s;
        for (int i = 0; i < n; ++i) s.push_back(SpecStrategy{dkt[3 * i], dkt[3 * i + 1], dkt[3 * i + 2]});
        std::vector<int> t(thr, thr + n_thr);
        *rc = 0;
        return new BegMabState(beg_initialize(s, t, eps, window));
    } catch (...) {
        *rc = code_of(std::current_exception());
        return nullptr;
    }
}
void ref_mab_destroy(void* m) { delete static_cast<BegMabState*>(m); }
int ref_mab_select(void* m, int batch, void* rng) {
    try {
        auto* st = static_cast<BegMabState*>(m);
        const SpecStrategy& s = beg_select(*st, batch, *static_cast<RngStream*>(rng));
        for (size_t i = 0; i < st->arms().size(); ++i)
            if (&st->arms()[i].strategy == &s) return static_cast<int>(i);
        return -3;
    } catch (...) {
        return code_of(std::current_exception());
    }
}
int ref_mab_record(void* m, int d, int k, int t, double elapsed, const int32_t* lens, int n_lens, int batch) {
    try {
        std::vector<int> a(lens, lens + n_lens);
        beg_record(*static_cast<BegMabState*>(m), SpecStrategy{d, k, t}, elapsed, a, batch);
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}
int ref_mab_stats(void* m, int arm, double* median_reward, long long* selections, int* n, double* last_reward,
                  double* last_accept) {
    auto* st = static_cast<BegMabState*>(m);
    const auto& a = st->arms()[static_cast<size_t>(arm)];
    *median_reward = BegMabState::median(a.rewards);
    *selections = a.selections;
    *n = static_cast<int>(a.rewards.size());
    *last_reward = a.rewards.empty() ? 0.0 : a.rewards.back();
    *last_accept = a.accept_lens.empty() ? 0.0 : a.accept_lens.back();
    return 0;
}

// ------------------------------------------------------- capture plan
int ref_plan_captures(const int32_t* dkt, int n, const int32_t* thr, int n_thr, int max_batch, int vanilla,
                      int32_t* out6, double* mem, int max_out, double* total) {
    try {
        std::vector<SpecStrategy> s;
        for (int i = 0; i < n; ++i) s.push_back(SpecStrategy{dkt[3 * i], dkt[3 * i + 1], dkt[3 * i + 2]});
        BucketSpec spec{std::vector<int>(thr, thr + n_thr), max_batch};
        CapturePlan p = vanilla ? plan_captures_vanilla(s, spec) : plan_captures(s, spec);
        if (static_cast<int>(p.entries.size()) > max_out) return -3;
        for (size_t i = 0; i < p.entries.size(); ++i) {
            const auto& e = p.entries[i];
            int32_t* o = out6 + 6 * i;
            o[0] = e.side == CaptureSide::Target ? 0 : 1;
            o[1] = e.bucket_lo;
            o[2] = e.bucket_hi;
            o[3] = e.tokens_to_verify;
            o[4] = e.top_k;
            o[5] = e.draft_depth;
            mem[i] = e.memory_units;
        }
        *total = p.total_memory_units;
        return static_cast<int>(p.entries.size());
    } catch (...) {
        return code_of(std::current_exception());
    }
}

int ref_should_enable_sd(int active, int threshold) {
    try {
        return should_enable_sd(active, threshold) ? 1 : 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}
double ref_step_latency(int batch, int tokens, int d, int k, int t, int has_sd) {
    CostModelParams c;
    std::optional<SpecStrategy> s;
    if (has_sd) s = SpecStrategy{d, k, t};
    return step_latency(c, batch, tokens, s);
}

// ----------------------------------------------- Markov fixtures (model_gen)
void* ref_make_random_model(int vocab, int order, double temperature, double conc, double eos, void* rng) {
    return new MarkovTargetModel(make_random_model(vocab, order, temperature, conc, eos, *static_cast<RngStream*>(rng)));
}
void* ref_make_cyclic_model(int vocab, const int32_t* cycle, int n) {
    return new MarkovTargetModel(make_cyclic_model(vocab, TokenSeq(cycle, cycle + n)));
}
void ref_model_destroy(void* m) { delete static_cast<MarkovTargetModel*>(m); }
// raw_row for (ctx ++ path): user = {model, ctx, ctx_len}
struct RefRowUser {
    void* model;
    const int32_t* ctx;
    int ctx_len;
};
int ref_markov_row(void* user, const int32_t* path, int n, double* out) {
    auto* u = static_cast<RefRowUser*>(user);
    auto* m = static_cast<MarkovTargetModel*>(u->model);
    TokenSeq c(u->ctx, u->ctx + u->ctx_len);
    c.insert(c.end(), path, path + n);
    const Distribution& d = m->raw_row(c);
    std::memcpy(out, d.probs.data(), sizeof(double) * d.probs.size());
    return 0;
}
// Reference spec_generate (greedy tree, count-free drafter given by f).
int ref_spec_generate_greedy(void* model, row_fn draft_f, void* draft_user, const int32_t* prompt, int plen,
                             int max_len, int D, int k, int T, int32_t* out_tokens, int* out_len, int32_t* accept_lens,
                             int* n_steps) {
    try {
        auto* m = static_cast<MarkovTargetModel*>(model);
        const size_t base = static_cast<size_t>(plen);
        (void)base;
        DraftPlanner planner = [&](const TokenSeq& ctx, const SpecStrategy& s, RngStream&) {
            auto next = [&](const TokenSeq& c) {
                Distribution d{std::vector<double>(static_cast<size_t>(m->vocab_size()))};
                draft_f(draft_user, c.data(), static_cast<int>(c.size()), d.probs.data());
                return d;
            };
            return build_draft_tree(next, ctx, s);
        };
        RngStream rng(1, 0);
        SpecResult r = spec_generate(*m, planner, std::span<const TokenId>(prompt, static_cast<size_t>(plen)), max_len,
                                     SpecStrategy{D, k, T}, DecodeMode::GreedyTree, rng);
        for (size_t i = 0; i < r.tokens.size(); ++i) out_tokens[i] = r.tokens[i];
        *out_len = static_cast<int>(r.tokens.size());
        for (size_t i = 0; i < r.accept_lens.size(); ++i) accept_lens[i] = r.accept_lens[i];
        *n_steps = static_cast<int>(r.accept_lens.size());
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}
int ref_generate_autoregressive(void* model, const int32_t* prompt, int plen, int max_len, uint64_t seed,
                                int32_t* out, int* out_len) {
    RngStream rng(seed, 0);
    TokenSeq t = generate_autoregressive(*static_cast<MarkovTargetModel*>(model),
                                         std::span<const TokenId>(prompt, static_cast<size_t>(plen)), max_len, rng);
    for (size_t i = 0; i < t.size(); ++i) out[i] = t[i];
    *out_len = static_cast<int>(t.size());
    return 0;
}

// ---- n-gram fallback drafter (ngram.hpp:13-103, NgramTracker rollout.hpp:103-120)
void* ref_ngram_create(int n, int cont) {
    try {
        auto* t = new detail::NgramTracker;
        t->index = NgramIndex(n, cont);
        return t;
    } catch (...) {
        return nullptr;
    }
}
void ref_ngram_destroy(void* t) { delete static_cast<detail::NgramTracker*>(t); }
int ref_ngram_insert(void* t, const int32_t* r, int len, long long step) {
    auto* tr = static_cast<detail::NgramTracker*>(t);
    tr->index = ngram_insert(tr->index, std::span<const TokenId>(r, static_cast<std::size_t>(len)), step);
    return 0;
}
int ref_ngram_extend(void* t, const int32_t* r, int len, long long step) {
    static_cast<detail::NgramTracker*>(t)->extend(TokenSeq(r, r + len), step);
    return 0;
}
int ref_ngram_draft(void* t, const int32_t* ctx, int len, int depth, int32_t* out) {
    try {
        auto v = ngram_draft(static_cast<detail::NgramTracker*>(t)->index,
                             std::span<const TokenId>(ctx, static_cast<std::size_t>(len)), depth);
        std::copy(v.begin(), v.end(), out);
        return static_cast<int>(v.size());
    } catch (...) {
        return code_of(std::current_exception());
    }
}
long long ref_ngram_size(void* t) { return (long long)static_cast<detail::NgramTracker*>(t)->index.size(); }

// ------------------------------------------------------- spot training (f3)
void* ref_databuf_create(long long retention) { return new DataBuffer(retention); }
void ref_databuf_destroy(void* b) { delete static_cast<DataBuffer*>(b); }
// sequences back to back: toks, lens[n]
void ref_databuf_insert(void* b, long long step, const int32_t* toks, const int32_t* lens, int n) {
    std::vector<TokenSeq> seqs;
    for (int i = 0, off = 0; i < n; off += lens[i], ++i) seqs.emplace_back(toks + off, toks + off + lens[i]);
    static_cast<DataBuffer*>(b)->insert(step, seqs);
}
int ref_databuf_size(void* b) { return (int)static_cast<DataBuffer*>(b)->entries().size(); }
// sample -> concatenated tokens + lens; returns the number of sequences (or -1 if cap is too small)
int ref_databuf_sample(void* b, long long step, long long budget, int32_t* toks, int32_t* lens, int cap_seqs,
                       long long cap_toks) {
    auto s = static_cast<DataBuffer*>(b)->sample(step, (std::size_t)budget);
    if ((int)s.size() > cap_seqs) return -1;
    long long off = 0;
    for (size_t i = 0; i < s.size(); ++i) {
        if (off + (long long)s[i].size() > cap_toks) return -1;
        std::copy(s[i].begin(), s[i].end(), toks + off);
        lens[i] = (int32_t)s[i].size();
        off += (long long)s[i].size();
    }
    return (int)s.size();
}
// pack_sequences -> per pack: member lengths (bounds, -1 separates packs) and the pack tokens back to back
int ref_pack(const int32_t* toks, const int32_t* lens, int n, long long capacity, int32_t* bounds, int cap_bounds,
             int32_t* out_toks, long long cap_toks) {
    std::vector<TokenSeq> seqs;
    for (int i = 0, off = 0; i < n; off += lens[i], ++i) seqs.emplace_back(toks + off, toks + off + lens[i]);
    PackedBatch p;
    try {
        p = pack_sequences(seqs, (std::size_t)capacity);
    } catch (const std::exception&) {
        return -2;
    }
    int nb = 0;
    long long nt = 0;
    for (size_t k = 0; k < p.packs.size(); ++k) {
        for (size_t m : p.boundaries[k]) {
            if (nb >= cap_bounds) return -1;
            bounds[nb++] = (int32_t)m;
        }
        if (nb >= cap_bounds) return -1;
        bounds[nb++] = -1;
        for (TokenId t : p.packs[k]) {
            if (nt >= cap_toks) return -1;
            out_toks[nt++] = t;
        }
    }
    return nb;
}
unsigned long long ref_fnv1a64(const uint8_t* data, unsigned long long len) { return detail::fnv1a64(data, len); }

}  // extern "C"
