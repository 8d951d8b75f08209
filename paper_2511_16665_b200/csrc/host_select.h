// Host-side strategy selection and capture planning (product code, C++).
// Semantics follow the reference exactly (cited per function); only the
// elapsed time fed to beg_record changes: it is the measured device time of
// the step (CUDA events) instead of the simulated step_latency.
#pragma once
#include <algorithm>
#include <cstdint>
#include <deque>
#include <limits>
#include <map>
#include <random>
#include <vector>

#include "../../include/tlt_b200.h"
#include "tlt_internal.h"

namespace tlt {

// RngStream (rng.hpp:34-86): std::mt19937_64 seeded through SplitMix64.
class Rng {
public:
    Rng(uint64_t seed, uint64_t stream) : seed_(seed), stream_(stream) {
        uint64_t x = seed ^ mix_label(0x5bf03635d0d0183dULL, stream);
        eng_.seed(splitmix(x));
    }
    Rng fork(uint64_t label) const { return Rng(seed_, mix_label(stream_ + 0x9e3779b97f4a7c15ULL, label)); }
    uint64_t next_u64() { return eng_(); }
    double uniform01() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    uint64_t uniform_int(uint64_t n) { return next_u64() % n; }
    uint64_t seed() const { return seed_; }
    uint64_t stream_id() const { return stream_; }

private:
    static uint64_t splitmix(uint64_t& x) {
        x += 0x9e3779b97f4a7c15ULL;
        uint64_t z = x;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    static uint64_t mix_label(uint64_t state, uint64_t label) {
        uint64_t x = state ^ (0x9e3779b97f4a7c15ULL + label);
        splitmix(x);
        return x;
    }
    uint64_t seed_, stream_;
    std::mt19937_64 eng_;
};

inline bool same(const tlt_strategy& a, const tlt_strategy& b) {
    return a.draft_depth == b.draft_depth && a.top_k == b.top_k && a.tokens_to_verify == b.tokens_to_verify;
}

inline long long max_tree_nodes(const tlt_strategy& s) {  // spec_decode.hpp:25-34
    long long total = 0, level = 1;
    for (int d = 0; d < s.draft_depth; ++d) {
        if (level > (1LL << 40) / std::max(s.top_k, 1)) return 1LL << 40;
        level *= s.top_k;
        total += level;
        if (total > (1LL << 40)) return 1LL << 40;
    }
    return total;
}
inline void validate(const tlt_strategy& s) {  // spec_decode.hpp:36-42
    if (s.draft_depth < 1) throw ConfigErr("draft_depth", "must be >= 1");
    if (s.top_k < 1) throw ConfigErr("top_k", "must be >= 1");
    if (s.tokens_to_verify < 1) throw ConfigErr("tokens_to_verify", "must be >= 1");
    if (s.tokens_to_verify > max_tree_nodes(s))
        throw ConfigErr("tokens_to_verify", "exceeds tree capacity for (top_k, draft_depth)");
}

// CostModelParams (cost_model.hpp:16-33): all-zero = the reference defaults;
// otherwise every field must be > 0 (validate, :24-32).
inline tlt_cost_model cost_or_default(const tlt_cost_model& c) {
    if (c.t_launch == 0 && c.model_bytes == 0 && c.mem_bw == 0 && c.flops_per_token == 0 && c.peak_flops == 0 &&
        c.drafter_step_cost == 0)
        return tlt_cost_model{0.05, 1.0, 1.0, 1.0, 377.0, 0.046};
    if (!(c.t_launch > 0.0)) throw ConfigErr("cost_model.t_launch", "must be > 0");
    if (!(c.model_bytes > 0.0)) throw ConfigErr("cost_model.model_bytes", "must be > 0");
    if (!(c.mem_bw > 0.0)) throw ConfigErr("cost_model.mem_bw", "must be > 0");
    if (!(c.flops_per_token > 0.0)) throw ConfigErr("cost_model.flops_per_token", "must be > 0");
    if (!(c.peak_flops > 0.0)) throw ConfigErr("cost_model.peak_flops", "must be > 0");
    if (!(c.drafter_step_cost > 0.0)) throw ConfigErr("cost_model.drafter_step_cost", "must be > 0");
    return c;
}
// step_latency (cost_model.hpp:38-48): launch + max(weight stream, compute)
// + one drafter pass per draft level.
inline double step_latency(const tlt_cost_model& c, int batch, int tokens_per_request, const tlt_strategy* sd) {
    if (batch < 1) throw ConfigErr("batch", "must be >= 1");
    const int tokens = sd ? sd->tokens_to_verify : tokens_per_request;
    const double memory_time = c.model_bytes / c.mem_bw;
    const double compute_time = static_cast<double>(batch) * static_cast<double>(tokens) * c.flops_per_token / c.peak_flops;
    double t = c.t_launch + std::max(memory_time, compute_time);
    if (sd) t += static_cast<double>(sd->draft_depth) * c.drafter_step_cost;
    return t;
}

// BEG-MAB state (beg_mab.hpp:28-69).
struct Mab {
    struct Arm {
        tlt_strategy strategy;
        std::deque<double> rewards, accept_lens;
        int64_t selections = 0;
    };
    std::vector<Arm> arms;
    std::vector<int> thresholds;
    std::vector<std::vector<size_t>> groups;
    double epsilon = 0.1;
    int window = 20;

    static double median(const std::deque<double>& d) {  // :47-54
        if (d.empty()) return std::numeric_limits<double>::infinity();
        std::vector<double> v(d.begin(), d.end());
        std::sort(v.begin(), v.end());
        const size_t mid = v.size() / 2;
        return v.size() % 2 ? v[mid] : 0.5 * (v[mid - 1] + v[mid]);
    }

    // beg_initialize (:74-106)
    Mab(const std::vector<tlt_strategy>& s, const std::vector<int>& thr, double eps, int w) {
        if (s.empty()) throw ConfigErr("strategies", "must not be empty");
        if (eps < 0.0 || eps > 1.0) throw ConfigErr("epsilon", "must be in [0, 1]");
        if (w < 1) throw ConfigErr("window", "must be >= 1");
        if (thr.empty()) throw ConfigErr("thresholds", "must not be empty");
        for (size_t i = 0; i + 1 < thr.size(); ++i)
            if (thr[i] >= thr[i + 1]) throw ConfigErr("thresholds", "must be strictly ascending");
        epsilon = eps;
        window = w;
        thresholds = thr;
        for (auto& x : s) {
            validate(x);
            arms.push_back(Arm{x, {}, {}, 0});
        }
        std::map<int, std::vector<size_t>, std::greater<int>> by_verify;
        for (size_t i = 0; i < arms.size(); ++i) by_verify[arms[i].strategy.tokens_to_verify].push_back(i);
        if (by_verify.size() != thr.size())
            throw ConfigErr("thresholds", "count must equal the number of tokens_to_verify groups");
        for (auto& kv : by_verify) groups.push_back(kv.second);
    }

    // beg_record (:111-134): a_bar = sum/bs + 1, r = a_bar * bs / elapsed
    void record(const tlt_strategy& s, double elapsed, const int32_t* lens, int batch) {
        if (batch < 1) throw ConfigErr("batch_size", "must be >= 1");
        if (!(elapsed > 0.0)) throw ConfigErr("elapsed_time", "must be > 0");
        for (auto& arm : arms) {
            if (!same(arm.strategy, s)) continue;
            double sum = 0.0;
            for (int i = 0; i < batch; ++i) sum += lens[i];
            const double a_bar = sum / static_cast<double>(batch) + 1.0;
            push(arm, a_bar * static_cast<double>(batch) / elapsed, a_bar);
            return;
        }
        throw ConfigErr("strategy", "not a configured strategy");
    }
    // C1 log: every record pushed by beg_record on this replica since the last
    // take (arm, reward, a_bar), for the cross-rank merge
    struct LogRec {
        int arm;
        double reward, a_bar;
    };
    std::vector<LogRec> log;
    void push(Arm& arm, double reward, double a_bar, bool logged = true) {
        if (logged) log.push_back(LogRec{(int)(&arm - arms.data()), reward, a_bar});
        arm.rewards.push_back(reward);
        arm.accept_lens.push_back(a_bar);
        while (arm.rewards.size() > static_cast<size_t>(window)) arm.rewards.pop_front();
        while (arm.accept_lens.size() > static_cast<size_t>(window)) arm.accept_lens.pop_front();
    }

    // beg_select (:140-170)
    size_t select(int batch, Rng& rng) {
        if (thresholds.empty() || batch < thresholds.front())
            throw RoutingErr("batch size below the smallest bucket threshold");
        size_t bucket = thresholds.size() - 1;
        for (size_t i = 0; i + 1 < thresholds.size(); ++i)
            if (batch >= thresholds[i] && batch < thresholds[i + 1]) {
                bucket = i;
                break;
            }
        const auto& c = groups[bucket];
        size_t pick;
        if (c.size() == 1) {
            pick = c[0];
        } else if (rng.uniform01() < epsilon) {
            pick = c[rng.uniform_int(c.size())];
        } else {
            pick = c[0];
            double best = median(arms[pick].rewards);
            for (size_t i = 1; i < c.size(); ++i) {
                const double m = median(arms[c[i]].rewards);
                if (m > best) {
                    best = m;
                    pick = c[i];
                }
            }
        }
        arms[pick].selections += 1;
        return pick;
    }
};

// plan_captures / plan_captures_vanilla (capture_plan.hpp:58-155)
inline std::vector<tlt_capture_entry> plan_captures(const std::vector<tlt_strategy>& s, const std::vector<int>& thr,
                                                    int max_batch, bool vanilla, double* total) {
    if (thr.empty()) throw ConfigErr("thresholds", "must not be empty");
    for (size_t i = 0; i + 1 < thr.size(); ++i)
        if (thr[i] >= thr[i + 1]) throw ConfigErr("thresholds", "must be strictly ascending");
    if (max_batch < thr.back()) throw ConfigErr("max_batch", "must cover the last threshold");
    std::vector<std::pair<int, int>> ranges;
    for (size_t i = 0; i < thr.size(); ++i)
        ranges.emplace_back(thr[i], i + 1 < thr.size() ? thr[i + 1] - 1 : max_batch);
    std::vector<tlt_capture_entry> out;
    double tot = 0.0;
    auto add = [&](tlt_capture_entry e) {
        const int width = e.side == 0 ? e.tokens_to_verify : e.top_k;
        e.memory_units = static_cast<double>(e.bucket_hi) * static_cast<double>(width);
        tot += e.memory_units;
        out.push_back(e);
    };
    for (auto& x : s) validate(x);
    if (vanilla) {
        for (auto& x : s)
            for (auto [lo, hi] : ranges) {
                add(tlt_capture_entry{0, lo, hi, x.tokens_to_verify, 0, 0, 0.0});
                add(tlt_capture_entry{1, lo, hi, 0, x.top_k, x.draft_depth, 0.0});
            }
    } else {
        std::map<int, std::vector<tlt_strategy>, std::greater<int>> groups;
        for (auto& x : s) groups[x.tokens_to_verify].push_back(x);
        if (groups.size() != ranges.size())
            throw ConfigErr("thresholds", "count must equal the number of tokens_to_verify groups");
        size_t b = 0;
        for (auto& [verify, members] : groups) {
            auto [lo, hi] = ranges[b];
            add(tlt_capture_entry{0, lo, hi, verify, 0, 0, 0.0});
            std::map<std::pair<int, int>, bool> seen;
            for (auto& m : members) {
                auto key = std::make_pair(m.top_k, m.draft_depth);
                if (seen.count(key)) continue;
                seen[key] = true;
                add(tlt_capture_entry{1, lo, hi, 0, m.top_k, m.draft_depth, 0.0});
            }
            ++b;
        }
    }
    if (total) *total = tot;
    return out;
}

// Model-free n-gram fallback drafter (reference ngram.hpp:13-103 and the
// per-request NgramTracker, rollout.hpp:103-120). Keys are the last n tokens;
// each key holds its distinct continuations in first-seen order with a
// frequency and the latest step id. draft() picks (frequency desc, step id
// desc, continuation lexicographically asc) and truncates to depth; the chain
// it returns is verified on the GPU (Engine::sd_step_chain).
struct Ngram {
    struct Entry {
        std::vector<int32_t> cont;
        uint64_t freq = 0;
        int64_t last_step = 0;
    };
    int n = 2, cont_len = 8;
    size_t next_key_start = 0;  // tracker cursor over the request stream
    std::map<std::vector<int32_t>, std::vector<Entry>> entries;

    Ngram(int n_, int cont_len_) : n(n_), cont_len(cont_len_) {
        if (n < 1) throw ConfigErr("n", "must be >= 1");
        if (cont_len < 1) throw ConfigErr("continuation_len", "must be >= 1");
    }
    size_t size() const {
        size_t t = 0;
        for (auto& kv : entries) t += kv.second.size();
        return t;
    }
    // ngram.hpp:40-51
    void record(std::vector<int32_t> key, std::vector<int32_t> cont, int64_t step) {
        auto& list = entries[std::move(key)];
        for (auto& e : list)
            if (e.cont == cont) {
                e.freq += 1;
                e.last_step = std::max(e.last_step, step);
                return;
            }
        list.push_back(Entry{std::move(cont), 1, step});
    }
    // ngram_insert, ngram.hpp:62-78 (every n-gram of the response, truncated continuation)
    void insert(const int32_t* r, size_t len, int64_t step) {
        const size_t nn = (size_t)n;
        if (len < nn + 1) return;
        for (size_t s = 0; s + nn < len; ++s) {
            const size_t ce = std::min(len, s + nn + (size_t)cont_len);
            record(std::vector<int32_t>(r + s, r + s + nn), std::vector<int32_t>(r + s + nn, r + ce), step);
        }
    }
    // NgramTracker::extend, rollout.hpp:107-118 (only complete windows)
    void extend(const int32_t* stream, size_t len, int64_t step) {
        const size_t nn = (size_t)n, c = (size_t)cont_len;
        while (next_key_start + nn + c <= len) {
            const int32_t* k = stream + next_key_start;
            record(std::vector<int32_t>(k, k + nn), std::vector<int32_t>(k + nn, k + nn + c), step);
            ++next_key_start;
        }
    }
    // ngram_draft, ngram.hpp:83-101
    std::vector<int32_t> draft(const int32_t* ctx, size_t len, int depth) const {
        if (depth < 1) throw ConfigErr("depth", "must be >= 1");
        const size_t nn = (size_t)n;
        if (len < nn) return {};
        auto it = entries.find(std::vector<int32_t>(ctx + len - nn, ctx + len));
        if (it == entries.end()) return {};
        const Entry* best = nullptr;
        for (auto& e : it->second)
            if (!best || e.freq > best->freq || (e.freq == best->freq && e.last_step > best->last_step) ||
                (e.freq == best->freq && e.last_step == best->last_step && e.cont < best->cont))
                best = &e;
        std::vector<int32_t> out = best->cont;
        if (out.size() > (size_t)depth) out.resize((size_t)depth);
        return out;
    }
};

}  // namespace tlt
