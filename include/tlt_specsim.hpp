// tlt_specsim.hpp — reference-side adapter (what a specsim maintainer adds).
//
// Maps the reference C++ types (specsim::SpecStrategy, DraftTree,
// AcceptResult, CaptureEntry; /root/reference/proj/include/specsim) onto the
// C-ABI of libtlt_b200.so. Header-only; include it after the specsim headers.
// The batched calls replace the per-request loop body of run_rollout
// (rollout.hpp:191-241): one tlt_sd_step serves every running request.
#pragma once
#include <stdexcept>
#include <string>
#include <vector>

#include "tlt_b200.h"

namespace tlt_specsim {

// Re-throw C-ABI status codes as the reference exception types (errors.hpp:9-34).
template <class ConfigError, class RoutingError>
inline void check(int rc) {
    if (rc == TLT_OK) return;
    const std::string msg = tlt_last_error(nullptr);
    if (rc == TLT_ERR_CONFIG) throw ConfigError("", msg);
    if (rc == TLT_ERR_ROUTING) throw RoutingError(msg);
    throw std::runtime_error(msg);
}

inline tlt_strategy to_c(int draft_depth, int top_k, int tokens_to_verify) {
    return tlt_strategy{draft_depth, top_k, tokens_to_verify};
}

// One batched greedy tree-SD engine step for `slots`; fills the reference's
// DraftTree and AcceptResult per request (spec_decode.hpp:61-80).
template <class Strategy, class DraftTree, class AcceptResult, class ConfigError, class RoutingError>
void sd_step(tlt_engine* e, const Strategy& s, const std::vector<int>& slots, std::vector<DraftTree>& trees,
             std::vector<AcceptResult>& results) {
    const int b = static_cast<int>(slots.size()), T = s.tokens_to_verify, D = s.draft_depth;
    std::vector<int32_t> tok(b * T), par(b * T), dep(b * T), n(b), acc(b * D), alen(b), bonus(b);
    std::vector<double> prob(b * T), pp(b * T);
    tlt_tree_out to{tok.data(), par.data(), dep.data(), prob.data(), pp.data(), n.data()};
    tlt_accept_out ao{acc.data(), nullptr, alen.data(), bonus.data(), nullptr, nullptr, nullptr};
    const tlt_strategy cs = to_c(s.draft_depth, s.top_k, s.tokens_to_verify);
    check<ConfigError, RoutingError>(tlt_sd_step(e, &cs, b, slots.data(), &to, &ao));
    trees.assign(b, {});
    results.assign(b, {});
    for (int i = 0; i < b; ++i) {
        for (int j = 0; j < n[i]; ++j) {
            typename decltype(trees[i].nodes)::value_type node;
            node.token = tok[i * T + j];
            node.parent = par[i * T + j];
            node.depth = dep[i * T + j];
            node.prob = prob[i * T + j];
            node.path_prob = pp[i * T + j];
            trees[i].nodes.push_back(node);
        }
        results[i].accept_length = alen[i];
        results[i].bonus = bonus[i];
        results[i].accepted.assign(acc.begin() + i * D, acc.begin() + i * D + alen[i]);
    }
}

}  // namespace tlt_specsim
