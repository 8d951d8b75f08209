// tlt_specsim.hpp — reference-side adapter (what a specsim maintainer adds).
//
// Maps the reference C++ types (specsim::SpecStrategy, DraftTree,
// AcceptResult, CaptureEntry; /root/reference/proj/include/specsim) onto the
// C-ABI of libtlt_b200.so. Header-only; include it after the specsim headers.
// The batched calls replace the per-request loop body of run_rollout
// (rollout.hpp:191-241): one tlt_sd_step serves every running request.
#pragma once
#include <functional>
#include <stdexcept>
#include <type_traits>
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

// ---- the per-request seam: DraftPlanner + verify_greedy over the GPU ------
// Reference: using DraftPlanner = std::function<DraftTree(const TokenSeq&,
// const SpecStrategy&, RngStream&)> (spec_decode.hpp:319-320) and
// verify_greedy(target, ctx, tree) -> AcceptResult (:245-268). The engine
// holds each request's context in its KV cache (slot), so the planner's ctx
// argument must be that slot's committed tokens + the pending root.

// build_draft_tree for one request on the GPU drafter (tlt_draft, b = 1).
template <class DraftTree, class Strategy, class ConfigError, class RoutingError>
DraftTree draft_tree(tlt_engine* e, int slot, const Strategy& s) {
    const int T = s.tokens_to_verify;
    std::vector<int32_t> tok(T), par(T), dep(T);
    std::vector<double> prob(T), pp(T);
    int32_t n = 0;
    tlt_tree_out to{tok.data(), par.data(), dep.data(), prob.data(), pp.data(), &n};
    const tlt_strategy cs = to_c(s.draft_depth, s.top_k, s.tokens_to_verify);
    const int32_t sl = slot;
    check<ConfigError, RoutingError>(tlt_draft(e, &cs, 1, &sl, &to));
    DraftTree tree;
    for (int j = 0; j < n; ++j) {
        typename decltype(tree.nodes)::value_type node;
        node.token = tok[j];
        node.parent = par[j];
        node.depth = dep[j];
        node.prob = prob[j];
        node.path_prob = pp[j];
        tree.nodes.push_back(node);
    }
    return tree;
}

// verify_greedy + KV commit of an arbitrary DraftTree for one request
// (tlt_verify_accept_commit with the tree uploaded from the host).
template <class AcceptResult, class DraftTree, class ConfigError, class RoutingError>
AcceptResult verify_greedy(tlt_engine* e, int slot, const DraftTree& tree) {
    const int n = static_cast<int>(tree.nodes.size()), stride = n > 0 ? n : 1;
    std::vector<int32_t> tok(stride), par(stride), acc(stride);
    std::vector<double> prob(stride), pp(stride);
    for (int j = 0; j < n; ++j) {
        tok[j] = tree.nodes[j].token;
        par[j] = tree.nodes[j].parent;
        prob[j] = tree.nodes[j].prob;
        pp[j] = tree.nodes[j].path_prob;
    }
    const int32_t nn = n, sl = slot;
    int32_t alen = 0, bonus = 0;
    tlt_tree_in ti{tok.data(), par.data(), prob.data(), pp.data(), &nn, stride};
    tlt_accept_out ao{acc.data(), nullptr, &alen, &bonus, nullptr, nullptr, nullptr};
    check<ConfigError, RoutingError>(tlt_verify_accept_commit(e, 1, &sl, &ti, &ao));
    AcceptResult r;
    r.accept_length = alen;
    r.bonus = bonus;
    r.accepted.assign(acc.begin(), acc.begin() + alen);
    return r;
}

// A reference DraftPlanner whose trees come from the GPU EAGLE drafter
// (drop-in for make_adaptive_tree_planner, spec_decode.hpp:322-327).
template <class DraftPlanner, class DraftTree, class ConfigError, class RoutingError>
DraftPlanner make_eagle_tree_planner(tlt_engine* e, int slot) {
    return [e, slot](const auto& ctx, const auto& s, auto&) {
        int32_t len = 0;
        check<ConfigError, RoutingError>(tlt_slot_len(e, slot, &len));
        if (static_cast<long long>(ctx.size()) != static_cast<long long>(len) + 1)
            throw ConfigError("ctx", "does not match the engine slot's committed tokens + root");
        return draft_tree<DraftTree, std::decay_t<decltype(s)>, ConfigError, RoutingError>(e, slot, s);
    };
}

}  // namespace tlt_specsim
