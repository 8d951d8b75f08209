// Executed reference-side integration (GPU test tests/test_gpu_adapter.py):
// the reference's own types (specsim::SpecStrategy, DraftPlanner, DraftTree,
// AcceptResult, RngStream; /root/reference/proj/include/specsim, unmodified)
// drive the GPU engine through include/tlt_specsim.hpp. The loop is the body
// of specsim::spec_generate (spec_decode.hpp:351-380) with its two leaves
// swapped: the DraftPlanner is make_eagle_tree_planner (tlt_draft) and
// verify_greedy is the GPU target (tlt_verify_accept_commit of the planner's
// tree, uploaded from the host). Built by oracle/Makefile (test
// infrastructure) into oracle/_ref/adapter_run.
//
//   adapter_run <max_len> <D> <k> <T> <prompt tokens...>
// prints "tokens t0 t1 ..." and "accept_lens a0 a1 ...".
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "specsim/spec_decode.hpp"
#include "tlt_specsim.hpp"

int main(int argc, char** argv) {
    if (argc < 6) {
        std::fprintf(stderr, "usage: adapter_run max_len D k T prompt...\n");
        return 2;
    }
    const int max_len = std::atoi(argv[1]);
    specsim::SpecStrategy s{std::atoi(argv[2]), std::atoi(argv[3]), std::atoi(argv[4])};
    specsim::TokenSeq prompt;
    for (int i = 5; i < argc; ++i) prompt.push_back(std::atoi(argv[i]));
    // BASELINE config 1: tiny Llama-style target + EAGLE drafter (engine.py MODELS/INITS "tiny")
    tlt_model_cfg cfg{4096, 256, 2, 4, 2, 64, 688, 1, 1e4f, 1e-6f, 1, 512};
    tlt_init_cfg ini{42, 1.0f, 10.0f, 0.9f, 1.0f, 0.05f, 0};
    tlt_engine* e = nullptr;
    using CE = specsim::ConfigError;
    using RE = specsim::RoutingError;
    tlt_specsim::check<CE, RE>(tlt_engine_create(&cfg, &ini, 0, &e));
    const int32_t slot = 0, len = static_cast<int32_t>(prompt.size());
    tlt_specsim::check<CE, RE>(tlt_prefill(e, 1, &slot, &len, prompt.data()));

    s.validate();
    specsim::DraftPlanner planner =
        tlt_specsim::make_eagle_tree_planner<specsim::DraftPlanner, specsim::DraftTree, CE, RE>(e, slot);
    specsim::RngStream rng(0, 0);
    specsim::SpecResult out;
    specsim::TokenSeq ctx = prompt;
    while (static_cast<int>(out.tokens.size()) < max_len) {  // spec_generate, GreedyTree mode
        specsim::DraftTree tree = planner(ctx, s, rng);
        specsim::AcceptResult res =
            tlt_specsim::verify_greedy<specsim::AcceptResult, specsim::DraftTree, CE, RE>(e, slot, tree);
        out.accept_lens.push_back(res.accept_length);
        specsim::TokenSeq emitted = res.accepted;
        emitted.push_back(res.bonus);
        bool done = false;
        for (specsim::TokenId t : emitted) {
            out.tokens.push_back(t);
            ctx.push_back(t);
            if (t == specsim::kEosToken || static_cast<int>(out.tokens.size()) >= max_len) {
                done = true;
                break;
            }
        }
        if (done) break;
    }
    std::printf("tokens");
    for (auto t : out.tokens) std::printf(" %d", t);
    std::printf("\naccept_lens");
    for (auto a : out.accept_lens) std::printf(" %d", a);
    std::printf("\n");
    tlt_engine_destroy(e);
    return 0;
}
