// Compile-and-link check of include/tlt_specsim.hpp against the UNMODIFIED
// reference types (built by tests/test_integration_adapter.py; not run).
#include "specsim/beg_mab.hpp"
#include "specsim/spec_decode.hpp"
#include "tlt_specsim.hpp"

int main(int argc, char**) {
    if (argc > 100) {  // never executed: proves the instantiation type-checks and links
        std::vector<specsim::DraftTree> trees;
        std::vector<specsim::AcceptResult> res;
        specsim::SpecStrategy s{4, 4, 16};
        tlt_specsim::sd_step<specsim::SpecStrategy, specsim::DraftTree, specsim::AcceptResult, specsim::ConfigError,
                             specsim::RoutingError>(nullptr, s, std::vector<int>{0}, trees, res);
    }
    return 0;
}
