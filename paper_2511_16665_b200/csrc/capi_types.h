// Opaque C-ABI handle types shared by the C-ABI translation units.
#pragma once
#include <memory>

#include "engine.h"
#include "host_select.h"

struct tlt_engine {
    std::unique_ptr<tlt::Engine> e;
};
struct tlt_mab {
    std::unique_ptr<tlt::Mab> m;
};
struct tlt_rng {
    tlt::Rng r;
};
struct tlt_ngram {
    tlt::Ngram g;
};
