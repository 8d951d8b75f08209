// Device-side row / group metadata shared by the engine kernels.
//
// Every forward (prefill chunk, drafter level, target verify, AR decode) is a
// set of ROWS grouped per request with a STATIC row stride (rows_per_req), so
// a CUDA graph captured at bucket_hi replays for any batch in the bucket:
// padding rows carry slot = -1 and are skipped by every side effect.
// Attention visibility of a row = the request's committed prefix [0, Lc) plus
// a bitmask over the "tail" cache entries [tail0, tail0 + n_tail) (tree nodes,
// expansion slots, or the causal block of a prefill chunk).
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

namespace tlt {

constexpr int kMaskWords = 32;  // up to 1024 tail entries per group
constexpr int kMaxTopK = 8;
constexpr int kMaxDepth = 16;
constexpr int kMaxT = 128;

struct StepIn {  // host-uploaded per batch index
    int slot;
    int lt;  // target committed KV length (root position)
    int ld;  // drafter committed KV length
    int pad;
};

struct Rows {            // SoA row metadata, capacity R
    int* tok;            // token id
    int* pos;            // RoPE position
    int* slot;           // request slot, -1 = padding row
    int* cidx;           // KV-cache index inside the slot
    int* fkind;          // drafter input feature source: 0 zero, 1 target history, 2 drafter row
    long long* fidx;     // element offset (units of hidden) into that source
    uint32_t* mask;      // [R][kMaskWords] visibility of tail entries
};

struct Groups {          // per request in the batch
    int* slot;           // request slot, -1 = inactive group
    int* lc;             // committed prefix length visible to all rows
    int* tail0;          // cache index of tail entry 0
    int* ntail;          // number of tail entries
};

// Drafter tree arena entry (reference detail::Candidate, spec_decode.hpp:84-91)
struct Cand {
    double pp;    // path_prob
    double prob;  // p
    int token;
    int parent;   // arena index, -1 root
    int depth;
    int birth;    // arena index == creation order
    int row;      // drafter expansion row (global row id) if expanded, else -1
    int eslot;    // expansion slot (tail index) if expanded
};

}  // namespace tlt
