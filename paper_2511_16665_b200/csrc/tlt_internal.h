// Internal host-side declarations shared by the CUDA translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "gemm.cuh"

namespace tlt {

// Maps onto TLT_ERR_CUDA at the C-ABI boundary.
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
// Maps onto TLT_ERR_CONFIG (reference specsim::ConfigError, errors.hpp:9-19).
struct ConfigErr : std::runtime_error {
    std::string field;
    ConfigErr(std::string f, const std::string& m)
        : std::runtime_error(f.empty() ? m : f + ": " + m), field(std::move(f)) {}
};
// Maps onto TLT_ERR_ROUTING (reference specsim::RoutingError, errors.hpp:32-34).
struct RoutingErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define CUDA_CHECK(expr)                                                                     \
    do {                                                                                     \
        cudaError_t e_ = (expr);                                                             \
        if (e_ != cudaSuccess)                                                               \
            throw ::tlt::CudaError(std::string(#expr) + ": " + cudaGetErrorString(e_) + " @" + \
                                   __FILE__ + ":" + std::to_string(__LINE__));               \
    } while (0)

struct GemmPlan {
    int bn = 16, n_ttiles = 1, n_wtiles = 1, kb_total = 1, kb_per_split = 1, splits = 1, stages = 4;
    int smem = 0;
    unsigned tmem_cols = 32;
    int wm = 1;  // 128-row weight sub-tiles per CTA (1 or 2)
    int pair = 1;      // 2: cta_group::2 CTA pair per 256-row tile
    int box_rows = 16; // token rows per TMA box of the activation tensor map (bn / pair)
    int l2pf = 0;      // weight k-blocks prefetched into L2 ahead of the smem ring
    int persist = 0;   // 1: persistent kernel (double-buffered TMEM accumulators)
    int fp8 = 0;       // 1: e4m3 operands (kind::f8f6f4), per-row / per-token scales in the epilogue
    int mc = 1;        // CTA pairs per cluster sharing one weight k-block by TMA multicast (pair plans)
    int wn = 1;        // token sub-tiles (MMAs of N = bn / wn) sharing each weight k-block (bn up to 512)
    bool same_as(const GemmPlan& o) const {
        return bn == o.bn && n_ttiles == o.n_ttiles && n_wtiles == o.n_wtiles && splits == o.splits &&
               stages == o.stages && wm == o.wm && pair == o.pair && persist == o.persist && mc == o.mc &&
               wn == o.wn;
    }
};

int num_sms();
CUtensorMap make_tmap_bf16(const void* base, int rows, int cols, long long row_stride_elems, int box_rows);
GemmPlan plan_gemm(int m_tok, int n_out, int k, int variant = 0);
void gemm_one_wave(GemmPlan& g);  // TLT_GEMM_ONE_WAVE: <= 1 CTA per SM with the full smem ring
GemmPlan plan_gemm_e4m3(int m_tok, int n_out, int k);
CUtensorMap make_tmap_e4m3(const void* base, int rows, int cols, long long row_stride_elems, int box_rows);
int* gemm_norm_counter();
void launch_gemm(const GemmPlan& g, const CUtensorMap& tmW, const CUtensorMap& tmX, const EpiParams& ep,
                 float* workspace, size_t workspace_elems, cudaStream_t st);

}  // namespace tlt
