// Kernel-level entry points used by the GPU unit tests (plain pointers, C-ABI).
#include <cuda_runtime.h>
#include "tlt_internal.h"
#include "engine_kernels.h"
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>
#include "../../include/tlt_b200.h"

using namespace tlt;

static int dev_gemm(const void* x, int m, int k, const void* w, int n, int kind, float* y_f32, void* y_bf16,
                    float* ws, long long ws_elems, int max_splits, const int* dyn_n) {
    try {
        GemmPlan g = plan_gemm(m, n, k, std::getenv("TLT_GEMM_FORCE_VARIANT") ? std::atoi(std::getenv("TLT_GEMM_FORCE_VARIANT")) : 0);
        if (max_splits > 0 && g.splits > max_splits) {
            g.kb_per_split = (g.kb_total + max_splits - 1) / max_splits;
            g.splits = (g.kb_total + g.kb_per_split - 1) / g.kb_per_split;
        }
        CUtensorMap tw = make_tmap_bf16(w, n, k, k, 128);
        CUtensorMap tx = make_tmap_bf16(x, m, k, k, g.box_rows);
        EpiParams ep{};
        ep.kind = kind;
        ep.n_out = n;
        ep.m_tok = m;
        ep.out_f32 = y_f32;
        ep.ld_f32 = kind == EPI_SWIGLU ? n / 2 : n;
        ep.out_bf16 = static_cast<__nv_bfloat16*>(y_bf16);
        ep.ld_bf16 = kind == EPI_SWIGLU ? n / 2 : n;
        ep.dyn_n = dyn_n;
        ep.dyn_rpr = 1;
        launch_gemm(g, tw, tx, ep, ws, static_cast<size_t>(ws_elems), 0);
        CUDA_CHECK(cudaDeviceSynchronize());
        return g.splits;
    } catch (const std::exception& e) {
        tlt_set_last_error(e.what());
        return -1;
    }
}

extern "C" TLT_API int tlt_dev_gemm(const void* x, int m, int k, const void* w, int n, int kind, float* y_f32,
                                    void* y_bf16, float* ws, long long ws_elems, int max_splits) {
    return dev_gemm(x, m, k, w, n, kind, y_f32, y_bf16, ws, ws_elems, max_splits, nullptr);
}

// As tlt_dev_gemm with a device-resident live-row count (the bucketed graph
// pool's padding skip): rows >= *live_rows may be left unwritten.
extern "C" TLT_API int tlt_dev_gemm_live(const void* x, int m, int k, const void* w, int n, int kind, float* y_f32,
                                         void* y_bf16, float* ws, long long ws_elems, const int* live_rows) {
    return dev_gemm(x, m, k, w, n, kind, y_f32, y_bf16, ws, ws_elems, 0, live_rows);
}

// LM head with the fused top-k epilogue (EPI_TOPK, whole-K accumulators) and
// the per-row merge, as Engine::lm_topk runs it: logits never leave the SM.
// part: [ceil(n/128)][m][2 + 2k] floats; thr: null or [m] zeroed uints (the
// per-row k-th-value bounds, left zeroed by the merge). Returns the plan's
// CTA-pair factor.
extern "C" TLT_API int tlt_dev_lm_topk(const void* x, int m, int k, const void* w, int n, int topk, float* part,
                                       int* out_tok, float* out_logit, float* out_M, float* out_S, unsigned* thr) {
    try {
        if (topk < 1 || topk > 8) throw ConfigErr("topk", "must be in [1, 8]");
        GemmPlan g = plan_gemm(m, n, k, std::getenv("TLT_GEMM_FORCE_VARIANT") ? std::atoi(std::getenv("TLT_GEMM_FORCE_VARIANT")) : 0);
        g.kb_per_split = g.kb_total;
        g.splits = 1;
        CUtensorMap tw = make_tmap_bf16(w, n, k, k, 128);
        CUtensorMap tx = make_tmap_bf16(x, m, k, k, g.box_rows);
        EpiParams ep{};
        ep.kind = EPI_TOPK;
        ep.n_out = n;
        ep.m_tok = m;
        ep.out_f32 = part;
        ep.topk_k = topk;
        ep.topk_thr = topk > 1 ? thr : nullptr;
        launch_gemm(g, tw, tx, ep, nullptr, 0, 0);
        launch_topk_merge(part, (n + 127) / 128, m, topk, nullptr, out_tok, out_logit, out_M, out_S, 0, ep.topk_thr);
        CUDA_CHECK(cudaDeviceSynchronize());
        return g.pair;
    } catch (const std::exception& e) {
        tlt_set_last_error(e.what());
        return -1;
    }
}

// Average device time of one GEMM launch (incl. its split-K reduce), `iters`
// back-to-back launches on a private stream bracketed by CUDA events.
extern "C" TLT_API int tlt_dev_time_gemm(const void* x, int m, int k, const void* w, int n, int kind, float* y_f32,
                                         void* y_bf16, float* ws, long long ws_elems, int iters, float* avg_ms) {
    try {
        GemmPlan g = plan_gemm(m, n, k, std::getenv("TLT_GEMM_FORCE_VARIANT") ? std::atoi(std::getenv("TLT_GEMM_FORCE_VARIANT")) : 0);
        CUtensorMap tw = make_tmap_bf16(w, n, k, k, 128);
        CUtensorMap tx = make_tmap_bf16(x, m, k, k, g.box_rows);
        EpiParams ep{};
        ep.kind = kind;
        ep.n_out = n;
        ep.m_tok = m;
        ep.out_f32 = y_f32;
        ep.ld_f32 = kind == EPI_SWIGLU ? n / 2 : n;
        ep.out_bf16 = static_cast<__nv_bfloat16*>(y_bf16);
        ep.ld_bf16 = kind == EPI_SWIGLU ? n / 2 : n;
        cudaStream_t st;
        CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        cudaEvent_t e0, e1;
        CUDA_CHECK(cudaEventCreate(&e0));
        CUDA_CHECK(cudaEventCreate(&e1));
        for (int i = 0; i < 3; ++i) launch_gemm(g, tw, tx, ep, ws, static_cast<size_t>(ws_elems), st);
        CUDA_CHECK(cudaEventRecord(e0, st));
        for (int i = 0; i < iters; ++i) launch_gemm(g, tw, tx, ep, ws, static_cast<size_t>(ws_elems), st);
        CUDA_CHECK(cudaEventRecord(e1, st));
        CUDA_CHECK(cudaEventSynchronize(e1));
        float ms = 0.f;
        CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
        *avg_ms = ms / iters;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaStreamDestroy(st);
        return g.splits;
    } catch (const std::exception& e) {
        tlt_set_last_error(e.what());
        return -1;
    }
}

// Row top-k over materialised fp32 logits (chunked scan + merge), timed with
// CUDA events over `iters` launches; outputs of the last launch.
extern "C" TLT_API int tlt_dev_row_topk(const float* logits, int R, int V, int k, float* part, int* out_tok,
                                        float* out_logit, float* out_M, float* out_S, int iters, float* avg_ms) {
    try {
        cudaStream_t st;
        CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        cudaEvent_t e0, e1;
        CUDA_CHECK(cudaEventCreate(&e0));
        CUDA_CHECK(cudaEventCreate(&e1));
        int nch = 0;
        CUDA_CHECK(cudaEventRecord(e0, st));
        for (int i = 0; i < std::max(1, iters); ++i) {
            nch = launch_row_topk_chunked(logits, R, V, nullptr, k, part, st);
            launch_topk_merge(part, nch, R, k, nullptr, out_tok, out_logit, out_M, out_S, st);
        }
        CUDA_CHECK(cudaEventRecord(e1, st));
        CUDA_CHECK(cudaEventSynchronize(e1));
        float ms = 0.f;
        CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
        if (avg_ms) *avg_ms = ms / std::max(1, iters);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaStreamDestroy(st);
        return nch;
    } catch (const std::exception& e) {
        tlt_set_last_error(e.what());
        return -1;
    }
}

// Tree-masked attention over explicit buffers (unit tests): q [R][H*hd],
// kc/vc [slots][KV][cap][hd] bf16, out [R][H*hd]; rows: slot[R], mask[R][32];
// groups: slot/lc/tail0/ntail[n_groups]; R = n_groups * rows_per_req.
// kernel: 0 mma.sync tree/decode kernels, 1 tcgen05 kernel (when eligible).
extern "C" TLT_API int tlt_dev_attention(const void* q, const void* kc, const void* vc, void* out, int n_groups,
                                         int rows_per_req, int H, int KV, int hd, int cap, const int* row_slot,
                                         const unsigned* row_mask, const int* g_slot, const int* g_lc,
                                         const int* g_tail0, const int* g_ntail, int max_keys, int kernel) {
    try {
        const int R = n_groups * rows_per_req;
        AttnParams p{};
        p.q = static_cast<const __nv_bfloat16*>(q);
        p.out = static_cast<__nv_bfloat16*>(out);
        p.kc = static_cast<const __nv_bfloat16*>(kc);
        p.vc = static_cast<const __nv_bfloat16*>(vc);
        p.rows.slot = const_cast<int*>(row_slot);
        p.rows.mask = const_cast<unsigned*>(row_mask);
        p.g.slot = const_cast<int*>(g_slot);
        p.g.lc = const_cast<int*>(g_lc);
        p.g.tail0 = const_cast<int*>(g_tail0);
        p.g.ntail = const_cast<int*>(g_ntail);
        p.rows_per_req = rows_per_req;
        p.n_groups = n_groups;
        p.H = H;
        p.KV = KV;
        p.hd = hd;
        p.cap = cap;
        p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)hd));
        p.impl = 1;
        // kernel 0/1: fixed 256-key splits (legacy / tcgen05 kernels); 2/3/4:
        // the engine's split plan (flash-decode or tree kernel)
        if (kernel >= 2) {
            attention_plan_splits(p, max_keys);
        } else {
            p.chunk = attention_mma_split();
            p.max_splits = std::max(1, (max_keys + p.chunk - 1) / p.chunk);
        }
        p.qv_cap = rows_per_req * (H / KV);
        const size_t need = (size_t)n_groups * p.max_splits * p.qv_cap * KV;
        float *wm = nullptr, *wl = nullptr, *wo = nullptr;
        CUDA_CHECK(cudaMalloc(&wm, need * sizeof(float)));
        CUDA_CHECK(cudaMalloc(&wl, need * sizeof(float)));
        CUDA_CHECK(cudaMalloc(&wo, need * hd * sizeof(float)));
        p.ws_m = wm;
        p.ws_l = wl;
        p.ws_o = wo;
        (void)R;
        const char* prev = std::getenv("TLT_ATTN_TC");
        (void)prev;
        if (kernel == 1) {
            if (!attention_tc_shape_ok(p)) throw ConfigErr("kernel", "shape not eligible for the tcgen05 kernel");
            launch_attention_tc(p, 0);
            launch_attn_combine_only(p, 0);
        } else if (kernel == 2 || kernel == 3) {
            // flash-decode kernel as the engine sizes it (<= 16 query vectors per
            // request and KV head); 3 = split combine fused into the last CTA
            int* ctr = nullptr;
            if (rows_per_req * (H / KV) > 16) throw ConfigErr("kernel", "decode kernel needs <= 16 query vectors");
            if (!p.dec) throw ConfigErr("kernel", "decode kernel disabled (TLT_ATTN_DEC=0)");
            if (kernel == 3) {
                CUDA_CHECK(cudaMalloc(&ctr, sizeof(int) * n_groups * KV));
                CUDA_CHECK(cudaMemset(ctr, 0, sizeof(int) * n_groups * KV));
                p.counters = ctr;
            }
            launch_attention(p, 0);
            CUDA_CHECK(cudaDeviceSynchronize());
            if (ctr) {  // the last CTA must have reset every counter (graph-replay invariant)
                std::vector<int> h(n_groups * KV);
                CUDA_CHECK(cudaMemcpy(h.data(), ctr, sizeof(int) * h.size(), cudaMemcpyDeviceToHost));
                cudaFree(ctr);
                for (int v : h)
                    if (v != 0) throw ConfigErr("counters", "fused combine left a non-zero counter");
            }
        } else if (kernel == 4) {
            // tree kernel as the engine plans it (per-request splits, direct
            // single-split outputs, separate combine)
            if (rows_per_req * (H / KV) <= 16) throw ConfigErr("kernel", "tree kernel needs > 16 query vectors");
            launch_attention(p, 0);
        } else if (kernel == 7) {
            // tcgen05 / TMEM tree attention (attn_tc5.cu) with the engine's split plan
            if (!attention_tma_enabled(p) || !attention_tree_tc_eligible(p))
                throw ConfigErr("kernel", "shape not eligible for the tcgen05 tree kernel");
            const long long rows = (long long)n_groups * KV * cap;
            const CUtensorMap tk = make_tmap_kv(kc, rows, hd), tv = make_tmap_kv(vc, rows, hd);
            launch_attention_tree_tc(tk, tv, p, 0);
            CUDA_CHECK(cudaDeviceSynchronize());
        } else if (kernel == 5 || kernel == 6) {
            // TMA-fed kernel (attn_tma.cu) with the engine's split plan; 6 =
            // split combine fused into the last CTA (decode shapes)
            if (!attention_tma_enabled(p)) throw ConfigErr("kernel", "shape not eligible for the TMA kernel");
            int* ctr = nullptr;
            if (kernel == 6) {
                const long long n = (long long)n_groups * KV * ((rows_per_req * (H / KV) + 15) / 16);
                CUDA_CHECK(cudaMalloc(&ctr, sizeof(int) * n));
                CUDA_CHECK(cudaMemset(ctr, 0, sizeof(int) * n));
                p.counters = ctr;
            }
            const long long rows = (long long)n_groups * KV * cap;  // caches hold n_groups slots
            const CUtensorMap tk = make_tmap_kv(kc, rows, hd), tv = make_tmap_kv(vc, rows, hd);
            launch_attention_tma(tk, tv, p, 0);
            CUDA_CHECK(cudaDeviceSynchronize());
            if (ctr) cudaFree(ctr);
        } else {
            p.impl = 1;
            launch_attention_legacy(p, 0);
        }
        CUDA_CHECK(cudaDeviceSynchronize());
        cudaFree(wm);
        cudaFree(wl);
        cudaFree(wo);
        return 0;
    } catch (const std::exception& e) {
        tlt_set_last_error(e.what());
        return -1;
    }
}

// e4m3 GEMM through the production path: x [m][k], w [n][k] bf16 are
// quantised per row (launch_quant_rows_e4m3), then y = (qx qw^T) * sx * sw
// (fp32) with the kind::f8f6f4 kernel. Also returns the quantised operands
// and scales for the reference. Returns the CTA-pair factor used.
extern "C" TLT_API int tlt_dev_gemm_e4m3(const void* x, int m, int k, const void* w, int n, float* y, void* qx,
                                         float* sx, void* qw, float* sw) {
    try {
        launch_quant_rows_e4m3(static_cast<const __nv_bfloat16*>(x), m, k, k, qx, sx, 0);
        launch_quant_rows_e4m3(static_cast<const __nv_bfloat16*>(w), n, k, k, qw, sw, 0);
        // the GEMM streams its weight stages before griddepcontrol.wait (weights
        // are static in the engine): here they were just written, so finish first
        CUDA_CHECK(cudaDeviceSynchronize());
        GemmPlan g = plan_gemm_e4m3(m, n, k);
        CUtensorMap tw = make_tmap_e4m3(qw, n, k, k, 128);
        CUtensorMap tx = make_tmap_e4m3(qx, m, k, k, g.box_rows);
        EpiParams ep{};
        ep.kind = EPI_F32;
        ep.n_out = n;
        ep.m_tok = m;
        ep.out_f32 = y;
        ep.ld_f32 = n;
        ep.row_scale = sw;
        ep.tok_scale = sx;
        launch_gemm(g, tw, tx, ep, nullptr, 0, 0);
        CUDA_CHECK(cudaDeviceSynchronize());
        return g.pair;
    } catch (const std::exception& e) {
        tlt_set_last_error(e.what());
        return -1;
    }
}
