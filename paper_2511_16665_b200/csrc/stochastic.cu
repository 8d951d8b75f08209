// Rejection-sampling SD on the GPU (K9): the drafter samples a linear chain
// (build_sampled_chain, spec_decode.hpp:202-223) and the target accepts with
// min(1, p/q), resampling the normalized residual (p - q)^+ on rejection and
// drawing the bonus from p after a full accept (verify_stochastic,
// spec_decode.hpp:275-313). Uniforms are the reference RngStream draws,
// host-generated per request in consumption order and uploaded.
//
// Distributions: a row's raw distribution is p_i = exp((double)(l_i - M)) / S
// (M = row max, S = sum expf(l - M), fp32) — the same definition the greedy
// path exports; tempering (token_model.hpp:161-173) is applied in double.
// Inverse CDF (token_model.hpp:83-91) uses a fixed blocked double scan: each
// thread owns a contiguous segment, segments are prefix-summed in thread
// order; when u falls within a rigorous rounding bound of a CDF boundary the
// pick is redone with the reference's sequential sum, so the result is the
// reference's pick by construction (inverse_cdf_block).
#include <cuda_runtime.h>
#include <math_constants.h>

#include "engine_kernels.h"
#include "kernels.cuh"
#include "pdl.cuh"

namespace tlt {

namespace {
constexpr int kST = 256;  // threads per row CTA

// block-wide double sum in fixed order (thread order)
__device__ double block_sum_fixed(double v, double* sh) {
    sh[threadIdx.x] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < (int)blockDim.x; ++i) s += sh[i];
        sh[kST] = s;
    }
    __syncthreads();
    const double r = sh[kST];
    __syncthreads();
    return r;
}

// inverse CDF over a probability row held in global memory (double):
// min{t : u < cum(t)}, fallback V-1 (token_model.hpp:83-91), bit-exact with
// the reference's SEQUENTIAL cumulative sum.
//
// Fast path: a blocked scan (each thread owns a contiguous segment, segment
// sums exclusive-scanned in thread order) picks t*. The blocked prefix sums
// cumB and the reference's sequential ones cumR are both sums of <= V
// non-negative doubles totalling ~1, so each is within V * 2^-53 * (1 + tiny)
// of the exact prefix and |cumB(t) - cumR(t)| < delta = V * 2^-51 (2x
// margin). cumR is monotone (adding p >= 0 never decreases a double), so
// t* is the reference's pick whenever u >= cumB(t*-1) + delta and
// u < cumB(t*) - delta. Otherwise u sits within rounding of a CDF boundary
// and one thread replays the reference's sequential sum exactly (rare: the
// window is ~1e-10 wide).
__device__ int inverse_cdf_block(const double* p, int V, double u, double* sh, int* ish) {
    __shared__ double s_lo, s_hi;
    const int per = (V + kST - 1) / kST;
    const int a = threadIdx.x * per, b = min(V, a + per);
    double seg = 0.0;
    for (int i = a; i < b; ++i) seg += p[i];
    sh[threadIdx.x] = seg;
    __syncthreads();
    if (threadIdx.x == 0) {  // exclusive scan of segment sums, thread order
        double c = 0.0;
        for (int i = 0; i < (int)blockDim.x; ++i) {
            const double s = sh[i];
            sh[i] = c;
            c += s;
        }
        ish[0] = V - 1;
    }
    __syncthreads();
    double cum = sh[threadIdx.x], lo = cum, hi = cum;
    int found = 0x7fffffff;
    for (int i = a; i < b && i < V - 1; ++i) {
        lo = cum;
        cum += p[i];
        if (u < cum) {
            found = i;
            hi = cum;
            break;
        }
    }
    if (found != 0x7fffffff) atomicMin(ish, found);
    __syncthreads();
    const int r = ish[0];
    if (found == r) {  // the winning thread: cumB(t*-1), cumB(t*)
        s_lo = lo;
        s_hi = hi;
    }
    if (r == V - 1 && a <= V - 2 && V - 2 < b) {  // no pick below V-1: cumB(V-2) bounds it
        s_lo = cum;
        s_hi = CUDART_INF;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const double delta = (double)V * 0x1p-51;
        const bool lo_ok = r == 0 || u - s_lo >= delta;
        const bool hi_ok = r == V - 1 || s_hi - u > delta;
        if (!(lo_ok && hi_ok)) {  // boundary window: the reference's own loop
            double c = 0.0;
            int t = V - 1;
            for (int i = 0; i < V - 1; ++i) {
                c += p[i];
                if (u < c) {
                    t = i;
                    break;
                }
            }
            ish[0] = t;
        }
    }
    __syncthreads();
    const int res = ish[0];
    __syncthreads();
    return res;
}

// raw row from logits into dst (double), returns nothing; M/S via block reductions
__device__ void raw_row(const float* lg, int V, double* dst, float* fsh, double* dsh, float* outM, float* outS) {
    float m = -CUDART_INF_F;
    for (int i = threadIdx.x; i < V; i += blockDim.x) m = fmaxf(m, lg[i]);
    fsh[threadIdx.x] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        float mm = fsh[0];
        for (int i = 1; i < (int)blockDim.x; ++i) mm = fmaxf(mm, fsh[i]);
        fsh[kST] = mm;
    }
    __syncthreads();
    const float M = fsh[kST];
    // normalizer in double (fixed thread order) so the row sums to 1 within
    // 1e-15, as a reference Distribution must (token_model.hpp:34-41)
    double s = 0.0;
    for (int i = threadIdx.x; i < V; i += blockDim.x) {
        const double e = exp((double)(lg[i] - M));
        dst[i] = e;
        s += e;
    }
    const double S = block_sum_fixed(s, dsh);
    for (int i = threadIdx.x; i < V; i += blockDim.x) dst[i] /= S;
    if (threadIdx.x == 0) {
        if (outM) *outM = M;
        if (outS) *outS = (float)S;  // the tree kernel re-derives p from (logit, M, S)
    }
    __syncthreads();
}

// temper in place (target_next_dist): t == 1 raw; t == 0 one-hot argmax
// (lowest id); else p^(1/t) normalized (fixed-order double sum)
__device__ void temper_row(double* p, int V, double t, double* sh, int* ish) {
    if (t == 1.0) return;
    if (t == 0.0) {
        // argmax, lowest id on ties
        double bv = -1.0;
        int bi = 0x7fffffff;
        for (int i = threadIdx.x; i < V; i += blockDim.x)
            if (p[i] > bv) {
                bv = p[i];
                bi = i;
            }
        sh[threadIdx.x] = bv;
        ish[threadIdx.x] = bi;
        __syncthreads();
        if (threadIdx.x == 0) {
            double b = sh[0];
            int ix = ish[0];
            for (int i = 1; i < (int)blockDim.x; ++i)
                if (sh[i] > b || (sh[i] == b && ish[i] < ix)) {
                    b = sh[i];
                    ix = ish[i];
                }
            ish[0] = ix;
        }
        __syncthreads();
        const int a = ish[0];
        for (int i = threadIdx.x; i < V; i += blockDim.x) p[i] = i == a ? 1.0 : 0.0;
        __syncthreads();
        return;
    }
    const double inv = 1.0 / t;
    double s = 0.0;
    const int per = (V + kST - 1) / kST;
    const int a0 = threadIdx.x * per, b0 = min(V, a0 + per);
    for (int i = a0; i < b0; ++i) {
        const double v = p[i] > 0.0 ? pow(p[i], inv) : 0.0;
        p[i] = v;
        s += v;
    }
    const double tot = block_sum_fixed(s, sh);
    if (tot <= 0.0) {
        for (int i = threadIdx.x; i < V; i += blockDim.x) p[i] = 1.0 / (double)V;
    } else {
        for (int i = threadIdx.x; i < V; i += blockDim.x) p[i] /= tot;
    }
    __syncthreads();
}
}  // namespace

// Drafter chain level: per request, the distribution of its (single) row is
// written to q[i][level] (double) and a token is drawn with the level's
// uniform. Outputs follow the top-k interface (k = 1) consumed by the tree
// kernel: token, its logit, M and S.
__global__ void __launch_bounds__(kST) k_chain_sample(const float* __restrict__ logits, int V, const int* live,
                                                      double* __restrict__ q, int level, int D,
                                                      const double* __restrict__ uni, int uni_stride,
                                                      int* __restrict__ out_tok, float* __restrict__ out_logit,
                                                      float* __restrict__ out_M, float* __restrict__ out_S) {
    pdl_wait();
    __shared__ float fsh[kST + 2];
    __shared__ double dsh[kST + 1];
    __shared__ int ish[kST];
    const int r = blockIdx.x;  // request index (one LM row per request)
    if (live && live[r] < 0) return;
    const float* lg = logits + (long long)r * V;
    double* qr = q + ((long long)r * D + (level - 1)) * V;
    raw_row(lg, V, qr, fsh, dsh, out_M + r, out_S + r);
    const double u = uni[(long long)r * uni_stride + (level - 1)];
    const int t = inverse_cdf_block(qr, V, u, dsh, ish);
    if (threadIdx.x == 0) {
        out_tok[r] = t;
        out_logit[r] = lg[t];
    }
}
void launch_chain_sample(const float* logits, int R, int V, const int* live, double* q, int level, int D,
                         const double* uni, int uni_stride, int* out_tok, float* out_logit, float* out_M, float* out_S,
                         cudaStream_t st) {
    launch_pdl(k_chain_sample, R, kST, 0, st, logits, V, live, q, level, D, uni, uni_stride, out_tok, out_logit,
               out_M, out_S);
}

// raw rows of arbitrary logits rows with the exact device code the accept
// kernel uses (parity export)
__global__ void __launch_bounds__(kST) k_raw_rows(const float* __restrict__ logits, int V, double* __restrict__ out) {
    pdl_wait();
    __shared__ float fsh[kST + 2];
    __shared__ double dsh[kST + 1];
    const int r = blockIdx.x;
    raw_row(logits + (long long)r * V, V, out + (long long)r * V, fsh, dsh, nullptr, nullptr);
}
void launch_raw_rows(const float* logits, int R, int V, double* out, cudaStream_t st) {
    launch_pdl(k_raw_rows, R, kST, 0, st, logits, V, out);
}

// Plain-decode sampling (rollout.hpp:252-253): token = inverse CDF of the
// tempered target row with the request's next uniform.
__global__ void __launch_bounds__(kST) k_sample_rows(const float* __restrict__ logits, int V, const int* live,
                                                     double temperature, const double* __restrict__ uni,
                                                     double* __restrict__ pbuf, int* __restrict__ out_tok) {
    pdl_wait();
    __shared__ float fsh[kST + 2];
    __shared__ double dsh[kST + 1];
    __shared__ int ish[kST];
    const int r = blockIdx.x;
    if (live && live[r] < 0) return;
    double* p = pbuf + (long long)r * V;
    raw_row(logits + (long long)r * V, V, p, fsh, dsh, nullptr, nullptr);
    temper_row(p, V, temperature, dsh, ish);
    const int t = inverse_cdf_block(p, V, uni[r], dsh, ish);
    if (threadIdx.x == 0) out_tok[r] = t;
}
void launch_sample_rows(const float* logits, int R, int V, const int* live, double temperature, const double* uni,
                        double* pbuf, int* out_tok, cudaStream_t st) {
    launch_pdl(k_sample_rows, R, kST, 0, st, logits, V, live, temperature, uni, pbuf, out_tok);
}

// verify_stochastic over the chain of request i (one CTA): verify rows are
// i*(D+1) + j (row 0 = root). Writes acc_len, accepted tokens/nodes, bonus,
// the number of uniforms consumed, and the raw target rows (for the parity
// export) into praw when non-null.
__global__ void __launch_bounds__(kST) k_accept_stochastic(const StepIn* __restrict__ step, int b, int D, int V,
                                                           double temperature, const float* __restrict__ vlogits,
                                                           const double* __restrict__ q, const int* __restrict__ chain,
                                                           const int* __restrict__ chain_n,
                                                           const double* __restrict__ uni, int uni_stride,
                                                           double* __restrict__ pbuf, int* __restrict__ acc_nodes,
                                                           int* __restrict__ acc_tok, int* __restrict__ acc_len,
                                                           int* __restrict__ bonus, int* __restrict__ consumed,
                                                           int maxD, int chain_stride, int cur0) {
    pdl_wait();
    __shared__ float fsh[kST + 2];
    __shared__ double dsh[kST + 1];
    __shared__ int ish[kST];
    __shared__ int s_dec;
    const int i = blockIdx.x;
    if (i >= b || step[i].slot < 0) return;
    const int n = chain_n[i];
    const double* ur = uni + (long long)i * uni_stride;
    int cur = cur0;  // sampled chains: the D chain draws come first; n-gram chains draw none
    // q == nullptr: host-proposed (n-gram) chain, empty draft_dist -> q is
    // one-hot at the drafted token (spec_decode.hpp:282, 296-298)
    double* p = pbuf + (long long)i * V;
    int a = 0;
    for (int j = 0; j <= n; ++j) {
        raw_row(vlogits + ((long long)i * (D + 1) + j) * V, V, p, fsh, dsh, nullptr, nullptr);
        temper_row(p, V, temperature, dsh, ish);
        if (j == n) {  // full accept: bonus ~ p (spec_decode.hpp:311)
            const int t = inverse_cdf_block(p, V, ur[cur], dsh, ish);
            cur += 1;
            if (threadIdx.x == 0) bonus[i] = t;
            break;
        }
        const int x = chain[(long long)i * chain_stride + j];
        const double* qr = q ? q + ((long long)i * kMaxDepth + j) * V : nullptr;  // layout of k_chain_sample
        if (threadIdx.x == 0) {
            const double qx = qr ? qr[x] : 1.0, px = p[x];
            const double ap = qx > 0.0 ? (px / qx < 1.0 ? px / qx : 1.0) : 0.0;
            s_dec = ur[cur] < ap ? 1 : 0;  // spec_decode.hpp:285
        }
        __syncthreads();
        cur += 1;
        if (s_dec) {
            if (threadIdx.x == 0) {
                acc_nodes[(long long)i * maxD + a] = j;
                acc_tok[(long long)i * maxD + a] = x;
            }
            ++a;
            __syncthreads();
            continue;
        }
        // residual (p - q)^+ normalized (:291-307), in place in p
        double s = 0.0;
        const int per = (V + kST - 1) / kST;
        const int a0 = threadIdx.x * per, b0 = min(V, a0 + per);
        for (int k = a0; k < b0; ++k) {
            const double diff = p[k] - (qr ? qr[k] : (k == x ? 1.0 : 0.0));
            const double v = diff > 0.0 ? diff : 0.0;
            p[k] = v;  // tentatively the residual
            s += v;
        }
        const double tot = block_sum_fixed(s, dsh);
        if (tot <= 0.0) {
            // p == q pointwise: the residual is p itself -> recompute p
            raw_row(vlogits + ((long long)i * (D + 1) + j) * V, V, p, fsh, dsh, nullptr, nullptr);
            temper_row(p, V, temperature, dsh, ish);
        } else {
            for (int k = threadIdx.x; k < V; k += blockDim.x) p[k] /= tot;
            __syncthreads();
        }
        const int t = inverse_cdf_block(p, V, ur[cur], dsh, ish);
        cur += 1;
        if (threadIdx.x == 0) bonus[i] = t;
        break;
    }
    if (threadIdx.x == 0) {
        acc_len[i] = a;
        consumed[i] = cur;
    }
}
void launch_accept_stochastic(const StepIn* step, int b, int D, int V, double temperature, const float* vlogits,
                              const double* q, const int* chain, const int* chain_n, const double* uni,
                              int uni_stride, double* pbuf, int* acc_nodes, int* acc_tok, int* acc_len, int* bonus,
                              int* consumed, int maxD, int chain_stride, int cur0, cudaStream_t st) {
    launch_pdl(k_accept_stochastic, b, kST, 0, st, step, b, D, V, temperature, vlogits, q, chain, chain_n, uni,
               uni_stride, pbuf, acc_nodes, acc_tok, acc_len, bonus, consumed, maxD, chain_stride, cur0);
}

}  // namespace tlt
