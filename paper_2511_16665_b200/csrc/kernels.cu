#include <algorithm>
// Engine kernels: weight init, gathers, RMSNorm, tree-masked attention,
// row top-k / argmax, drafter tree select (K6), greedy accept (K7), KV
// compaction + commit (K8), row-metadata builders. The GEMMs are in gemm.cu.
#include <cuda_bf16.h>
#include <cuda_fp8.h>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <math_constants.h>

#include "../../include/tlt_init.h"
#include "engine_kernels.h"
#include "kernels.cuh"
#include "pdl.cuh"

namespace tlt {

using bf16 = __nv_bfloat16;

// ------------------------------------------------------------------ init
__global__ void k_init_weights(uint16_t* dst, long long n, tlt_init_params p, int tensor, int layer) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        dst[i] = tlt_init_elem(&p, tensor, layer, i);
}
void launch_init(uint16_t* dst, long long n, const tlt_init_params& p, int tensor, int layer, cudaStream_t st) {
    k_init_weights<<<148 * 8, 256, 0, st>>>(dst, n, p, tensor, layer);
}

// ------------------------------------------------------------- gathers
__global__ void k_embed(const int* __restrict__ tok, const int* __restrict__ slot, const bf16* __restrict__ E, int d,
                        float* __restrict__ x) {
    pdl_wait();
    const int r = blockIdx.x;
    const bool live = slot[r] >= 0;
    const bf16* e = E + (long long)(live ? tok[r] : 0) * d;
    for (int i = threadIdx.x; i < d; i += blockDim.x) x[(long long)r * d + i] = live ? __bfloat162float(e[i]) : 0.f;
}
void launch_embed(const Rows& rows, int R, const bf16* E, int d, float* x, cudaStream_t st) {
    launch_pdl(k_embed, R, 256, 0, st, rows.tok, rows.slot, E, d, x);
}

// X2[r] = [prev feature || embed(tok)] (drafter fc input)
__global__ void k_draft_in(Rows rows, const bf16* __restrict__ E, int d, const bf16* __restrict__ hist,
                           const bf16* __restrict__ dfeat, bf16* __restrict__ X2) {
    pdl_wait();
    const int r = blockIdx.x;
    const bool live = rows.slot[r] >= 0;
    const int kind = live ? rows.fkind[r] : 0;
    const bf16* src = kind == 1 ? hist + rows.fidx[r] * d : (kind == 2 ? dfeat + rows.fidx[r] * d : nullptr);
    const bf16* e = E + (long long)(live ? rows.tok[r] : 0) * d;
    bf16* o = X2 + (long long)r * 2 * d;
    const bf16 z = __float2bfloat16(0.f);
    if ((d & 7) == 0) {  // 16-byte copies (rows are 16-byte aligned when d % 8 == 0)
        const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
        for (int i = threadIdx.x * 8; i < d; i += blockDim.x * 8) {
            *reinterpret_cast<uint4*>(o + i) = src ? *reinterpret_cast<const uint4*>(src + i) : z4;
            *reinterpret_cast<uint4*>(o + d + i) = live ? *reinterpret_cast<const uint4*>(e + i) : z4;
        }
        return;
    }
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        o[i] = src ? src[i] : z;
        o[d + i] = live ? e[i] : z;
    }
}
void launch_draft_in(const Rows& rows, int R, const bf16* E, int d, const bf16* hist, const bf16* dfeat, bf16* X2,
                     cudaStream_t st) {
    launch_pdl(k_draft_in, R, 256, 0, st, rows, E, d, hist, dfeat, X2);
}

// out[r] = x[src[r]] for gathering the level-1 root rows
__global__ void k_gather_rows(const float* __restrict__ x, const int* __restrict__ src, int d, float* __restrict__ out) {
    pdl_wait();
    const int r = blockIdx.x;
    const int s = src[r];
    for (int i = threadIdx.x; i < d; i += blockDim.x) out[(long long)r * d + i] = s >= 0 ? x[(long long)s * d + i] : 0.f;
}
void launch_gather_rows(const float* x, const int* src, int n, int d, float* out, cudaStream_t st) {
    launch_pdl(k_gather_rows, n, 256, 0, st, x, src, d, out);
}

__global__ void k_to_bf16(const float* __restrict__ x, long long n, bf16* __restrict__ out) {
    pdl_wait();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[i] = __float2bfloat16_rn(x[i]);
}
void launch_to_bf16(const float* x, long long n, bf16* out, cudaStream_t st) {
    int blocks = (int)((n + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    launch_pdl(k_to_bf16, blocks, 256, 0, st, x, n, out);
}

// ------------------------------------------------------------- RMSNorm
// out = bf16(x * (1/sqrt(mean(x^2) + eps)) * g), one CTA per row, fixed
// reduction tree (deterministic).
__global__ void k_rmsnorm(const float* __restrict__ x, int d, const bf16* __restrict__ g, float eps,
                          bf16* __restrict__ out) {
    pdl_wait();
    __shared__ float red[32];
    const int r = blockIdx.x;
    const float* xr = x + (long long)r * d;
    float ss = 0.f;
    for (int i = threadIdx.x; i < d; i += blockDim.x) ss += xr[i] * xr[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    const float inv = 1.0f / sqrtf(red[0] / (float)d + eps);
    for (int i = threadIdx.x; i < d; i += blockDim.x)
        out[(long long)r * d + i] = __float2bfloat16_rn(xr[i] * inv * __bfloat162float(g[i]));
}
// Vectorised variant (d % 4 == 0): the row is read ONCE with 16-byte loads
// into registers (VPT float4 per thread), reduced in a fixed order, and
// written as 8-byte groups of four bf16 — one HBM pass over x, no re-read.
template <int VPT>
__global__ void __launch_bounds__(256) k_rmsnorm_vec(const float* __restrict__ x, int d, const bf16* __restrict__ g,
                                                     float eps, bf16* __restrict__ out) {
    pdl_wait();
    __shared__ float red[8];
    const int r = blockIdx.x;
    const int d4 = d >> 2;
    const float4* xr = reinterpret_cast<const float4*>(x + (long long)r * d);
    float4 v[VPT];
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
        const int i = threadIdx.x + j * blockDim.x;
        v[j] = i < d4 ? __ldg(xr + i) : make_float4(0.f, 0.f, 0.f, 0.f);
        ss += v[j].x * v[j].x + v[j].y * v[j].y + v[j].z * v[j].z + v[j].w * v[j].w;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    float tot = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];  // fixed order
    const float inv = 1.0f / sqrtf(tot / (float)d + eps);
    uint2* orow = reinterpret_cast<uint2*>(out + (long long)r * d);
    const uint2* g4 = reinterpret_cast<const uint2*>(g);
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
        const int i = threadIdx.x + j * blockDim.x;
        if (i >= d4) break;
        const uint2 gw = __ldg(g4 + i);
        const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gw);
        const float2 ga = __bfloat1622float2(g2[0]), gb = __bfloat1622float2(g2[1]);
        uint2 o;
        __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
        o2[0] = __floats2bfloat162_rn(v[j].x * inv * ga.x, v[j].y * inv * ga.y);
        o2[1] = __floats2bfloat162_rn(v[j].z * inv * gb.x, v[j].w * inv * gb.y);
        orow[i] = o;
    }
}

void launch_rmsnorm(const float* x, int R, int d, const bf16* g, float eps, bf16* out, cudaStream_t st) {
    const int d4 = d / 4;
    if (d % 4 == 0 && d4 <= 8 * 256) {
        const int threads = d4 <= 8 * 128 ? 128 : 256;
        const int vpt = (d4 + threads - 1) / threads;
        switch (vpt) {
#define TLT_NORM_CASE(V) \
    case V: launch_pdl(k_rmsnorm_vec<V>, R, threads, 0, st, x, d, g, eps, out); return;
            TLT_NORM_CASE(1) TLT_NORM_CASE(2) TLT_NORM_CASE(3) TLT_NORM_CASE(4)
            TLT_NORM_CASE(5) TLT_NORM_CASE(6) TLT_NORM_CASE(7) TLT_NORM_CASE(8)
#undef TLT_NORM_CASE
            default: break;
        }
    }
    launch_pdl(k_rmsnorm, R, 256, 0, st, x, d, g, eps, out);
}

// Split-K reduce + residual add + RMSNorm of the updated row, one CTA per
// token row (the O-proj / down-proj epilogue at long-tail batch sizes):
//   x[r] += sum_z ws[z][r]   (fixed z order);  h[r] = bf16(x[r] * inv_rms * g)
// splits == 0: RMSNorm only (the residual add already happened in the GEMM
// epilogue), still spread over the cluster for the few-row long-tail case.
// One 8-CTA thread-block cluster per token row: each CTA owns d/8 features
// (so a single long-tail row still spreads over 8 SMs), the row's sum of
// squares is combined through distributed shared memory in fixed rank order.
constexpr int kNormCluster = 8;
__global__ void __cluster_dims__(kNormCluster, 1, 1) __launch_bounds__(256)
    k_reduce_resid_norm(const float* __restrict__ ws, long long plane, int splits, int d, float* __restrict__ x,
                        const bf16* __restrict__ g, float eps, bf16* __restrict__ out) {
    pdl_wait();
    __shared__ float red[32];
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int crank = (int)cluster.block_rank();
    const int r = blockIdx.y;
    const int per = (d + kNormCluster - 1) / kNormCluster;
    const int i0 = crank * per, i1 = min(d, i0 + per);
    float* xr = x + (long long)r * d;
    const float* wr = ws + (long long)r * d;
    float ss = 0.f;
    for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        float v = 0.f;
        for (int z = 0; z < splits; ++z) v += wr[z * plane + i];
        const float nx = xr[i] + v;
        if (splits) xr[i] = nx;
        ss += nx * nx;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
        float v = 0.f;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[w];
        red[16] = v;
    }
    cluster.sync();
    if (threadIdx.x == 0) {
        float tot = 0.f;
        for (int c = 0; c < kNormCluster; ++c) tot += *cluster.map_shared_rank(&red[16], c);  // fixed order
        red[17] = tot;
    }
    cluster.sync();  // remote reads done before any CTA of the cluster exits
    if (!g) return;
    const float inv = 1.0f / sqrtf(red[17] / (float)d + eps);
    for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x)
        out[(long long)r * d + i] = __float2bfloat16_rn(xr[i] * inv * __bfloat162float(g[i]));
}

// (single-CTA variant kept for reference / cross-checks)
__global__ void k_reduce_resid_norm_1cta(const float* __restrict__ ws, long long plane, int splits, int d,
                                         float* __restrict__ x, const bf16* __restrict__ g, float eps,
                                         bf16* __restrict__ out) {
    pdl_wait();
    __shared__ float red[32];
    const int r = blockIdx.x;
    float* xr = x + (long long)r * d;
    const float* wr = ws + (long long)r * d;
    float ss = 0.f;
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        float v = 0.f;
        for (int z = 0; z < splits; ++z) v += wr[z * plane + i];
        const float nx = xr[i] + v;
        xr[i] = nx;
        ss += nx * nx;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    if (!g) return;
    const float inv = 1.0f / sqrtf(red[0] / (float)d + eps);
    for (int i = threadIdx.x; i < d; i += blockDim.x)
        out[(long long)r * d + i] = __float2bfloat16_rn(xr[i] * inv * __bfloat162float(g[i]));
}
void launch_reduce_resid_norm(const float* ws, long long plane, int splits, int R, int d, float* x, const bf16* g,
                              float eps, bf16* out, cudaStream_t st) {
    launch_pdl(k_reduce_resid_norm, dim3(kNormCluster, R), dim3(256), 0, st, ws, plane, splits, d, x, g, eps, out);
}

// ----------------------------------------------------------- attention
// Tree-masked GQA attention over the per-slot KV cache, split along keys in
// fixed 512-key chunks aligned to absolute key indices (so a row's result
// does not depend on how many other rows share the launch). One CTA handles
// 16 query vectors (row x q-head of one KV head) against one key chunk; K/V
// tiles of 32 keys are staged in shared memory, the tree mask is read as
// 32-bit words per row. Partials (m, l, o) are merged by k_attn_combine.
constexpr int kAttnQV = 16;
constexpr int kAttnKeys = 32;

template <int HD>
__global__ void __launch_bounds__(128) k_attention(AttnParams p) {
    pdl_wait();
    constexpr int DPL = HD / 32;  // output dims per lane
    __shared__ float qs[kAttnQV][HD];
    __shared__ uint32_t ks[kAttnKeys][HD / 2 + 1];
    __shared__ __align__(16) bf16 vs[kAttnKeys][HD];
    __shared__ int s_row[kAttnQV], s_head[kAttnQV];

    const int G = p.H / p.KV;
    const int kvh = blockIdx.y;
    const int grp = blockIdx.z / p.max_splits;
    const int split = blockIdx.z % p.max_splits;
    const int qv0 = blockIdx.x * kAttnQV;
    const int nqv = p.rows_per_req * G;
    const int slot = p.g.slot[grp];
    const int lc = p.g.lc[grp], tail0 = p.g.tail0[grp], ntail = p.g.ntail[grp];
    const int total = slot >= 0 ? lc + ntail : 0;
    const int k0 = split * p.chunk;
    const int k1 = min(total, k0 + p.chunk);

    if (threadIdx.x < kAttnQV) {
        const int gqv = qv0 + threadIdx.x;
        int row = -1, head = 0;
        if (gqv < nqv) {
            row = grp * p.rows_per_req + gqv / G;
            head = kvh * G + gqv % G;
            if (p.rows.slot[row] < 0) row = -1;
        }
        s_row[threadIdx.x] = row;
        s_head[threadIdx.x] = head;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < kAttnQV * HD; idx += blockDim.x) {
        const int l = idx / HD, e = idx % HD;
        const int row = s_row[l];
        qs[l][e] = row >= 0 ? __bfloat162float(p.q[(long long)row * p.H * HD + s_head[l] * HD + e]) * p.scale_log2 : 0.f;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float m[4], l[4], acc[4][DPL];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        m[a] = -CUDART_INF_F;
        l[a] = 0.f;
#pragma unroll
        for (int e = 0; e < DPL; ++e) acc[a][e] = 0.f;
    }
    const long long slot_base = ((long long)(slot < 0 ? 0 : slot) * p.KV + kvh) * p.cap;
    for (int kb = k0; kb < k1; kb += kAttnKeys) {
        const int nk = min(kAttnKeys, k1 - kb);
        __syncthreads();
        // stage K (padded u32 pairs) and V for up to 32 keys: 16-byte chunks
        constexpr int CPK = HD * 2 / 16;  // 16B chunks per key row
        for (int c = threadIdx.x; c < kAttnKeys * CPK; c += blockDim.x) {
            const int j = c / CPK, w = c % CPK;
            uint4 kv = make_uint4(0, 0, 0, 0), vv = make_uint4(0, 0, 0, 0);
            if (j < nk) {
                const int v = kb + j;
                const long long ci = v < lc ? v : tail0 + (v - lc);
                const long long off = (slot_base + ci) * HD;
                kv = reinterpret_cast<const uint4*>(p.kc + off)[w];
                vv = reinterpret_cast<const uint4*>(p.vc + off)[w];
            }
            ks[j][w * 4 + 0] = kv.x;
            ks[j][w * 4 + 1] = kv.y;
            ks[j][w * 4 + 2] = kv.z;
            ks[j][w * 4 + 3] = kv.w;
            reinterpret_cast<uint4*>(&vs[j][0])[w] = vv;
        }
        __syncthreads();
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const int lq = warp * 4 + a;
            const int row = s_row[lq];
            if (row < 0) continue;  // warp-uniform
            float s = -CUDART_INF_F;
            const int v = kb + lane;
            if (lane < nk) {
                bool vis = v < lc;
                if (!vis) {
                    const int t = v - lc;
                    vis = (p.rows.mask[(long long)row * kMaskWords + (t >> 5)] >> (t & 31)) & 1u;
                }
                if (vis) {
                    float dot = 0.f;
#pragma unroll 8
                    for (int w = 0; w < HD / 2; ++w) {
                        const uint32_t kk = ks[lane][w];
                        const float k0f = __uint_as_float(kk << 16), k1f = __uint_as_float(kk & 0xffff0000u);
                        dot = fmaf(qs[lq][2 * w], k0f, dot);
                        dot = fmaf(qs[lq][2 * w + 1], k1f, dot);
                    }
                    s = dot;
                }
            }
            float mx = s;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            const float m_new = fmaxf(m[a], mx);
            if (m_new == -CUDART_INF_F) continue;
            const float pr = exp2f(s - m_new);
            float sum = pr;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            const float corr = exp2f(m[a] - m_new);
            l[a] = l[a] * corr + sum;
#pragma unroll
            for (int e = 0; e < DPL; ++e) acc[a][e] *= corr;
            for (int jj = 0; jj < nk; ++jj) {
                const float pj = __shfl_sync(0xffffffffu, pr, jj);
#pragma unroll
                for (int e = 0; e < DPL; ++e) acc[a][e] = fmaf(pj, __bfloat162float(vs[jj][lane * DPL + e]), acc[a][e]);
            }
            m[a] = m_new;
        }
    }
    // partials
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int lq = warp * 4 + a;
        const int gqv = qv0 + lq;
        if (gqv >= nqv) continue;
        const long long pidx = ((long long)(grp * p.max_splits + split) * p.qv_cap + gqv) * p.KV + kvh;
        if (lane == 0) {
            p.ws_m[pidx] = m[a];
            p.ws_l[pidx] = l[a];
        }
#pragma unroll
        for (int e = 0; e < DPL; ++e) p.ws_o[pidx * HD + lane * DPL + e] = acc[a][e];
    }
}

template <int HD>
__global__ void k_attn_combine(AttnParams p) {
    pdl_wait();
    // one warp per (group, query vector, kv head)
    const int G = p.H / p.KV;
    const int nqv = p.rows_per_req * G;
    const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const long long total = (long long)p.n_groups * nqv * p.KV;
    if (gw >= total) return;
    const int kvh = (int)(gw % p.KV);
    const int gqv = (int)((gw / p.KV) % nqv);
    const int grp = (int)(gw / ((long long)p.KV * nqv));
    const int row = grp * p.rows_per_req + gqv / G;
    const int head = kvh * G + gqv % G;
    const int slot = p.rows.slot[row], lc = p.g.lc[grp], nt = p.g.ntail[grp];  // loads in flight together
    if (slot < 0) return;
    const int nsplit = split_count(p, lc + nt);
    if (nsplit <= 1 && p.direct1) return;  // written by the attention kernel itself
    constexpr int DPL = HD / 32;
    constexpr int kB = 16;  // splits whose partials are loaded in one round trip
    float M = -CUDART_INF_F;
    float L = 0.f, o[DPL];
#pragma unroll
    for (int e = 0; e < DPL; ++e) o[e] = 0.f;
    const long long pbase = ((long long)grp * p.max_splits * p.qv_cap + gqv) * p.KV + kvh;
    const long long pstride = (long long)p.qv_cap * p.KV;
    if (nsplit <= kB) {
        // every partial (m, l, o) of the <= 16 splits loaded at once (one
        // dependent L2 round trip instead of two per split), then the same
        // arithmetic as the loop below: max over all splits, fixed-order sum
        float ms[kB], ls[kB], ov[kB][DPL];
#pragma unroll
        for (int s = 0; s < kB; ++s) {
            ms[s] = -CUDART_INF_F;
            ls[s] = 0.f;
#pragma unroll
            for (int e = 0; e < DPL; ++e) ov[s][e] = 0.f;
            if (s < nsplit) {
                const long long pidx = pbase + s * pstride;
                ms[s] = p.ws_m[pidx];
                ls[s] = p.ws_l[pidx];
#pragma unroll
                for (int e = 0; e < DPL; ++e) ov[s][e] = p.ws_o[pidx * HD + lane * DPL + e];
            }
        }
#pragma unroll
        for (int s = 0; s < kB; ++s) M = fmaxf(M, ms[s]);
#pragma unroll
        for (int s = 0; s < kB; ++s) {  // fixed order
            if (s >= nsplit || ms[s] == -CUDART_INF_F) continue;
            const float w = exp2f(ms[s] - M);
            L += ls[s] * w;
#pragma unroll
            for (int e = 0; e < DPL; ++e) o[e] += ov[s][e] * w;
        }
    } else {
        for (int s = 0; s < nsplit; ++s) M = fmaxf(M, p.ws_m[pbase + s * pstride]);
        for (int s = 0; s < nsplit; ++s) {  // fixed order
            const long long pidx = pbase + s * pstride;
            const float ms = p.ws_m[pidx];
            if (ms == -CUDART_INF_F) continue;
            const float w = exp2f(ms - M);
            L += p.ws_l[pidx] * w;
#pragma unroll
            for (int e = 0; e < DPL; ++e) o[e] += p.ws_o[pidx * HD + lane * DPL + e] * w;
        }
    }
    const float inv = L > 0.f ? 1.0f / L : 0.f;
#pragma unroll
    for (int e = 0; e < DPL; ++e)
        p.out[(long long)row * p.H * HD + head * HD + lane * DPL + e] = __float2bfloat16_rn(o[e] * inv);
}

void launch_attn_combine_only(const AttnParams& p, cudaStream_t st) {
    const int G = p.H / p.KV;
    const long long warps = (long long)p.n_groups * p.rows_per_req * G * p.KV;
    const int cblocks = (int)((warps * 32 + 255) / 256);
    if (p.hd == 128)
        launch_pdl(k_attn_combine<128>, cblocks, 256, 0, st, p);
    else
        launch_pdl(k_attn_combine<64>, cblocks, 256, 0, st, p);
}
void launch_attention_legacy(const AttnParams& p, cudaStream_t st) {
    launch_attention_mma(p, st, false);
    launch_attn_combine_only(p, st);
}

void launch_attention(const AttnParams& p, cudaStream_t st) {
    const int G = p.H / p.KV;
    const int nqv = p.rows_per_req * G;
    dim3 grid((nqv + kAttnQV - 1) / kAttnQV, p.KV, p.n_groups * p.max_splits);
    const long long warps = (long long)p.n_groups * nqv * p.KV;
    const int cblocks = (int)((warps * 32 + 255) / 256);
    if (p.impl == 1) {
        launch_attention_mma(p, st);  // tensor-core path (attn_mma.cu), chunk = 256 keys
        if (p.counters) return;       // split combine fused into the attention kernel
        if (p.dec && p.max_splits == 1) return;  // decode kernel wrote the output itself
    } else if (p.hd == 128) {
        launch_pdl(k_attention<128>, grid, 128, 0, st, p);
    } else {
        launch_pdl(k_attention<64>, grid, 128, 0, st, p);
    }
    if (p.hd == 128)
        launch_pdl(k_attn_combine<128>, cblocks, 256, 0, st, p);
    else
        launch_pdl(k_attn_combine<64>, cblocks, 256, 0, st, p);
}

// ------------------------------------------------------- row top-k / argmax
// Top-k by (logit desc, id asc) — the reference child order (stable_sort over
// ascending id, spec_decode.hpp:121-125) — plus the row max M and
// S = sum_i exp(l_i - M). Everything stays in registers: per-thread sorted
// K-lists with static-index insertion, then K rounds of warp arg-max
// (shuffle butterfly over a strict total order, so every lane agrees) and one
// more warp merge over the per-warp lists. (m, s) pairs are combined with
// max-rescaling in a fixed order: deterministic.
template <int K>
struct TopK {
    float v[K];
    int id[K];
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int i = 0; i < K; ++i) {
            v[i] = -CUDART_INF_F;
            id[i] = 0x7fffffff;
        }
    }
    __device__ __forceinline__ static bool better(float a, int ia, float b, int ib) {
        return a > b || (a == b && ia < ib);
    }
    __device__ __forceinline__ void push(float x, int ix) {
        if (!better(x, ix, v[K - 1], id[K - 1])) return;
        bool placed = false;
#pragma unroll
        for (int s = K - 1; s > 0; --s) {
            const bool shift = !placed && better(x, ix, v[s - 1], id[s - 1]);
            const bool put = !placed && !shift;
            const float nv = shift ? v[s - 1] : (put ? x : v[s]);
            const int ni = shift ? id[s - 1] : (put ? ix : id[s]);
            v[s] = nv;
            id[s] = ni;
            placed = placed || put;
        }
        if (!placed) {
            v[0] = x;
            id[0] = ix;
        }
    }
    // After the call every lane holds the warp's top-K (sorted).
    __device__ __forceinline__ void warp_merge() {
        float ov[K];
        int oi[K];
#pragma unroll
        for (int r = 0; r < K; ++r) {
            float bv = v[0];
            int bi = id[0];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float xv = __shfl_xor_sync(0xffffffffu, bv, o);
                const int xi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (better(xv, xi, bv, bi)) {
                    bv = xv;
                    bi = xi;
                }
            }
            ov[r] = bv;
            oi[r] = bi;
            if (id[0] == bi && v[0] == bv) {  // this lane's head won: pop it
#pragma unroll
                for (int s = 0; s < K - 1; ++s) {
                    v[s] = v[s + 1];
                    id[s] = id[s + 1];
                }
                v[K - 1] = -CUDART_INF_F;
                id[K - 1] = 0x7fffffff;
            }
        }
#pragma unroll
        for (int r = 0; r < K; ++r) {
            v[r] = ov[r];
            id[r] = oi[r];
        }
    }
};

// online (max, sum-exp) pair
__device__ __forceinline__ void ms_add(float& m, float& s, float x) {
    if (x > m) {
        s = (m == -CUDART_INF_F ? 0.f : s * __expf(m - x)) + 1.f;
        m = x;
    } else if (x != -CUDART_INF_F) {
        s += __expf(x - m);
    }
}
__device__ __forceinline__ void ms_merge(float& m, float& s, float om, float os) {
    const float nm = fmaxf(m, om);
    const float a = m == -CUDART_INF_F ? 0.f : s * __expf(m - nm);
    const float b = om == -CUDART_INF_F ? 0.f : os * __expf(om - nm);
    m = nm;
    s = a + b;
}

// Block-level finish (256 threads = 8 warps): warp merges, then warp 0 merges
// the 8 per-warp lists. Result (top-K, M, S) valid in warp 0 afterwards.
template <int K>
__device__ __forceinline__ void block_topk_finish(TopK<K>& t, float& m, float& s, float* sv, int* si, float* sm,
                                                  float* ss) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float om = __shfl_xor_sync(0xffffffffu, m, o);
        const float os = __shfl_xor_sync(0xffffffffu, s, o);
        ms_merge(m, s, om, os);
    }
    t.warp_merge();
    if (lane == 0) {
        sm[warp] = m;
        ss[warp] = s;
#pragma unroll
        for (int r = 0; r < K; ++r) {
            sv[warp * K + r] = t.v[r];
            si[warp * K + r] = t.id[r];
        }
    }
    __syncthreads();
    if (warp == 0) {
        t.init();
        for (int e = lane; e < 8 * K; e += 32) t.push(sv[e], si[e]);
        t.warp_merge();
        m = sm[0];
        s = ss[0];
        for (int w = 1; w < 8; ++w) ms_merge(m, s, sm[w], ss[w]);  // fixed warp order
    }
}

// Stage 1 of the multi-CTA row top-k (k > 1) over materialized logits: CTA
// (chunk c, row r) reduces an 8192-entry chunk to the same partial record the
// EPI_TOPK epilogue writes (chunk max m, sum exp(l - m), sorted top-k), so
// k_topk_merge finishes both. Chunk order is fixed -> deterministic.
// Stage 1 of the multi-CTA row top-k (k > 1) over materialised logits: CTA
// (chunk c, row r) reduces an 8192-entry chunk (held in registers, 32 per
// thread, all loads in flight at once) to the partial record the EPI_TOPK
// epilogue writes (chunk max m, sum exp(l - m), sorted top-k), so
// k_topk_merge finishes both. Selection: the K-th largest of the 256
// per-thread maxima is a lower bound of the chunk's K-th value (K distinct
// entries reach it), entries at or above it are appended to a small smem
// candidate list (typically ~K of 8192) and only those are ranked. Ties are
// ranked by id, so the result is deterministic whatever the append order.
constexpr int kTopkChunk = 8192;
constexpr int kTopkPer = kTopkChunk / 256;
constexpr int kTopkCap = 512;
template <int K>
__global__ void __launch_bounds__(256, 3) k_row_topk_chunk(const float* __restrict__ logits, int V, const int* live,
                                                        int k, float* __restrict__ part, int R) {
    pdl_wait();
    __shared__ float sv[8 * K];
    __shared__ int si[8 * K];
    __shared__ float sm[8], ss[8];
    __shared__ float s_thr, s_max;
    __shared__ float cv[kTopkCap];
    __shared__ int ci[kTopkCap];
    __shared__ int s_cnt;
    const int c = blockIdx.x, r = blockIdx.y;
    if (live && live[r] < 0) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float* lr = logits + (long long)r * V;
    const int i0 = c * kTopkChunk, i1 = min(V, i0 + kTopkChunk);
    float x[kTopkPer];
    float mx = -CUDART_INF_F;
#pragma unroll
    for (int u = 0; u < kTopkPer; ++u) {
        const int i = i0 + u * 256 + threadIdx.x;
        x[u] = i < i1 ? __ldcs(lr + i) : -CUDART_INF_F;
        mx = fmaxf(mx, x[u]);
    }
    if (threadIdx.x == 0) s_cnt = 0;
    {  // per warp: bitonic sort (descending) of the 32 lane maxima
        float v = mx;
#pragma unroll
        for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                const float o = __shfl_xor_sync(0xffffffffu, v, stride);
                const bool desc = (lane & size) == 0 || size == 32;
                const bool lower = (lane & stride) == 0;
                v = (lower == desc) ? fmaxf(v, o) : fminf(v, o);
            }
        }
        // the warp's K-th largest lane maximum bounds the chunk's K-th value
        const float kth = __shfl_sync(0xffffffffu, v, K - 1);
        const float wmax = __shfl_sync(0xffffffffu, v, 0);
        if (lane == 0) {
            sm[warp] = kth;
            ss[warp] = wmax;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            float t0 = sm[0], m0 = ss[0];
            for (int w = 1; w < 8; ++w) {
                t0 = fmaxf(t0, sm[w]);
                m0 = fmaxf(m0, ss[w]);
            }
            s_thr = t0;
            s_max = m0;
        }
        __syncthreads();
    }
    const float thr = s_thr, M = s_max;
    float s = 0.f;
    if (M != -CUDART_INF_F) {
#pragma unroll
        for (int u = 0; u < kTopkPer; ++u) s += __expf(x[u] - M);  // exp(-inf) = 0
    }
#pragma unroll
    for (int u = 0; u < kTopkPer; ++u) {
        if (x[u] >= thr) {
            const int p = atomicAdd(&s_cnt, 1);
            if (p < kTopkCap) {
                cv[p] = x[u];
                ci[p] = i0 + u * 256 + threadIdx.x;
            }
        }
    }
    // s: fixed-order block sum
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    __syncthreads();  // candidates complete; sm/ss reused
    if (lane == 0) ss[warp] = s;
    const int cnt = s_cnt;
    TopK<K> t;
    t.init();
    float m = M;
    if (cnt <= kTopkCap) {
        __syncthreads();
        if (warp != 0) return;
        for (int e = lane; e < cnt; e += 32) t.push(cv[e], ci[e]);
        t.warp_merge();
        s = ss[0];
        for (int w = 1; w < 8; ++w) s += ss[w];
    } else {  // pathological ties at the threshold: rank every thread's entries
#pragma unroll
        for (int u = 0; u < kTopkPer; ++u)
            if (x[u] >= thr) t.push(x[u], i0 + u * 256 + threadIdx.x);
        __syncthreads();
        float tot = ss[0];
        for (int w = 1; w < 8; ++w) tot += ss[w];
        __syncthreads();  // ss is scratch of block_topk_finish below
        float mm = M, s0 = 0.f;
        block_topk_finish<K>(t, mm, s0, sv, si, sm, ss);  // (m, s) of this call unused
        s = tot;
        if (warp != 0) return;
    }
    const int W = 2 + 2 * k;
    float* out = part + ((long long)c * R + r) * W;
    if (threadIdx.x == 0) {
        out[0] = m;
        out[1] = s;
    }
    if (threadIdx.x < 32) {
#pragma unroll
        for (int j = 0; j < K; ++j)
            if (threadIdx.x == j && j < k) {
                out[2 + j] = t.v[j];
                out[2 + k + j] = __int_as_float(t.id[j]);
            }
    }
}
int launch_row_topk_chunked(const float* logits, int R, int V, const int* live, int k, float* part, cudaStream_t st) {
    const int nch = (V + kTopkChunk - 1) / kTopkChunk;
    const dim3 grid(nch, R);
    if (k <= 2)
        launch_pdl(k_row_topk_chunk<2>, grid, dim3(256), 0, st, logits, V, live, k, part, R);
    else if (k <= 4)
        launch_pdl(k_row_topk_chunk<4>, grid, dim3(256), 0, st, logits, V, live, k, part, R);
    else
        launch_pdl(k_row_topk_chunk<8>, grid, dim3(256), 0, st, logits, V, live, k, part, R);
    return nch;
}

// Merge of the partial records (LM-head EPI_TOPK tiles or top-k chunks) of
// each row, one CTA per row: M and S by max-rescaled combination in a fixed
// order, top-k of the per-tile sorted candidate lists by (logit desc, id asc).
template <int K>
__global__ void __launch_bounds__(256) k_topk_merge(const float* __restrict__ part, int n_tiles, int m_tok, int k,
                                                    const int* __restrict__ live, int* __restrict__ out_tok,
                                                    float* __restrict__ out_logit, float* __restrict__ out_M,
                                                    float* __restrict__ out_S, unsigned* __restrict__ thr_reset) {
    pdl_wait();
    __shared__ float sv[8 * K];
    __shared__ int si[8 * K];
    __shared__ float sm[8], ss[8];
    const int r = blockIdx.x;
    // the LM head's per-row k-th-value bound (EpiParams::topk_thr) is spent:
    // clear it for the next launch, dead rows included
    if (thr_reset && threadIdx.x == 0) thr_reset[r] = 0u;
    if (live && live[r] < 0) return;
    const int W = 2 + 2 * k;
    float m = -CUDART_INF_F, s = 0.f;
    TopK<K> t;
    t.init();
    if (K == 1) {
        for (int i = threadIdx.x; i < n_tiles; i += blockDim.x) {
            const float* pp = part + ((long long)i * m_tok + r) * W;
            ms_merge(m, s, pp[0], pp[1]);
            t.push(pp[2], __float_as_int(pp[2 + k]));
        }
        block_topk_finish<K>(t, m, s, sv, si, sm, ss);
    } else {
        // K > 1: the K-th largest per-lane best (within a warp) bounds the
        // row's K-th value; only list entries at or above it are ranked
        __shared__ float cv[kTopkCap];
        __shared__ int ci[kTopkCap];
        __shared__ int s_cnt;
        __shared__ float s_thr;
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        float best = -CUDART_INF_F;
        for (int i = threadIdx.x; i < n_tiles; i += blockDim.x) {
            const float* pp = part + ((long long)i * m_tok + r) * W;
            ms_merge(m, s, pp[0], pp[1]);
            best = fmaxf(best, pp[2]);
        }
        if (threadIdx.x == 0) s_cnt = 0;
        float v = best;
#pragma unroll
        for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                const float o = __shfl_xor_sync(0xffffffffu, v, stride);
                const bool desc = (lane & size) == 0 || size == 32;
                const bool lower = (lane & stride) == 0;
                v = (lower == desc) ? fmaxf(v, o) : fminf(v, o);
            }
        }
        const float kth = __shfl_sync(0xffffffffu, v, K - 1);
        if (lane == 0) sv[warp] = kth;
        __syncthreads();
        if (threadIdx.x == 0) {
            float tt = sv[0];
            for (int w = 1; w < 8; ++w) tt = fmaxf(tt, sv[w]);
            s_thr = tt;
        }
        __syncthreads();
        const float thr = s_thr;
        for (int i = threadIdx.x; i < n_tiles; i += blockDim.x) {
            const float* pp = part + ((long long)i * m_tok + r) * W;
            if (pp[2] < thr) continue;
            for (int c = 0; c < k; ++c) {
                const float x = pp[2 + c];
                if (x < thr) break;  // tile lists are sorted
                const int p = atomicAdd(&s_cnt, 1);
                if (p < kTopkCap) {
                    cv[p] = x;
                    ci[p] = __float_as_int(pp[2 + k + c]);
                }
            }
        }
        __syncthreads();
        const int cnt = s_cnt;
        if (cnt <= kTopkCap) {
            for (int e = threadIdx.x; e < cnt; e += blockDim.x) t.push(cv[e], ci[e]);
        } else {  // pathological ties: rank every entry at or above the bound
            for (int i = threadIdx.x; i < n_tiles; i += blockDim.x) {
                const float* pp = part + ((long long)i * m_tok + r) * W;
                for (int c = 0; c < k; ++c)
                    if (pp[2 + c] >= thr) t.push(pp[2 + c], __float_as_int(pp[2 + k + c]));
            }
        }
        __syncthreads();
        block_topk_finish<K>(t, m, s, sv, si, sm, ss);
    }
    if (threadIdx.x < 32) {
#pragma unroll
        for (int j = 0; j < K; ++j)
            if (threadIdx.x == j && j < k) {
                out_tok[(long long)r * k + j] = t.id[j];
                out_logit[(long long)r * k + j] = t.v[j];
            }
    }
    if (threadIdx.x == 0) {
        if (out_M) out_M[r] = m;
        if (out_S) out_S[r] = s;
    }
}
void launch_topk_merge(const float* part, int n_tiles, int R, int k, const int* live, int* out_tok, float* out_logit,
                       float* out_M, float* out_S, cudaStream_t st, unsigned* thr_reset) {
    if (k <= 1)
        launch_pdl(k_topk_merge<1>, R, 256, 0, st, part, n_tiles, R, k, live, out_tok, out_logit, out_M, out_S,
                   thr_reset);
    else if (k <= 2)
        launch_pdl(k_topk_merge<2>, R, 256, 0, st, part, n_tiles, R, k, live, out_tok, out_logit, out_M, out_S,
                   thr_reset);
    else if (k <= 4)
        launch_pdl(k_topk_merge<4>, R, 256, 0, st, part, n_tiles, R, k, live, out_tok, out_logit, out_M, out_S,
                   thr_reset);
    else
        launch_pdl(k_topk_merge<8>, R, 256, 0, st, part, n_tiles, R, k, live, out_tok, out_logit, out_M, out_S,
                   thr_reset);
}

// full fp64 distribution of a row (parity/debug export): p = exp((double)(l-M))/S
__global__ void k_row_probs(const float* __restrict__ logits, int V, const float* __restrict__ M,
                            const float* __restrict__ S, double* __restrict__ out) {
    pdl_wait();
    const int r = blockIdx.x;
    const float m = M[r];
    const double s = (double)S[r];
    for (int i = threadIdx.x; i < V; i += blockDim.x)
        out[(long long)r * V + i] = exp((double)(logits[(long long)r * V + i] - m)) / s;
}
void launch_row_probs(const float* logits, int R, int V, const float* M, const float* S, double* out, cudaStream_t st) {
    launch_pdl(k_row_probs, R, 256, 0, st, logits, V, M, S, out);
}

// ------------------------------------------------------------ row builders
// Drafter level 1: pending committed positions [ld, lt) (target features
// known) + the root at lt, causal among themselves. Stride D1 per request.
__global__ void k_rows_level1(const StepIn* __restrict__ st, int b, int b_hi, int D1, Rows rows, Groups g,
                              int* __restrict__ root_row, const int* __restrict__ tok_hist, int cap,
                              int drafter_cap) {
    pdl_wait();
    const int i = blockIdx.x;
    const int j = threadIdx.x;
    if (j >= D1) return;
    const int r = i * D1 + j;
    const bool live = i < b && st[i].slot >= 0;
    const int pend = live ? st[i].lt - st[i].ld + 1 : 0;
    uint32_t* mk = rows.mask + (long long)r * kMaskWords;
    for (int w = 0; w < kMaskWords; ++w) mk[w] = 0u;
    if (live && j < pend) {
        const int slot = st[i].slot, pos = st[i].ld + j;
        rows.tok[r] = tok_hist[(long long)slot * cap + pos];
        rows.pos[r] = pos;
        rows.slot[r] = slot;
        rows.cidx[r] = pos;
        rows.fkind[r] = pos > 0 ? 1 : 0;
        rows.fidx[r] = (long long)slot * cap + pos - 1;
        for (int t = 0; t <= j; ++t) mk[t >> 5] |= 1u << (t & 31);
    } else {
        rows.tok[r] = 0;
        rows.pos[r] = 0;
        rows.slot[r] = -1;
        rows.cidx[r] = 0;
        rows.fkind[r] = 0;
        rows.fidx[r] = 0;
    }
    if (j == 0) {
        g.slot[i] = live ? st[i].slot : -1;
        g.lc[i] = live ? st[i].ld : 0;
        g.tail0[i] = live ? st[i].ld : 0;
        g.ntail[i] = pend;
        root_row[i] = live ? i * D1 + pend - 1 : -1;
    }
    (void)b_hi;
    (void)drafter_cap;
}
void launch_rows_level1(const StepIn* st, int b, int b_hi, int D1, const Rows& rows, const Groups& g, int* root_row,
                        const int* tok_hist, int cap, cudaStream_t s) {
    launch_pdl(k_rows_level1, b_hi, 32 * ((D1 + 31) / 32), 0, s, st, b, b_hi, D1, rows, g, root_row, tok_hist, cap, 0);
}

// AR decode: one row per request (the root), visible prefix [0, lt) + self.
__global__ void k_rows_ar(const StepIn* __restrict__ st, int b, int b_hi, Rows rows, Groups g,
                          const int* __restrict__ tok_hist, int cap) {
    pdl_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= b_hi) return;
    const bool live = i < b && st[i].slot >= 0;
    uint32_t* mk = rows.mask + (long long)i * kMaskWords;
    for (int w = 0; w < kMaskWords; ++w) mk[w] = 0u;
    mk[0] = 1u;
    const int slot = live ? st[i].slot : -1, lt = live ? st[i].lt : 0;
    rows.tok[i] = live ? tok_hist[(long long)slot * cap + lt] : 0;
    rows.pos[i] = lt;
    rows.slot[i] = slot;
    rows.cidx[i] = lt;
    rows.fkind[i] = 0;
    rows.fidx[i] = 0;
    g.slot[i] = slot;
    g.lc[i] = lt;
    g.tail0[i] = lt;
    g.ntail[i] = live ? 1 : 0;
}
void launch_rows_ar(const StepIn* st, int b, int b_hi, const Rows& rows, const Groups& g, const int* tok_hist, int cap,
                    cudaStream_t s) {
    launch_pdl(k_rows_ar, (b_hi + 127) / 128, 128, 0, s, st, b, b_hi, rows, g, tok_hist, cap);
}

// ------------------------------------------------------------ tree (K6)
__device__ __forceinline__ bool rank_before(const Cand& a, const Cand& b) {  // spec_decode.hpp:96-101
    if (a.pp != b.pp) return a.pp > b.pp;
    if (a.depth != b.depth) return a.depth < b.depth;
    if (a.token != b.token) return a.token < b.token;
    return a.birth < b.birth;
}

constexpr int kTreeThreads = 256;
constexpr int kSortCap = 2048;

// bitonic sort of idx[0..n) (n <= kSortCap, padded with -1) by rank_before over cand[]
__device__ void bitonic_rank_sort(int* idx, int n_pad, const Cand* cand) {
    for (int size = 2; size <= n_pad; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < n_pad / 2; t += blockDim.x) {
                const int lo = 2 * t - (t & (stride - 1));
                const int hi = lo + stride;
                const bool up = ((lo & size) == 0);
                const int a = idx[lo], b = idx[hi];
                // -1 (padding) ranks last
                bool a_first;
                if (a < 0) a_first = false;
                else if (b < 0) a_first = true;
                else a_first = rank_before(cand[a], cand[b]);
                const bool swap = up ? !a_first : a_first;
                if (swap && !(a < 0 && b < 0)) {
                    idx[lo] = b;
                    idx[hi] = a;
                }
            }
            __syncthreads();
        }
    }
}

// One drafter level of build_draft_tree (spec_decode.hpp:118-169) for one
// request per CTA: append the children of this level's expanded rows (top-k
// in child-rank order, p > 0, births in expansion order), sort them by
// rank_before, merge into the running global top-T (the final selection of
// :171-179, computed incrementally — exact under the strict total order),
// and emit the cut frontier (:154-160) as the next level's drafter rows.
__global__ void __launch_bounds__(kTreeThreads) k_tree_level(TreeParams p) {
    pdl_wait();
    extern __shared__ __align__(16) unsigned char tree_smem[];
    Cand* sc = reinterpret_cast<Cand*>(tree_smem);                       // kept (first n_kept) + new children
    int* sidx = reinterpret_cast<int*>(tree_smem + sizeof(Cand) * kSortCap);
    __shared__ int s_cnt[kTreeThreads + 1];
    __shared__ int s_n_new, s_n_kept;
    const int i = blockIdx.x;
    const bool live = i < p.b && p.step[i].slot >= 0;
    const int lt = live ? p.step[i].lt : 0;
    const int slot = live ? p.step[i].slot : -1;
    Cand* arena = p.arena + (long long)i * p.arena_cap;
    int* kept = p.kept + (long long)i * p.T;

    if (p.level == 1 && threadIdx.x == 0) {
        p.arena_n[i] = 0;
        p.kept_n[i] = 0;
        p.exp_n[i] = 0;
        p.done[i] = live ? 0 : 1;
    }
    __syncthreads();
    const bool active = live && !p.done[i];
    // ---- collect children of this level's rows (row j of this request)
    const int F = p.lm_F;
    int my_valid = 0;
    const int j = threadIdx.x;
    int node = -1;
    int lm_row = i * F + j;
    bool row_live = false;
    if (active && j < F) {
        if (p.level == 1) {
            row_live = true;
            node = -1;
        } else {
            const int grow = p.lvl_base + lm_row;
            row_live = p.rows.slot[grow] >= 0;
            node = row_live ? p.row_node[grow] : -1;
        }
        if (row_live) {
            for (int c = 0; c < p.k; ++c) {
                const float lg = p.tk_logit[(long long)lm_row * p.k + c];
                const double pr = exp((double)(lg - p.tk_M[lm_row])) / (double)p.tk_S[lm_row];
                if (!(pr > 0.0)) break;
                ++my_valid;
            }
        }
    }
    if (j < kTreeThreads) s_cnt[j] = my_valid;
    __syncthreads();
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int t = 0; t < kTreeThreads; ++t) {
            const int v = s_cnt[t];
            s_cnt[t] = acc;
            acc += v;
        }
        s_cnt[kTreeThreads] = acc;
        s_n_new = acc;
        s_n_kept = active ? p.kept_n[i] : 0;
    }
    __syncthreads();
    const int n_new = s_n_new, n_kept = s_n_kept;
    const int count0 = active ? p.arena_n[i] : 0;
    if (active && my_valid > 0) {
        const double ppar = node < 0 ? 1.0 : arena[node].pp;
        for (int c = 0; c < my_valid; ++c) {
            const float lg = p.tk_logit[(long long)lm_row * p.k + c];
            const double pr = exp((double)(lg - p.tk_M[lm_row])) / (double)p.tk_S[lm_row];
            Cand cd;
            cd.pp = ppar * pr;  // spec_decode.hpp:132
            cd.prob = pr;
            cd.token = p.tk_tok[(long long)lm_row * p.k + c];
            cd.parent = node;
            cd.depth = p.level;
            cd.birth = count0 + s_cnt[j] + c;
            cd.row = -1;
            cd.eslot = -1;
            arena[cd.birth] = cd;
        }
    }
    __syncthreads();
    // ---- sort the new children (indices into sc: kept at [0,n_kept), new at [n_kept, n_kept+n_new))
    for (int t = threadIdx.x; t < n_kept; t += blockDim.x) sc[t] = arena[kept[t]];
    for (int t = threadIdx.x; t < n_new; t += blockDim.x) sc[n_kept + t] = arena[count0 + t];
    int n_pad = 1;
    while (n_pad < n_new && n_pad < (1 << 20)) n_pad <<= 1;
    for (int t = threadIdx.x; t < n_pad; t += blockDim.x) sidx[t] = t < n_new ? n_kept + t : -1;
    __syncthreads();
    if (n_new > 1) bitonic_rank_sort(sidx, n_pad, sc);
    // frontier = first min(T, n_new) new children in rank order (:154-160)
    const int n_front = (p.level < p.D) ? min(p.T, n_new) : 0;
    if (active && p.level < p.D) {
        const int e0 = p.exp_n[i];
        for (int f = threadIdx.x; f < p.nxt_F; f += blockDim.x) {
            const int r = p.nxt_base + i * p.nxt_F + f;
            uint32_t* mk = p.rows.mask + (long long)r * kMaskWords;
            if (f < n_front) {
                const int a = sidx[f] - n_kept;  // index among the new children
                const int an = count0 + a;       // arena index
                const Cand& cd = sc[n_kept + a];
                const int e = e0 + f;
                const int prow = cd.parent < 0 ? p.root_row[i] : arena[cd.parent].row;
                p.rows.tok[r] = cd.token;
                p.rows.pos[r] = lt + cd.depth;
                p.rows.slot[r] = slot;
                p.rows.cidx[r] = lt + 1 + e;
                p.rows.fkind[r] = 2;
                p.rows.fidx[r] = prow;
                const uint32_t* pm = cd.parent < 0 ? nullptr : p.rows.mask + (long long)prow * kMaskWords;
                for (int w = 0; w < kMaskWords; ++w) mk[w] = pm ? pm[w] : 0u;
                mk[e >> 5] |= 1u << (e & 31);
                p.row_node[r] = an;
                arena[an].row = r;
                arena[an].eslot = e;
            } else {
                p.rows.slot[r] = -1;
                p.rows.tok[r] = 0;
                p.rows.pos[r] = 0;
                p.rows.cidx[r] = 0;
                p.rows.fkind[r] = 0;
                p.row_node[r] = -1;
                for (int w = 0; w < kMaskWords; ++w) mk[w] = 0u;
            }
        }
        if (threadIdx.x == 0) {
            p.g_next.slot[i] = n_front > 0 ? slot : -1;
            p.g_next.lc[i] = lt + 1;
            p.g_next.tail0[i] = lt + 1;
            p.g_next.ntail[i] = e0 + n_front;
        }
    } else if (!active && p.level < p.D) {
        for (int f = threadIdx.x; f < p.nxt_F; f += blockDim.x) {
            const int r = p.nxt_base + i * p.nxt_F + f;
            p.rows.slot[r] = -1;
            p.rows.tok[r] = 0;
            p.rows.pos[r] = 0;
            p.rows.cidx[r] = 0;
            p.rows.fkind[r] = 0;
            p.row_node[r] = -1;
        }
        if (threadIdx.x == 0) {
            p.g_next.slot[i] = -1;
            p.g_next.ntail[i] = 0;
        }
    }
    __syncthreads();
    // ---- merge: top-T of (kept U new) under rank_before
    if (active) {
        const int n_all = n_kept + n_new;
        int m_pad = 1;
        while (m_pad < n_all && m_pad < (1 << 20)) m_pad <<= 1;
        // reuse sidx: kept then new (unsorted is fine: full sort)
        __syncthreads();
        for (int t = threadIdx.x; t < m_pad; t += blockDim.x) sidx[t] = t < n_all ? t : -1;
        __syncthreads();
        if (n_all > 1) bitonic_rank_sort(sidx, m_pad, sc);
        const int nk = min(p.T, n_all);
        for (int t = threadIdx.x; t < nk; t += blockDim.x) {
            const int s = sidx[t];
            kept[t] = sc[s].birth;  // birth == arena index
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            p.kept_n[i] = nk;
            p.arena_n[i] = count0 + n_new;
            p.exp_n[i] += n_front;
            if (n_new == 0 || p.level >= p.D) p.done[i] = 1;  // :167 `if (next.empty()) break;`
        }
    }
}

// Final tree (spec_decode.hpp:171-196): kept list in rank order with parents
// remapped, plus the verify rows: root at lt, node n at cache lt+1+n with
// position lt+depth, visibility = root + ancestors + self.
__global__ void k_tree_final(TreeParams p) {
    pdl_wait();
    const int i = blockIdx.x;
    const bool live = i < p.b && p.step[i].slot >= 0;
    const int T = p.T, T1 = p.T + 1;
    const int n = live ? p.kept_n[i] : 0;
    const Cand* arena = p.arena + (long long)i * p.arena_cap;
    const int* kept = p.kept + (long long)i * T;
    const int lt = live ? p.step[i].lt : 0, slot = live ? p.step[i].slot : -1;
    __shared__ int s_par[kMaxT];
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        const Cand& c = arena[kept[t]];
        int par = -1;
        if (c.parent >= 0)
            for (int u = 0; u < t; ++u)
                if (kept[u] == c.parent) par = u;
        s_par[t] = par;
        p.tree_tok[(long long)i * T + t] = c.token;
        p.tree_par[(long long)i * T + t] = par;
        p.tree_dep[(long long)i * T + t] = c.depth;
        p.tree_prob[(long long)i * T + t] = c.prob;
        p.tree_pp[(long long)i * T + t] = c.pp;
    }
    __syncthreads();
    if (threadIdx.x == 0) p.tree_n[i] = n;
    // verify rows
    for (int t = threadIdx.x; t < T1; t += blockDim.x) {
        const int r = i * T1 + t;
        uint32_t* mk = p.vrows.mask + (long long)r * kMaskWords;
        for (int w = 0; w < kMaskWords; ++w) mk[w] = 0u;
        if (live && t <= n) {
            mk[0] = 1u;  // root
            if (t == 0) {
                p.vrows.tok[r] = p.tok_hist[(long long)slot * p.cap + lt];
                p.vrows.pos[r] = lt;
            } else {
                const int nd = t - 1;
                p.vrows.tok[r] = p.tree_tok[(long long)i * T + nd];
                p.vrows.pos[r] = lt + p.tree_dep[(long long)i * T + nd];
                // bounded walk (a tree path has <= D nodes): malformed input cannot spin
                for (int a = nd, g = 0; a >= 0 && a < T && g <= kMaxDepth; a = s_par[a], ++g)
                    mk[(a + 1) >> 5] |= 1u << ((a + 1) & 31);
            }
            p.vrows.slot[r] = slot;
            p.vrows.cidx[r] = lt + t;
        } else {
            p.vrows.slot[r] = -1;
            p.vrows.tok[r] = 0;
            p.vrows.pos[r] = 0;
            p.vrows.cidx[r] = 0;
        }
        p.vrows.fkind[r] = 0;
        p.vrows.fidx[r] = 0;
    }
    if (threadIdx.x == 0) {
        p.vg.slot[i] = live ? slot : -1;
        p.vg.lc[i] = lt;
        p.vg.tail0[i] = lt;
        p.vg.ntail[i] = live ? n + 1 : 0;
    }
}

void launch_tree_level(const TreeParams& p, cudaStream_t st) {
    static bool attr = false;
    const int smem = (int)(sizeof(Cand) * kSortCap + sizeof(int) * kSortCap);
    if (!attr) {
        cudaFuncSetAttribute(k_tree_level, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    launch_pdl(k_tree_level, p.b_hi, kTreeThreads, smem, st, p);
}
void launch_tree_final(const TreeParams& p, cudaStream_t st) { launch_pdl(k_tree_final, p.b_hi, 128, 0, st, p); }

// ---------------------------------------------------------- accept (K7)
// verify_greedy (spec_decode.hpp:245-268): from the root, accept the child
// whose token equals the target argmax at the current node (lowest index; a
// node's children carry distinct tokens), else emit that argmax as the bonus.
// One warp per request; children are found with a ballot over the tree.
__global__ void k_accept_greedy(AcceptParams p) {
    pdl_wait();
    const int i = blockIdx.x;
    const int lane = threadIdx.x;
    const bool live = i < p.b && p.step[i].slot >= 0;
    if (!live) {
        if (lane == 0 && i < p.b_hi) {
            p.acc_len[i] = 0;
            p.bonus[i] = 0;
        }
        return;
    }
    const int T = p.T, T1 = p.T + 1;
    const int n = p.tree_n[i];
    const int* tok = p.tree_tok + (long long)i * T;
    const int* par = p.tree_par + (long long)i * T;
    int node = -1, a = 0;
    int want;
    // the accepted path is a root-to-leaf chain of the tree: at most D nodes
    // (children always follow their parent in rank order, so `found` strictly
    // increases); the bound also makes a malformed tree unable to spin
    for (int depth = 0;; ++depth) {
        const int vrow = i * T1 + (node < 0 ? 0 : node + 1);
        want = p.argmax[vrow];
        int found = -1;
        for (int c0 = 0; c0 < n && found < 0; c0 += 32) {
            const int c = c0 + lane;
            const bool hit = c < n && par[c] == node && tok[c] == want;
            const unsigned bal = __ballot_sync(0xffffffffu, hit);
            if (bal) found = c0 + __ffs(bal) - 1;
        }
        if (found < 0 || found <= node || depth >= p.maxD) break;
        if (lane == 0) {
            p.acc_nodes[(long long)i * p.maxD + a] = found;
            p.acc_tok[(long long)i * p.maxD + a] = want;
        }
        ++a;
        node = found;
    }
    if (lane == 0) {
        p.acc_len[i] = a;
        p.bonus[i] = want;
    }
}
void launch_accept_greedy(const AcceptParams& p, cudaStream_t st) { launch_pdl(k_accept_greedy, p.b_hi, 32, 0, st, p); }

// ------------------------------------------------- commit / compaction (K8)
// grid (b_hi, layers + 1): blocks y < layers compact that layer's target KV
// (tree slot lt+1+n_j -> lt+1+j, all sources read before any write), block y
// == layers commits tokens (accepted ++ bonus) and target features of the
// root + accepted rows into the per-slot histories.
__global__ void __launch_bounds__(256) k_commit(CommitParams p) {
    pdl_wait();
    const int i = blockIdx.x;
    const bool live = i < p.b && p.step[i].slot >= 0;
    if (!live) return;
    const int slot = p.step[i].slot, lt = p.step[i].lt;
    const int a = p.acc_len[i];
    const int y = blockIdx.y;
    if (y < p.layers) {
        // 16-byte chunks of (K|V, accepted j, head h, chunk w): every source is
        // read into registers before any destination is written (in-place
        // compaction: a destination may be another accepted node's source)
        const int cph = p.hd / 8;                  // chunks per head row
        const int total = 2 * a * p.KV * cph;
        constexpr int kPer = 16;                   // chunks per thread (2 * kMaxDepth * KV * cph <= 16 * 256)
        uint4 v[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int c = threadIdx.x + u * 256;
            if (c < total) {
                const int which = c / (a * p.KV * cph), rem = c % (a * p.KV * cph);
                const int jj = rem / (p.KV * cph), r2 = rem % (p.KV * cph);
                const int h = r2 / cph, w = r2 % cph;
                const int src = lt + 1 + p.acc_nodes[(long long)i * p.maxD + jj];
                const bf16* cache = which == 0 ? p.kc[y] : p.vc[y];
                v[u] = reinterpret_cast<const uint4*>(cache + (((long long)slot * p.KV + h) * p.cap + src) * p.hd)[w];
            }
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int c = threadIdx.x + u * 256;
            if (c < total) {
                const int which = c / (a * p.KV * cph), rem = c % (a * p.KV * cph);
                const int jj = rem / (p.KV * cph), r2 = rem % (p.KV * cph);
                const int h = r2 / cph, w = r2 % cph;
                bf16* cache = which == 0 ? p.kc[y] : p.vc[y];
                reinterpret_cast<uint4*>(cache + (((long long)slot * p.KV + h) * p.cap + lt + 1 + jj) * p.hd)[w] = v[u];
            }
        }
    } else {
        // tokens: accepted at lt+1.., bonus at lt+1+a
        for (int t = threadIdx.x; t <= a; t += blockDim.x) {
            const int tokv = t < a ? p.acc_tok[(long long)i * p.maxD + t] : p.bonus[i];
            p.tok_hist[(long long)slot * p.cap + lt + 1 + t] = tokv;
        }
        // features of root (verify row 0) and accepted nodes at positions lt..lt+a (16-byte chunks)
        const int cpr = p.d / 8;
        for (int c = threadIdx.x; c < (a + 1) * cpr; c += blockDim.x) {
            const int t = c / cpr, w = c % cpr;
            const int vrow = i * p.row_stride + (t == 0 ? 0 : 1 + p.acc_nodes[(long long)i * p.maxD + t - 1]);
            reinterpret_cast<uint4*>(p.feat_hist + ((long long)slot * p.cap + lt + t) * p.d)[w] =
                reinterpret_cast<const uint4*>(p.vfeat + (long long)vrow * p.d)[w];
        }
        if (threadIdx.x == 0 && p.kv_len) p.kv_len[i] = lt + 1 + a;
    }
}
void launch_commit(const CommitParams& p, cudaStream_t st) {
    if (2 * p.maxD * p.KV * (p.hd / 8) > 16 * 256 || (p.hd % 8) || (p.d % 8))
        throw CudaError("k_commit: per-thread chunk budget exceeded");
    dim3 grid(p.b_hi, p.layers + 1);
    launch_pdl(k_commit, grid, 256, 0, st, p);
}

// AR commit: token at lt+1, feature at lt
__global__ void k_commit_ar(const StepIn* __restrict__ st, int b, const int* __restrict__ argmax,
                            const bf16* __restrict__ feat, int d, int* tok_hist, bf16* feat_hist, int cap,
                            int* __restrict__ out_tok) {
    pdl_wait();
    const int i = blockIdx.x;
    if (i >= b || st[i].slot < 0) return;
    const int slot = st[i].slot, lt = st[i].lt;
    if (threadIdx.x == 0) {
        tok_hist[(long long)slot * cap + lt + 1] = argmax[i];
        out_tok[i] = argmax[i];
    }
    for (int e = threadIdx.x; e < d; e += blockDim.x)
        feat_hist[((long long)slot * cap + lt) * d + e] = feat[(long long)i * d + e];
}
void launch_commit_ar(const StepIn* st, int b, const int* argmax, const bf16* feat, int d, int* tok_hist,
                      bf16* feat_hist, int cap, int* out_tok, cudaStream_t s) {
    if (b > 0) launch_pdl(k_commit_ar, b, 256, 0, s, st, b, argmax, feat, d, tok_hist, feat_hist, cap, out_tok);
}

}  // namespace tlt

namespace tlt {
// e4m3 quantisation with one fp32 scale per row (weights: per output
// feature; activations: per token): scale = amax / 448 (1 for an all-zero
// row), q = e4m3(x / scale), round-to-nearest-even, saturating. One warp per
// row; the oracle (orc_neural.c) applies the identical arithmetic.
// One CTA per row (a warp per row left a few warps on the GPU, ~12 us per
// drafter level at b <= 8). The row is read once into registers with 16-byte
// loads, all in flight together (a strided scalar loop was a chain of
// dependent L2 round trips: 14 us for 8 rows of 3584 under ncu), its amax by a
// block max (order-free, so the scale is that of any reduction order), then
// each thread quantises its own elements and stores them 8 bytes at a time.
// Bit-identical to the oracle's orc_e4m3_quant_row.
constexpr int kQuantVec = 4;  // uint4 (8 bf16) per thread: rows up to 256 x 32 = 8192 columns
__global__ void __launch_bounds__(256) k_quant_rows_e4m3(const bf16* __restrict__ x, int rows, int cols, long long ld,
                                                         __nv_fp8_storage_t* __restrict__ q, float* __restrict__ scale) {
    pdl_wait();
    __shared__ float red[8];
    const int r = blockIdx.x;
    if (r >= rows) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bf16* xr = x + (long long)r * ld;
    __nv_fp8_storage_t* qr = q + (long long)r * cols;
    const bool vec = (cols & 7) == 0 && (ld & 7) == 0 && cols <= (int)blockDim.x * 8 * kQuantVec;
    uint4 v[kQuantVec];
    float amax = 0.f;
    if (vec) {
#pragma unroll
        for (int u = 0; u < kQuantVec; ++u) {
            const int i = (threadIdx.x + u * blockDim.x) * 8;
            v[u] = i < cols ? *reinterpret_cast<const uint4*>(xr + i) : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int u = 0; u < kQuantVec; ++u) {
            const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&v[u]);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2 f = __bfloat1622float2(h2[j]);
                amax = fmaxf(amax, fmaxf(fabsf(f.x), fabsf(f.y)));
            }
        }
    } else {
        for (int c = threadIdx.x; c < cols; c += blockDim.x) amax = fmaxf(amax, fabsf(__bfloat162float(xr[c])));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if (lane == 0) red[warp] = amax;
    __syncthreads();
    amax = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) amax = fmaxf(amax, red[w]);
    const float s = amax > 0.f ? __fdiv_rn(amax, 448.0f) : 1.0f;  // IEEE division (the oracle computes the same)
    if (vec) {
#pragma unroll
        for (int u = 0; u < kQuantVec; ++u) {
            const int i = (threadIdx.x + u * blockDim.x) * 8;
            if (i >= cols) break;
            const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&v[u]);
            uint2 o;
            uint8_t* ob = reinterpret_cast<uint8_t*>(&o);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2 f = __bfloat1622float2(h2[j]);
                ob[2 * j] = __nv_cvt_float_to_fp8(__fdiv_rn(f.x, s), __NV_SATFINITE, __NV_E4M3);
                ob[2 * j + 1] = __nv_cvt_float_to_fp8(__fdiv_rn(f.y, s), __NV_SATFINITE, __NV_E4M3);
            }
            *reinterpret_cast<uint2*>(qr + i) = o;
        }
    } else {
        for (int c = threadIdx.x; c < cols; c += blockDim.x)
            qr[c] = __nv_cvt_float_to_fp8(__fdiv_rn(__bfloat162float(xr[c]), s), __NV_SATFINITE, __NV_E4M3);
    }
    if (threadIdx.x == 0) scale[r] = s;
}
void launch_quant_rows_e4m3(const bf16* x, int rows, int cols, long long ld, void* q, float* scale, cudaStream_t st) {
    launch_pdl(k_quant_rows_e4m3, rows, 256, 0, st, x, rows, cols, ld, static_cast<__nv_fp8_storage_t*>(q), scale);
}
}  // namespace tlt
