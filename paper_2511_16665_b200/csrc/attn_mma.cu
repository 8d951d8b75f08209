// Tree-masked GQA flash-decode attention on the tensor cores (mma.sync
// m16n8k16 bf16 -> fp32, ldmatrix for V^T).
//
// Work unit (CTA): one request group x one KV head x 16 query vectors (the
// (row, q-head) pairs of that KV head, GQA-packed) x one 256-key split aligned
// to absolute key indices. Each of the 4 warps owns a 64-key quarter of the
// split (keys across warps, so a single decode row still spreads over the SM),
// stages 32 keys of K and V at a time in its own padded shared-memory slice
// (cp.async 16B), runs S = Q K^T, applies the tree mask (bits per query row
// staged in shared memory), an online exp2 softmax, O += P V, and the four
// warps merge (m, l, O) in shared memory into one split partial for
// k_attn_combine. Key layout per slot/head is contiguous [cap][hd] so every
// 32-key tile is 8 KB of coalesced loads.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdlib>

#include "engine_kernels.h"
#include "kernels.cuh"
#include "pdl.cuh"
#include "ptx.cuh"

namespace tlt {

using bf16 = __nv_bfloat16;

namespace {
constexpr int kQV = 16;         // query vectors per CTA (one m16 tile)
constexpr int kSplit = 256;     // keys per CTA split
constexpr int kWarpKeys = 64;   // keys per warp per split
constexpr int kTile = 32;       // keys per warp iteration

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4_trans(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3,
                                              const void* p) {
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(a));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    const int sz = pred ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
}  // namespace


// Fused split combine: the last CTA (of the non-empty split CTAs that share this
// (request, KV head, query-vector tile)) merges every split's (m, l, O) in
// fixed split order — the same arithmetic as k_attn_combine — and writes the
// bf16 output, so no separate combine launch is needed. Called by all
// threads of the CTA at the very end of the attention kernels.
template <int kHD>
__device__ __forceinline__ void attn_fused_combine(const AttnParams& p, int grp, int kvh, int qtile, int qv_lo,
                                                   int qv_hi) {
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    const int n_qt = gridDim.x;
    const long long cidx = ((long long)grp * p.KV + kvh) * n_qt + qtile;
    const int n_active = split_count(p, p.g.lc[grp] + p.g.ntail[grp]);
    if (n_active <= 1 && p.direct1) return;  // the single split wrote the final output itself
    if (threadIdx.x == 0) s_last = atomicAdd(p.counters + cidx, 1) == n_active - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int G = p.H / p.KV;
    const int nqv = p.rows_per_req * G;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int total_keys = p.g.lc[grp] + p.g.ntail[grp];
    const int nsplit = n_active;
    (void)total_keys;
    constexpr int DPL = kHD / 32;
    for (int gqv = qv_lo + warp; gqv < min(qv_hi, nqv); gqv += nw) {
        const int row = grp * p.rows_per_req + gqv / G;
        const int head = kvh * G + gqv % G;
        if (p.rows.slot[row] < 0) continue;
        float M = -CUDART_INF_F;
        for (int sp = 0; sp < nsplit; ++sp) {
            const long long pidx = ((long long)(grp * p.max_splits + sp) * p.qv_cap + gqv) * p.KV + kvh;
            M = fmaxf(M, __ldcg(p.ws_m + pidx));
        }
        float L = 0.f, o[DPL];
#pragma unroll
        for (int e = 0; e < DPL; ++e) o[e] = 0.f;
        for (int sp = 0; sp < nsplit; ++sp) {  // fixed order
            const long long pidx = ((long long)(grp * p.max_splits + sp) * p.qv_cap + gqv) * p.KV + kvh;
            const float ms = __ldcg(p.ws_m + pidx);
            if (ms == -CUDART_INF_F) continue;
            const float w = exp2f(ms - M);
            L += __ldcg(p.ws_l + pidx) * w;
#pragma unroll
            for (int e = 0; e < DPL; ++e) o[e] += __ldcg(p.ws_o + pidx * kHD + lane * DPL + e) * w;
        }
        const float inv = L > 0.f ? 1.0f / L : 0.f;
#pragma unroll
        for (int e = 0; e < DPL; ++e)
            p.out[(long long)row * p.H * kHD + head * kHD + lane * DPL + e] = __float2bfloat16_rn(o[e] * inv);
    }
    if (threadIdx.x == 0) p.counters[cidx] = 0;  // ready for the next launch / graph replay
}

template <int kHD>
__global__ void __launch_bounds__(128) k_attention_mma(AttnParams p) {
    pdl_wait();
    l2_prefetch_slice(p.pf, p.pf_bytes);
    constexpr int kStride = kHD + 8;  // padded smem row (elements): conflict-free fragments
    constexpr int KS = kHD / 16;      // k-steps over head_dim
    constexpr int NT = kHD / 8;       // n-tiles of the output
    extern __shared__ __align__(16) unsigned char sm_raw[];
    bf16* Qs = reinterpret_cast<bf16*>(sm_raw);                       // [16][kStride]
    bf16* KVs = Qs + kQV * kStride;                                   // per warp: K[32][kStride], V[32][kStride]
    uint32_t* Ms = reinterpret_cast<uint32_t*>(KVs + 4 * 2 * kTile * kStride);  // [16][kMaskWords]
    float* red = reinterpret_cast<float*>(KVs);                       // merge scratch (aliases K/V after the loop)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int G = p.H / p.KV;
    const int kvh = blockIdx.y;
    const int grp = blockIdx.z / p.max_splits;
    const int split = blockIdx.z % p.max_splits;
    const int qv0 = blockIdx.x * kQV;
    const int nqv = p.rows_per_req * G;
    const int slot = p.g.slot[grp];
    const int lc = p.g.lc[grp], tail0 = p.g.tail0[grp], ntail = p.g.ntail[grp];
    const int total = slot >= 0 ? lc + ntail : 0;
    const int k0 = split * kSplit;
    if (k0 >= total) return;  // empty split: nothing reads its partial (combine stops at the last non-empty one)

    // ---- stage Q (bf16) and the query rows' tail masks
    __shared__ int s_row[kQV];
    if (threadIdx.x < kQV) {
        const int gqv = qv0 + threadIdx.x;
        int row = -1;
        if (gqv < nqv) {
            row = grp * p.rows_per_req + gqv / G;
            if (p.rows.slot[row] < 0) row = -1;
        }
        s_row[threadIdx.x] = row;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < kQV * (kHD / 8); c += blockDim.x) {
        const int l = c / (kHD / 8), w = c % (kHD / 8);
        const int row = s_row[l];
        uint4 v = make_uint4(0, 0, 0, 0);
        if (row >= 0) {
            const int head = kvh * G + (qv0 + l) % G;
            v = reinterpret_cast<const uint4*>(p.q + (long long)row * p.H * kHD + head * kHD)[w];
        }
        *reinterpret_cast<uint4*>(Qs + l * kStride + w * 8) = v;
    }
    const int mw = (ntail + 31) >> 5;
    for (int c = threadIdx.x; c < kQV * kMaskWords; c += blockDim.x) {
        const int l = c / kMaskWords, w = c % kMaskWords;
        const int row = s_row[l];
        Ms[c] = (row >= 0 && w < mw) ? p.rows.mask[(long long)row * kMaskWords + w] : 0u;
    }
    __syncthreads();

    // Q fragments (A operand), 8 k-steps over head_dim
    uint32_t qa[KS][4];
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
        qa[kk][0] = *reinterpret_cast<const uint32_t*>(Qs + g * kStride + kk * 16 + 2 * t);
        qa[kk][1] = *reinterpret_cast<const uint32_t*>(Qs + (g + 8) * kStride + kk * 16 + 2 * t);
        qa[kk][2] = *reinterpret_cast<const uint32_t*>(Qs + g * kStride + kk * 16 + 8 + 2 * t);
        qa[kk][3] = *reinterpret_cast<const uint32_t*>(Qs + (g + 8) * kStride + kk * 16 + 8 + 2 * t);
    }
    const bool live0 = s_row[g] >= 0, live1 = s_row[g + 8] >= 0;

    float o[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float m0 = -CUDART_INF_F, m1 = -CUDART_INF_F, l0 = 0.f, l1 = 0.f;

    bf16* Ks = KVs + warp * 2 * kTile * kStride;
    bf16* Vs = Ks + kTile * kStride;
    const long long slot_base = ((long long)(slot < 0 ? 0 : slot) * p.KV + kvh) * p.cap;
    const int wk0 = k0 + warp * kWarpKeys;
    const int wk1 = min(total, wk0 + kWarpKeys);
    for (int kb = wk0; kb < wk1; kb += kTile) {
        const int nk = min(kTile, wk1 - kb);
        // ---- stage 32 keys of K and V (16B chunks), zero-fill past nk
#pragma unroll 4
        for (int c = lane; c < kTile * (kHD / 8); c += 32) {
            const int j = c / (kHD / 8), w = c % (kHD / 8);
            const bool ok = j < nk;
            const int v = kb + j;
            const long long ci = ok ? (v < lc ? v : tail0 + (v - lc)) : 0;
            const long long off = (slot_base + ci) * kHD + w * 8;
            cp_async16(Ks + j * kStride + w * 8, p.kc + off, ok);
            cp_async16(Vs + j * kStride + w * 8, p.vc + off, ok);
        }
        cp_async_wait_all();
        __syncwarp();
        // ---- S = Q K^T  (16 x 32)
        float s[4][4];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
            s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
            for (int kk = 0; kk < KS; ++kk) {
                const bf16* kr = Ks + (nt * 8 + g) * kStride + kk * 16 + 2 * t;
                mma16816(s[nt], qa[kk], *reinterpret_cast<const uint32_t*>(kr),
                         *reinterpret_cast<const uint32_t*>(kr + 8));
            }
        }
        // ---- scale + visibility (prefix, or tree-mask bit of the query row)
        float mx0 = -CUDART_INF_F, mx1 = -CUDART_INF_F;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int col = nt * 8 + 2 * t + (e & 1);
                const int r = e < 2 ? g : g + 8;
                const int v = kb + col;
                bool vis = col < nk && (e < 2 ? live0 : live1);
                if (vis && v >= lc) {
                    const int tt = v - lc;
                    vis = (Ms[r * kMaskWords + (tt >> 5)] >> (tt & 31)) & 1u;
                }
                const float x = vis ? s[nt][e] * p.scale_log2 : -CUDART_INF_F;
                s[nt][e] = x;
                if (e < 2) mx0 = fmaxf(mx0, x);
                else mx1 = fmaxf(mx1, x);
            }
        }
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
        const float nm0 = fmaxf(m0, mx0), nm1 = fmaxf(m1, mx1);
        const float c0 = nm0 == -CUDART_INF_F ? 1.f : exp2f(m0 - nm0);
        const float c1 = nm1 == -CUDART_INF_F ? 1.f : exp2f(m1 - nm1);
        m0 = nm0;
        m1 = nm1;
        l0 *= c0;
        l1 *= c1;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            o[n][0] *= c0;
            o[n][1] *= c0;
            o[n][2] *= c1;
            o[n][3] *= c1;
        }
        uint32_t pa[2][4];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
            const float p0 = m0 == -CUDART_INF_F ? 0.f : exp2f(s[nt][0] - m0);
            const float p1 = m0 == -CUDART_INF_F ? 0.f : exp2f(s[nt][1] - m0);
            const float p2 = m1 == -CUDART_INF_F ? 0.f : exp2f(s[nt][2] - m1);
            const float p3 = m1 == -CUDART_INF_F ? 0.f : exp2f(s[nt][3] - m1);
            l0 += p0 + p1;
            l1 += p2 + p3;
            const int j = nt >> 1;
            if ((nt & 1) == 0) {
                pa[j][0] = pack_bf16(p0, p1);
                pa[j][1] = pack_bf16(p2, p3);
            } else {
                pa[j][2] = pack_bf16(p0, p1);
                pa[j][3] = pack_bf16(p2, p3);
            }
        }
        // ---- O += P V  (k = 32 keys in two k16 steps, 16 n-tiles of head dims)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
#pragma unroll
            for (int nd = 0; nd < NT; nd += 2) {
                // matrices: (keys 16j..+7, dims nd*8), (keys 16j+8.., nd*8), (.., (nd+1)*8) x2
                const int mi = lane >> 3, r = lane & 7;
                const int key = 16 * j + (mi & 1) * 8 + r;
                const int dim = (nd + (mi >> 1)) * 8;
                uint32_t b0, b1, b2, b3;
                ldsm_x4_trans(b0, b1, b2, b3, Vs + key * kStride + dim);
                mma16816(o[nd], pa[j], b0, b1);
                mma16816(o[nd + 1], pa[j], b2, b3);
            }
        }
        __syncwarp();
    }
    // quad-reduce l
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);

    // ---- merge the 4 warps' partials (fixed order) in shared memory
    __syncthreads();
    float* wm = red;                      // [4][16]
    float* wl = wm + 4 * kQV;             // [4][16]
    float* wo = wl + 4 * kQV;             // [4][16][kHD]
    if (t == 0) {
        wm[warp * kQV + g] = m0;
        wm[warp * kQV + g + 8] = m1;
        wl[warp * kQV + g] = l0;
        wl[warp * kQV + g + 8] = l1;
    }
#pragma unroll
    for (int n = 0; n < NT; ++n) {
        float* r0 = wo + (warp * kQV + g) * kHD + n * 8 + 2 * t;
        float* r1 = wo + (warp * kQV + g + 8) * kHD + n * 8 + 2 * t;
        r0[0] = o[n][0];
        r0[1] = o[n][1];
        r1[0] = o[n][2];
        r1[1] = o[n][3];
    }
    __syncthreads();
    for (int c = threadIdx.x; c < kQV * kHD; c += blockDim.x) {
        const int q = c / kHD, e = c % kHD;
        const int gqv = qv0 + q;
        if (gqv >= nqv) continue;
        float M = -CUDART_INF_F;
        for (int w = 0; w < 4; ++w) M = fmaxf(M, wm[w * kQV + q]);
        float L = 0.f, O = 0.f;
        if (M != -CUDART_INF_F)
            for (int w = 0; w < 4; ++w) {
                const float sc = exp2f(wm[w * kQV + q] - M);
                L += wl[w * kQV + q] * sc;
                O += wo[(w * kQV + q) * kHD + e] * sc;
            }
        const long long pidx = ((long long)(grp * p.max_splits + split) * p.qv_cap + gqv) * p.KV + kvh;
        p.ws_o[pidx * kHD + e] = O;
        if (e == 0) {
            p.ws_m[pidx] = M;
            p.ws_l[pidx] = L;
        }
    }
    if (p.counters) attn_fused_combine<kHD>(p, grp, kvh, blockIdx.x, qv0, qv0 + kQV);
}

// ---------------------------------------------------------------------------
// Multi-row variant for tree verify / drafter levels (many query vectors per
// request and KV head): CTA = (128 query vectors, KV head, request, 256-key
// split), 8 warps, warp w owns query m16-tile w. K/V tiles of 64 keys are
// staged ONCE per CTA in shared memory (cp.async, double-buffered) and shared
// by all 8 warps, so each K/V byte is read once per 128 query vectors instead
// of once per 16 (7 query heads x T+1 rows of a request share one KV head).
// Same split alignment and partial layout as k_attention_mma, so
// k_attn_combine merges either.
constexpr int kTKeys = 64;  // keys per stage

// QV query vectors per CTA (QV / 16 warps): 128 shares each K/V tile widest,
// 64 fits two CTAs per SM (more latency hiding when there are few CTAs)
template <int kHD, int QV>
__global__ void __launch_bounds__(QV * 2, QV == 64 ? 2 : 1) k_attention_tree(AttnParams p) {
    constexpr int kTQV = QV;
    constexpr int kTRows = kTQV / 2 + 2;  // >= distinct rows covered by QV qv (G >= 2)
    constexpr int kThreads = QV * 2;
    pdl_wait();
    l2_prefetch_slice(p.pf, p.pf_bytes);
    constexpr int kStride = kHD + 8;
    constexpr int KS = kHD / 16;
    constexpr int NT = kHD / 8;
    extern __shared__ __align__(16) unsigned char sm_raw[];
    bf16* Qs = reinterpret_cast<bf16*>(sm_raw);            // [128][kStride]
    bf16* Kb = Qs + kTQV * kStride;                        // [2][64][kStride]
    bf16* Vb = Kb + 2 * kTKeys * kStride;                  // [2][64][kStride]
    uint32_t* Ms = reinterpret_cast<uint32_t*>(Vb + 2 * kTKeys * kStride);  // [kTRows][kMaskWords]
    __shared__ int s_lrow[kTQV];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int G = p.H / p.KV;
    const int kvh = blockIdx.y;
    const int grp = blockIdx.z / p.max_splits;
    const int split = blockIdx.z % p.max_splits;
    const int qv0 = blockIdx.x * kTQV;
    const int nqv = p.rows_per_req * G;
    const int slot = p.g.slot[grp];
    const int lc = p.g.lc[grp], tail0 = p.g.tail0[grp], ntail = p.g.ntail[grp];
    const int total = slot >= 0 ? lc + ntail : 0;
    // per-request split size (whole 64-key tiles) from the request's own key count
    const int chunk = p.dyn_splits > 0 ? split_chunk(p, total) : kSplit;
    const int k0 = split * chunk;
    if (k0 >= total) return;  // empty split: nothing reads its partial (combine stops at the last non-empty one)
    const int k1 = min(total, k0 + chunk);
    const bool single = p.direct1 && split_count(p, total) == 1;  // write the normalised output directly
    const int row_base = qv0 / G;  // first request-local row of this CTA

    // ---- K/V tile loader (all threads): 64 keys x kHD of K and of V
    const long long slot_base = ((long long)(slot < 0 ? 0 : slot) * p.KV + kvh) * p.cap;
    auto load_tile = [&](int kb, int buf) {
        bf16* Kd = Kb + buf * kTKeys * kStride;
        bf16* Vd = Vb + buf * kTKeys * kStride;
        const int nk = min(kTKeys, k1 - kb);
#pragma unroll
        for (int c = threadIdx.x; c < kTKeys * (kHD / 8); c += kThreads) {
            const int j = c / (kHD / 8), w = c % (kHD / 8);
            const bool ok = j < nk;
            const int v = kb + j;
            const long long ci = ok ? (v < lc ? v : tail0 + (v - lc)) : 0;
            const long long off = (slot_base + ci) * kHD + w * 8;
            cp_async16(Kd + j * kStride + w * 8, p.kc + off, ok);
            cp_async16(Vd + j * kStride + w * 8, p.vc + off, ok);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    load_tile(k0, 0);  // first K/V tile in flight while Q and the masks are staged

    // ---- stage Q (async, zero-filled for padding rows) and the rows' tail masks
    if (threadIdx.x < kTQV) {
        const int gqv = qv0 + threadIdx.x;
        int lr = -1;
        if (gqv < nqv) {
            const int row = grp * p.rows_per_req + gqv / G;
            if (p.rows.slot[row] >= 0) lr = gqv / G - row_base;
        }
        s_lrow[threadIdx.x] = lr;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < kTQV * (kHD / 8); c += blockDim.x) {
        const int l = c / (kHD / 8), w = c % (kHD / 8);
        const bool ok = s_lrow[l] >= 0;
        const int gqv = qv0 + l;
        const int row = ok ? grp * p.rows_per_req + gqv / G : 0;
        const int head = kvh * G + gqv % G;
        cp_async16(Qs + l * kStride + w * 8, p.q + (long long)row * p.H * kHD + head * kHD + w * 8, ok);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    const int nrows = min(kTRows, p.rows_per_req - row_base);
    const int mw = (ntail + 31) >> 5;
    for (int c = threadIdx.x; c < nrows * (kMaskWords / 4); c += blockDim.x) {
        const int l = c / (kMaskWords / 4), w4 = c % (kMaskWords / 4);
        const int row = grp * p.rows_per_req + row_base + l;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (w4 * 4 < mw) v = reinterpret_cast<const uint4*>(p.rows.mask + (long long)row * kMaskWords)[w4];
        const int w = w4 * 4;
        if (w + 0 >= mw) v.x = 0u;
        if (w + 1 >= mw) v.y = 0u;
        if (w + 2 >= mw) v.z = 0u;
        if (w + 3 >= mw) v.w = 0u;
        *reinterpret_cast<uint4*>(Ms + l * kMaskWords + w) = v;
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");  // Q (and K/V tile 0)
    __syncthreads();  // Q / masks staged

    // this warp's 16 query vectors
    const int wq0 = warp * 16;
    const bool active = qv0 + wq0 < nqv;
    uint32_t qa[KS][4];
    int lr0 = -1, lr1 = -1;
    if (active) {
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
            qa[kk][0] = *reinterpret_cast<const uint32_t*>(Qs + (wq0 + g) * kStride + kk * 16 + 2 * t);
            qa[kk][1] = *reinterpret_cast<const uint32_t*>(Qs + (wq0 + g + 8) * kStride + kk * 16 + 2 * t);
            qa[kk][2] = *reinterpret_cast<const uint32_t*>(Qs + (wq0 + g) * kStride + kk * 16 + 8 + 2 * t);
            qa[kk][3] = *reinterpret_cast<const uint32_t*>(Qs + (wq0 + g + 8) * kStride + kk * 16 + 8 + 2 * t);
        }
        lr0 = s_lrow[wq0 + g];
        lr1 = s_lrow[wq0 + g + 8];
    }
    float o[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float m0 = -CUDART_INF_F, m1 = -CUDART_INF_F, l0 = 0.f, l1 = 0.f;

    int buf = 0;
    for (int kb = k0; kb < k1; kb += kTKeys, buf ^= 1) {
        if (kb + kTKeys < k1) {
            load_tile(kb + kTKeys, buf ^ 1);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        if (active) {
            const bf16* Ks = Kb + buf * kTKeys * kStride;
            const bf16* Vs = Vb + buf * kTKeys * kStride;
            const int nk = min(kTKeys, k1 - kb);
            // ---- S = Q K^T (16 x 64)
            float s[8][4];
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) {
                s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
                for (int kk = 0; kk < KS; ++kk) {
                    const bf16* kr = Ks + (nt * 8 + g) * kStride + kk * 16 + 2 * t;
                    mma16816(s[nt], qa[kk], *reinterpret_cast<const uint32_t*>(kr),
                             *reinterpret_cast<const uint32_t*>(kr + 8));
                }
            }
            // ---- scale + visibility (committed prefix, or the row's tree-mask bit)
            float mx0 = -CUDART_INF_F, mx1 = -CUDART_INF_F;
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int col = nt * 8 + 2 * t + (e & 1);
                    const int lr = e < 2 ? lr0 : lr1;
                    const int v = kb + col;
                    bool vis = col < nk && lr >= 0;
                    if (vis && v >= lc) {
                        const int tt = v - lc;
                        vis = (Ms[lr * kMaskWords + (tt >> 5)] >> (tt & 31)) & 1u;
                    }
                    const float x = vis ? s[nt][e] * p.scale_log2 : -CUDART_INF_F;
                    s[nt][e] = x;
                    if (e < 2) mx0 = fmaxf(mx0, x);
                    else mx1 = fmaxf(mx1, x);
                }
            }
            mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
            mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
            mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
            mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
            const float nm0 = fmaxf(m0, mx0), nm1 = fmaxf(m1, mx1);
            const float c0 = nm0 == -CUDART_INF_F ? 1.f : exp2f(m0 - nm0);
            const float c1 = nm1 == -CUDART_INF_F ? 1.f : exp2f(m1 - nm1);
            m0 = nm0;
            m1 = nm1;
            l0 *= c0;
            l1 *= c1;
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                o[n][0] *= c0;
                o[n][1] *= c0;
                o[n][2] *= c1;
                o[n][3] *= c1;
            }
            uint32_t pa[4][4];
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) {
                const float p0 = m0 == -CUDART_INF_F ? 0.f : exp2f(s[nt][0] - m0);
                const float p1 = m0 == -CUDART_INF_F ? 0.f : exp2f(s[nt][1] - m0);
                const float p2 = m1 == -CUDART_INF_F ? 0.f : exp2f(s[nt][2] - m1);
                const float p3 = m1 == -CUDART_INF_F ? 0.f : exp2f(s[nt][3] - m1);
                l0 += p0 + p1;
                l1 += p2 + p3;
                const int j = nt >> 1;
                if ((nt & 1) == 0) {
                    pa[j][0] = pack_bf16(p0, p1);
                    pa[j][1] = pack_bf16(p2, p3);
                } else {
                    pa[j][2] = pack_bf16(p0, p1);
                    pa[j][3] = pack_bf16(p2, p3);
                }
            }
            // ---- O += P V (64 keys = 4 k16 steps)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
#pragma unroll
                for (int nd = 0; nd < NT; nd += 2) {
                    const int mi = lane >> 3, r = lane & 7;
                    const int key = 16 * j + (mi & 1) * 8 + r;
                    const int dim = (nd + (mi >> 1)) * 8;
                    uint32_t b0, b1, b2, b3;
                    ldsm_x4_trans(b0, b1, b2, b3, Vs + key * kStride + dim);
                    mma16816(o[nd], pa[j], b0, b1);
                    mma16816(o[nd + 1], pa[j], b2, b3);
                }
            }
        }
        __syncthreads();  // buffer `buf` is refilled by the next iteration's prefetch
    }
    if (active) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
    // ---- split partial of each of this warp's query vectors (or, for a
    // request served by one split, its final output)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int gqv = qv0 + wq0 + g + 8 * h;
        if (gqv >= nqv) continue;
        if (single) {
            if ((h ? lr1 : lr0) < 0) continue;  // padding row
            const float inv = (h ? l1 : l0) > 0.f ? 1.0f / (h ? l1 : l0) : 0.f;
            const int row = grp * p.rows_per_req + gqv / G;
            bf16* dst = p.out + (long long)row * p.H * kHD + (kvh * G + gqv % G) * kHD;
#pragma unroll
            for (int n = 0; n < NT; ++n)
                *reinterpret_cast<__nv_bfloat162*>(dst + n * 8 + 2 * t) =
                    __floats2bfloat162_rn(o[n][2 * h] * inv, o[n][2 * h + 1] * inv);
            continue;
        }
        const long long pidx = ((long long)(grp * p.max_splits + split) * p.qv_cap + gqv) * p.KV + kvh;
        float* dst = p.ws_o + pidx * kHD;
#pragma unroll
        for (int n = 0; n < NT; ++n)
            *reinterpret_cast<float2*>(dst + n * 8 + 2 * t) = make_float2(o[n][2 * h], o[n][2 * h + 1]);
        if (t == 0) {
            p.ws_m[pidx] = h ? m1 : m0;
            p.ws_l[pidx] = h ? l1 : l0;
        }
    }
    }  // active
    if (p.counters && !single) attn_fused_combine<kHD>(p, grp, kvh, blockIdx.x, qv0, qv0 + kTQV);
}

template <int kHD, int QV>
void launch_attention_tree_t(const AttnParams& p, cudaStream_t st) {
    constexpr int kStride = kHD + 8;
    const size_t smem = sizeof(bf16) * (QV + 4 * kTKeys) * kStride + sizeof(uint32_t) * (QV / 2 + 2) * kMaskWords;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_attention_tree<kHD, QV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    const int G = p.H / p.KV;
    const int nqv = p.rows_per_req * G;
    dim3 grid((nqv + QV - 1) / QV, p.KV, p.n_groups * p.max_splits);
    launch_pdl(k_attention_tree<kHD, QV>, grid, QV * 2, smem, st, p);
}

// ---------------------------------------------------------------------------
// Decode variant (<= 16 query vectors per request and KV head, e.g. plain AR
// decode: 1 row x 7 q-heads): CTA = (KV head, request, key split of p.chunk
// keys, a multiple of 256 chosen so the grid covers the SMs ~2x). All 128
// threads stage 64-key K/V tiles into a 3-deep cp.async ring (contiguous
// 16-byte chunks: committed-prefix keys are consecutive rows), and warp w
// consumes keys [16w, 16w+16) of every tile (ldmatrix fragments), keeping its
// own online-softmax state; the 4 warps merge in smem at the end. One
// partial per split -> fused combine.
constexpr int kDKeys = 64;
constexpr int kDStages = 3;

__device__ __forceinline__ void ldsm_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, const void* p) {
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(a));
}

template <int kHD>
__global__ void __launch_bounds__(128) k_attention_dec(AttnParams p) {
    pdl_wait();
    l2_prefetch_slice(p.pf, p.pf_bytes);
    constexpr int kStride = kHD + 8;
    constexpr int KS = kHD / 16;
    constexpr int NT = kHD / 8;
    constexpr int CPR = kHD / 8;  // 16-byte chunks per key row
    extern __shared__ __align__(16) unsigned char sm_raw[];
    bf16* Qs = reinterpret_cast<bf16*>(sm_raw);                 // [16][kStride]
    bf16* Kb = Qs + kQV * kStride;                              // [stages][64][kStride]
    bf16* Vb = Kb + kDStages * kDKeys * kStride;                // [stages][64][kStride]
    uint32_t* Ms = reinterpret_cast<uint32_t*>(Vb + kDStages * kDKeys * kStride);  // [16][kMaskWords]
    float* red = reinterpret_cast<float*>(Kb);                  // merge scratch (aliases the ring after the loop)
    __shared__ int s_row[kQV];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int G = p.H / p.KV;
    const int kvh = blockIdx.y;
    const int grp = blockIdx.z / p.max_splits;
    const int split = blockIdx.z % p.max_splits;
    const int nqv = p.rows_per_req * G;
    const int slot = p.g.slot[grp];
    const int lc = p.g.lc[grp], tail0 = p.g.tail0[grp], ntail = p.g.ntail[grp];
    const int total = slot >= 0 ? lc + ntail : 0;
    const int chunk = split_chunk(p, total);
    const int k0 = split * chunk;
    if (k0 >= total) return;  // empty split
    const int k1 = min(total, k0 + chunk);
    const bool single = p.max_splits == 1 || (p.direct1 && split_count(p, total) == 1);
    const int ntiles = (k1 - k0 + kDKeys - 1) / kDKeys;
    const long long slot_base = ((long long)slot * p.KV + kvh) * p.cap;

    auto load_tile = [&](int ti) {
        const int st = ti % kDStages;
        const int kb = k0 + ti * kDKeys;
        const int nk = min(kDKeys, k1 - kb);
        bf16* Kd = Kb + st * kDKeys * kStride;
        bf16* Vd = Vb + st * kDKeys * kStride;
#pragma unroll
        for (int c = threadIdx.x; c < kDKeys * CPR; c += 128) {
            const int j = c / CPR, w = c % CPR;
            const bool ok = j < nk;
            const int v = kb + j;
            const long long ci = ok ? (v < lc ? v : tail0 + (v - lc)) : 0;
            const long long off = (slot_base + ci) * kHD + w * 8;
            cp_async16(Kd + j * kStride + w * 8, p.kc + off, ok);
            cp_async16(Vd + j * kStride + w * 8, p.vc + off, ok);
        }
    };
    // prologue: first stages in flight before Q / masks are staged
#pragma unroll
    for (int i = 0; i < kDStages - 1; ++i) {
        if (i < ntiles) load_tile(i);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    if (threadIdx.x < kQV) {
        const int gqv = threadIdx.x;
        int row = -1;
        if (gqv < nqv) {
            row = grp * p.rows_per_req + gqv / G;
            if (p.rows.slot[row] < 0) row = -1;
        }
        s_row[threadIdx.x] = row;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < kQV * CPR; c += 128) {
        const int l = c / CPR, w = c % CPR;
        const int row = s_row[l];
        uint4 v = make_uint4(0, 0, 0, 0);
        if (row >= 0) v = reinterpret_cast<const uint4*>(p.q + (long long)row * p.H * kHD + (kvh * G + l % G) * kHD)[w];
        *reinterpret_cast<uint4*>(Qs + l * kStride + w * 8) = v;
    }
    const int mw = (ntail + 31) >> 5;
    for (int c = threadIdx.x; c < kQV * kMaskWords; c += 128) {
        const int l = c / kMaskWords, w = c % kMaskWords;
        const int row = s_row[l];
        Ms[c] = (row >= 0 && w < mw) ? p.rows.mask[(long long)row * kMaskWords + w] : 0u;
    }
    __syncthreads();
    uint32_t qa[KS][4];
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
        qa[kk][0] = *reinterpret_cast<const uint32_t*>(Qs + g * kStride + kk * 16 + 2 * t);
        qa[kk][1] = *reinterpret_cast<const uint32_t*>(Qs + (g + 8) * kStride + kk * 16 + 2 * t);
        qa[kk][2] = *reinterpret_cast<const uint32_t*>(Qs + g * kStride + kk * 16 + 8 + 2 * t);
        qa[kk][3] = *reinterpret_cast<const uint32_t*>(Qs + (g + 8) * kStride + kk * 16 + 8 + 2 * t);
    }
    const bool live0 = s_row[g] >= 0, live1 = s_row[g + 8] >= 0;
    float o[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float m0 = -CUDART_INF_F, m1 = -CUDART_INF_F, l0 = 0.f, l1 = 0.f;

    for (int ti = 0; ti < ntiles; ++ti) {
        if (ti + kDStages - 1 < ntiles) load_tile(ti + kDStages - 1);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        asm volatile("cp.async.wait_group %0;\n" ::"n"(kDStages - 1) : "memory");
        __syncthreads();
        const int st = ti % kDStages;
        const bf16* Ks = Kb + st * kDKeys * kStride + warp * 16 * kStride;  // this warp's 16 keys
        const bf16* Vs = Vb + st * kDKeys * kStride + warp * 16 * kStride;
        const int kb = k0 + ti * kDKeys + warp * 16;
        const int nk = min(16, k1 - kb);
        if (nk > 0) {
            // ---- S = Q K^T (16 x 16): ldmatrix x4 = (keys 0-7 | 8-15) x (dims k | k+8)
            float s[2][4];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
            const int mi = lane >> 3, r = lane & 7;
#pragma unroll
            for (int kk = 0; kk < KS; ++kk) {
                uint32_t b0, b1, b2, b3;
                // matrices: 0 = keys 0-7 dims kk*16+0..7, 1 = keys 0-7 dims +8, 2 = keys 8-15 dims +0, 3 = keys 8-15 dims +8
                ldsm_x4(b0, b1, b2, b3, Ks + ((mi >> 1) * 8 + r) * kStride + kk * 16 + (mi & 1) * 8);
                mma16816(s[0], qa[kk], b0, b1);
                mma16816(s[1], qa[kk], b2, b3);
            }
            float mx0 = -CUDART_INF_F, mx1 = -CUDART_INF_F;
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int col = nt * 8 + 2 * t + (e & 1);
                    const int rr = e < 2 ? g : g + 8;
                    const int v = kb + col;
                    bool vis = col < nk && (e < 2 ? live0 : live1);
                    if (vis && v >= lc) {
                        const int tt = v - lc;
                        vis = (Ms[rr * kMaskWords + (tt >> 5)] >> (tt & 31)) & 1u;
                    }
                    const float x = vis ? s[nt][e] * p.scale_log2 : -CUDART_INF_F;
                    s[nt][e] = x;
                    if (e < 2) mx0 = fmaxf(mx0, x);
                    else mx1 = fmaxf(mx1, x);
                }
            }
            mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
            mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
            mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
            mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
            const float nm0 = fmaxf(m0, mx0), nm1 = fmaxf(m1, mx1);
            const float c0 = nm0 == -CUDART_INF_F ? 1.f : exp2f(m0 - nm0);
            const float c1 = nm1 == -CUDART_INF_F ? 1.f : exp2f(m1 - nm1);
            m0 = nm0;
            m1 = nm1;
            l0 *= c0;
            l1 *= c1;
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                o[n][0] *= c0;
                o[n][1] *= c0;
                o[n][2] *= c1;
                o[n][3] *= c1;
            }
            uint32_t pa[4];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                const float p0 = m0 == -CUDART_INF_F ? 0.f : exp2f(s[nt][0] - m0);
                const float p1 = m0 == -CUDART_INF_F ? 0.f : exp2f(s[nt][1] - m0);
                const float p2 = m1 == -CUDART_INF_F ? 0.f : exp2f(s[nt][2] - m1);
                const float p3 = m1 == -CUDART_INF_F ? 0.f : exp2f(s[nt][3] - m1);
                l0 += p0 + p1;
                l1 += p2 + p3;
                pa[nt * 2 + 0] = pack_bf16(p0, p1);
                pa[nt * 2 + 1] = pack_bf16(p2, p3);
            }
            // A fragment order for m16n8k16: {rows g, k 0-7}, {rows g+8, k 0-7}, {rows g, k 8-15}, {rows g+8, k 8-15}
            const uint32_t pf[4] = {pa[0], pa[1], pa[2], pa[3]};
#pragma unroll
            for (int nd = 0; nd < NT; nd += 2) {
                const int key = (mi & 1) * 8 + r;
                const int dim = (nd + (mi >> 1)) * 8;
                uint32_t b0, b1, b2, b3;
                ldsm_x4_trans(b0, b1, b2, b3, Vs + key * kStride + dim);
                mma16816(o[nd], pf, b0, b1);
                mma16816(o[nd + 1], pf, b2, b3);
            }
        }
        __syncthreads();  // stage st is refilled by a later iteration's prefetch
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
    // ---- merge the 4 warps' partials (fixed order) in shared memory
    __syncthreads();
    float* wm = red;
    float* wl = wm + 4 * kQV;
    float* wo = wl + 4 * kQV;
    if (t == 0) {
        wm[warp * kQV + g] = m0;
        wm[warp * kQV + g + 8] = m1;
        wl[warp * kQV + g] = l0;
        wl[warp * kQV + g + 8] = l1;
    }
#pragma unroll
    for (int n = 0; n < NT; ++n) {
        *reinterpret_cast<float2*>(wo + (warp * kQV + g) * kHD + n * 8 + 2 * t) = make_float2(o[n][0], o[n][1]);
        *reinterpret_cast<float2*>(wo + (warp * kQV + g + 8) * kHD + n * 8 + 2 * t) = make_float2(o[n][2], o[n][3]);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < kQV * kHD; c += blockDim.x) {
        const int q = c / kHD, e = c % kHD;
        if (q >= nqv) continue;
        float M = -CUDART_INF_F;
        for (int w = 0; w < 4; ++w) M = fmaxf(M, wm[w * kQV + q]);
        float L = 0.f, O = 0.f;
        if (M != -CUDART_INF_F)
            for (int w = 0; w < 4; ++w) {
                const float sc = exp2f(wm[w * kQV + q] - M);
                L += wl[w * kQV + q] * sc;
                O += wo[(w * kQV + q) * kHD + e] * sc;
            }
        if (single) {  // single split: final normalised output, no combine
            const int row = s_row[q];
            if (row >= 0)
                p.out[(long long)row * p.H * kHD + (kvh * G + q % G) * kHD + e] =
                    __float2bfloat16_rn(L > 0.f ? O / L : 0.f);
            continue;
        }
        const long long pidx = ((long long)(grp * p.max_splits + split) * p.qv_cap + q) * p.KV + kvh;
        p.ws_o[pidx * kHD + e] = O;
        if (e == 0) {
            p.ws_m[pidx] = M;
            p.ws_l[pidx] = L;
        }
    }
    if (p.counters && !single) attn_fused_combine<kHD>(p, grp, kvh, 0, 0, kQV);
}

template <int kHD>
void launch_attention_dec_t(const AttnParams& p, cudaStream_t st) {
    constexpr int kStride = kHD + 8;
    const size_t ring = sizeof(bf16) * 2 * kDStages * kDKeys * kStride;
    const size_t merge = sizeof(float) * (8 * kQV + 4 * kQV * kHD);
    const size_t smem = sizeof(bf16) * kQV * kStride + (ring > merge ? ring : merge) + sizeof(uint32_t) * kQV * kMaskWords;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_attention_dec<kHD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    dim3 grid(1, p.KV, p.n_groups * p.max_splits);
    launch_pdl(k_attention_dec<kHD>, grid, 128, smem, st, p);
}

static int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v ? std::atoi(v) : dflt;
}

// Target split count per (request, KV head) for the per-request split sizing
// (split_chunk); 0 = per-request sizing off (TLT_ATTN_DEC_DYN=0). Knobs are
// read per call (host side, once per captured launch).
int attention_dec_target_splits(int n_groups, int kv) {
    if (!env_int("TLT_ATTN_DEC_DYN", 1)) return 0;
    const int target_ctas = env_int("TLT_ATTN_DEC_CTAS", 296);
    return n_groups * kv >= target_ctas ? 1 : std::max(1, target_ctas / std::max(1, n_groups * kv));
}

// Fixed split size (TLT_ATTN_DEC_DYN=0): chunk so that (groups x KV heads x
// splits) ~ 2 CTAs per SM. Any multiple of the 64-key tile works for this
// kernel: 64-key granularity balances the splits (b = 16: 4 x 320 keys
// instead of 2 x 512 + 1; 26.7 -> 22.6 us per layer), and a 256-key floor
// keeps the long-tail shapes from fragmenting into many tiny splits whose
// combine costs more than it saves (b = 1: 16.5 us vs 18.5 us at 64 keys;
// profiles/r1_attn_dec_granularity.txt). Returns 0 when the decode kernel is
// off (TLT_ATTN_DEC=0).
int attention_dec_chunk(int n_groups, int kv, int max_keys) {
    if (!env_int("TLT_ATTN_DEC", 1)) return 0;
    const int target_ctas = env_int("TLT_ATTN_DEC_CTAS", 296);
    const int gran = std::max(kDKeys, env_int("TLT_ATTN_DEC_GRAN", kDKeys) / kDKeys * kDKeys);
    const int min_chunk = std::max(kDKeys, env_int("TLT_ATTN_DEC_MIN_CHUNK", 256));
    const int chunks = std::max(1, (max_keys + gran - 1) / gran);
    // (request, head) pairs alone reach the CTA target: a single split (the
    // kernel then writes the normalised output itself, no partials, no combine)
    const int want_splits = n_groups * kv >= target_ctas ? 1 : std::max(1, target_ctas / std::max(1, n_groups * kv));
    if (env_int("TLT_ATTN_DEC_EVEN", 1) && max_keys <= min_chunk + min_chunk / 2) {
        // short contexts (<= 384 keys) run as ONE split: no remainder split,
        // no partials, no combine launch (b=1 ctx 257: 14.4 -> 13.1 us; b=4:
        // 16.5 -> 14.4 us; profiles/r1_attn_dec_even.txt)
        return std::max(gran, (max_keys + gran - 1) / gran * gran);
    }
    const int per = std::max(1, (chunks + want_splits - 1) / want_splits);
    return std::max(min_chunk, per * gran);
}

template <int kHD>
size_t attention_mma_smem() {
    constexpr int kStride = kHD + 8;
    const size_t kv = sizeof(bf16) * 4 * 2 * kTile * kStride;
    const size_t merge = sizeof(float) * (4 * kQV * 2 + 4 * kQV * kHD);
    return sizeof(bf16) * kQV * kStride + (kv > merge ? kv : merge) + sizeof(uint32_t) * kQV * kMaskWords;
}

template <int kHD>
void launch_attention_mma_t(const AttnParams& p, cudaStream_t st) {
    static bool attr = false;
    const size_t smem = attention_mma_smem<kHD>();
    if (!attr) {
        cudaFuncSetAttribute(k_attention_mma<kHD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    const int G = p.H / p.KV;
    const int nqv = p.rows_per_req * G;
    dim3 grid((nqv + kQV - 1) / kQV, p.KV, p.n_groups * p.max_splits);
    launch_pdl(k_attention_mma<kHD>, grid, 128, smem, st, p);
}

int attention_mma_split() { return kSplit; }

// Split plan of one attention launch over requests of up to max_keys keys
// (the grid is sized for that bound; each CTA sizes its split from its own
// request's key count, split_chunk). Decode (<= 16 query vectors per
// (request, KV head)): flash-decode kernel. Tree verify / drafter levels:
// the 64-query-vector tree kernel with (request, KV head, q-tile) x splits
// aiming at TLT_ATTN_TREE_CTAS CTAs (default 296 = 2 per SM, the kernel's
// occupancy), whole 64-key tiles, at least TLT_ATTN_TREE_MIN_CHUNK (128)
// keys per split: measured best over the verify / drafter shapes
// (profiles/r2_attn_sweep.txt: b=5 T=48 46.7 -> 39.0 us, b=16 T=16 51.2 ->
// 39.9 us, b=31 T=16 75.3 -> 59.5 us per layer vs the fixed 256-key splits
// sized for the cache capacity). A request served by one split writes its
// output directly (no partials, no combine).
void attention_plan_splits(AttnParams& p, int max_keys) {
    const int G = p.H / p.KV;
    const int nqv = p.rows_per_req * G;
    p.chunk = p.impl == 1 ? kSplit : 512;
    p.dec = 0;
    p.dyn_splits = 0;
    p.gran = kDKeys;
    p.min_chunk = kSplit;
    p.direct1 = 0;
    if (p.impl == 1 && nqv <= 16) {
        const int ch = attention_dec_chunk(p.n_groups, p.KV, max_keys);
        if (ch > 0) {
            p.chunk = ch;
            p.dec = 1;
            p.dyn_splits = attention_dec_target_splits(p.n_groups, p.KV);
            p.gran = std::max(kDKeys, env_int("TLT_ATTN_DEC_GRAN", kDKeys) / kDKeys * kDKeys);
            p.min_chunk = std::max(p.gran, env_int("TLT_ATTN_DEC_MIN_CHUNK", 256) / kDKeys * kDKeys);
            p.direct1 = 1;
        }
    } else if (p.impl == 1 && G >= 2 && nqv >= env_int("TLT_ATTN_TREE_MIN_QV", 17) && env_int("TLT_ATTN_TREE_DYN", 1)) {
        const int qv = env_int("TLT_ATTN_TREE_QV", 64);
        const long long pairs = (long long)p.n_groups * p.KV * ((nqv + qv - 1) / qv);
        const int target = env_int("TLT_ATTN_TREE_CTAS", 296);
        p.dyn_splits = pairs >= target ? 1 : (int)std::max(1LL, target / std::max(1LL, pairs));
        p.gran = kTKeys;
        p.min_chunk = std::max(kTKeys, env_int("TLT_ATTN_TREE_MIN_CHUNK", 128) / kTKeys * kTKeys);
        p.chunk = p.min_chunk;
        p.direct1 = 1;
    }
    p.max_splits = std::max(1, (max_keys + p.chunk - 1) / p.chunk);
    if (p.dyn_splits > 0) p.max_splits = std::max(1, std::min(p.dyn_splits, (max_keys + p.min_chunk - 1) / p.min_chunk));
}

void launch_attention_mma(const AttnParams& p, cudaStream_t st, bool allow_tc) {
    if (allow_tc && attention_tc_eligible(p)) {  // tcgen05 / TMEM kernel (attn_tc.cu)
        launch_attention_tc(p, st);
        return;
    }
    // many query vectors per (request, KV head): share each K/V tile across them
    static const int tree_min = [] {
        const char* v = std::getenv("TLT_ATTN_TREE_MIN_QV");
        return v ? std::atoi(v) : 17;
    }();
    // ... as long as that still yields enough CTAs to cover the SMs (at
    // batch 1 the 16-vector kernel's 8x more CTAs win)
    const int G = p.H / p.KV;
    static const int tree_qv = [] {
        const char* v = std::getenv("TLT_ATTN_TREE_QV");
        return v ? std::atoi(v) : 64;
    }();
    const long long tree_ctas =
        (long long)((p.rows_per_req * G + tree_qv - 1) / tree_qv) * p.KV * p.n_groups * p.max_splits;
    if (p.rows_per_req * G >= tree_min && G >= 2 && (tree_ctas >= 128 || p.dyn_splits > 0)) {
        if (tree_qv == 128) {
            if (p.hd == 128)
                launch_attention_tree_t<128, 128>(p, st);
            else
                launch_attention_tree_t<64, 128>(p, st);
        } else {
            if (p.hd == 128)
                launch_attention_tree_t<128, 64>(p, st);
            else
                launch_attention_tree_t<64, 64>(p, st);
        }
        return;
    }
    if (p.dec) {
        if (p.hd == 128)
            launch_attention_dec_t<128>(p, st);
        else
            launch_attention_dec_t<64>(p, st);
        return;
    }
    if (p.hd == 128)
        launch_attention_mma_t<128>(p, st);
    else
        launch_attention_mma_t<64>(p, st);
}

}  // namespace tlt
