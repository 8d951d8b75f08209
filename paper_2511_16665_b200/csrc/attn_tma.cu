// Tree-masked GQA flash-decode attention with TMA-fed K/V tiles (sm_100a).
//
// Same work decomposition and arithmetic as the mma.sync kernels of
// attn_mma.cu (QK^T and PV on mma.sync m16n8k16 bf16 -> fp32, online exp2
// softmax, fixed-order split merge), but the K/V stream is moved by the
// Tensor Memory Accelerator: one elected thread issues 2D cp.async.bulk.tensor
// loads of whole 64-key x 64-dim boxes (128-byte swizzle) into a ring of
// mbarrier-tracked stages, so the 128 consumer threads issue no load
// instructions for K/V at all and a CTA keeps STAGES x 32 KB in flight.
// The swizzle makes the ldmatrix reads of the tile conflict-free (16-byte
// chunk c of key row r lives at chunk c ^ (r & 7)).
//
// Key tiles: the committed prefix [0, lc) of the request in 64-key tiles from
// key 0, then the tree tail [0, ntail) in 64-key tiles starting at cache row
// tail0 (any row: TMA coordinates need no alignment). A split of the
// request's virtual key sequence (prefix ++ tail, split_chunk keys) maps to a
// run of prefix tiles followed by a run of tail tiles. Rows beyond the valid
// keys of a tile (or beyond the cache: zero-filled by TMA) are masked.
//
// DEC (<= 16 query vectors per (request, KV head), plain decode): the 4 warps
// split every tile's keys (16 each) and merge their (m, l, O) in shared
// memory at the end. TREE: 64 query vectors per CTA, warp w owns vectors
// [16w, 16w + 16) and consumes every key of the tile.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdlib>

#include "engine_kernels.h"
#include "kernels.cuh"
#include "pdl.cuh"
#include "ptx.cuh"
#include "tlt_internal.h"

namespace tlt {

using bf16 = __nv_bfloat16;

namespace {
constexpr int kTK = 64;  // keys per tile

__device__ __forceinline__ void mma16816t(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm4t(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
// byte offset of (key row, dim) inside one stage's K or V tile: halves of 64
// dims are separate 64 x 128 B boxes, 128-byte swizzle within each
template <int HD>
__device__ __forceinline__ uint32_t swz_off(int key, int dim) {
    const int h = dim >> 6, c = (dim & 63) >> 3;
    return (uint32_t)(h * (kTK * 128) + key * 128 + ((c ^ (key & 7)) << 4) + ((dim & 7) << 1));
}
}  // namespace

template <int HD>
__device__ __forceinline__ void attn_fused_combine_tma(const AttnParams& p, int grp, int kvh, int qtile, int qv_lo,
                                                       int qv_hi);

// SUBK: keys per S / P chunk of the TREE warps (64: one chunk per tile; 32:
// two, halving the S / P registers so 3 CTAs fit per SM with STAGES = 2)
template <int HD, bool DEC, int STAGES, int SUBK>
__global__ void __launch_bounds__(128, STAGES == 2 ? 3 : 2)
    k_attention_tma(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, AttnParams p) {
    constexpr int QV = DEC ? 16 : 64;      // query vectors per CTA
    constexpr int KS = HD / 16;            // k-steps over head_dim (QK^T)
    constexpr int NT = HD / 8;             // output n-tiles (PV)
    constexpr int TILE_B = kTK * HD * 2;   // bytes of one K (or V) tile
    constexpr int kRows = DEC ? 16 : QV / 2 + 2;  // distinct rows covered (G >= 2)
    pdl_wait();
    l2_prefetch_slice(p.pf, p.pf_bytes);
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char* ring = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    uint32_t* Ms = reinterpret_cast<uint32_t*>(ring + STAGES * 2 * TILE_B);  // [kRows][kMaskWords]
    __shared__ uint64_t full[STAGES], empty[STAGES];
    __shared__ int s_row[QV];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int G = p.H / p.KV;
    const int kvh = blockIdx.y;
    const int grp = blockIdx.z / p.max_splits;
    const int split = blockIdx.z % p.max_splits;
    const int qv0 = blockIdx.x * QV;
    const int nqv = p.rows_per_req * G;
    const int slot = p.g.slot[grp];
    const int lc = p.g.lc[grp], tail0 = p.g.tail0[grp], ntail = p.g.ntail[grp];
    const int total = slot >= 0 ? lc + ntail : 0;
    const int chunk = split_chunk(p, total);
    const int k0 = split * chunk;
    if (k0 >= total) return;  // empty split
    const int k1 = min(total, k0 + chunk);
    const bool single = p.max_splits == 1 || (p.direct1 && split_count(p, total) == 1);
    // tile runs: prefix [k0, pe) from key k0, tail [ta, te) from tail index ta
    const int pe = min(k1, lc);
    const int n_pt = pe > k0 ? (pe - k0 + kTK - 1) / kTK : 0;
    const int ta = max(k0, lc) - lc, te = k1 - lc;
    const int n_tt = te > ta ? (te - ta + kTK - 1) / kTK : 0;
    const int ntiles = n_pt + n_tt;
    const long long head_row = ((long long)slot * p.KV + kvh) * p.cap;

    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmK);
        tma_prefetch_desc(&tmV);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 4);  // one arrival per consumer warp
        }
        fence_barrier_init();
    }
    __syncthreads();
    const uint64_t pol = policy_evict_first();  // K/V are streamed once per step
    auto issue = [&](int i) {  // thread 0: loads of tile i into stage i % STAGES
        const int s = i % STAGES;
        const long long row = i < n_pt ? head_row + k0 + (long long)i * kTK
                                       : head_row + tail0 + ta + (long long)(i - n_pt) * kTK;
        unsigned char* kd = ring + s * 2 * TILE_B;
        mbar_arrive_expect_tx(&full[s], 2 * TILE_B);
#pragma unroll
        for (int h = 0; h < HD / 64; ++h) {
            tma_load_2d(kd + h * (kTK * 128), &tmK, &full[s], h * 64, (int)row, pol);
            tma_load_2d(kd + TILE_B + h * (kTK * 128), &tmV, &full[s], h * 64, (int)row, pol);
        }
    };
    if (threadIdx.x == 0)
        for (int i = 0; i < min(STAGES, ntiles); ++i) issue(i);

    // ---- query rows and their tail masks (overlaps the first loads)
    if (threadIdx.x < QV) {
        const int gqv = qv0 + threadIdx.x;
        int row = -1;
        if (gqv < nqv) {
            row = grp * p.rows_per_req + gqv / G;
            if (p.rows.slot[row] < 0) row = -1;
        }
        s_row[threadIdx.x] = row;
    }
    __syncthreads();
    const int row_base = qv0 / G;  // first request-local row of this CTA
    const int nrows = min(kRows, p.rows_per_req - row_base);
    const int mw = (ntail + 31) >> 5;
    for (int c = threadIdx.x; c < nrows * kMaskWords; c += blockDim.x) {
        const int l = c / kMaskWords, w = c % kMaskWords;
        const int row = grp * p.rows_per_req + row_base + l;
        Ms[c] = w < mw ? p.rows.mask[(long long)row * kMaskWords + w] : 0u;
    }
    // Q fragments straight from global (each query vector is read once)
    const int wq0 = DEC ? 0 : warp * 16;  // this warp's 16 query vectors
    const bool active = qv0 + wq0 < nqv;
    uint32_t qa[KS][4];
    const int ra = s_row[wq0 + g], rb = s_row[wq0 + g + 8];
    {
        const int ha = kvh * G + (qv0 + wq0 + g) % G, hb = kvh * G + (qv0 + wq0 + g + 8) % G;
        const uint32_t* qA = ra >= 0 ? reinterpret_cast<const uint32_t*>(p.q + (long long)ra * p.H * HD + ha * HD) : nullptr;
        const uint32_t* qB = rb >= 0 ? reinterpret_cast<const uint32_t*>(p.q + (long long)rb * p.H * HD + hb * HD) : nullptr;
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
            qa[kk][0] = qA ? qA[(kk * 16 + 2 * t) >> 1] : 0u;
            qa[kk][1] = qB ? qB[(kk * 16 + 2 * t) >> 1] : 0u;
            qa[kk][2] = qA ? qA[(kk * 16 + 8 + 2 * t) >> 1] : 0u;
            qa[kk][3] = qB ? qB[(kk * 16 + 8 + 2 * t) >> 1] : 0u;
        }
    }
    const int lr0 = ra >= 0 ? (qv0 + wq0 + g) / G - row_base : -1;
    const int lr1 = rb >= 0 ? (qv0 + wq0 + g + 8) / G - row_base : -1;
    __syncthreads();  // masks staged

    float o[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float m0 = -CUDART_INF_F, m1 = -CUDART_INF_F, l0 = 0.f, l1 = 0.f;
    const int mi = lane >> 3, r8 = lane & 7;

    for (int i = 0; i < ntiles; ++i) {
        const int s = i % STAGES;
        const bool tail = i >= n_pt;
        const int kb = tail ? ta + (i - n_pt) * kTK : k0 + i * kTK;  // first key (tail: tail index)
        const int nk = tail ? min(kTK, te - kb) : min(kTK, pe - kb);
        mbar_wait(&full[s], (uint32_t)((i / STAGES) & 1));
        const uint32_t kbase = smem_u32(ring + s * 2 * TILE_B), vbase = kbase + TILE_B;
        // keys of this warp within the tile: DEC 16 (warp-sliced), TREE all
        // 64 in chunks of SUBK
        constexpr int WK = DEC ? 16 : SUBK;
        const int wk0 = DEC ? warp * 16 : 0, wk1 = DEC ? warp * 16 + 16 : kTK;
        const bool zfix = active && wk0 < nk && nk < wk1;
        if (zfix) {
            // rows past the tile's valid keys hold whatever the cache has there
            // (later positions, never-written memory: possibly NaN bit patterns):
            // P is 0 for them but 0 * NaN is NaN, so zero this warp's V rows
            // [nk, wk1) first (other warps write the same zeros)
            uint4* vz = reinterpret_cast<uint4*>(ring + s * 2 * TILE_B + TILE_B);
            constexpr int CPR = 8 * (HD / 64);  // 16-byte chunks per key row (both halves)
            const int z0 = nk, z1 = wk1;
            for (int c = lane; c < (z1 - z0) * CPR; c += 32) {
                const int r = z0 + c / CPR, rem = c % CPR;
                vz[((rem >> 3) * (kTK * 128) + r * 128 + (rem & 7) * 16) >> 4] = make_uint4(0u, 0u, 0u, 0u);
            }
            __syncwarp();
        }
#pragma unroll 1
        for (int key0 = wk0; key0 < wk1; key0 += WK)
        if (active && key0 < nk) {
            float sc[WK / 8][4];
#pragma unroll
            for (int nt = 0; nt < WK / 8; ++nt) sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
#pragma unroll
            for (int kk = 0; kk < KS; ++kk) {
#pragma unroll
                for (int np = 0; np < WK / 16; ++np) {
                    // matrices: (keys +0..7, dims +0..7) (keys +0..7, dims +8..15) (keys +8..15, ...)
                    uint32_t b0, b1, b2, b3;
                    const int key = key0 + np * 16 + (mi >> 1) * 8 + r8;
                    ldsm4(b0, b1, b2, b3, kbase + swz_off<HD>(key, kk * 16 + (mi & 1) * 8));
                    mma16816t(sc[2 * np], qa[kk], b0, b1);
                    mma16816t(sc[2 * np + 1], qa[kk], b2, b3);
                }
            }
            // ---- scale + visibility (committed prefix, or the row's tree-mask bit)
            float mx0 = -CUDART_INF_F, mx1 = -CUDART_INF_F;
#pragma unroll
            for (int nt = 0; nt < WK / 8; ++nt) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int col = key0 + nt * 8 + 2 * t + (e & 1);
                    const int lr = e < 2 ? lr0 : lr1;
                    bool vis = col < nk && lr >= 0;
                    if (vis && tail) {
                        const int tt = kb + col;
                        vis = (Ms[lr * kMaskWords + (tt >> 5)] >> (tt & 31)) & 1u;
                    }
                    const float x = vis ? sc[nt][e] * p.scale_log2 : -CUDART_INF_F;
                    sc[nt][e] = x;
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
            uint32_t pa[WK / 16][4];
#pragma unroll
            for (int nt = 0; nt < WK / 8; ++nt) {
                const float p0 = m0 == -CUDART_INF_F ? 0.f : exp2f(sc[nt][0] - m0);
                const float p1 = m0 == -CUDART_INF_F ? 0.f : exp2f(sc[nt][1] - m0);
                const float p2 = m1 == -CUDART_INF_F ? 0.f : exp2f(sc[nt][2] - m1);
                const float p3 = m1 == -CUDART_INF_F ? 0.f : exp2f(sc[nt][3] - m1);
                l0 += p0 + p1;
                l1 += p2 + p3;
                const int j = nt >> 1;
                if ((nt & 1) == 0) {
                    pa[j][0] = pack2(p0, p1);
                    pa[j][1] = pack2(p2, p3);
                } else {
                    pa[j][2] = pack2(p0, p1);
                    pa[j][3] = pack2(p2, p3);
                }
            }
            // ---- O += P V
#pragma unroll
            for (int j = 0; j < WK / 16; ++j) {
#pragma unroll
                for (int nd = 0; nd < NT; nd += 2) {
                    const int key = key0 + 16 * j + (mi & 1) * 8 + r8;
                    const int dim = (nd + (mi >> 1)) * 8;
                    uint32_t b0, b1, b2, b3;
                    ldsm4t(b0, b1, b2, b3, vbase + swz_off<HD>(key, dim));
                    mma16816t(o[nd], pa[j], b0, b1);
                    mma16816t(o[nd + 1], pa[j], b2, b3);
                }
            }
        }
        if (zfix) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // zeros before the next TMA write
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (warp == 0) {  // refill the stage once every warp released it
            if (lane == 0 && i + STAGES < ntiles) {
                mbar_wait(&empty[s], (uint32_t)((i / STAGES) & 1));
                issue(i + STAGES);
            }
            __syncwarp();  // reconverge before the next tile's warp-collective ldmatrix / mma
        }
    }
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);

    if (DEC) {
        // ---- merge the 4 warps' key slices (fixed order) over the drained ring
        __syncthreads();  // every tile consumed: the ring is free
        float* wm = reinterpret_cast<float*>(ring);
        float* wl = wm + 4 * 16;
        float* wo = wl + 4 * 16;
        if (t == 0) {
            wm[warp * 16 + g] = m0;
            wm[warp * 16 + g + 8] = m1;
            wl[warp * 16 + g] = l0;
            wl[warp * 16 + g + 8] = l1;
        }
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            *reinterpret_cast<float2*>(wo + (warp * 16 + g) * HD + n * 8 + 2 * t) = make_float2(o[n][0], o[n][1]);
            *reinterpret_cast<float2*>(wo + (warp * 16 + g + 8) * HD + n * 8 + 2 * t) = make_float2(o[n][2], o[n][3]);
        }
        __syncthreads();
        for (int c = threadIdx.x; c < 16 * HD; c += blockDim.x) {
            const int q = c / HD, e = c % HD;
            if (q >= nqv) continue;
            float M = -CUDART_INF_F;
            for (int w = 0; w < 4; ++w) M = fmaxf(M, wm[w * 16 + q]);
            float L = 0.f, O = 0.f;
            if (M != -CUDART_INF_F)
                for (int w = 0; w < 4; ++w) {
                    const float sc = exp2f(wm[w * 16 + q] - M);
                    L += wl[w * 16 + q] * sc;
                    O += wo[(w * 16 + q) * HD + e] * sc;
                }
            if (single) {
                const int row = s_row[q];
                if (row >= 0)
                    p.out[(long long)row * p.H * HD + (kvh * G + q % G) * HD + e] = __float2bfloat16_rn(L > 0.f ? O / L : 0.f);
                continue;
            }
            const long long pidx = ((long long)(grp * p.max_splits + split) * p.qv_cap + q) * p.KV + kvh;
            p.ws_o[pidx * HD + e] = O;
            if (e == 0) {
                p.ws_m[pidx] = M;
                p.ws_l[pidx] = L;
            }
        }
        if (p.counters && !single) attn_fused_combine_tma<HD>(p, grp, kvh, 0, 0, 16);
        return;
    }
    if (active) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int gqv = qv0 + wq0 + g + 8 * h;
            if (gqv >= nqv) continue;
            if (single) {
                if ((h ? lr1 : lr0) < 0) continue;  // padding row
                const float inv = (h ? l1 : l0) > 0.f ? 1.0f / (h ? l1 : l0) : 0.f;
                const int row = grp * p.rows_per_req + gqv / G;
                bf16* dst = p.out + (long long)row * p.H * HD + (kvh * G + gqv % G) * HD;
#pragma unroll
                for (int n = 0; n < NT; ++n)
                    *reinterpret_cast<__nv_bfloat162*>(dst + n * 8 + 2 * t) =
                        __floats2bfloat162_rn(o[n][2 * h] * inv, o[n][2 * h + 1] * inv);
                continue;
            }
            const long long pidx = ((long long)(grp * p.max_splits + split) * p.qv_cap + gqv) * p.KV + kvh;
            float* dst = p.ws_o + pidx * HD;
#pragma unroll
            for (int n = 0; n < NT; ++n)
                *reinterpret_cast<float2*>(dst + n * 8 + 2 * t) = make_float2(o[n][2 * h], o[n][2 * h + 1]);
            if (t == 0) {
                p.ws_m[pidx] = h ? m1 : m0;
                p.ws_l[pidx] = h ? l1 : l0;
            }
        }
    }
    if (p.counters && !single) attn_fused_combine_tma<HD>(p, grp, kvh, blockIdx.x, qv0, qv0 + QV);
}

// Fused split combine (same arithmetic and order as k_attn_combine): the last
// non-empty split CTA of a (request, KV head, q-tile) merges every split.
template <int HD>
__device__ __forceinline__ void attn_fused_combine_tma(const AttnParams& p, int grp, int kvh, int qtile, int qv_lo,
                                                       int qv_hi) {
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    const long long cidx = ((long long)grp * p.KV + kvh) * gridDim.x + qtile;
    const int n_active = split_count(p, p.g.lc[grp] + p.g.ntail[grp]);
    if (n_active <= 1 && p.direct1) return;
    if (threadIdx.x == 0) s_last = atomicAdd(p.counters + cidx, 1) == n_active - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int G = p.H / p.KV;
    const int nqv = p.rows_per_req * G;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    constexpr int DPL = HD / 32;
    for (int gqv = qv_lo + warp; gqv < min(qv_hi, nqv); gqv += nw) {
        const int row = grp * p.rows_per_req + gqv / G;
        const int head = kvh * G + gqv % G;
        if (p.rows.slot[row] < 0) continue;
        float M = -CUDART_INF_F;
        for (int sp = 0; sp < n_active; ++sp) {
            const long long pidx = ((long long)(grp * p.max_splits + sp) * p.qv_cap + gqv) * p.KV + kvh;
            M = fmaxf(M, __ldcg(p.ws_m + pidx));
        }
        float L = 0.f, o[DPL];
#pragma unroll
        for (int e = 0; e < DPL; ++e) o[e] = 0.f;
        for (int sp = 0; sp < n_active; ++sp) {
            const long long pidx = ((long long)(grp * p.max_splits + sp) * p.qv_cap + gqv) * p.KV + kvh;
            const float ms = __ldcg(p.ws_m + pidx);
            if (ms == -CUDART_INF_F) continue;
            const float w = exp2f(ms - M);
            L += __ldcg(p.ws_l + pidx) * w;
#pragma unroll
            for (int e = 0; e < DPL; ++e) o[e] += __ldcg(p.ws_o + pidx * HD + lane * DPL + e) * w;
        }
        const float inv = L > 0.f ? 1.0f / L : 0.f;
#pragma unroll
        for (int e = 0; e < DPL; ++e)
            p.out[(long long)row * p.H * HD + head * HD + lane * DPL + e] = __float2bfloat16_rn(o[e] * inv);
    }
    if (threadIdx.x == 0) p.counters[cidx] = 0;  // ready for the next launch / graph replay
}

// 2D view of one layer's cache [slots * KV * cap rows][hd] bf16, 64 x 64 boxes, 128B swizzle.
CUtensorMap make_tmap_kv(const void* base, long long rows, int hd) {
    return make_tmap_bf16(base, (int)rows, hd, hd, 64);
}

template <int HD, bool DEC, int STAGES, int SUBK>
static void launch_tma_t(const CUtensorMap& tk, const CUtensorMap& tv, const AttnParams& p, cudaStream_t st) {
    constexpr int TILE_B = kTK * HD * 2;
    constexpr int kRows = DEC ? 16 : 34;
    const size_t smem = 1024 + (size_t)STAGES * 2 * TILE_B + sizeof(uint32_t) * kRows * kMaskWords;
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(k_attention_tma<HD, DEC, STAGES, SUBK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
        attr = true;
    }
    const int G = p.H / p.KV;
    const int nqv = p.rows_per_req * G;
    constexpr int QV = DEC ? 16 : 64;
    dim3 grid((nqv + QV - 1) / QV, p.KV, p.n_groups * p.max_splits);
    launch_pdl(k_attention_tma<HD, DEC, STAGES, SUBK>, grid, 128, smem, st, tk, tv, p);
}

// TMA attention for a plan from attention_plan_splits (dec: <= 16 query
// vectors per (request, KV head); otherwise the 64-vector tree tiling),
// followed by the split combine unless it is fused or every request is
// served by a single split.
void launch_attention_tma(const CUtensorMap& tk, const CUtensorMap& tv, const AttnParams& p, cudaStream_t st) {
    if (p.hd != 128 && p.hd != 64) throw CudaError("attention (TMA): head_dim must be 64 or 128");
    static const int tree_v = [] {  // TREE variant: 0 = 3 stages x 64-key chunks (2 CTAs/SM), 1 = 2 stages x 32 (3/SM)
        const char* v = std::getenv("TLT_ATTN_TMA_TREE");
        return v ? std::atoi(v) : 0;
    }();
    if (p.dec) {
        if (p.hd == 128)
            launch_tma_t<128, true, 3, 16>(tk, tv, p, st);
        else
            launch_tma_t<64, true, 3, 16>(tk, tv, p, st);
    } else if (tree_v == 1) {
        if (p.hd == 128)
            launch_tma_t<128, false, 2, 32>(tk, tv, p, st);
        else
            launch_tma_t<64, false, 2, 32>(tk, tv, p, st);
    } else {
        if (p.hd == 128)
            launch_tma_t<128, false, 3, 64>(tk, tv, p, st);
        else
            launch_tma_t<64, false, 3, 64>(tk, tv, p, st);
    }
    if (p.counters || p.max_splits == 1) return;
    launch_attn_combine_only(p, st);
}

bool attention_tma_enabled(const AttnParams& p) {
    const char* v = std::getenv("TLT_ATTN_TMA");
    if (v && std::atoi(v) == 0) return false;
    return p.impl == 1 && (p.hd == 128 || p.hd == 64) && (p.dec || p.dyn_splits > 0) && p.H / p.KV >= 2;
}

}  // namespace tlt
