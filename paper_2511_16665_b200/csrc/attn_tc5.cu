// Tree-masked attention on tcgen05 / TMEM with TMA-fed K/V (sm_100a), for the
// multi-row forwards (tree verify, drafter levels): S = Q K^T and O += P V run
// on the 5th-gen tensor cores, S and O live in TMEM, and the three roles of a
// CTA are warp-specialised:
//   warp 5      TMA producer: 64-key x 64-dim boxes (128-byte swizzle) of the
//               layer's [slots * KV * cap][hd] K and V views into a 3-stage
//               mbarrier ring (prefix tiles from key k0, then tree-tail tiles
//               from cache row tail0 — same tile runs as attn_tma.cu);
//   warp 4      MMA issuer (one elected thread): S_i = Q K_i^T (M = 128 query
//               vectors, N = 64 keys, K = 128 dims) into a double-buffered TMEM
//               S, then O += P_{i-1} V_{i-1} (N = 128 dims, K = 64 keys, V as
//               the MN-major operand), so the tensor core computes S_{i+1}
//               while the softmax warps work on S_i;
//   warps 0-3   softmax: thread = query vector = TMEM lane; reads its 64 scores
//               (tcgen05.ld), applies the committed-prefix / tree-mask
//               visibility, keeps an online max with LAZY rescaling (O in TMEM
//               is rescaled, by tcgen05.ld / st, only when a row's max grows by
//               more than 2^8 — exact: P and l are always relative to the max
//               actually used), writes P (bf16, swizzled K-major) to a double-
//               buffered smem tile, zeroes the V rows past the tile's valid
//               keys (stale cache rows may hold NaN: 0 * NaN = NaN), and at the
//               end writes the normalised output or the split partial.
// Splits, partial layout and the combine are those of attn_tma.cu.
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

namespace {
using bf16 = __nv_bfloat16;
constexpr int kQ5 = 128;      // query vectors per CTA (TMEM lanes, MMA M)
constexpr int kK5 = 64;       // keys per tile
constexpr int kHD5 = 128;     // head dim
constexpr int kSt5 = 3;       // K/V ring stages
constexpr int kRows5 = kQ5 / 2 + 2;
constexpr int kTileB5 = kK5 * kHD5 * 2;  // one K (or V) tile: 16 KB = 2 halves of 64 rows x 128 B
constexpr float kRescale = 8.0f;         // log2 growth that forces an O rescale

__device__ __forceinline__ uint32_t sw128_5(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }
__device__ __forceinline__ uint64_t desc_k5(uint32_t saddr) {  // SW128 K-major, SBO 1 KB
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= 1ull << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= 1ull << 46;
    d |= 2ull << 61;
    return d;
}
__device__ __forceinline__ uint64_t desc_mn5(uint32_t saddr, uint32_t lbo) {  // SW128 MN-major
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= 1ull << 46;
    d |= 2ull << 61;
    return d;
}
__host__ __device__ constexpr uint32_t idesc5(uint32_t M, uint32_t N, uint32_t b_mn_major) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (b_mn_major << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ void cp_async16_5(uint32_t saddr, const void* gmem, bool pred) {
    const int sz = pred ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem), "r"(sz));
}
}  // namespace

__global__ void __launch_bounds__(192, 1)
    k_attention_tree_tc(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, AttnParams p) {
    pdl_wait_only();  // dependents are released after the TMEM allocation below
    extern __shared__ __align__(1024) uint8_t smem5[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem5) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = sm;                                   // [2 halves][128 rows][128 B]      32 KB
    uint8_t* ring = sQ + 2 * kQ5 * 128;                 // [stage][K 16 KB | V 16 KB]       96 KB
    uint8_t* sP = ring + kSt5 * 2 * kTileB5;            // [2][128 rows][128 B]             32 KB
    uint32_t* Ms = reinterpret_cast<uint32_t*>(sP + 2 * kQ5 * 128);  // [kRows5][kMaskWords]
    __shared__ uint64_t full[kSt5], empty[kSt5], sfull[2], sfree[2], pready[2], pvdone[2];
    __shared__ uint32_t tmem_holder;
    __shared__ int s_lrow[kQ5];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = p.H / p.KV;
    const int kvh = blockIdx.y;
    const int grp = blockIdx.z / p.max_splits;
    const int split = blockIdx.z % p.max_splits;
    const int qv0 = blockIdx.x * kQ5;
    const int nqv = p.rows_per_req * G;
    const int slot = p.g.slot[grp];
    const int lc = p.g.lc[grp], tail0 = p.g.tail0[grp], ntail = p.g.ntail[grp];
    const int total = slot >= 0 ? lc + ntail : 0;
    const int chunk = split_chunk(p, total);
    const int k0 = split * chunk;
    if (k0 >= total) return;  // exited CTAs count as having released the dependents
    const int k1 = min(total, k0 + chunk);
    const bool single = p.max_splits == 1 || (p.direct1 && split_count(p, total) == 1);
    const int pe = min(k1, lc);
    const int n_pt = pe > k0 ? (pe - k0 + kK5 - 1) / kK5 : 0;
    const int ta = max(k0, lc) - lc, te = k1 - lc;
    const int n_tt = te > ta ? (te - ta + kK5 - 1) / kK5 : 0;
    const int ntiles = n_pt + n_tt;
    const long long head_row = ((long long)slot * p.KV + kvh) * p.cap;
    const int row_base = qv0 / G;

    // ---- setup: barriers, TMEM (S0 | S1 | O = 256 columns), Q rows, masks
    if (threadIdx.x == 0) {
        for (int s = 0; s < kSt5; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&sfull[b], 1);
            mbar_init(&sfree[b], kQ5);
            mbar_init(&pready[b], kQ5);
            mbar_init(&pvdone[b], 1);
        }
        fence_barrier_init();
    }
    if (warp == 4) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                         smem_u32(&tmem_holder))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x < kQ5) {
        const int gqv = qv0 + threadIdx.x;
        int lr = -1;
        if (gqv < nqv) {
            const int row = grp * p.rows_per_req + gqv / G;
            if (p.rows.slot[row] >= 0) lr = gqv / G - row_base;
        }
        s_lrow[threadIdx.x] = lr;
        // this query vector's 256-byte row -> two swizzled 128-byte halves (zero for padding)
        const int row = lr >= 0 ? grp * p.rows_per_req + gqv / G : 0;
        const int head = kvh * G + gqv % G;
        const bf16* src = p.q + (long long)row * p.H * kHD5 + head * kHD5;
#pragma unroll
        for (int w = 0; w < 16; ++w)
            cp_async16_5(smem_u32(sQ) + (uint32_t)((w >> 3) * kQ5 * 128) + sw128_5(threadIdx.x, w & 7), src + w * 8,
                         lr >= 0);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    const int nrows = min(kRows5, p.rows_per_req - row_base);
    const int mw = (ntail + 31) >> 5;
    for (int c = threadIdx.x; c < nrows * kMaskWords; c += blockDim.x) {
        const int l = c / kMaskWords, w = c % kMaskWords;
        Ms[c] = w < mw ? p.rows.mask[(long long)(grp * p.rows_per_req + row_base + l) * kMaskWords + w] : 0u;
    }
    if (threadIdx.x < kQ5) asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // Q (generic writes) -> tensor core
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_launch_dependents();  // this CTA holds its TMEM: dependents may start allocating theirs
    const uint32_t tmem = tmem_holder;
    const uint32_t tS[2] = {tmem, tmem + 64}, tO = tmem + 128;
    const uint32_t aQ = smem_u32(sQ), aRing = smem_u32(ring), aP = smem_u32(sP);

    if (warp == 5) {
        // ---------------- TMA producer
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            for (int i = 0; i < ntiles; ++i) {
                const int s = i % kSt5;
                if (i >= kSt5) mbar_wait(&empty[s], (uint32_t)(((i / kSt5) - 1) & 1));
                const long long row = i < n_pt ? head_row + k0 + (long long)i * kK5
                                               : head_row + tail0 + ta + (long long)(i - n_pt) * kK5;
                uint8_t* kd = ring + s * 2 * kTileB5;
                mbar_arrive_expect_tx(&full[s], 2 * kTileB5);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    tma_load_2d(kd + h * (kK5 * 128), &tmK, &full[s], h * 64, (int)row, pol);
                    tma_load_2d(kd + kTileB5 + h * (kK5 * 128), &tmV, &full[s], h * 64, (int)row, pol);
                }
            }
        }
    } else if (warp == 4) {
        // ---------------- MMA issuer
        const uint32_t idS = idesc5(128, 64, 0), idO = idesc5(128, 128, 1);
        auto issue_pv = [&](int j) {  // O += P_j V_j, then release P_j's buffer and K/V stage j
            mbar_wait(&pready[j & 1], (uint32_t)((j >> 1) & 1));
            tc_fence_after();
            if (elect_one()) {
                const uint32_t aV = aRing + (j % kSt5) * 2 * kTileB5 + kTileB5;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    tc_mma_bf16(tO, desc_k5(aP + (j & 1) * kQ5 * 128 + kk * 32), desc_mn5(aV + kk * 16 * 128, kK5 * 128),
                                idO, (j | kk) != 0);
                tc_commit(&pvdone[j & 1]);
                tc_commit(&empty[j % kSt5]);
            }
            __syncwarp();
        };
        for (int i = 0; i < ntiles; ++i) {
            const int s = i % kSt5;
            mbar_wait(&full[s], (uint32_t)((i / kSt5) & 1));
            if (i >= 2) mbar_wait(&sfree[i & 1], (uint32_t)(((i - 2) >> 1) & 1));
            tc_fence_after();
            if (elect_one()) {
                const uint32_t aK = aRing + s * 2 * kTileB5;
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        tc_mma_bf16(tS[i & 1], desc_k5(aQ + h * kQ5 * 128 + kk * 32),
                                    desc_k5(aK + h * (kK5 * 128) + kk * 32), idS, (h | kk) != 0);
                tc_commit(&sfull[i & 1]);
            }
            __syncwarp();
            if (i >= 1) issue_pv(i - 1);
        }
        if (ntiles > 0) issue_pv(ntiles - 1);
    } else {
        // ---------------- softmax warps: thread = query vector = TMEM lane
        const int l = warp * 32 + lane;
        const int lr = s_lrow[l];
        const uint32_t trow = (uint32_t)(warp * 32) << 16;
        float m = -CUDART_INF_F, lsum = 0.f;
        for (int i = 0; i < ntiles; ++i) {
            const bool tail = i >= n_pt;
            const int kb = tail ? ta + (i - n_pt) * kK5 : k0 + i * kK5;
            const int nk = tail ? min(kK5, te - kb) : min(kK5, pe - kb);
            mbar_wait(&sfull[i & 1], (uint32_t)((i >> 1) & 1));
            tc_fence_after();
            uint32_t r[4][16];
#pragma unroll
            for (int u = 0; u < 4; ++u) tmem_ld16_nowait(tS[i & 1] + trow + 16 * u, r[u]);
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(&sfree[i & 1]);  // S buffer may be overwritten by S_{i+2}
            // visibility as one 64-bit mask per row (valid keys of the tile, and for
            // tree-tail tiles the row's mask bits kb .. kb+63), then scale; NaN-safe:
            // invisible scores never enter the max or P
            uint64_t vis = lr < 0 ? 0ull : (nk >= 64 ? ~0ull : ((1ull << nk) - 1ull));
            if (tail && vis) {
                const uint32_t* mr = Ms + lr * kMaskWords;
                const int w0 = kb >> 5, sh = kb & 31;
                const uint32_t a0 = mr[w0], a1 = w0 + 1 < kMaskWords ? mr[w0 + 1] : 0u,
                               a2 = w0 + 2 < kMaskWords ? mr[w0 + 2] : 0u;
                const uint64_t lo = ((uint64_t)a1 << 32) | a0, hi = a2;
                vis &= sh ? ((lo >> sh) | (hi << (64 - sh))) : lo;
            }
            float x[64];
            float mt = -CUDART_INF_F;
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int col = 16 * u + j;
                    x[col] = ((vis >> col) & 1ull) ? __uint_as_float(r[u][j]) * p.scale_log2 : -CUDART_INF_F;
                    mt = fmaxf(mt, x[col]);
                }
            // lazy rescale: move the max only when it grows by > 2^8 (or from -inf)
            const bool grow = mt > -CUDART_INF_F && (m == -CUDART_INF_F || mt > m + kRescale);
            const float m_new = grow ? mt : m;
            if (__any_sync(0xffffffffu, grow && m != -CUDART_INF_F && i > 0)) {
                // O holds sum_{j < i} P_j V_j: wait for PV_{i-1}, then scale this warp's rows
                mbar_wait(&pvdone[(i - 1) & 1], (uint32_t)(((i - 1) >> 1) & 1));
                tc_fence_after();
                const float f = (grow && m != -CUDART_INF_F) ? exp2f(m - m_new) : 1.f;
#pragma unroll
                for (int c = 0; c < kHD5; c += 64) {
                    uint32_t o[4][16];
#pragma unroll
                    for (int u = 0; u < 4; ++u) tmem_ld16_nowait(tO + trow + c + 16 * u, o[u]);
                    tmem_ld_wait();
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
#pragma unroll
                        for (int j = 0; j < 16; ++j) o[u][j] = __float_as_uint(__uint_as_float(o[u][j]) * f);
                        tmem_st16(tO + trow + c + 16 * u, o[u]);
                    }
                }
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                lsum *= f;
            }
            m = m_new;
            // P (bf16) for this row, relative to the max in use
            // ex2(-inf) = +0 for invisible keys; a row with no visible key so far
            // (m = -inf) contributes nothing
            uint32_t pk[32];
            const float mm = m == -CUDART_INF_F ? CUDART_INF_F : m;
#pragma unroll
            for (int j = 0; j < 64; j += 2) {
                const float p0 = ex2_approx(x[j] - mm);
                const float p1 = ex2_approx(x[j + 1] - mm);
                lsum += p0 + p1;
                __nv_bfloat162 h = __floats2bfloat162_rn(p0, p1);
                pk[j >> 1] = *reinterpret_cast<uint32_t*>(&h);
            }
            if (i >= 2) mbar_wait(&pvdone[i & 1], (uint32_t)(((i - 2) >> 1) & 1));  // PV_{i-2} read this P buffer
            uint8_t* prow = sP + (i & 1) * kQ5 * 128;
#pragma unroll
            for (int c = 0; c < 8; ++c)
                *reinterpret_cast<uint4*>(prow + sw128_5(l, c)) = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2],
                                                                             pk[4 * c + 3]);
            if (nk < kK5) {  // V rows past the tile's valid keys: zero (stale cache rows may hold NaN)
                uint4* vz = reinterpret_cast<uint4*>(ring + (i % kSt5) * 2 * kTileB5 + kTileB5);
                for (int c = l; c < (kK5 - nk) * 16; c += kQ5) {
                    const int rr = nk + (c >> 4), rem = c & 15;
                    vz[((rem >> 3) * (kK5 * 128) + rr * 128 + (rem & 7) * 16) >> 4] = make_uint4(0u, 0u, 0u, 0u);
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // P / zeros -> tensor core
            tc_fence_before();
            mbar_arrive(&pready[i & 1]);
        }
        // ---- epilogue: wait for the last PV, read this row's O
        if (ntiles > 0) mbar_wait(&pvdone[(ntiles - 1) & 1], (uint32_t)(((ntiles - 1) >> 1) & 1));
        tc_fence_after();
        const int gqv = qv0 + l;
        const bool wr = lr >= 0 && gqv < nqv;
        const int row = grp * p.rows_per_req + gqv / G, head = kvh * G + gqv % G;
        const long long pidx = ((long long)(grp * p.max_splits + split) * p.qv_cap + (wr ? gqv : 0)) * p.KV + kvh;
        const float inv = lsum > 0.f ? 1.0f / lsum : 0.f;
#pragma unroll
        for (int c = 0; c < kHD5; c += 64) {
            uint32_t o[4][16];
#pragma unroll
            for (int u = 0; u < 4; ++u) tmem_ld16_nowait(tO + trow + c + 16 * u, o[u]);
            tmem_ld_wait();
            if (!wr) continue;
            if (single) {
                bf16* dst = p.out + (long long)row * p.H * kHD5 + head * kHD5 + c;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    uint4 pk4[2];
                    uint32_t* w = reinterpret_cast<uint32_t*>(pk4);
#pragma unroll
                    for (int j = 0; j < 16; j += 2) {
                        __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(o[u][j]) * inv,
                                                                 __uint_as_float(o[u][j + 1]) * inv);
                        w[j >> 1] = *reinterpret_cast<uint32_t*>(&h);
                    }
                    *reinterpret_cast<uint4*>(dst + 16 * u) = pk4[0];
                    *reinterpret_cast<uint4*>(dst + 16 * u + 8) = pk4[1];
                }
            } else {
                float* dst = p.ws_o + pidx * kHD5 + c;
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int j = 0; j < 16; j += 4)
                        *reinterpret_cast<float4*>(dst + 16 * u + j) =
                            make_float4(__uint_as_float(o[u][j]), __uint_as_float(o[u][j + 1]),
                                        __uint_as_float(o[u][j + 2]), __uint_as_float(o[u][j + 3]));
            }
        }
        if (wr && !single) {
            p.ws_m[pidx] = m;
            p.ws_l[pidx] = lsum;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 4)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

bool attention_tree_tc_eligible(const AttnParams& p) {
    // default on for every hd = 128 multi-row forward: with the 64-bit
    // visibility mask + ex2.approx softmax it beats the mma.sync TMA kernel at
    // every verify / drafter shape measured (profiles/r2_probe_tree_{tma2,tc2}.txt:
    // b = 31 T = 16 46.9 -> 20.7 us, ctx 2000 117.7 -> 40.8 us, b = 5 T = 48
    // 32.9 -> 22.1 us, b = 1 T = 64 20.6 -> 19.8 us); TLT_ATTN_TREE_TC=0 off
    const char* v = std::getenv("TLT_ATTN_TREE_TC");
    if (v && std::atoi(v) == 0) return false;
    return p.hd == kHD5 && !p.dec && p.dyn_splits > 0 && p.H / p.KV >= 2;
}

void launch_attention_tree_tc(const CUtensorMap& tk, const CUtensorMap& tv, const AttnParams& p, cudaStream_t st) {
    const size_t smem = 1024 + 2 * kQ5 * 128 + (size_t)kSt5 * 2 * kTileB5 + 2 * kQ5 * 128 +
                        sizeof(uint32_t) * kRows5 * kMaskWords;
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(k_attention_tree_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    const int G = p.H / p.KV;
    const int nqv = p.rows_per_req * G;
    dim3 grid((nqv + kQ5 - 1) / kQ5, p.KV, p.n_groups * p.max_splits);
    launch_pdl(k_attention_tree_tc, grid, 192, smem, st, tk, tv, p);
    if (p.max_splits > 1) launch_attn_combine_only(p, st);
}

}  // namespace tlt
