// Tree-masked attention on the 5th-gen tensor cores (tcgen05 + TMEM) for the
// multi-row forwards (tree verify, drafter levels, prefill chunks).
//
// CTA = (128 query vectors, KV head, request group, 256-key split) — the same
// split alignment and (m, l, O) partial layout as the mma.sync kernels, so
// k_attn_combine merges the splits. Per CTA, with S and O in TMEM:
//   1. Q [128 x 128], K [256 x 128], V [256 x 128] bf16 staged in smem in the
//      128B-swizzled UMMA layouts (cp.async, the tail-key index remap applied
//      per 16-byte chunk);
//   2. S = Q K^T: 8 x tcgen05.mma M=128 N=256 K=16 into TMEM columns [0, 256);
//   3. softmax by the 4 warps, thread = query row (its 256 scores read with
//      tcgen05.ld): scale, committed-prefix / tree-mask visibility, row max,
//      p = exp2(x - m) -> bf16 P written in the swizzled K-major layout over
//      the (consumed) K tile, l = sum p. Two passes over the split's 256
//      scores, so no online rescaling of O is needed;
//   4. O = P V: 16 x tcgen05.mma M=128 N=128 K=16 with V as an MN-major B
//      operand (dims contiguous), TMEM columns [256, 384);
//   5. each thread writes its row's (m, l, O) partial.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdlib>

#include "engine_kernels.h"
#include "kernels.cuh"
#include "pdl.cuh"
#include "ptx.cuh"

namespace tlt {

namespace {
using bf16 = __nv_bfloat16;
constexpr int kQ = 128;     // query vectors per CTA (TMEM lanes / MMA M)
constexpr int kKeys = 256;  // keys per split (= attention_mma_split())
constexpr int kHDt = 128;   // head dim
constexpr int kRows = kQ / 2 + 2;

__device__ __forceinline__ void cp_async16_tc(uint32_t saddr, const void* gmem, bool pred) {
    const int sz = pred ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem), "r"(sz));
}
// byte offset of 16-byte chunk c (0..7) of row r inside a 128B-swizzled
// [rows x 128 B] block (1 KB atoms of 8 rows, 16 B granules XOR row % 8)
__device__ __forceinline__ uint32_t sw128(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }

// SW128 descriptor, K-major (SBO = 1 KB per 8 rows)
__device__ __forceinline__ uint64_t desc_k(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= 1ull << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= 1ull << 46;
    d |= 2ull << 61;
    return d;
}
// SW128 descriptor, MN-major: 64-element MN groups LBO bytes apart, 8-row K
// groups SBO = 1 KB apart (canonical ((8,8,m),(8,k)):((1,8,LBO),(64,SBO)))
__device__ __forceinline__ uint64_t desc_mn(uint32_t saddr, uint32_t lbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= 1ull << 46;
    d |= 2ull << 61;
    return d;
}
__device__ __forceinline__ float ex2_fast(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__host__ __device__ constexpr uint32_t idesc_tc(uint32_t M, uint32_t N, uint32_t b_mn_major) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (b_mn_major << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
}  // namespace

__global__ void __launch_bounds__(256, 1) k_attention_tc(AttnParams p, int dbg_stage) {
    pdl_wait_only();  // dependents are released after the TMEM allocation (pdl.cuh)
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    // layout: Q 2 x 16 KB | K (later P) 64 KB | V 64 KB | masks | barriers
    uint8_t* sQ = sm;                       // [2 dim blocks][128 rows][128 B]
    uint8_t* sK = sm + 32768;               // [2 dim blocks][256 keys][128 B]; P: [4 key blocks][128 rows][128 B]
    uint8_t* sV = sm + 32768 + 65536;       // [2 dim blocks][256 keys][128 B]
    uint32_t* Ms = reinterpret_cast<uint32_t*>(sm + 32768 + 2 * 65536);  // [kRows][kMaskWords]
    uint64_t* bars = reinterpret_cast<uint64_t*>(Ms + kRows * kMaskWords);  // s_full, o_full
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2);
    __shared__ int s_lrow[kQ];
    __shared__ float s_part[2][kQ];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = p.H / p.KV;
    const int kvh = blockIdx.y;
    const int grp = blockIdx.z / p.max_splits;
    const int split = blockIdx.z % p.max_splits;
    const int qv0 = blockIdx.x * kQ;
    const int nqv = p.rows_per_req * G;
    const int slot = p.g.slot[grp];
    const int lc = p.g.lc[grp], tail0 = p.g.tail0[grp], ntail = p.g.ntail[grp];
    const int total = slot >= 0 ? lc + ntail : 0;
    const int k0 = split * kKeys;
    if (k0 >= total) return;  // empty split
    const int k1 = min(total, k0 + kKeys);
    const int row_base = qv0 / G;

    // ---- 1. stage K, V (tail remap per key), Q, masks
    const long long slot_base = ((long long)slot * p.KV + kvh) * p.cap;
    const uint32_t aK = smem_u32(sK), aV = smem_u32(sV), aQ = smem_u32(sQ);
    for (int c = threadIdx.x; c < kKeys * 16; c += 256) {
        const int j = c >> 4, w = c & 15;  // key j, 16-byte chunk w of its 256-byte row
        const int v = k0 + j;
        const bool ok = v < k1;
        const long long ci = ok ? (v < lc ? v : tail0 + (v - lc)) : 0;
        const long long off = (slot_base + ci) * kHDt + w * 8;
        const uint32_t dst = (uint32_t)((w >> 3) * kKeys * 128) + sw128(j, w & 7);
        cp_async16_tc(aK + dst, p.kc + off, ok);
    }
    if (threadIdx.x < kQ) {
        const int gqv = qv0 + threadIdx.x;
        int lr = -1;
        if (gqv < nqv) {
            const int row = grp * p.rows_per_req + gqv / G;
            if (p.rows.slot[row] >= 0) lr = gqv / G - row_base;
        }
        s_lrow[threadIdx.x] = lr;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < kQ * 16; c += 256) {
        const int l = c >> 4, w = c & 15;
        const bool ok = s_lrow[l] >= 0;
        const int gqv = qv0 + l;
        const int row = ok ? grp * p.rows_per_req + gqv / G : 0;
        const int head = kvh * G + gqv % G;
        cp_async16_tc(aQ + (uint32_t)((w >> 3) * kQ * 128) + sw128(l, w & 7),
                      p.q + (long long)row * p.H * kHDt + head * kHDt + w * 8, ok);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");  // group 0: K + Q
    for (int c = threadIdx.x; c < kKeys * 16; c += 256) {      // group 1: V (needed only after the softmax)
        const int j = c >> 4, w = c & 15;
        const int v = k0 + j;
        const bool ok = v < k1;
        const long long ci = ok ? (v < lc ? v : tail0 + (v - lc)) : 0;
        const long long off = (slot_base + ci) * kHDt + w * 8;
        cp_async16_tc(aV + (uint32_t)((w >> 3) * kKeys * 128) + sw128(j, w & 7), p.vc + off, ok);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    const int nrows = min(kRows, p.rows_per_req - row_base);
    const int mw = (ntail + 31) >> 5;
    for (int c = threadIdx.x; c < nrows * kMaskWords; c += 256) {
        const int l = c / kMaskWords, w = c % kMaskWords;
        const int row = grp * p.rows_per_req + row_base + l;
        Ms[c] = w < mw ? p.rows.mask[(long long)row * kMaskWords + w] : 0u;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         smem_u32(tmem_holder))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_barrier_init();
    }
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // K + Q landed (V may still be in flight)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // cp.async writes -> tensor-core reads
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_launch_dependents();
    const uint32_t tmem = *tmem_holder;
    const uint32_t tS = tmem, tO = tmem + 256;
    if (dbg_stage == 1) { tc_fence_before(); __syncthreads(); if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory"); return; }

    // ---- 2. S = Q K^T (M = 128 qv, N = 256 keys, K = 128 dims)
    if (warp == 0) {
        if (elect_one()) {
            const uint32_t id = idesc_tc(128, 256, 0);
#pragma unroll
            for (int kb = 0; kb < 2; ++kb)
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    tc_mma_bf16(tS, desc_k(aQ + kb * kQ * 128 + kk * 32), desc_k(aK + kb * kKeys * 128 + kk * 32),
                                id, (kb | kk) != 0);
            tc_commit(&bars[0]);
        }
        __syncwarp();
    }
    mbar_wait(&bars[0], 0);
    tc_fence_after();
    if (dbg_stage == 2) { tc_fence_before(); __syncthreads(); if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory"); return; }

    // ---- 3. softmax: 2 threads per query row l (TMEM lane): warps w and w+4
    //         share a lane quarter, each owns 128 of the 256 score columns
    const int q4 = warp & 3, hh = warp >> 2;
    const int l = q4 * 32 + lane;
    const int lr = s_lrow[l];
    const uint32_t trow = (uint32_t)(q4 * 32) << 16;
    const int cbase = hh * (kKeys / 2);
    auto visible = [&](int col) {
        const int v = k0 + col;
        if (lr < 0 || v >= k1) return false;
        if (v < lc) return true;
        const int tt = v - lc;
        return ((Ms[lr * kMaskWords + (tt >> 5)] >> (tt & 31)) & 1u) != 0;
    };
    const int vis_all = min(lc, k1);  // keys below this are visible to every valid row
    float m = -CUDART_INF_F;
    for (int c = cbase; c < cbase + kKeys / 2; c += 64) {
        uint32_t r[4][16];
#pragma unroll
        for (int u = 0; u < 4; ++u) tmem_ld16_nowait(tS + trow + c + 16 * u, r[u]);
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int cc = c + 16 * u;
            if (lr >= 0 && k0 + cc + 16 <= vis_all) {  // committed prefix: every key visible
                float mm = __uint_as_float(r[u][0]);
#pragma unroll
                for (int j = 1; j < 16; ++j) mm = fmaxf(mm, __uint_as_float(r[u][j]));
                m = fmaxf(m, mm * p.scale_log2);
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (visible(cc + j)) m = fmaxf(m, __uint_as_float(r[u][j]) * p.scale_log2);
            }
        }
    }
    s_part[hh][l] = m;
    __syncthreads();
    m = fmaxf(s_part[0][l], s_part[1][l]);
    float lsum = 0.f;
    const uint32_t aP = aK;  // P overwrites K (S MMAs complete: s_full)
    for (int c = cbase; c < cbase + kKeys / 2; c += 64) {
        uint32_t r[4][16];
#pragma unroll
        for (int u = 0; u < 4; ++u) tmem_ld16_nowait(tS + trow + c + 16 * u, r[u]);
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int cc = c + 16 * u;
            uint32_t pk[8];
            const bool all = lr >= 0 && k0 + cc + 16 <= vis_all && m != -CUDART_INF_F;
#pragma unroll
            for (int j = 0; j < 16; j += 2) {
                float p0, p1;
                if (all) {
                    p0 = ex2_fast(__uint_as_float(r[u][j]) * p.scale_log2 - m);
                    p1 = ex2_fast(__uint_as_float(r[u][j + 1]) * p.scale_log2 - m);
                } else {
                    p0 = (m != -CUDART_INF_F && visible(cc + j)) ? ex2_fast(__uint_as_float(r[u][j]) * p.scale_log2 - m)
                                                                 : 0.f;
                    p1 = (m != -CUDART_INF_F && visible(cc + j + 1))
                             ? ex2_fast(__uint_as_float(r[u][j + 1]) * p.scale_log2 - m) : 0.f;
                }
                lsum += p0 + p1;
                __nv_bfloat162 h = __floats2bfloat162_rn(p0, p1);
                pk[j >> 1] = *reinterpret_cast<uint32_t*>(&h);
            }
            // keys cc..cc+15 = key block cc/64, 16-byte chunks (cc%64)/8 and +1 of row l
            const int kb = cc >> 6, ch = (cc & 63) >> 3;
            uint8_t* base = sK + kb * kQ * 128;
            *reinterpret_cast<uint4*>(base + sw128(l, ch)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            *reinterpret_cast<uint4*>(base + sw128(l, ch + 1)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        }
    }
    __syncthreads();  // s_part reads done
    s_part[hh][l] = lsum;
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");       // V landed
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // P + V -> tensor core
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    lsum = s_part[0][l] + s_part[1][l];  // fixed order

    // ---- 4. O = P V (M = 128 qv, N = 128 dims, K = 256 keys), V MN-major
    if (warp == 0) {
        if (elect_one()) {
            const uint32_t id = idesc_tc(128, 128, 1);
#pragma unroll
            for (int kb = 0; kb < 4; ++kb)
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    tc_mma_bf16(tO, desc_k(aP + kb * kQ * 128 + kk * 32),
                                desc_mn(aV + (kb * 64 + kk * 16) * 128, kKeys * 128), id, (kb | kk) != 0);
            tc_commit(&bars[1]);
        }
        __syncwarp();
    }
    mbar_wait(&bars[1], 0);
    tc_fence_after();
    if (dbg_stage == 4) { tc_fence_before(); __syncthreads(); if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory"); return; }

    // ---- 5. this row's split partial (tcgen05.ld is warp-collective: every
    //         lane loads, only valid rows store)
    const int gqv = qv0 + l;
    const bool wr = lr >= 0 && gqv < nqv;
    const long long pidx = ((long long)(grp * p.max_splits + split) * p.qv_cap + (wr ? gqv : 0)) * p.KV + kvh;
    float* dst = p.ws_o + pidx * kHDt;
    {
        uint32_t r[4][16];
#pragma unroll
        for (int u = 0; u < 4; ++u) tmem_ld16_nowait(tO + trow + hh * 64 + 16 * u, r[u]);
        tmem_ld_wait();
        if (wr) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int j = 0; j < 16; j += 4)
                    *reinterpret_cast<float4*>(dst + hh * 64 + 16 * u + j) =
                        make_float4(__uint_as_float(r[u][j]), __uint_as_float(r[u][j + 1]),
                                    __uint_as_float(r[u][j + 2]), __uint_as_float(r[u][j + 3]));
        }
    }
    if (wr && hh == 0) {
        p.ws_m[pidx] = m;
        p.ws_l[pidx] = lsum;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

size_t attention_tc_smem() { return 1024 + 32768 + 2 * 65536 + kRows * kMaskWords * 4 + 64; }

bool attention_tc_shape_ok(const AttnParams& p) {
    const int G = p.H / p.KV;
    return p.hd == kHDt && G >= 2 && p.rows_per_req > 1 && p.rows_per_req * G > 16 && !p.dec && p.chunk == kKeys;
}

bool attention_tc_eligible(const AttnParams& p) {
    static const int on = [] {
        // off by default: correct (tests/test_gpu_attention.py) but measured
        // 1.05-1.3x slower than the mma.sync tree kernel at the verify and
        // prefill shapes (serial stage/MMA/softmax phases, 1 CTA per SM)
        const char* v = std::getenv("TLT_ATTN_TC");
        return v ? std::atoi(v) : 0;
    }();
    return on && attention_tc_shape_ok(p);
}

void launch_attention_tc(const AttnParams& p, cudaStream_t st) {
    static bool attr = false;
    const size_t smem = attention_tc_smem();
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(k_attention_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    const int G = p.H / p.KV;
    const int nqv = p.rows_per_req * G;
    dim3 grid((nqv + kQ - 1) / kQ, p.KV, p.n_groups * p.max_splits);
    static const int dbg = [] {
        const char* v = std::getenv("TLT_ATTN_TC_DBG");
        return v ? std::atoi(v) : 0;
    }();
    launch_pdl(k_attention_tc, grid, 256, smem, st, p, dbg);
}

}  // namespace tlt
