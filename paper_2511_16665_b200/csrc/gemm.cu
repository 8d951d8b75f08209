// tcgen05 swap-AB GEMM kernel + split-K reduce + host-side planner/launcher.
// See gemm.cuh for the operand mapping and the fused epilogues.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cooperative_groups.h>
#include <math_constants.h>

#include <algorithm>
#include <cstdio>
#include <mutex>
#include <stdexcept>
#include <string>

#include "gemm.cuh"
#include "ptx.cuh"
#include "pdl.cuh"
#include "tlt_internal.h"

namespace tlt {

constexpr int kBlockM = 128;  // weight rows per tile (MMA M)
constexpr int kBlockK = 64;   // 64 bf16 = one 128-byte swizzle row
constexpr int kABytes = kBlockM * kBlockK * 2;
constexpr int kMaxSplits = 16;  // split-K cluster size (> 8 needs the non-portable cluster attribute)
constexpr int kPeerBatch = 8;   // peers whose partials are loaded together in the DSMEM reduction

// LM-head epilogue (EPI_TOPK) for one 128-vocab x bn-token accumulator tile.
// Per 16-token chunk the 4 epilogue warps transpose the accumulators through
// shared memory; then 8 threads per token scan 16 vocab rows each (local max,
// sum-exp, sorted top-K by (logit desc, id asc)) and merge with a 3-step
// butterfly inside the warp. The merge is symmetric (commutative adds, strict
// total order), so all 8 lanes hold identical results and the output is
// deterministic. One partial (M, S, K values, K ids) per (tile, token).
template <int KM>
__device__ __forceinline__ void topk_insert(float (&v)[KM], int (&id)[KM], float x, int ix) {
    if (!(x > v[KM - 1] || (x == v[KM - 1] && ix < id[KM - 1]))) return;
    // branch-free insertion with static indices only (keeps the list in registers)
    bool placed = false;
#pragma unroll
    for (int s = KM - 1; s > 0; --s) {
        const bool shift = !placed && (x > v[s - 1] || (x == v[s - 1] && ix < id[s - 1]));
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

template <int KM>
__device__ __forceinline__ void epi_topk_tile(const EpiParams& ep, uint32_t tmem, int q, int lane, int n0, int t0,
                                              int bn, float* tr, int tile) {
    const int K = ep.topk_k;
    const int W = 2 + 2 * K;
    const int ep_tid = threadIdx.x - 64;  // 0..127
    const int col = ep_tid >> 3, part = ep_tid & 7;
    for (int c = 0; c < bn; c += 16) {
        if (t0 + c >= ep.m_tok) break;
        float v[16];
        tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + c, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) tr[j * 128 + q * 32 + lane] = v[j];
        asm volatile("bar.sync 1, 128;" ::: "memory");
        float m = -CUDART_INF_F, s = 0.f;
        float lv[KM];
        int li[KM];
#pragma unroll
        for (int r = 0; r < KM; ++r) {
            lv[r] = -CUDART_INF_F;
            li[r] = 0x7fffffff;
        }
        const float* src = tr + col * 128 + part * 16;
        float xs[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int id = n0 + part * 16 + i;
            xs[i] = id < ep.n_out ? src[i] : -CUDART_INF_F;
            m = fmaxf(m, xs[i]);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (xs[i] != -CUDART_INF_F) s += __expf(xs[i] - m);
            topk_insert<KM>(lv, li, xs[i], n0 + part * 16 + i);
        }
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const float om = __shfl_xor_sync(0xffffffffu, m, o);
            const float os = __shfl_xor_sync(0xffffffffu, s, o);
            const float nm = fmaxf(m, om);
            const float a = m == -CUDART_INF_F ? 0.f : s * __expf(m - nm);
            const float b = om == -CUDART_INF_F ? 0.f : os * __expf(om - nm);
            s = a + b;
            m = nm;
            float ov[KM];
            int oi[KM];
#pragma unroll
            for (int r = 0; r < KM; ++r) {
                ov[r] = __shfl_xor_sync(0xffffffffu, lv[r], o);
                oi[r] = __shfl_xor_sync(0xffffffffu, li[r], o);
            }
#pragma unroll
            for (int r = 0; r < KM; ++r) topk_insert<KM>(lv, li, ov[r], oi[r]);
        }
        const int tok = t0 + c + col;
        if (part == 0 && tok < ep.m_tok) {
            float* out = ep.out_f32 + ((long long)tile * ep.m_tok + tok) * W;
            out[0] = m;
            out[1] = s;
#pragma unroll
            for (int r = 0; r < KM; ++r) {  // static indices: lv/li stay in registers
                if (r < K) {
                    out[2 + r] = lv[r];
                    out[2 + K + r] = __int_as_float(li[r]);
                }
            }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
    }
}

// order-preserving float <-> uint (x < y  <=>  ord(x) < ord(y); ord > 0)
__device__ __forceinline__ unsigned float_to_ord(float f) {
    const unsigned u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord_to_float(unsigned o) {
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

// k > 1 (drafter children, k <= 8): the same partial record by K extraction
// rounds instead of per-element sorted insertion. Each of the 8 threads of a
// token keeps only its current best of its 16 entries; a round is a 3-step
// butterfly argmax over the 8 threads (logit desc, id asc), the winning
// thread drops that entry and rescans its 16. About a third of the
// instructions of the insertion merge, so the epilogue of one tile hides
// under the co-resident CTA's mainloop and the drafter's fp32 logits never
// reach HBM. With ep.topk_thr the rounds stop once the winner falls below the
// token's running k-th-value bound (most vocabulary tiles after the first
// wave stop after round 0); the record is then padded with -inf, which the
// merge ignores, so the merged top-k (and M, S, computed in full) does not
// depend on which tiles stopped early.
template <int KM>
__device__ __forceinline__ void epi_topk_tile_rounds(const EpiParams& ep, uint32_t tmem, int q, int lane, int n0,
                                                     int t0, int bn, float* tr, int tile) {
    const int K = ep.topk_k;
    const int W = 2 + 2 * K;
    const int ep_tid = threadIdx.x - 64;  // 0..127
    const int col = ep_tid >> 3, part = ep_tid & 7;
    const int id0 = n0 + part * 16;
    for (int c = 0; c < bn; c += 16) {
        if (t0 + c >= ep.m_tok) break;
        float v[16];
        tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + c, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) tr[j * 128 + q * 32 + lane] = v[j];
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const float* src = tr + col * 128 + part * 16;
        float xs[16];
        float bv = -CUDART_INF_F;
        int bi = 0;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            xs[i] = id0 + i < ep.n_out ? src[i] : -CUDART_INF_F;
            if (xs[i] > bv) {  // strict: the lowest index among equal values
                bv = xs[i];
                bi = i;
            }
        }
        // (m, s) of the tile's 128 entries for this token
        float m = bv, s = 0.f;
        if (m != -CUDART_INF_F) {
#pragma unroll
            for (int i = 0; i < 16; ++i) s += __expf(xs[i] - m);  // exp(-inf) = 0
        }
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const float om = __shfl_xor_sync(0xffffffffu, m, o);
            const float os = __shfl_xor_sync(0xffffffffu, s, o);
            const float nm = fmaxf(m, om);
            const float a = m == -CUDART_INF_F ? 0.f : s * __expf(m - nm);
            const float b = om == -CUDART_INF_F ? 0.f : os * __expf(om - nm);
            s = a + b;
            m = nm;
        }
        const int tok = t0 + c + col;
        // entries below a proven lower bound of the token's k-th largest
        // logit (some finished tile's k-th value) cannot reach the top-k
        float thr_v = -CUDART_INF_F;
        if (ep.topk_thr && tok < ep.m_tok) {
            const unsigned o = __ldcg(ep.topk_thr + tok);
            if (o) thr_v = ord_to_float(o);
        }
        float lv[KM];
        int li[KM];
#pragma unroll
        for (int r = 0; r < KM; ++r) {
            lv[r] = -CUDART_INF_F;
            li[r] = 0x7fffffff;
        }
        bool stop = false;
#pragma unroll
        for (int r = 0; r < KM; ++r) {
            float wv = bv;
            int wi = bv == -CUDART_INF_F ? 0x7fffffff : id0 + bi;
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) {
                const float ov = __shfl_xor_sync(0xffffffffu, wv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, wi, o);
                if (ov > wv || (ov == wv && oi < wi)) {
                    wv = ov;
                    wi = oi;
                }
            }
            if (!stop) {
                lv[r] = wv;
                li[r] = wi;
            }
            stop = stop || wv == -CUDART_INF_F || wv < thr_v;
            if (r + 1 < KM && !stop && wi == id0 + bi) {  // this thread's entry won: next best
#pragma unroll
                for (int i = 0; i < 16; ++i) xs[i] = i == bi ? -CUDART_INF_F : xs[i];
                bv = -CUDART_INF_F;
                bi = 0;
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    if (xs[i] > bv) {
                        bv = xs[i];
                        bi = i;
                    }
            }
            if (__all_sync(0xffffffffu, stop)) break;  // the warp's 4 tokens are done
        }
        if (ep.topk_thr && part == 0 && tok < ep.m_tok) {
            float kth = -CUDART_INF_F;
#pragma unroll
            for (int r = 0; r < KM; ++r)
                if (r == K - 1) kth = lv[r];
            if (kth != -CUDART_INF_F && kth > thr_v) atomicMax(ep.topk_thr + tok, float_to_ord(kth));
        }
        if (part == 0 && tok < ep.m_tok) {
            float* out = ep.out_f32 + ((long long)tile * ep.m_tok + tok) * W;
            out[0] = m;
            out[1] = s;
#pragma unroll
            for (int r = 0; r < KM; ++r) {
                if (r < K) {
                    out[2 + r] = lv[r];
                    out[2 + K + r] = __int_as_float(li[r]);
                }
            }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
    }
}

__device__ __forceinline__ float* align16f(void* p) {
    return reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
}

// Epilogue of one 128-row x bn-token accumulator tile (4 epilogue warps,
// 128 threads, named barrier 1). Per 16-token chunk: TMEM -> registers ->
// smem [16 tokens][128 rows] fp32 (lane = row: conflict-free), then every
// thread applies the fused op to units of 8 consecutive rows of one token and
// writes them with 16-byte stores (row-contiguous output, fully coalesced).
__device__ __forceinline__ void epi_tile_staged(const EpiParams& ep, uint32_t acc, int q, int lane, int n0, int t0,
                                                int bn, float* tr) {
    const int ep_tid = threadIdx.x - 64;  // 0..127
    for (int c = 0; c < bn; c += 16) {
        if (t0 + c >= ep.m_tok) break;
        float v[16];
        tmem_ld16(acc + (static_cast<uint32_t>(q * 32) << 16) + c, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) tr[j * 128 + q * 32 + lane] = v[j];
        asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int unit = ep_tid + 128 * u;  // 16 tokens x 16 row-octets
            const int tk = unit >> 4, r8 = (unit & 15) * 8;
            const float4 a = *reinterpret_cast<const float4*>(tr + tk * 128 + r8);
            const float4 b = *reinterpret_cast<const float4*>(tr + tk * 128 + r8 + 4);
            const float w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
            epi_vec8(ep, t0 + c + tk, n0 + r8, w);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
    }
}

// PAIR == 2: a thread-block cluster of two CTAs on one TPC computes a
// 256-row x bn-token tile with tcgen05.mma.cta_group::2 (M = 256): each CTA
// stages its own 128 weight rows and HALF of the token tile, the leader CTA
// issues the MMAs, each CTA's TMEM holds the accumulators of its 128 rows for
// all bn tokens. Per SM this halves the token-operand smem traffic and the
// L2->SMEM re-reads of the activations (the tensor-bound regime, M >~ 256).
template <int PAIR, int FP8 = 0>
__global__ void __launch_bounds__(192, 1)
    k_gemm_swapab(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                  int bn, int stages, int kb_total, int kb_per_split, uint32_t tmem_cols, int wm, int l2pf,
                  int mc, int wn, EpiParams ep) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int b_rows = bn / PAIR;  // token rows staged by this CTA
    const int b_bytes = b_rows * kBlockK * 2;
    // wn token sub-tiles of bn / wn tokens (one MMA of N = bn / wn each) share
    // every weight k-block: a token tile of up to 512 tokens reads each
    // weight tile once (TMEM columns = token offset within the tile). Pair:
    // each sub-tile is itself split between the two CTAs.
    const int bn_sub = bn / wn;
    const int sub_rows = bn_sub / PAIR;
    const int sub_bytes = sub_rows * kBlockK * 2;
    const int a_bytes = wm * kABytes;  // wm weight sub-tiles of 128 rows share every token tile
    uint8_t* sA = smem;
    uint8_t* sB = smem + stages * a_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + stages * b_bytes);
    uint64_t* empty = full + stages;
    uint64_t* tfull = empty + stages;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tfull + 1);

    constexpr int kKel = FP8 ? 2 * kBlockK : kBlockK;  // elements per 128-byte k-block row
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    // pair: rank = position in the CTA pair (cluster x); with split-K the
    // cluster is (2, 1, splits) and the pair of split z has cluster ranks
    // (2z, 2z+1): the leader (MMA issuer, full barriers) is rank 2z
    const uint32_t rank = PAIR == 2 ? (blockIdx.x & 1u) : 0u;
    // weight multicast (PAIR, mc > 1): a (2 mc, 1, 1) cluster holds mc CTA
    // pairs on the same weight tile and consecutive token tiles; pair 0 loads
    // each weight k-block once and multicasts it to the mc pairs, every
    // pair's MMA completion releases the stage in all of them
    const uint32_t mpair = (PAIR == 2 && mc > 1) ? (uint32_t)((blockIdx.x >> 1) % mc) : 0u;
    const uint32_t lead_rank = PAIR == 2 ? (mc > 1 ? 2u * mpair : 2u * blockIdx.z) : 0u;
    const uint16_t pair_mask = (uint16_t)(0x3u << lead_rank);
    const uint16_t all_mask = (uint16_t)((1u << (2 * mc)) - 1u);
    const uint16_t w_mask = (uint16_t)(0x5555u & all_mask) << rank;  // CTAs of the same pair rank
    const bool w_issuer = mc <= 1 || mpair == 0;
    // token tiles vary fastest: the CTAs sharing one weight tile run together,
    // so the weight tile is fetched from HBM once and re-read from L2
    const int n0 = (blockIdx.y * PAIR + rank) * kBlockM * wm;
    const int t0 = (blockIdx.x / PAIR) * bn;
    const int z = blockIdx.z;
    const int kb0 = z * kb_per_split;
    // padding token tile of a bucketed graph: no loads, no MMA, no epilogue.
    // Every CTA of a pair / split-K cluster shares t0, so they skip together;
    // a multicast cluster spans mc token tiles and must skip as a whole (its
    // weight issuer signals every pair's barriers): it skips only when its
    // first token tile is padding, otherwise all its pairs run
    const int m_live = epi_live_rows(ep);
    const int t_first = mc > 1 ? (int)((blockIdx.x / PAIR) / mc * mc) * bn : t0;
    const bool skip = t_first >= m_live;
    const int nkb = skip ? 0 : min(kb_total, kb0 + kb_per_split) - kb0;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmW);
        tma_prefetch_desc(&tmX);
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], mc > 1 ? mc : 1);
        }
        mbar_init(tfull, 1);
        fence_barrier_init();
    }
    if (warp == 1) {
        if (PAIR == 2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_holder)),
                         "r"(tmem_cols)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_holder)),
                         "r"(tmem_cols)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
    }
    tc_fence_before();
    if (PAIR == 2)
        cluster_sync_all();  // peer barriers initialised before any cross-CTA signal
    else
        __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_holder;
    // Weights do not depend on the previous kernel: the producer issues the
    // weight tiles of the first pipeline stages BEFORE griddepcontrol.wait, so
    // under PDL the weight stream overlaps the previous kernel's tail.
    const int npre = min(stages, nkb);
    const uint64_t pol_w = policy_evict_first();  // weights: streamed once
    const uint64_t pol_x = policy_evict_last();   // activations: re-read by every weight tile
    const uint32_t full_bar0 = PAIR == 2 ? mapa_shared(smem_u32(&full[0]), lead_rank) : 0u;
    if (warp == 0 && lane == 0) {
        // weight tiles beyond the smem ring: L2 prefetch l2pf k-blocks ahead
        if (w_issuer)
            for (int i = npre; i < min(nkb, npre + l2pf); ++i)
                for (int a = 0; a < wm; ++a) tma_prefetch_l2_2d(&tmW, (kb0 + i) * kKel, n0 + a * kBlockM);
        for (int i = 0; i < npre; ++i) {
            const int kc = (kb0 + i) * kKel;
            if (PAIR == 2) {
                if (rank == 0) mbar_arrive_expect_tx(&full[i], 2 * (a_bytes + b_bytes));
                if (mc > 1) {
                    if (w_issuer) tma_load_2d_pair_mc(sA + i * a_bytes, &tmW, &full[i], kc, n0, w_mask, pol_w);
                } else {
                    for (int a = 0; a < wm; ++a)
                        tma_load_2d_pair(sA + i * a_bytes + a * kABytes, &tmW, full_bar0 + 8u * i, kc,
                                         n0 + a * kBlockM, pol_w);
                }
            } else {
                mbar_arrive_expect_tx(&full[i], a_bytes + b_bytes);
                for (int a = 0; a < wm; ++a)
                    tma_load_2d(sA + i * a_bytes + a * kABytes, &tmW, &full[i], kc, n0 + a * kBlockM, pol_w);
            }
        }
    }
    pdl_wait();  // setup above overlaps the previous kernel's tail (PDL)

    if (warp == 0) {
        // ---------------- TMA producer (one per CTA; pair: both count on the leader's full barrier)
        if (lane == 0) {
            for (int i = 0; i < nkb; ++i) {
                const int s = i % stages;
                const uint32_t ph = (i / stages) & 1;
                const int kc = (kb0 + i) * kKel;
                auto load_x = [&] {  // this CTA's rows of every token sub-tile
                    for (int j = 0; j < wn; ++j) {
                        if (PAIR == 2)
                            tma_load_2d_pair(sB + s * b_bytes + j * sub_bytes, &tmX, full_bar0 + 8u * s, kc,
                                             t0 + j * bn_sub + (int)rank * sub_rows, pol_x);
                        else
                            tma_load_2d(sB + s * b_bytes + j * sub_bytes, &tmX, &full[s], kc, t0 + j * bn_sub, pol_x);
                    }
                };
                if (i < npre) {  // weight tile already in flight: activations only
                    load_x();
                    continue;
                }
                if (w_issuer && i + l2pf < nkb)
                    for (int a = 0; a < wm; ++a) tma_prefetch_l2_2d(&tmW, kc + l2pf * kKel, n0 + a * kBlockM);
                mbar_wait(&empty[s], ph ^ 1);
                if (PAIR == 2) {
                    if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * (a_bytes + b_bytes));
                    if (mc > 1) {
                        if (w_issuer) tma_load_2d_pair_mc(sA + s * a_bytes, &tmW, &full[s], kc, n0, w_mask, pol_w);
                    } else {
                        for (int a = 0; a < wm; ++a)
                            tma_load_2d_pair(sA + s * a_bytes + a * kABytes, &tmW, full_bar0 + 8u * s, kc,
                                             n0 + a * kBlockM, pol_w);
                    }
                    load_x();
                } else {
                    mbar_arrive_expect_tx(&full[s], a_bytes + b_bytes);
                    for (int a = 0; a < wm; ++a)
                        tma_load_2d(sA + s * a_bytes + a * kABytes, &tmW, &full[s], kc, n0 + a * kBlockM, pol_w);
                    load_x();
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (single elected thread; pair: leader CTA only)
        if (PAIR == 1 || rank == 0) {
            const uint32_t idesc =
                FP8 ? idesc_e4m3_f32(kBlockM * PAIR, bn_sub) : idesc_bf16_f32(kBlockM * PAIR, bn_sub);
            for (int i = 0; i < nkb; ++i) {
                const int s = i % stages;
                const uint32_t ph = (i / stages) & 1;
                mbar_wait(&full[s], ph);
                tc_fence_after();
                if (elect_one()) {
                    for (int a = 0; a < wm; ++a) {
                        const uint64_t da = sdesc_kmajor_sw128(sA + s * a_bytes + a * kABytes);
                        for (int j = 0; j < wn; ++j) {
                        const uint64_t db = sdesc_kmajor_sw128(sB + s * b_bytes + j * sub_bytes);
                        const uint32_t acc = tmem + a * bn + j * bn_sub;
#pragma unroll
                        for (int kk = 0; kk < kBlockK / 16; ++kk) {
                            // +32 bytes along K inside the 128B swizzle row == +2 in the >>4 address field
                            if (ep.dbg & 1) continue;  // diagnostics: loads only
                            if (FP8) {
                                if (PAIR == 2)
                                    tc_mma_e4m3_pair(acc, da + 2 * kk, db + 2 * kk, idesc, (i | kk) != 0);
                                else
                                    tc_mma_e4m3(acc, da + 2 * kk, db + 2 * kk, idesc, (i | kk) != 0);
                            } else if (PAIR == 2) {
                                tc_mma_bf16_pair(acc, da + 2 * kk, db + 2 * kk, idesc, (i | kk) != 0);
                            } else {
                                tc_mma_bf16(acc, da + 2 * kk, db + 2 * kk, idesc, (i | kk) != 0);
                            }
                        }
                        }  // j
                    }
                    if (PAIR == 2) {
                        tc_commit_pair_mc(&empty[s], mc > 1 ? all_mask : pair_mask);
                        if (i == nkb - 1) tc_commit_pair_mc(tfull, pair_mask);
                    } else {
                        tc_commit(&empty[s]);
                        if (i == nkb - 1) tc_commit(tfull);
                    }
                }
                __syncwarp();
            }
        }
    } else {
        // ---------------- epilogue: warps 2..5 own TMEM lane quarters (warp % 4)
        if (!skip) {
            mbar_wait(tfull, 0);
            tc_fence_after();
        }
        const int q = warp & 3;
        if (skip || (ep.dbg & 2)) {
            // diagnostics: no epilogue
        } else if (gridDim.z > 1) {
            // split-K: stage this CTA's fp32 partial in the (now idle) pipeline
            // smem, [token][128 weight rows]; the cluster reduces it below
            float* P = reinterpret_cast<float*>(smem);
            for (int c = 0; c < bn; c += 16) {
                if (t0 + c >= ep.m_tok) break;
                float v[16];
                tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + c, v);
#pragma unroll
                for (int j = 0; j < 16; ++j) P[(c + j) * kBlockM + q * 32 + lane] = v[j];
            }
        } else {
        for (int a = 0; a < wm; ++a) {
        const int na = n0 + a * kBlockM;
        if (na >= ep.n_out) break;  // second sub-tile entirely out of range
        const uint32_t tm_a = tmem + a * bn;
        const int row = na + q * 32 + lane;
        const int n_even = row & ~1;
        if (ep.kind == EPI_TOPK) {
            float* tr = reinterpret_cast<float*>(smem);  // [16 cols][128 vocab rows] over the drained ring
            const int tile = (blockIdx.y * PAIR + rank) * wm + a;
            if (ep.topk_k <= 1)
                epi_topk_tile<1>(ep, tm_a, q, lane, na, t0, bn, tr, tile);
            else
                epi_topk_tile_rounds<kEpiTopkMax>(ep, tm_a, q, lane, na, t0, bn, tr, tile);
        } else {
            epi_tile_staged(ep, tm_a, q, lane, na, t0, bn, reinterpret_cast<float*>(smem));
        }
        (void)n_even;
        }  // a
        }
    }
    if (gridDim.z > 1 && !(ep.dbg & 2)) {
        // Split-K finish inside the thread-block cluster (cluster = the
        // gridDim.z CTAs of one output tile): every CTA sums one contiguous
        // slice of (token, row-pair) elements over all peers' partials through
        // distributed shared memory, in fixed rank order (deterministic), and
        // applies the epilogue to it. No global partials, no second launch.
        namespace cg = cooperative_groups;
        cg::cluster_group cluster = cg::this_cluster();
        cluster.sync();
        const int S = (int)gridDim.z;
        const int tv = min(bn, m_live - t0);
        // units of 8 consecutive rows of one token: all S remote float4 pairs
        // are loaded before the fixed-order sum (DSMEM latency overlapped),
        // then the vectorised epilogue
        const int nunits = max(tv, 0) * (kBlockM / 8);
        const int per = (nunits + S - 1) / S;
        const int u0 = z * per, u1 = min(nunits, u0 + per);
        float* P = reinterpret_cast<float*>(smem);
        for (int u = u0 + (int)threadIdx.x; u < u1; u += (int)blockDim.x) {
            const int c = u / (kBlockM / 8);
            const int r8 = (u % (kBlockM / 8)) * 8;
            const int off4 = (c * kBlockM + r8) >> 2;
            float w[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            for (int zb = 0; zb < S; zb += kPeerBatch) {
                float4 va[kPeerBatch], vb[kPeerBatch];
#pragma unroll
                for (int zz = 0; zz < kPeerBatch; ++zz)
                    if (zb + zz < S) {
                        const float4* pr = reinterpret_cast<const float4*>(
                            cluster.map_shared_rank(P, (int)rank + PAIR * (zb + zz)));
                        va[zz] = pr[off4];
                        vb[zz] = pr[off4 + 1];
                    }
#pragma unroll
                for (int zz = 0; zz < kPeerBatch; ++zz)  // fixed split order: deterministic
                    if (zb + zz < S) {
                        w[0] += va[zz].x; w[1] += va[zz].y; w[2] += va[zz].z; w[3] += va[zz].w;
                        w[4] += vb[zz].x; w[5] += vb[zz].y; w[6] += vb[zz].z; w[7] += vb[zz].w;
                    }
            }
            epi_vec8(ep, t0 + c, n0 + r8, w);
        }
        cluster.sync();  // peers' smem stays alive until every remote read is done
    }
    if (ep.norm_w) {
        // Fused RMSNorm of the updated rows (long-tail M): the last CTA to
        // finish its epilogue normalises out_f32[0..m_tok) into norm_out.
        __shared__ int s_last;
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) {
            const int total = (int)(gridDim.x * gridDim.y * gridDim.z);
            s_last = atomicAdd(ep.norm_counter, 1) == total - 1;
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            const int d = ep.n_out;
            const int nw = blockDim.x >> 5;
            for (int t = warp; t < m_live; t += nw) {  // one warp per live token row
                const float* xr = ep.out_f32 + (long long)t * ep.ld_f32;
                float ss = 0.f;
                for (int i = lane * 4; i < d; i += 128) {
                    const float4 v = __ldcg(reinterpret_cast<const float4*>(xr + i));
                    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
                const float inv = 1.0f / sqrtf(ss / (float)d + ep.norm_eps);
                __nv_bfloat16* hr = ep.norm_out + (long long)t * d;
                for (int i = lane * 4; i < d; i += 128) {
                    const float4 v = __ldcg(reinterpret_cast<const float4*>(xr + i));
                    const uint2 gw = *reinterpret_cast<const uint2*>(ep.norm_w + i);
                    const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gw);
                    const float2 ga = __bfloat1622float2(g2[0]), gb = __bfloat1622float2(g2[1]);
                    uint2 o;
                    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
                    o2[0] = __floats2bfloat162_rn(v.x * inv * ga.x, v.y * inv * ga.y);
                    o2[1] = __floats2bfloat162_rn(v.z * inv * gb.x, v.w * inv * gb.y);
                    *reinterpret_cast<uint2*>(hr + i) = o;
                }
            }
            if (threadIdx.x == 0) *ep.norm_counter = 0;  // ready for the next launch / graph replay
        }
    }
    tc_fence_before();
    if (PAIR == 2)
        cluster_sync_all();
    else
        __syncthreads();
    if (warp == 1) {
        if (PAIR == 2)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols)
                         : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols)
                         : "memory");
    }
}


// ------------------------------------------------------------------ persistent
// Persistent variant for the multi-wave regime (output tiles >= CTA slots):
// one CTA (PAIR == 2: one CTA pair) per SM loops over output tiles
// (token tile fastest, so co-running CTAs share weight tiles through L2).
// The TMA producer streams k-blocks across tile boundaries without pausing;
// the MMA issuer alternates between two TMEM accumulators, so the epilogue of
// tile j (tcgen05.ld -> fused epilogue -> global) overlaps the mainloop of
// tile j+1. Barriers: smem ring full/empty; per accumulator tfull (MMA ->
// epilogue) and tempty (epilogue -> MMA, 4 warps per CTA of the pair arrive
// on the leader's barrier).
template <int PAIR>
__global__ void __launch_bounds__(192, 1)
    k_gemm_persist(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, int bn,
                   int stages, int kb_total, int n_ttiles, int n_tiles, uint32_t tmem_cols, EpiParams ep) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int b_rows = bn / PAIR;
    const int b_bytes = b_rows * kBlockK * 2;
    const int a_bytes = kABytes;
    uint8_t* sA = smem;
    uint8_t* sB = smem + stages * a_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + stages * b_bytes);
    uint64_t* empty = full + stages;
    uint64_t* tfull = empty + stages;  // [2]
    uint64_t* tempty = tfull + 2;      // [2]
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = PAIR == 2 ? cluster_ctarank() : 0u;
    const int cid = blockIdx.x / PAIR, ncl = gridDim.x / PAIR;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmW);
        tma_prefetch_desc(&tmX);
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 4 * PAIR);
        }
        fence_barrier_init();
    }
    if (warp == 1) {
        if (PAIR == 2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_holder)),
                         "r"(tmem_cols)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_holder)),
                         "r"(tmem_cols)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
    }
    tc_fence_before();
    if (PAIR == 2)
        cluster_sync_all();
    else
        __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_holder;
    const uint64_t pol_w = policy_evict_first();
    const uint64_t pol_x = policy_evict_last();
    const uint32_t full_bar0 = PAIR == 2 ? mapa_shared(smem_u32(&full[0]), 0) : 0u;
    // bucketed graphs: only the token tiles holding live rows are scheduled
    // (same tile order, the padding tiles dropped from the static schedule)
    {
        const int n_wt = n_tiles / n_ttiles;
        n_ttiles = min(n_ttiles, (epi_live_rows(ep) + bn - 1) / bn);
        n_tiles = n_ttiles * n_wt;
    }
    // first tile's weight stages before griddepcontrol.wait (weights are not
    // produced by the previous kernel)
    const int npre = (cid < n_tiles) ? min(stages, kb_total) : 0;
    if (warp == 0 && lane == 0 && npre > 0) {
        const int n0 = ((cid / n_ttiles) * PAIR + rank) * kBlockM;
        for (int i = 0; i < npre; ++i) {
            if (PAIR == 2) {
                if (rank == 0) mbar_arrive_expect_tx(&full[i], 2 * (a_bytes + b_bytes));
                tma_load_2d_pair(sA + i * a_bytes, &tmW, full_bar0 + 8u * i, i * kBlockK, n0, pol_w);
            } else {
                mbar_arrive_expect_tx(&full[i], a_bytes + b_bytes);
                tma_load_2d(sA + i * a_bytes, &tmW, &full[i], i * kBlockK, n0, pol_w);
            }
        }
    }
    pdl_wait();

    if (warp == 0) {
        if (lane == 0) {
            int it = 0;
            for (int t = cid; t < n_tiles; t += ncl) {
                const int n0 = ((t / n_ttiles) * PAIR + rank) * kBlockM;
                const int t0 = (t % n_ttiles) * bn;
                for (int kb = 0; kb < kb_total; ++kb, ++it) {
                    const int s = it % stages;
                    const uint32_t ph = (it / stages) & 1;
                    const int kc = kb * kBlockK;
                    if (it < npre) {  // weight tile already in flight
                        if (PAIR == 2)
                            tma_load_2d_pair(sB + s * b_bytes, &tmX, full_bar0 + 8u * s, kc, t0 + (int)rank * b_rows,
                                             pol_x);
                        else
                            tma_load_2d(sB + s * b_bytes, &tmX, &full[s], kc, t0, pol_x);
                        continue;
                    }
                    mbar_wait(&empty[s], ph ^ 1);
                    if (PAIR == 2) {
                        if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * (a_bytes + b_bytes));
                        tma_load_2d_pair(sA + s * a_bytes, &tmW, full_bar0 + 8u * s, kc, n0, pol_w);
                        tma_load_2d_pair(sB + s * b_bytes, &tmX, full_bar0 + 8u * s, kc, t0 + (int)rank * b_rows,
                                         pol_x);
                    } else {
                        mbar_arrive_expect_tx(&full[s], a_bytes + b_bytes);
                        tma_load_2d(sA + s * a_bytes, &tmW, &full[s], kc, n0, pol_w);
                        tma_load_2d(sB + s * b_bytes, &tmX, &full[s], kc, t0, pol_x);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (PAIR == 1 || rank == 0) {
            const uint32_t idesc = idesc_bf16_f32(kBlockM * PAIR, bn);
            int it = 0, j = 0;
            for (int t = cid; t < n_tiles; t += ncl, ++j) {
                const int b = j & 1;
                mbar_wait(&tempty[b], ((j >> 1) & 1) ^ 1);  // accumulator b drained by the epilogue
                tc_fence_after();
                const uint32_t acc = tmem + b * bn;
                for (int kb = 0; kb < kb_total; ++kb, ++it) {
                    const int s = it % stages;
                    const uint32_t ph = (it / stages) & 1;
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint64_t da = sdesc_kmajor_sw128(sA + s * a_bytes);
                        const uint64_t db = sdesc_kmajor_sw128(sB + s * b_bytes);
#pragma unroll
                        for (int kk = 0; kk < kBlockK / 16; ++kk) {
                            if (ep.dbg & 1) continue;
                            if (PAIR == 2)
                                tc_mma_bf16_pair(acc, da + 2 * kk, db + 2 * kk, idesc, (kb | kk) != 0);
                            else
                                tc_mma_bf16(acc, da + 2 * kk, db + 2 * kk, idesc, (kb | kk) != 0);
                        }
                        if (PAIR == 2) {
                            tc_commit_pair_mc(&empty[s], 0x3);
                            if (kb == kb_total - 1) tc_commit_pair_mc(&tfull[b], 0x3);
                        } else {
                            tc_commit(&empty[s]);
                            if (kb == kb_total - 1) tc_commit(&tfull[b]);
                        }
                    }
                    __syncwarp();
                }
            }
        }
    } else {
        // epilogue warps 2..5: TMEM lane quarter q = warp % 4
        const int q = warp & 3;
        float* tr = align16f(tmem_holder + 4);  // EPI_TOPK transpose scratch
        const uint32_t tempty_leader = PAIR == 2 ? mapa_shared(smem_u32(&tempty[0]), 0) : 0u;
        int j = 0;
        for (int t = cid; t < n_tiles; t += ncl, ++j) {
            const int b = j & 1;
            const int n0 = ((t / n_ttiles) * PAIR + rank) * kBlockM;
            const int t0 = (t % n_ttiles) * bn;
            mbar_wait(&tfull[b], (j >> 1) & 1);
            tc_fence_after();
            const uint32_t acc = tmem + b * bn;
            if (!(ep.dbg & 2) && n0 < ep.n_out) {
                if (ep.kind == EPI_TOPK) {
                    const int tile = (t / n_ttiles) * PAIR + rank;
                    if (ep.topk_k <= 1)
                        epi_topk_tile<1>(ep, acc, q, lane, n0, t0, bn, tr, tile);
                    else
                        epi_topk_tile_rounds<kEpiTopkMax>(ep, acc, q, lane, n0, t0, bn, tr, tile);
                } else {
                    epi_tile_staged(ep, acc, q, lane, n0, t0, bn, tr);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (PAIR == 2)
                    mbar_arrive_cluster(tempty_leader + 8u * b);
                else
                    mbar_arrive(&tempty[b]);
            }
        }
    }
    tc_fence_before();
    if (PAIR == 2)
        cluster_sync_all();
    else
        __syncthreads();
    if (warp == 1) {
        if (PAIR == 2)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols)
                         : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols)
                         : "memory");
    }
}

// ------------------------------------------------------------------ host side

static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
    return fn;
}

// 2D bf16 K-major tensor map: rows x cols (cols = K, contiguous), box = box_rows x 64.
CUtensorMap make_tmap_bf16(const void* base, int rows, int cols, long long row_stride_elems, int box_rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(row_stride_elems * 2)};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(kBlockK), static_cast<cuuint32_t>(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = get_encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                                 strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return m;
}

// 2D e4m3 (one-byte) K-major map: box = box_rows x 128 elements (128 bytes).
CUtensorMap make_tmap_e4m3(const void* base, int rows, int cols, long long row_stride_elems, int box_rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(row_stride_elems)};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(2 * kBlockK), static_cast<cuuint32_t>(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = get_encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (e4m3) failed: " + std::to_string(r));
    return m;
}

static int g_num_sms = 0;
int num_sms() {
    if (!g_num_sms) {
        int dev = 0;
        CUDA_CHECK(cudaGetDevice(&dev));
        CUDA_CHECK(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    return g_num_sms;
}

static int env_knob(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v ? std::atoi(v) : dflt;
}

// per-device zeroed counter for the fused-norm "last CTA" election (each last
// CTA resets it, so the buffer stays zero between launches / graph replays)
int* gemm_norm_counter() {
    static int* ptrs[64] = {nullptr};
    int dev = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    if (!ptrs[dev]) {
        CUDA_CHECK(cudaMalloc(&ptrs[dev], sizeof(int) * 32));
        CUDA_CHECK(cudaMemset(ptrs[dev], 0, sizeof(int) * 32));
    }
    return ptrs[dev];
}

int gemm_dbg_flags() {
    static const int f = env_knob("TLT_GEMM_DBG", 0);
    return f;
}

// Weight-streaming plans (single-CTA tiles, split-K over few weight tiles):
// TLT_GEMM_ONE_WAVE=1 caps the split count so every CTA gets its own SM
// (tiles x splits <= #SMs; the 2-per-SM packing otherwise leaves half the
// SMs with twice the bytes to stream) and gives each CTA the whole smem ring
// (up to 12 stages, ~200 KB of weight tiles in flight per SM).
void gemm_one_wave(GemmPlan& g) {
    static const int on = env_knob("TLT_GEMM_ONE_WAVE", 0);
    if (!on || g.pair != 1 || g.persist || g.wm != 1 || g.fp8 || g.mc != 1) return;
    const int tiles = g.n_wtiles * g.n_ttiles;
    if (tiles > num_sms()) return;
    int splits = g.splits;
    if (tiles * splits > num_sms()) {
        splits = std::max(1, num_sms() / tiles);
        g.kb_per_split = (g.kb_total + splits - 1) / splits;
        g.splits = (g.kb_total + g.kb_per_split - 1) / g.kb_per_split;
    }
    const int fixed = 1024 + 256;
    const int stage_bytes = kABytes + g.box_rows * kBlockK * 2;
    g.stages = std::max(2, std::min(12, (220 * 1024 - fixed) / stage_bytes));
    g.smem = g.stages * stage_bytes + fixed;
}

GemmPlan plan_gemm(int m_tok, int n_out, int k, int variant) {
    GemmPlan g;
    static const int l2pf = env_knob("TLT_GEMM_L2PF", 0);
    g.l2pf = l2pf;
    g.kb_total = (k + kBlockK - 1) / kBlockK;
    // ring + barriers + alignment slack; the epilogue's 8 KB staging reuses
    // the drained ring (all MMAs complete before the epilogue starts)
    const int fixed = 1024 + 256;
    // Tensor-bound regime: CTA pairs (cta_group::2, 256 weight rows x up to
    // 256 tokens per pair), no split-K.
    static const int pair_min_m_env = env_knob("TLT_GEMM_PAIR_MIN_M", 192);
    static const int pair_bn_max_env = env_knob("TLT_GEMM_PAIR_BN_MAX", 256);
    // 4 = CTA pairs with <= 128-token tiles (more tiles: fills the SMs on
    // small-N shapes), 6 = the pair split-K plan with 4 splits
    const int pair_bn_max = variant == 4 ? 128 : pair_bn_max_env;
    static const int pair_cps_env = env_knob("TLT_GEMM_PAIR_CPS", 2);
    // plan variants (the engine's per-shape autotuner times them once and
    // keeps the fastest): 1 = CTA pairs with a deep 1-CTA/SM ring, 2 = the
    // persistent CTA-pair kernel, 3 = no CTA pairs (single-CTA tiles)
    const int pair_min_m = variant == 3 ? 0 : pair_min_m_env;
    const int pair_cps = variant == 1 ? 1 : pair_cps_env;
    // 1: persistent kernel for CTA-pair plans; 2: also for single-CTA plans
    // measured (profiles/r1_gemm_knobs_*.txt): with the staged epilogue the
    // 2-CTA/SM non-persistent kernel wins below ~768 tokens, the persistent
    // CTA-pair kernel above; the single-CTA persistent kernel never wins
    static const int persist = env_knob("TLT_GEMM_PERSIST", 1);
    static const int pair_persist_min_m_env = env_knob("TLT_GEMM_PAIR_PERSIST_MIN_M", 768);
    const int pair_persist_min_m = variant == 2 ? 1 : pair_persist_min_m_env;
    static const int persist1_min_m = env_knob("TLT_GEMM_PERSIST1_MIN_M", 48);
    // pairs only when they still put >= 1 CTA on every SM (else the 1-CTA
    // plan with in-cluster split-K fills the machine better)
    const int pair_ctas = 2 * ((n_out + 2 * kBlockM - 1) / (2 * kBlockM)) * ((m_tok + pair_bn_max - 1) / pair_bn_max);
    static const int pair_min_ctas = env_knob("TLT_GEMM_PAIR_MIN_CTAS", 148);
    static const int pair_split = env_knob("TLT_GEMM_PAIR_SPLIT", 1);
    if (variant == 8 && m_tok > 256) {
        // CTA pairs with token tiles of up to 512 tokens as two MMA sub-tiles
        // (N = bn / 2 each, 2 x bn TMEM columns -> 1 CTA per SM): each weight
        // tile is read once per 512 tokens instead of once per <= 256, which
        // cuts the L2 -> SM traffic (the limit at mid M: ~6.3 KB/clk chip-wide
        // L2 throughput) by up to a third; split-K in a (2, 1, splits) cluster
        // when the weight tiles alone cannot fill the SMs
        const int n_tt = (m_tok + 511) / 512;
        const int per = (m_tok + n_tt - 1) / n_tt;
        const int bn_sub = std::max(32, ((per + 1) / 2 + 15) / 16 * 16);
        g.pair = 2;
        g.wm = 1;
        g.wn = 2;
        g.bn = 2 * bn_sub;
        g.box_rows = bn_sub / 2;
        g.n_ttiles = (m_tok + g.bn - 1) / g.bn;
        g.n_wtiles = (n_out + 2 * kBlockM - 1) / (2 * kBlockM);
        const int stage_bytes = kABytes + (g.bn / 2) * kBlockK * 2;
        g.stages = std::max(2, std::min(8, (220 * 1024 - fixed) / stage_bytes));
        g.smem = g.stages * stage_bytes + fixed;
        g.tmem_cols = g.bn <= 256 ? 256 : 512;
        const int pairs = g.n_wtiles * g.n_ttiles;
        int splits = 1;
        if (pairs < num_sms() / 2) splits = std::max(1, std::min({(num_sms() / 2) / pairs, g.kb_total / 4, 4}));
        if (splits > 1 && g.stages * stage_bytes < g.bn * kBlockM * 4) splits = 1;  // partials must fit the ring
        g.kb_per_split = (g.kb_total + splits - 1) / splits;
        g.splits = (g.kb_total + g.kb_per_split - 1) / g.kb_per_split;
        return g;
    }
    if (pair_split && (variant == 0 || variant == 6) && pair_min_m > 0 && m_tok >= pair_min_m &&
        (pair_ctas < pair_min_ctas || variant == 6)) {
        // few weight tiles (N = d): CTA pairs with <= 128-token tiles and
        // split-K across a (2, 1, splits) cluster, reduced through DSMEM
        const int n_tt = (m_tok + 127) / 128;
        int bn = (m_tok + n_tt - 1) / n_tt;
        bn = std::max(32, (bn + 15) / 16 * 16);
        const int n_wt = (n_out + 2 * kBlockM - 1) / (2 * kBlockM);
        const int ctas = 2 * n_wt * ((m_tok + bn - 1) / bn);
        int splits = std::max(1, std::min({(2 * num_sms()) / ctas, g.kb_total / 4, 4}));
        if (variant == 6) splits = std::max(1, std::min(4, g.kb_total / 4));
        const int stage_bytes = kABytes + (bn / 2) * kBlockK * 2;
        const int stages = std::max(2, std::min(8, (112 * 1024 - fixed) / stage_bytes));
        if (splits > 1 && stages * stage_bytes >= bn * kBlockM * 4) {
            g.pair = 2;
            g.wm = 1;
            g.bn = bn;
            g.box_rows = bn / 2;
            g.n_ttiles = (m_tok + bn - 1) / bn;
            g.n_wtiles = n_wt;
            g.stages = stages;
            g.smem = stages * stage_bytes + fixed;
            g.tmem_cols = bn <= 32 ? 32 : bn <= 64 ? 64 : 128;
            g.kb_per_split = (g.kb_total + splits - 1) / splits;
            g.splits = (g.kb_total + g.kb_per_split - 1) / g.kb_per_split;
            return g;
        }
    }
    if (pair_min_m > 0 && m_tok >= pair_min_m &&
        (pair_ctas >= pair_min_ctas || variant == 1 || variant == 2 || variant == 4 || variant == 7)) {
        g.pair = 2;
        g.wm = 1;
        static const int pair_wm2 = env_knob("TLT_GEMM_PAIR_WM2", 0);  // measured slower (exposed epilogue, 1 CTA/SM)
        // two 256-row pair tiles per cluster (512 weight rows x bn tokens,
        // 1 CTA/SM): halves the token-tile TMA traffic per FLOP, the bound of
        // the 2-CTA/SM plan at mid M (chip TMA throughput)
        if (pair_wm2 && m_tok >= 384 && (n_out + 4 * kBlockM - 1) / (4 * kBlockM) * 2 >= num_sms() / 2) g.wm = 2;
        const int n_tt = (m_tok + pair_bn_max - 1) / pair_bn_max;
        int bn = (m_tok + n_tt - 1) / n_tt;
        bn = std::max(32, (bn + 15) / 16 * 16);
        g.bn = bn;
        g.box_rows = bn / 2;
        g.n_ttiles = (m_tok + bn - 1) / bn;
        g.n_wtiles = (n_out + 2 * kBlockM * g.wm - 1) / (2 * kBlockM * g.wm);
        const int stage_bytes = g.wm * kABytes + g.box_rows * kBlockK * 2;
        g.kb_per_split = g.kb_total;
        g.splits = 1;
        if (g.wm == 2) {
            g.stages = std::max(2, std::min(8, (220 * 1024 - fixed) / stage_bytes));
            g.smem = g.stages * stage_bytes + fixed;
            g.tmem_cols = 2 * bn <= 256 ? 256 : 512;
            return g;
        }
        if (variant == 7) {
            // weight multicast across the token tiles of one weight tile: a
            // (2 mc, 1, 1) cluster, each weight k-block read from L2 once per
            // cluster instead of once per token tile
            int mc = 1;
            for (int c = 4; c >= 2; --c)
                if (g.n_ttiles % c == 0) {
                    mc = c;
                    break;
                }
            if (mc > 1) {
                g.mc = mc;
                const int budget = (pair_cps == 2 ? 112 * 1024 : 220 * 1024) - fixed;
                g.stages = std::max(2, std::min(8, budget / stage_bytes));
                g.smem = g.stages * stage_bytes + fixed;
                g.tmem_cols = bn <= 32 ? 32 : bn <= 64 ? 64 : bn <= 128 ? 128 : 256;
                return g;
            }
        }
        if (persist >= 1 && m_tok >= pair_persist_min_m) {
            // persistent: one pair per 2 SMs, full smem ring, 2 TMEM accumulators
            const int pfixed = 1024 + 32 * 8 + 16 + 16 * 128 * 4;
            g.persist = 1;
            g.stages = std::max(2, std::min(12, (220 * 1024 - pfixed) / stage_bytes));
            g.smem = g.stages * stage_bytes + pfixed;
            const int cols = 2 * bn;
            g.tmem_cols = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
            return g;
        }
        const int budget = (pair_cps == 2 ? 112 * 1024 : 220 * 1024) - fixed;
        g.stages = std::max(2, std::min(8, budget / stage_bytes));
        g.smem = g.stages * stage_bytes + fixed;
        g.tmem_cols = bn <= 32 ? 32 : bn <= 64 ? 64 : bn <= 128 ? 128 : 256;
        return g;
    }
    // Measured on B200 (tools/gemm_sweep.sh, profiles/): two co-resident CTAs
    // per SM (one's epilogue/prologue overlapping the other's mainloop) beat
    // deeper pipelines and larger tiles: token tiles <= 128, <= ~110 KB smem.
    static const int bn_max = env_knob("TLT_GEMM_BN_MAX", 128);
    static const int force_wm = env_knob("TLT_GEMM_WM", 0);
    static const int force_stages = env_knob("TLT_GEMM_STAGES", 0);
    const int n_ttiles = (m_tok + bn_max - 1) / bn_max;
    int bn = (m_tok + n_ttiles - 1) / n_ttiles;
    bn = std::max(16, (bn + 15) / 16 * 16);
    g.bn = bn;
    g.box_rows = bn;
    g.n_ttiles = (m_tok + bn - 1) / bn;
    g.wm = 1;  // 2 measured slower at every shape (fewer co-resident CTAs); kept behind TLT_GEMM_WM
    if (force_wm) g.wm = force_wm;
    g.n_wtiles = (n_out + kBlockM * g.wm - 1) / (kBlockM * g.wm);
    const int stage_bytes = g.wm * kABytes + bn * kBlockK * 2;
    const int ctas_per_sm = (bn <= 128 && g.wm == 1) ? 2 : 1;
    // per-CTA budget incl. barriers, alignment slack and the EPI_TOPK merge
    // scratch, so that 2 CTAs/SM really fit in the 228 KB SM carve-out
    const int budget = (ctas_per_sm == 2 ? 112 * 1024 : 220 * 1024) - fixed;
    g.stages = std::max(2, std::min(8, budget / stage_bytes));
    if (force_stages) g.stages = std::min(force_stages, std::max(2, (220 * 1024 - fixed) / stage_bytes));
    g.smem = g.stages * stage_bytes + fixed;
    const int cols = g.wm * bn;
    g.tmem_cols = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
    const int tiles = g.n_wtiles * g.n_ttiles;
    const int slots = num_sms() * ctas_per_sm;
    int splits = 1;
    if (tiles < slots) splits = std::max(1, std::min(slots / tiles, g.kb_total / 4));
    // split-K CTAs of a tile form one cluster (portable size <= 8) and park
    // their fp32 partial in the pipeline smem for the DSMEM reduction
    static const int max_splits = env_knob("TLT_GEMM_MAX_SPLITS", 8);
    splits = std::min({splits, kMaxSplits, std::max(1, max_splits)});
    if (g.wm != 1 || g.stages * stage_bytes < bn * kBlockM * 4) splits = 1;
    g.kb_per_split = (g.kb_total + splits - 1) / splits;
    g.splits = (g.kb_total + g.kb_per_split - 1) / g.kb_per_split;
    gemm_one_wave(g);
    if (g.splits == 1 && persist >= 2 && g.wm == 1 && m_tok >= persist1_min_m) {
        const int pfixed = 1024 + 32 * 8 + 16 + 16 * 128 * 4;
        g.persist = 1;
        g.stages = std::max(2, std::min(12, (220 * 1024 - pfixed) / stage_bytes));
        g.smem = g.stages * stage_bytes + pfixed;
        const int c2 = 2 * bn;
        g.tmem_cols = c2 <= 32 ? 32 : c2 <= 64 ? 64 : c2 <= 128 ? 128 : c2 <= 256 ? 256 : 512;
    }
    return g;
}

GemmPlan plan_gemm_e4m3(int m_tok, int n_out, int k) {
    // one-byte operands: a k-block (128 bytes) holds 128 elements, i.e. the
    // bf16 planner with k/2; single split (the large-N LM head fills the SMs)
    GemmPlan g = plan_gemm(m_tok, n_out, (k + 1) / 2);
    if (g.persist || g.splits != 1 || g.wm != 1) {
        const int fixed = 1024 + 256;
        const int stage_bytes = kABytes + g.box_rows * kBlockK * 2;
        g.persist = 0;
        g.wm = 1;
        g.splits = 1;
        g.kb_per_split = g.kb_total;
        g.stages = std::max(2, std::min(8, ((g.pair == 2 || g.bn <= 128 ? 112 : 220) * 1024 - fixed) / stage_bytes));
        g.smem = g.stages * stage_bytes + fixed;
        const int cols = g.bn;
        g.tmem_cols = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : 256;
    }
    g.fp8 = 1;
    return g;
}

void launch_gemm(const GemmPlan& g, const CUtensorMap& tmW, const CUtensorMap& tmX, const EpiParams& ep,
                 float* workspace, size_t workspace_elems, cudaStream_t st) {
    (void)workspace;
    (void)workspace_elems;
    static bool attr_set = false;
    if (!attr_set) {
        // 226 KB: leaves room for the kernel's few static shared words
        CUDA_CHECK(cudaFuncSetAttribute(k_gemm_swapab<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
        CUDA_CHECK(cudaFuncSetAttribute(k_gemm_swapab<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        CUDA_CHECK(cudaFuncSetAttribute(k_gemm_swapab<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
        CUDA_CHECK(cudaFuncSetAttribute(k_gemm_swapab<2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        CUDA_CHECK(cudaFuncSetAttribute(k_gemm_swapab<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
        CUDA_CHECK(cudaFuncSetAttribute(k_gemm_swapab<2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
        attr_set = true;
    }
    if (ep.kind == EPI_TOPK && g.splits > 1) throw CudaError("EPI_TOPK needs whole-K accumulators");
    if (g.splits > kMaxSplits) throw CudaError("split-K cluster larger than the portable cluster size");
    if (g.pair == 2 && ((g.wm != 1 && (g.splits != 1 || g.persist)) || g.bn % 16 || g.bn < 32 ||
                        g.bn > 256 * g.wn || (g.splits > 1 && g.bn > 128 && g.wn == 1) || 2 * g.splits > kMaxSplits))
        throw CudaError("invalid CTA-pair GEMM plan");
    if (g.wn != 1 && (g.wn != 2 || g.persist || g.mc != 1 || g.wm != 1 || (g.bn / g.wn) % 16 ||
                      g.wm * g.bn > (int)g.tmem_cols || g.fp8))
        throw CudaError("invalid token sub-tile GEMM plan");
    if (g.splits > 1 && (g.wm != 1 || g.stages * (kABytes + g.bn / g.pair * kBlockK * 2) < g.bn * kBlockM * 4))
        throw CudaError("split-K partial does not fit the pipeline smem");
    dim3 grid(g.n_ttiles * g.pair, g.n_wtiles, g.splits);
    EpiParams epd = ep;
    epd.dbg = gemm_dbg_flags();
    if (ep.norm_w && (g.persist || g.pair != 1 || ep.kind != EPI_RESID_ADD || (ep.n_out & 3) || ep.ld_f32 != ep.n_out))
        throw CudaError("fused RMSNorm epilogue needs a single-CTA residual-add plan");
    if (ep.norm_w) epd.norm_counter = gemm_norm_counter();
    if (g.persist) {
        static bool pattr = false;
        if (!pattr) {
            CUDA_CHECK(cudaFuncSetAttribute(k_gemm_persist<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
            CUDA_CHECK(cudaFuncSetAttribute(k_gemm_persist<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
            pattr = true;
        }
        const int n_tiles = g.n_ttiles * g.n_wtiles;
        const int groups = std::min(n_tiles, num_sms() / g.pair);
        cudaLaunchConfig_t pc = {};
        pc.gridDim = dim3(groups * g.pair, 1, 1);
        pc.blockDim = dim3(192);
        pc.dynamicSmemBytes = g.smem;
        pc.stream = st;
        cudaLaunchAttribute pa[2];
        int npa = 0;
        if (pdl_enabled(1)) {
            pa[npa].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            pa[npa].val.programmaticStreamSerializationAllowed = 1;
            ++npa;
        }
        pa[npa].id = cudaLaunchAttributeClusterDimension;
        pa[npa].val.clusterDim.x = g.pair;
        pa[npa].val.clusterDim.y = 1;
        pa[npa].val.clusterDim.z = 1;
        ++npa;
        pc.attrs = pa;
        pc.numAttrs = npa;
        cudaError_t e = cudaLaunchKernelEx(&pc, g.pair == 2 ? k_gemm_persist<2> : k_gemm_persist<1>, tmW, tmX, g.bn,
                                           g.stages, g.kb_total, g.n_ttiles, n_tiles, g.tmem_cols, epd);
        if (e != cudaSuccess) throw CudaError(std::string("gemm launch: ") + cudaGetErrorString(e));
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(192);
    cfg.dynamicSmemBytes = g.smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (pdl_enabled(1)) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    // the split-K CTAs of one output tile form one cluster (DSMEM reduction);
    // CTA pairs are (2, 1, 1) clusters
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = g.pair * g.mc;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = g.splits;
    ++na;
    cfg.attrs = at;
    cfg.numAttrs = na;
    auto kern = g.fp8 ? (g.pair == 2 ? k_gemm_swapab<2, 1> : k_gemm_swapab<1, 1>)
                      : (g.pair == 2 ? k_gemm_swapab<2, 0> : k_gemm_swapab<1, 0>);
    if (g.fp8 && (g.persist || g.splits != 1)) throw CudaError("e4m3 GEMM: only the single-split non-persistent plan");
    if (g.mc > 1 && (g.pair != 2 || g.splits != 1 || g.wm != 1 || g.n_ttiles % g.mc || g.mc > 4 || g.fp8))
        throw CudaError("invalid weight-multicast GEMM plan");
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tmW, tmX, g.bn, g.stages, g.kb_total, g.kb_per_split,
                                       g.tmem_cols, g.wm, g.l2pf, g.mc, g.wn, epd);
    if (e != cudaSuccess) throw CudaError(std::string("gemm launch: ") + cudaGetErrorString(e));
}

}  // namespace tlt
