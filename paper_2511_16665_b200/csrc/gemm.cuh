// Swap-AB tcgen05 GEMM for the verify / draft / decode linears.
//
//   Y[t][n] = sum_k X[t][k] * W[n][k]        (X: tokens x K, W: out-features x K, both bf16 K-major)
//
// Computed transposed on the tensor core: the weight tile (128 out-features)
// is the MMA "A" operand (M = 128, the only M the 1-CTA f16 path runs at full
// rate), and the token tile is the MMA "B" operand (N = BN in 16..256). At the
// long-tail batch sizes of the rollout (b*(T+1) = 17..600 tokens) this keeps the
// tensor core fully fed while every weight byte is streamed from HBM exactly
// once per token tile. Accumulators live in TMEM (128 lanes x BN fp32 columns),
// operands arrive by TMA (128B swizzle) through an mbarrier ring, and one
// elected thread issues tcgen05.mma. Epilogues (bias + RoPE + KV-cache write,
// residual add, SwiGLU, fp32 store, LM-head top-k) are fused; split-K partials
// are reduced inside a thread-block cluster through distributed shared memory and read the
// accumulator with tcgen05.ld.
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

namespace tlt {

enum EpiKind : int {
    EPI_F32 = 0,        // out_f32[t][n] = acc
    EPI_BF16 = 1,       // out_bf16[t][n] = bf16(acc)
    EPI_RESID_ADD = 2,  // out_f32[t][n] += acc  (fp32 residual stream)
    EPI_SWIGLU = 3,     // rows interleaved (gate, up): out_bf16[t][n/2] = bf16(silu(g) * u)
    EPI_QKV = 4,        // + bias, RoPE on q/k pairs, q -> out_bf16, k/v -> KV cache
    EPI_TOPK = 6,       // LM head: per (128-vocab tile, token) max, sum-exp and top-k (logit desc, id asc)
};

struct EpiParams {
    int kind;
    int n_out;            // valid output features (W rows)
    int m_tok;            // valid token rows
    float* out_f32;
    int ld_f32;
    __nv_bfloat16* out_bf16;
    int ld_bf16;
    // EPI_QKV
    const __nv_bfloat16* bias;  // [n_out] or null
    const float* rope_cos;      // [max_pos][head_dim/2]
    const float* rope_sin;
    const int* tok_pos;         // [m] absolute position (RoPE)
    const int* tok_slot;        // [m] request slot, <0 = padding row (no KV write)
    const int* tok_cidx;        // [m] KV-cache index within the slot
    __nv_bfloat16* kcache;      // layer base: [slots][n_kv][max_ctx][head_dim]
    __nv_bfloat16* vcache;
    int n_q;                    // H*hd rows of q
    int n_kvr;                  // KV*hd rows of k (and of v)
    int head_dim;
    int n_kv;
    int max_ctx;
    // EPI_TOPK: out_f32 = partials [n_wtiles][m_tok][2 + 2*topk_k] (m, s, vals[k], ids[k])
    int topk_k;
    // k > 1: per-token running lower bound of the row's k-th largest logit
    // (order-preserving uint encoding, 0 = none; atomicMax'ed by finished
    // tiles, reset to 0 by k_topk_merge): a tile whose maximum is below it
    // cannot contribute and skips its extraction rounds. Null: off.
    unsigned* topk_thr;
    int dbg;  // diagnostics (TLT_GEMM_DBG): bit0 skip MMA, bit1 skip epilogue
    // fused RMSNorm after EPI_RESID_ADD (long-tail M): the last CTA writes
    // norm_out[t] = bf16(rmsnorm(out_f32[t]) * norm_w) for every token row
    const __nv_bfloat16* norm_w;
    __nv_bfloat16* norm_out;
    float norm_eps;
    int* norm_counter;
    // e4m3 GEMM dequantisation: acc * row_scale[n] * tok_scale[t] (null: none)
    const float* row_scale;
    const float* tok_scale;
    // Bucketed CUDA graphs (capture_plan.hpp:87-126): a graph captured for
    // the bucket's largest batch is replayed for any batch in the bucket.
    // Rows are request-major and the padding requests come last, so only the
    // first (*dyn_n) * dyn_rpr token rows are live; token tiles entirely past
    // them are skipped (no weight stream, no MMA). dyn_n = null: all m_tok.
    const int* dyn_n;
    int dyn_rpr;
};
__device__ __forceinline__ int epi_live_rows(const EpiParams& p) {
    return p.dyn_n ? min(p.m_tok, *p.dyn_n * p.dyn_rpr) : p.m_tok;
}
constexpr int kEpiTopkMax = 8;

__device__ __forceinline__ float silu_f(float x) { return x / (1.0f + __expf(-x)); }

// Apply the epilogue to the adjacent output pair (n, n+1) of token t (n even).
__device__ __forceinline__ void epi_pair(const EpiParams& p, int t, int n, float v0, float v1, int split) {
    if (t >= p.m_tok || n >= p.n_out) return;
    const bool has1 = (n + 1) < p.n_out;
    if (p.row_scale && split >= 0) {
        v0 *= p.row_scale[n] * p.tok_scale[t];
        if (has1) v1 *= p.row_scale[n + 1] * p.tok_scale[t];
    }
    switch (p.kind) {
        case EPI_F32: {
            float* o = p.out_f32 + (long long)t * p.ld_f32 + n;
            o[0] = v0;
            if (has1) o[1] = v1;
        } break;
        case EPI_BF16: {
            __nv_bfloat16* o = p.out_bf16 + (long long)t * p.ld_bf16 + n;
            o[0] = __float2bfloat16_rn(v0);
            if (has1) o[1] = __float2bfloat16_rn(v1);
        } break;
        case EPI_RESID_ADD: {
            float* o = p.out_f32 + (long long)t * p.ld_f32 + n;
            o[0] += v0;
            if (has1) o[1] += v1;
        } break;
        case EPI_SWIGLU: {
            float g = v0, u = v1;
            p.out_bf16[(long long)t * p.ld_bf16 + (n >> 1)] = __float2bfloat16_rn(silu_f(g) * u);
        } break;
        case EPI_QKV: {
            if (p.tok_slot[t] < 0) return;  // padding row: no valid position
            if (p.bias) {
                v0 += __bfloat162float(p.bias[n]);
                v1 += __bfloat162float(p.bias[n + 1]);
            }
            const int hd = p.head_dim;
            if (n < p.n_q + p.n_kvr) {  // q or k: rotate the (2i, 2i+1) pair
                const int i = (n % hd) >> 1;
                const int pos = p.tok_pos[t];
                const float c = p.rope_cos[(long long)pos * (hd >> 1) + i];
                const float s = p.rope_sin[(long long)pos * (hd >> 1) + i];
                const float r0 = v0 * c - v1 * s;
                const float r1 = v0 * s + v1 * c;
                v0 = r0;
                v1 = r1;
            }
            if (n < p.n_q) {
                __nv_bfloat162 q2 = __floats2bfloat162_rn(v0, v1);
                *reinterpret_cast<__nv_bfloat162*>(p.out_bf16 + (long long)t * p.ld_bf16 + n) = q2;
            } else {
                const int slot = p.tok_slot[t];
                if (slot < 0) return;
                const bool is_k = n < p.n_q + p.n_kvr;
                const int r = n - p.n_q - (is_k ? 0 : p.n_kvr);
                const int h = r / hd, dd = r % hd;
                long long off = (((long long)slot * p.n_kv + h) * p.max_ctx + p.tok_cidx[t]) * hd + dd;
                __nv_bfloat16* dst = (is_k ? p.kcache : p.vcache) + off;
                *reinterpret_cast<__nv_bfloat162*>(dst) = __floats2bfloat162_rn(v0, v1);
            }
        } break;
    }
}


// Vectorised epilogue for the 8 consecutive output rows n..n+7 (n % 8 == 0)
// of token t, v[] = fp32 accumulators (rows interleaved exactly as the weight
// rows). Rows >= n_out are dropped. One 16-byte (bf16) or 2x16-byte (fp32)
// store per call where the layout allows it.
__device__ __forceinline__ void epi_vec8(const EpiParams& p, int t, int n, const float (&vin)[8]) {
    if (t >= p.m_tok || n >= p.n_out) return;
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = vin[i];
    if (p.row_scale) {
        const float ts = p.tok_scale[t];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] *= p.row_scale[min(n + i, p.n_out - 1)] * ts;
    }
    if (n + 8 > p.n_out) {  // ragged tail: scalar pairs
#pragma unroll
        for (int i = 0; i < 8; i += 2) epi_pair(p, t, n + i, v[i], v[i + 1], -1);  // already scaled
        return;
    }
    switch (p.kind) {
        case EPI_F32: {
            float4* o = reinterpret_cast<float4*>(p.out_f32 + (long long)t * p.ld_f32 + n);
            o[0] = make_float4(v[0], v[1], v[2], v[3]);
            o[1] = make_float4(v[4], v[5], v[6], v[7]);
        } break;
        case EPI_RESID_ADD: {
            float4* o = reinterpret_cast<float4*>(p.out_f32 + (long long)t * p.ld_f32 + n);
            float4 a = o[0], b = o[1];
            a.x += v[0]; a.y += v[1]; a.z += v[2]; a.w += v[3];
            b.x += v[4]; b.y += v[5]; b.z += v[6]; b.w += v[7];
            o[0] = a;
            o[1] = b;
        } break;
        case EPI_BF16: {
            uint4 u;
            __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
            for (int i = 0; i < 4; ++i) h2[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
            *reinterpret_cast<uint4*>(p.out_bf16 + (long long)t * p.ld_bf16 + n) = u;
        } break;
        case EPI_SWIGLU: {
            uint2 u;
            __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
            h2[0] = __floats2bfloat162_rn(silu_f(v[0]) * v[1], silu_f(v[2]) * v[3]);
            h2[1] = __floats2bfloat162_rn(silu_f(v[4]) * v[5], silu_f(v[6]) * v[7]);
            *reinterpret_cast<uint2*>(p.out_bf16 + (long long)t * p.ld_bf16 + (n >> 1)) = u;
        } break;
        case EPI_QKV: {
            // padding rows (slot < 0: unused tree slots, padding requests of a
            // bucketed graph) carry no valid position: nothing to rotate or write
            if (p.tok_slot[t] < 0) return;
            float w[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) w[i] = v[i];
            if (p.bias) {
                const uint4 bu = *reinterpret_cast<const uint4*>(p.bias + n);
                const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&bu);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float2 f = __bfloat1622float2(b2[i]);
                    w[2 * i] += f.x;
                    w[2 * i + 1] += f.y;
                }
            }
            const int hd = p.head_dim;
            if (n < p.n_q + p.n_kvr) {  // q or k: rotate the (2i, 2i+1) pairs
                const int i0 = (n % hd) >> 1;
                const long long rb = (long long)p.tok_pos[t] * (hd >> 1) + i0;
                const float4 c = *reinterpret_cast<const float4*>(p.rope_cos + rb);
                const float4 s = *reinterpret_cast<const float4*>(p.rope_sin + rb);
                const float cc[4] = {c.x, c.y, c.z, c.w}, ss[4] = {s.x, s.y, s.z, s.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float a = w[2 * i], b = w[2 * i + 1];
                    w[2 * i] = a * cc[i] - b * ss[i];
                    w[2 * i + 1] = a * ss[i] + b * cc[i];
                }
            }
            uint4 u;
            __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
            for (int i = 0; i < 4; ++i) h2[i] = __floats2bfloat162_rn(w[2 * i], w[2 * i + 1]);
            if (n < p.n_q) {
                *reinterpret_cast<uint4*>(p.out_bf16 + (long long)t * p.ld_bf16 + n) = u;
            } else {
                const int slot = p.tok_slot[t];
                if (slot < 0) return;
                const bool is_k = n < p.n_q + p.n_kvr;
                const int r = n - p.n_q - (is_k ? 0 : p.n_kvr);
                const int h = r / hd, dd = r % hd;
                const long long off = (((long long)slot * p.n_kv + h) * p.max_ctx + p.tok_cidx[t]) * hd + dd;
                *reinterpret_cast<uint4*>((is_k ? p.kcache : p.vcache) + off) = u;
            }
        } break;
        default: {
#pragma unroll
            for (int i = 0; i < 8; i += 2) epi_pair(p, t, n + i, v[i], v[i + 1], -1);  // already scaled
        } break;
    }
}

}  // namespace tlt
