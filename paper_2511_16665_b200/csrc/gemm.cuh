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
};
constexpr int kEpiTopkMax = 8;

__device__ __forceinline__ float silu_f(float x) { return x / (1.0f + __expf(-x)); }

// Apply the epilogue to the adjacent output pair (n, n+1) of token t (n even).
__device__ __forceinline__ void epi_pair(const EpiParams& p, int t, int n, float v0, float v1, int split) {
    if (t >= p.m_tok || n >= p.n_out) return;
    const bool has1 = (n + 1) < p.n_out;
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

}  // namespace tlt
