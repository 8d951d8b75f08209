/*
 * tlt_init.h — definition of the seeded synthetic random-init weights.
 *
 * There are no checkpoints offline, so the Qwen2.5-shaped target and the
 * EAGLE drafter are random-init. Every weight element is a pure function of
 * (seed, tensor id, layer, element index) through a counter hash, evaluated
 * with single, non-contracted fp32 operations and round-to-nearest-even to
 * bf16, so the GPU engine (init kernel) and the CPU oracle produce the SAME
 * bits without copying weights around. This header is the input definition
 * shared by both sides (like a seed), not the algorithm under test.
 *
 * Structure knob (SURVEY.md §7 "Random-init acceptance"): attention/MLP output
 * projections scale with layer_scale (small => the residual stream is
 * dominated by the token embedding), the LM head is lm_gain x a permuted copy
 * of the embedding plus lm_noise x noise (a bigram backbone), and the drafter
 * fc starts as the embedding passthrough plus fc_noise x noise. Target and
 * drafter then share the bigram argmax structure and disagree where the
 * context-dependent residual updates move the target's argmax.
 */
#ifndef TLT_INIT_H
#define TLT_INIT_H

#include <stdint.h>
#ifndef __CUDACC__
#include <math.h>
#endif

#ifdef __CUDACC__
#define TLT_HD __host__ __device__ __forceinline__
#else
#define TLT_HD static inline
#endif

/* tensor ids */
enum {
    TLT_W_EMBED = 0,      /* [V][d] */
    TLT_W_LM_HEAD = 1,    /* [V][d] */
    TLT_W_FINAL_NORM = 2, /* [d] */
    TLT_W_ATTN_NORM = 3,  /* [d] per layer */
    TLT_W_QKV = 4,        /* [(H+2KV)hd][d] rows: q heads, k heads, v heads */
    TLT_W_QKV_BIAS = 5,   /* [(H+2KV)hd] */
    TLT_W_O = 6,          /* [d][H hd] */
    TLT_W_MLP_NORM = 7,   /* [d] */
    TLT_W_GATE_UP = 8,    /* [2F][d] rows interleaved: 2f = gate_f, 2f+1 = up_f */
    TLT_W_DOWN = 9,       /* [d][F] */
    TLT_W_FC = 10         /* drafter [d][2d], input = [feature || embedding] */
};
#define TLT_DRAFTER_LAYER 1000 /* layer index of the EAGLE decoder layer */

/* LM-head backbone permutation: row y copies embedding row perm(y). */
#define TLT_PERM_A 1000003ULL
#define TLT_PERM_B 12345ULL
#define TLT_PERM_A2 999983ULL
#define TLT_PERM_B2 54321ULL

TLT_HD uint64_t tlt_mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xbf58476d1ce4e5b9ULL;
    z ^= z >> 27;
    z *= 0x94d049bb133111ebULL;
    z ^= z >> 31;
    return z;
}

/* uniform r in [-1, 1) with 24-bit resolution (exact in fp32) */
TLT_HD float tlt_hash_unit(uint64_t seed, int tensor, int layer, int64_t idx) {
    uint64_t base = tlt_mix64(seed ^ (0x100000001B3ULL * (uint64_t)(tensor * 4096 + layer + 1)));
    uint64_t h = tlt_mix64(base + (uint64_t)idx * 0x9E3779B97F4A7C15ULL);
    uint32_t u24 = (uint32_t)(h >> 40);
    return (float)((int32_t)u24 - (1 << 23)) * (1.0f / 8388608.0f);
}

TLT_HD uint16_t tlt_f32_to_bf16_bits(float f) {
    union {
        float f;
        uint32_t u;
    } v;
    v.f = f;
    if ((v.u & 0x7f800000u) == 0x7f800000u) return (uint16_t)((v.u >> 16) | ((v.u & 0xffffu) ? 0x40u : 0u));
    uint32_t lsb = (v.u >> 16) & 1u;
    v.u += 0x7fffu + lsb;
    return (uint16_t)(v.u >> 16);
}
TLT_HD float tlt_bf16_bits_to_f32(uint16_t b) {
    union {
        uint32_t u;
        float f;
    } v;
    v.u = ((uint32_t)b) << 16;
    return v.f;
}

/* explicit single-rounding ops (no FMA contraction on either side) */
#ifdef __CUDA_ARCH__
#define TLT_FMUL(a, b) __fmul_rn((a), (b))
#define TLT_FADD(a, b) __fadd_rn((a), (b))
#else
#define TLT_FMUL(a, b) ((float)((float)(a) * (float)(b)))
#define TLT_FADD(a, b) ((float)((float)(a) + (float)(b)))
#endif

typedef struct {
    uint64_t seed;
    float layer_scale, lm_gain, lm_alt, lm_noise, fc_noise;
    int vocab, hidden, heads, kv_heads, head_dim, ffn;
} tlt_init_params;

/* Weight element value as bf16 bits. `cols` is the row length of the tensor. */
TLT_HD uint16_t tlt_init_elem(const tlt_init_params* p, int tensor, int layer, int64_t idx) {
    const float sqrt3 = 1.7320508075688772f;
    const int d = p->hidden;
    float r = tlt_hash_unit(p->seed, tensor, layer, idx);
    float v;
    switch (tensor) {
        case TLT_W_EMBED:
            v = TLT_FMUL(sqrt3, r);
            break;
        case TLT_W_LM_HEAD: {
            int64_t y = idx / d, i = idx % d;
            if (y == 0) { /* EOS row: logit 0, never the argmax of the structured head */
                v = 0.0f;
                break;
            }
            /* two successors per token: y is the primary continuation of
             * perm1(y) and the alternative continuation of perm2(y) */
            int64_t s1 = (int64_t)((TLT_PERM_A * (uint64_t)y + TLT_PERM_B) % (uint64_t)p->vocab);
            int64_t s2 = (int64_t)((TLT_PERM_A2 * (uint64_t)y + TLT_PERM_B2) % (uint64_t)p->vocab);
            float e1 = tlt_bf16_bits_to_f32(
                tlt_f32_to_bf16_bits(TLT_FMUL(sqrt3, tlt_hash_unit(p->seed, TLT_W_EMBED, 0, s1 * d + i))));
            float e2 = tlt_bf16_bits_to_f32(
                tlt_f32_to_bf16_bits(TLT_FMUL(sqrt3, tlt_hash_unit(p->seed, TLT_W_EMBED, 0, s2 * d + i))));
            float a = TLT_FMUL(p->lm_gain, 1.0f / (float)d);
            float a2 = TLT_FMUL(a, p->lm_alt);
            float b = TLT_FMUL(p->lm_noise, 1.0f / (float)d);
            v = TLT_FADD(TLT_FADD(TLT_FMUL(a, e1), TLT_FMUL(a2, e2)), TLT_FMUL(TLT_FMUL(b, sqrt3), r));
        } break;
        case TLT_W_FINAL_NORM:
        case TLT_W_ATTN_NORM:
        case TLT_W_MLP_NORM:
            v = TLT_FADD(1.0f, TLT_FMUL(0.1f, r));
            break;
        case TLT_W_QKV:
        case TLT_W_GATE_UP:
            v = TLT_FMUL(TLT_FMUL(sqrt3, 1.0f / sqrtf((float)d)), r);
            break;
        case TLT_W_QKV_BIAS:
            v = TLT_FMUL(0.1f, r);
            break;
        case TLT_W_O:
            v = TLT_FMUL(TLT_FMUL(p->layer_scale, TLT_FMUL(sqrt3, 1.0f / sqrtf((float)(p->heads * p->head_dim)))), r);
            break;
        case TLT_W_DOWN:
            v = TLT_FMUL(TLT_FMUL(p->layer_scale, TLT_FMUL(sqrt3, 1.0f / sqrtf((float)p->ffn))), r);
            break;
        case TLT_W_FC: {
            int64_t row = idx / (2 * d), col = idx % (2 * d);
            float noise = TLT_FMUL(TLT_FMUL(p->fc_noise, TLT_FMUL(sqrt3, 1.0f / sqrtf((float)(2 * d)))), r);
            v = (col == d + row) ? TLT_FADD(1.0f, noise) : noise;
        } break;
        default:
            v = 0.0f;
    }
    return tlt_f32_to_bf16_bits(v);
}

#endif /* TLT_INIT_H */
