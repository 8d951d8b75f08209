/*
 * Neural leaf oracles (TEST INFRASTRUCTURE): a Llama/Qwen2-style target and a
 * one-layer EAGLE drafter in fp32 arithmetic over the same bf16 weights and
 * the same bf16 rounding points as the GPU engine. The reference contains no
 * neural model; these functions plug into the reference's own
 * seams restated in orc_discrete.c: the drafter is the NextDist of
 * build_draft_tree (spec_decode.hpp:111-113, :119) and the target provides
 * raw_row().argmax() for verify_greedy (spec_decode.hpp:251). The loop
 * orc_neural_spec_generate follows spec_generate (spec_decode.hpp:351-380).
 *
 * Model definition (shared with the GPU engine):
 *   x = embed[tok]                                   fp32 residual
 *   per layer: h = bf16(rmsnorm(x) * g_attn); qkv = h Wqkv^T (+bias), RoPE on
 *   interleaved (2i, 2i+1) pairs, q/k/v -> bf16; softmax(q k^T / sqrt(hd)) v
 *   -> bf16; x += o Wo^T; h = bf16(rmsnorm(x) * g_mlp); a = bf16(silu(g) u);
 *   x += a Wdown^T.  feature = bf16(x); logits = bf16(rmsnorm(x) * g_final) Wlm^T.
 *   Drafter row: x = [feature_prev || embed[tok]] Wfc^T, then one layer, then
 *   the shared final norm + LM head. feature_prev = the target feature of the
 *   previous position (committed positions) or the drafter output of the
 *   parent node (tree expansion, EAGLE self-feeding).
 */
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#include "../include/tlt_init.h"
#include "tlt_oracle.h"

#define TLT_EOS_TOKEN_ORC 0

typedef struct {
    uint16_t *attn_norm, *qkv, *qkv_b, *o, *mlp_norm, *gu, *down;
} orc_layer;

struct orc_model {
    orc_model_cfg c;
    tlt_init_params ip;
    uint16_t *embed, *lm_head, *final_norm, *fc;
    uint16_t* lm8;   /* drafter_lm_fp8: unscaled e4m3 values of lm_head rows (exact in bf16) */
    float* lm8_s;    /* [vocab] row scales */
    orc_layer* layers;
    orc_layer drafter;
    float *rope_cos, *rope_sin; /* [max_ctx][hd/2] */
    int n_threads;
};

struct orc_seq {
    orc_model* m;
    int32_t* tokens;
    int len;
    uint16_t **tk, **tv; /* per layer [KV][max_ctx][hd] */
    uint16_t *dk, *dv;   /* drafter layer */
    uint16_t* feat;      /* [max_ctx][d] target features */
    int tgt_kv_len, drf_kv_len;
    /* scratch */
    float *x, *h, *qkv, *att, *gu, *act, *logits;
    uint16_t* dfeat; /* drafter output features of scratch rows */
};

static inline float bf(uint16_t b) { return tlt_bf16_bits_to_f32(b); }
static inline float rbf(float f) { return tlt_bf16_bits_to_f32(tlt_f32_to_bf16_bits(f)); }

/* ------------------------------------------------------------ init ---- */
/* exact element init lives in orc_init.c (compiled with -ffp-contract=off) */
void orc_init_range(const tlt_init_params* p, uint16_t* dst, int tensor, int layer, int64_t lo, int64_t hi);

typedef struct {
    const tlt_init_params* p;
    uint16_t* dst;
    int tensor, layer;
    int64_t lo, hi;
} init_job;
static void* init_worker(void* a) {
    init_job* j = (init_job*)a;
    orc_init_range(j->p, j->dst, j->tensor, j->layer, j->lo, j->hi);
    return NULL;
}
static uint16_t* init_tensor(orc_model* m, int tensor, int layer, int64_t n) {
    uint16_t* t = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)n);
    if (!t) return NULL;
    int nt = m->n_threads > 1 && n > (1 << 20) ? m->n_threads : 1;
    pthread_t th[256];
    init_job jobs[256];
    for (int i = 0; i < nt; ++i) {
        jobs[i] = (init_job){&m->ip, t, tensor, layer, n * i / nt, n * (i + 1) / nt};
        if (nt > 1)
            pthread_create(&th[i], NULL, init_worker, &jobs[i]);
        else
            init_worker(&jobs[i]);
    }
    if (nt > 1)
        for (int i = 0; i < nt; ++i) pthread_join(th[i], NULL);
    return t;
}

static int init_layer(orc_model* m, orc_layer* L, int layer) {
    const orc_model_cfg* c = &m->c;
    int64_t d = c->hidden, nq = (int64_t)(c->heads + 2 * c->kv_heads) * c->head_dim;
    L->attn_norm = init_tensor(m, TLT_W_ATTN_NORM, layer, d);
    L->qkv = init_tensor(m, TLT_W_QKV, layer, nq * d);
    L->qkv_b = c->qkv_bias ? init_tensor(m, TLT_W_QKV_BIAS, layer, nq) : NULL;
    L->o = init_tensor(m, TLT_W_O, layer, d * c->heads * c->head_dim);
    L->mlp_norm = init_tensor(m, TLT_W_MLP_NORM, layer, d);
    L->gu = init_tensor(m, TLT_W_GATE_UP, layer, 2 * (int64_t)c->ffn * d);
    L->down = init_tensor(m, TLT_W_DOWN, layer, d * c->ffn);
    return (L->attn_norm && L->qkv && L->o && L->mlp_norm && L->gu && L->down) ? 0 : -1;
}

/* e4m3 (fn: bias 7, max 448, subnormal quantum 2^-9), round to nearest even,
 * saturating to +-448 -- __nv_cvt_float_to_fp8(x, __NV_SATFINITE, __NV_E4M3). */
static float e4m3_rne(float x) {
    const float a = fabsf(x);
    float q;
    if (!(a < 448.f)) {
        q = 448.f;
    } else if (a < 0.015625f) { /* below 2^-6: subnormals */
        q = nearbyintf(a * 512.f) / 512.f;
    } else {
        int e;
        frexpf(a, &e); /* a in [2^(e-1), 2^e) */
        const float quantum = ldexpf(1.f, e - 4);
        q = nearbyintf(a / quantum) * quantum;
    }
    return copysignf(q, x);
}

float orc_e4m3_quant_row(const float* x, int n, float* q) {
    float amax = 0.f;
    for (int i = 0; i < n; ++i) amax = fmaxf(amax, fabsf(x[i]));
    const float s = amax > 0.f ? amax / 448.0f : 1.0f; /* IEEE division, as the GPU's __fdiv_rn */
    for (int i = 0; i < n; ++i) q[i] = e4m3_rne(x[i] / s);
    return s;
}

typedef struct {
    orc_model* m;
    int64_t lo, hi;
} q8_job;
static void* q8_worker(void* a) {
    q8_job* j = (q8_job*)a;
    const int d = j->m->c.hidden;
    float* row = (float*)malloc(sizeof(float) * 2 * (size_t)d);
    if (!row) return (void*)1;
    for (int64_t v = j->lo; v < j->hi; ++v) {
        for (int i = 0; i < d; ++i) row[i] = bf(j->m->lm_head[v * d + i]);
        j->m->lm8_s[v] = orc_e4m3_quant_row(row, d, row + d);
        for (int i = 0; i < d; ++i) j->m->lm8[v * d + i] = tlt_f32_to_bf16_bits(row[d + i]); /* exact */
    }
    free(row);
    return NULL;
}

orc_model* orc_model_create(const orc_model_cfg* cfg, const orc_init_cfg* init, int n_threads) {
    orc_model* m = (orc_model*)calloc(1, sizeof(orc_model));
    if (!m) return NULL;
    m->c = *cfg;
    m->n_threads = n_threads < 1 ? 1 : (n_threads > 256 ? 256 : n_threads);
    m->ip = (tlt_init_params){init->seed, init->layer_scale, init->lm_gain, init->lm_alt, init->lm_noise, init->fc_noise,
                              cfg->vocab, cfg->hidden,      cfg->heads,    cfg->kv_heads,  cfg->head_dim, cfg->ffn};
    int64_t V = cfg->vocab, d = cfg->hidden;
    m->embed = init_tensor(m, TLT_W_EMBED, 0, V * d);
    m->lm_head = init_tensor(m, TLT_W_LM_HEAD, 0, V * d);
    m->final_norm = init_tensor(m, TLT_W_FINAL_NORM, 0, d);
    m->fc = init_tensor(m, TLT_W_FC, TLT_DRAFTER_LAYER, d * 2 * d);
    m->layers = (orc_layer*)calloc((size_t)cfg->layers, sizeof(orc_layer));
    int ok = m->embed && m->lm_head && m->final_norm && m->fc && m->layers;
    for (int l = 0; ok && l < cfg->layers; ++l) ok = init_layer(m, &m->layers[l], l) == 0;
    if (ok) ok = init_layer(m, &m->drafter, TLT_DRAFTER_LAYER) == 0;
    if (ok && init->drafter_lm_fp8) {
        m->lm8 = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(V * d));
        m->lm8_s = (float*)malloc(sizeof(float) * (size_t)V);
        ok = m->lm8 && m->lm8_s;
        int nt = m->n_threads;
        pthread_t th[256];
        q8_job jobs[256];
        for (int i = 0; ok && i < nt; ++i) {
            jobs[i] = (q8_job){m, V * i / nt, V * (i + 1) / nt};
            if (nt > 1)
                pthread_create(&th[i], NULL, q8_worker, &jobs[i]);
            else if (q8_worker(&jobs[i]) != NULL)
                ok = 0;
        }
        if (ok && nt > 1)
            for (int i = 0; i < nt; ++i) {
                void* rc = NULL;
                pthread_join(th[i], &rc);
                if (rc) ok = 0;
            }
    }
    /* RoPE table: angle = pos * theta^(-2i/hd) in double, stored fp32 */
    int half = cfg->head_dim / 2;
    m->rope_cos = (float*)malloc(sizeof(float) * (size_t)cfg->max_ctx * (size_t)half);
    m->rope_sin = (float*)malloc(sizeof(float) * (size_t)cfg->max_ctx * (size_t)half);
    if (!m->rope_cos || !m->rope_sin) ok = 0;
    for (int pos = 0; ok && pos < cfg->max_ctx; ++pos)
        for (int i = 0; i < half; ++i) {
            double inv = pow((double)cfg->rope_theta, -2.0 * (double)i / (double)cfg->head_dim);
            double ang = (double)pos * inv;
            m->rope_cos[(size_t)pos * half + i] = (float)cos(ang);
            m->rope_sin[(size_t)pos * half + i] = (float)sin(ang);
        }
    if (!ok) {
        orc_model_destroy(m);
        return NULL;
    }
    return m;
}

static void free_layer(orc_layer* L) {
    free(L->attn_norm);
    free(L->qkv);
    free(L->qkv_b);
    free(L->o);
    free(L->mlp_norm);
    free(L->gu);
    free(L->down);
}
void orc_model_set_threads(orc_model* m, int n_threads) {
    m->n_threads = n_threads < 1 ? 1 : (n_threads > 256 ? 256 : n_threads);
}

void orc_model_destroy(orc_model* m) {
    if (!m) return;
    free(m->embed);
    free(m->lm_head);
    free(m->lm8);
    free(m->lm8_s);
    free(m->final_norm);
    free(m->fc);
    if (m->layers)
        for (int l = 0; l < m->c.layers; ++l) free_layer(&m->layers[l]);
    free(m->layers);
    free_layer(&m->drafter);
    free(m->rope_cos);
    free(m->rope_sin);
    free(m);
}

int orc_model_weight(orc_model* m, int tensor_id, int layer, const uint16_t** ptr, int64_t* n) {
    const orc_model_cfg* c = &m->c;
    int64_t d = c->hidden, nq = (int64_t)(c->heads + 2 * c->kv_heads) * c->head_dim;
    orc_layer* L = layer == TLT_DRAFTER_LAYER ? &m->drafter : (layer >= 0 && layer < c->layers ? &m->layers[layer] : NULL);
    switch (tensor_id) {
        case TLT_W_EMBED: *ptr = m->embed; *n = (int64_t)c->vocab * d; return 0;
        case TLT_W_LM_HEAD: *ptr = m->lm_head; *n = (int64_t)c->vocab * d; return 0;
        case TLT_W_FINAL_NORM: *ptr = m->final_norm; *n = d; return 0;
        case TLT_W_FC: *ptr = m->fc; *n = 2 * d * d; return 0;
        default: break;
    }
    if (!L) return -1;
    switch (tensor_id) {
        case TLT_W_ATTN_NORM: *ptr = L->attn_norm; *n = d; return 0;
        case TLT_W_QKV: *ptr = L->qkv; *n = nq * d; return 0;
        case TLT_W_QKV_BIAS: *ptr = L->qkv_b; *n = L->qkv_b ? nq : 0; return 0;
        case TLT_W_O: *ptr = L->o; *n = d * c->heads * c->head_dim; return 0;
        case TLT_W_MLP_NORM: *ptr = L->mlp_norm; *n = d; return 0;
        case TLT_W_GATE_UP: *ptr = L->gu; *n = 2 * (int64_t)c->ffn * d; return 0;
        case TLT_W_DOWN: *ptr = L->down; *n = d * c->ffn; return 0;
        default: return -1;
    }
}

/* --------------------------------------------------------- matmul ---- */
/* y[t][j] = sum_k x[t][k] * W[j][k], W bf16, x/y fp32; threads split j. */
typedef struct {
    const float* x;
    int n, K;
    const uint16_t* W;
    int N;
    float* y;
    int lo, hi;
    int accumulate;
} mm_job;
static void* mm_worker(void* a) {
    mm_job* j = (mm_job*)a;
    float* wf = (float*)malloc(sizeof(float) * (size_t)j->K);
    for (int o = j->lo; o < j->hi; ++o) {
        const uint16_t* w = j->W + (size_t)o * (size_t)j->K;
        for (int k = 0; k < j->K; ++k) wf[k] = bf(w[k]);
        for (int t = 0; t < j->n; ++t) {
            const float* xr = j->x + (size_t)t * (size_t)j->K;
            /* 16 independent partial sums: vectorizable without reassociation */
            float acc[16] = {0};
            int k = 0;
            for (; k + 16 <= j->K; k += 16)
                for (int u = 0; u < 16; ++u) acc[u] += xr[k + u] * wf[k + u];
            float s = 0.f;
            for (int u = 0; u < 16; ++u) s += acc[u];
            for (; k < j->K; ++k) s += xr[k] * wf[k];
            if (j->accumulate)
                j->y[(size_t)t * j->N + o] += s;
            else
                j->y[(size_t)t * j->N + o] = s;
        }
    }
    free(wf);
    return NULL;
}
static void mm(orc_model* m, const float* x, int n, int K, const uint16_t* W, int N, float* y, int accumulate) {
    int nt = m->n_threads;
    if ((double)n * K * N < 4e6) nt = 1;
    if (nt > N) nt = N;
    pthread_t th[256];
    mm_job jobs[256];
    for (int i = 0; i < nt; ++i) {
        jobs[i] = (mm_job){x, n, K, W, N, y, (int)((int64_t)N * i / nt), (int)((int64_t)N * (i + 1) / nt), accumulate};
        if (nt > 1)
            pthread_create(&th[i], NULL, mm_worker, &jobs[i]);
        else
            mm_worker(&jobs[i]);
    }
    if (nt > 1)
        for (int i = 0; i < nt; ++i) pthread_join(th[i], NULL);
}

/* h = bf16(x * rsqrt(mean(x^2) + eps) * g) */
static void rmsnorm(const float* x, const uint16_t* g, int d, float eps, float* h) {
    float ss = 0.f;
    for (int i = 0; i < d; ++i) ss += x[i] * x[i];
    float r = 1.0f / sqrtf(ss / (float)d + eps);
    for (int i = 0; i < d; ++i) h[i] = rbf(x[i] * r * bf(g[i]));
}

/* -------------------------------------------------------- seq state ---- */
orc_seq* orc_seq_create(orc_model* m) {
    const orc_model_cfg* c = &m->c;
    orc_seq* s = (orc_seq*)calloc(1, sizeof(orc_seq));
    if (!s) return NULL;
    s->m = m;
    size_t kv = (size_t)c->kv_heads * (size_t)c->max_ctx * (size_t)c->head_dim;
    s->tokens = (int32_t*)calloc((size_t)c->max_ctx, sizeof(int32_t));
    s->tk = (uint16_t**)calloc((size_t)c->layers, sizeof(uint16_t*));
    s->tv = (uint16_t**)calloc((size_t)c->layers, sizeof(uint16_t*));
    for (int l = 0; l < c->layers; ++l) {
        s->tk[l] = (uint16_t*)calloc(kv, sizeof(uint16_t));
        s->tv[l] = (uint16_t*)calloc(kv, sizeof(uint16_t));
    }
    s->dk = (uint16_t*)calloc(kv, sizeof(uint16_t));
    s->dv = (uint16_t*)calloc(kv, sizeof(uint16_t));
    s->feat = (uint16_t*)calloc((size_t)c->max_ctx * (size_t)c->hidden, sizeof(uint16_t));
    int rows = 512; /* scratch rows per block */
    int nq = (c->heads + 2 * c->kv_heads) * c->head_dim;
    s->x = (float*)malloc(sizeof(float) * (size_t)rows * (size_t)(2 * c->hidden));
    s->h = (float*)malloc(sizeof(float) * (size_t)rows * (size_t)(2 * c->hidden));
    s->qkv = (float*)malloc(sizeof(float) * (size_t)rows * (size_t)nq);
    s->att = (float*)malloc(sizeof(float) * (size_t)rows * (size_t)(c->heads * c->head_dim));
    s->gu = (float*)malloc(sizeof(float) * (size_t)rows * (size_t)(2 * c->ffn));
    s->act = (float*)malloc(sizeof(float) * (size_t)rows * (size_t)c->ffn);
    s->logits = (float*)malloc(sizeof(float) * (size_t)c->vocab);
    s->dfeat = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(c->max_ctx) * (size_t)c->hidden);
    return s;
}
void orc_seq_destroy(orc_seq* s) {
    if (!s) return;
    for (int l = 0; l < s->m->c.layers; ++l) {
        free(s->tk[l]);
        free(s->tv[l]);
    }
    free(s->tk);
    free(s->tv);
    free(s->dk);
    free(s->dv);
    free(s->feat);
    free(s->tokens);
    free(s->x);
    free(s->h);
    free(s->qkv);
    free(s->att);
    free(s->gu);
    free(s->act);
    free(s->logits);
    free(s->dfeat);
    free(s);
}
int orc_seq_len(orc_seq* s) { return s->len; }
int orc_seq_append(orc_seq* s, const int32_t* toks, int n) {
    if (s->len + n > s->m->c.max_ctx) return -1;
    memcpy(s->tokens + s->len, toks, sizeof(int32_t) * (size_t)n);
    s->len += n;
    return 0;
}

/* One decoder layer over n rows at positions base..base+n-1 (causal among
 * them, full view of [0, base)). x: [n][d] fp32 residual, updated in place. */
static void layer_rows(orc_seq* s, const orc_layer* L, uint16_t* kc, uint16_t* vc, float* x, int n, int base) {
    orc_model* m = s->m;
    const orc_model_cfg* c = &m->c;
    const int d = c->hidden, H = c->heads, KV = c->kv_heads, hd = c->head_dim, F = c->ffn;
    const int nq = H * hd, nkv = KV * hd, ntot = nq + 2 * nkv, half = hd / 2;
    float* h = s->h;
    for (int t = 0; t < n; ++t) rmsnorm(x + (size_t)t * d, L->attn_norm, d, c->rms_eps, h + (size_t)t * d);
    mm(m, h, n, d, L->qkv, ntot, s->qkv, 0);
    for (int t = 0; t < n; ++t) {
        float* r = s->qkv + (size_t)t * ntot;
        int pos = base + t;
        for (int j = 0; j < ntot; j += 2) {
            float v0 = r[j], v1 = r[j + 1];
            if (L->qkv_b) {
                v0 += bf(L->qkv_b[j]);
                v1 += bf(L->qkv_b[j + 1]);
            }
            if (j < nq + nkv) {
                int i = (j % hd) >> 1;
                float cs = m->rope_cos[(size_t)pos * half + i], sn = m->rope_sin[(size_t)pos * half + i];
                float r0 = v0 * cs - v1 * sn, r1 = v0 * sn + v1 * cs;
                v0 = r0;
                v1 = r1;
            }
            r[j] = rbf(v0);
            r[j + 1] = rbf(v1);
        }
        for (int g = 0; g < KV; ++g)
            for (int e = 0; e < hd; ++e) {
                size_t off = ((size_t)g * c->max_ctx + pos) * hd + e;
                kc[off] = tlt_f32_to_bf16_bits(r[nq + g * hd + e]);
                vc[off] = tlt_f32_to_bf16_bits(r[nq + nkv + g * hd + e]);
            }
    }
    const float scale = 1.0f / sqrtf((float)hd);
    float* sc = (float*)malloc(sizeof(float) * (size_t)(base + n));
    for (int t = 0; t < n; ++t) {
        int pos = base + t;
        const float* q = s->qkv + (size_t)t * ntot;
        for (int hh = 0; hh < H; ++hh) {
            int g = hh / (H / KV);
            const float* qh = q + hh * hd;
            float mx = -INFINITY;
            for (int j = 0; j <= pos; ++j) {
                const uint16_t* kr = kc + ((size_t)g * c->max_ctx + j) * hd;
                float dot = 0.f;
                for (int e = 0; e < hd; ++e) dot += qh[e] * bf(kr[e]);
                sc[j] = dot * scale;
                if (sc[j] > mx) mx = sc[j];
            }
            float sum = 0.f;
            for (int j = 0; j <= pos; ++j) {
                sc[j] = expf(sc[j] - mx);
                sum += sc[j];
            }
            float* o = s->att + (size_t)t * nq + hh * hd;
            for (int e = 0; e < hd; ++e) o[e] = 0.f;
            for (int j = 0; j <= pos; ++j) {
                const uint16_t* vr = vc + ((size_t)g * c->max_ctx + j) * hd;
                float w = sc[j];
                for (int e = 0; e < hd; ++e) o[e] += w * bf(vr[e]);
            }
            for (int e = 0; e < hd; ++e) o[e] = rbf(o[e] / sum);
        }
    }
    free(sc);
    mm(m, s->att, n, nq, L->o, d, x, 1);
    for (int t = 0; t < n; ++t) rmsnorm(x + (size_t)t * d, L->mlp_norm, d, c->rms_eps, h + (size_t)t * d);
    mm(m, h, n, d, L->gu, 2 * F, s->gu, 0);
    for (int t = 0; t < n; ++t)
        for (int f = 0; f < F; ++f) {
            float g = s->gu[(size_t)t * 2 * F + 2 * f], u = s->gu[(size_t)t * 2 * F + 2 * f + 1];
            s->act[(size_t)t * F + f] = rbf(g / (1.0f + expf(-g)) * u);
        }
    mm(m, s->act, n, F, L->down, d, x, 1);
}

/* drafter && lm8: the e4m3 drafter LM head (engine drafter_logits with
 * drafter_fp8_): the normed row and the weight rows quantised per row, fp32
 * dot products of the e4m3 values, then x (row scale x token scale) as the
 * GEMM epilogue applies it (gemm.cuh epi_vec8, row_scale / tok_scale). */
static void lm_logits(orc_seq* s, const float* x_row, float* logits, int drafter) {
    orc_model* m = s->m;
    const int d = m->c.hidden;
    float* h = (float*)malloc(sizeof(float) * 2 * (size_t)d);
    rmsnorm(x_row, m->final_norm, d, m->c.rms_eps, h);
    if (drafter && m->lm8) {
        const float sh = orc_e4m3_quant_row(h, d, h + d);
        mm(m, h + d, 1, d, m->lm8, m->c.vocab, logits, 0);
        for (int v = 0; v < m->c.vocab; ++v) logits[v] *= m->lm8_s[v] * sh;
    } else {
        mm(m, h, 1, d, m->lm_head, m->c.vocab, logits, 0);
    }
    free(h);
}

/* Target rows for toks at positions base.. (writes KV there). Features of the
 * rows go to feat_out ([n][d] bf16) when non-NULL; logits of the last row. */
static int target_rows(orc_seq* s, const int32_t* toks, int n, int base, uint16_t* feat_out, float* logits) {
    orc_model* m = s->m;
    const int d = m->c.hidden;
    if (n > 512 || base + n > m->c.max_ctx) return -1;
    float* x = s->x;
    for (int t = 0; t < n; ++t)
        for (int i = 0; i < d; ++i) x[(size_t)t * d + i] = bf(m->embed[(size_t)toks[t] * d + i]);
    for (int l = 0; l < m->c.layers; ++l) layer_rows(s, &m->layers[l], s->tk[l], s->tv[l], x, n, base);
    if (feat_out)
        for (int t = 0; t < n; ++t)
            for (int i = 0; i < d; ++i) feat_out[(size_t)t * d + i] = tlt_f32_to_bf16_bits(x[(size_t)t * d + i]);
    if (logits) lm_logits(s, x + (size_t)(n - 1) * d, logits, 0);
    return 0;
}

/* Drafter rows: inputs (prev_feat[t], embed[toks[t]]) at positions base+t,
 * processed one block (causal). out_feat [n][d] bf16; logits of last row. */
static int drafter_rows(orc_seq* s, const uint16_t* prev_feat, const int32_t* toks, int n, int base,
                        uint16_t* out_feat, float* logits) {
    orc_model* m = s->m;
    const int d = m->c.hidden;
    if (n > 512 || base + n > m->c.max_ctx) return -1;
    float* in = s->h; /* [n][2d] reused before layer_rows overwrites s->h */
    float* x = s->x;
    for (int t = 0; t < n; ++t) {
        for (int i = 0; i < d; ++i) in[(size_t)t * 2 * d + i] = prev_feat ? bf(prev_feat[(size_t)t * d + i]) : 0.f;
        for (int i = 0; i < d; ++i) in[(size_t)t * 2 * d + d + i] = bf(m->embed[(size_t)toks[t] * d + i]);
    }
    /* copy input aside: mm reads `in` while writing x */
    float* xin = (float*)malloc(sizeof(float) * (size_t)n * 2 * d);
    memcpy(xin, in, sizeof(float) * (size_t)n * 2 * d);
    mm(m, xin, n, 2 * d, m->fc, d, x, 0);
    free(xin);
    layer_rows(s, &m->drafter, s->dk, s->dv, x, n, base);
    if (out_feat)
        for (int t = 0; t < n; ++t)
            for (int i = 0; i < d; ++i) out_feat[(size_t)t * d + i] = tlt_f32_to_bf16_bits(x[(size_t)t * d + i]);
    if (logits) lm_logits(s, x + (size_t)(n - 1) * d, logits, 1);
    return 0;
}

/* Commit target KV/features for positions [tgt_kv_len, len-1). */
static int ensure_target(orc_seq* s) {
    while (s->tgt_kv_len < s->len - 1) {
        int n = s->len - 1 - s->tgt_kv_len;
        if (n > 512) n = 512;
        const int d = s->m->c.hidden;
        if (target_rows(s, s->tokens + s->tgt_kv_len, n, s->tgt_kv_len, s->feat + (size_t)s->tgt_kv_len * d, NULL))
            return -1;
        s->tgt_kv_len += n;
    }
    return 0;
}
/* Commit drafter KV for positions [drf_kv_len, len-1) from target features. */
static int ensure_drafter(orc_seq* s) {
    if (ensure_target(s)) return -1;
    const int d = s->m->c.hidden;
    while (s->drf_kv_len < s->len - 1) {
        int n = s->len - 1 - s->drf_kv_len;
        if (n > 512) n = 512;
        int b = s->drf_kv_len;
        uint16_t* pf = (uint16_t*)calloc((size_t)n * d, sizeof(uint16_t));
        for (int t = 0; t < n; ++t)
            if (b + t > 0) memcpy(pf + (size_t)t * d, s->feat + (size_t)(b + t - 1) * d, sizeof(uint16_t) * (size_t)d);
        int rc = drafter_rows(s, pf, s->tokens + b, n, b, NULL, NULL);
        free(pf);
        if (rc) return -1;
        s->drf_kv_len += n;
    }
    return 0;
}

int orc_target_extend(orc_seq* s, const int32_t* toks, int n, float* logits_last) {
    if (orc_seq_append(s, toks, n)) return -1;
    if (ensure_target(s)) return -1;
    if (logits_last) return orc_target_logits_path(s, NULL, 0, logits_last);
    return 0;
}

int orc_target_logits_path(orc_seq* s, const int32_t* path, int n, float* logits) {
    if (s->len < 1 || ensure_target(s)) return -1;
    int32_t rows[512];
    if (n + 1 > 512) return -1;
    rows[0] = s->tokens[s->len - 1];
    for (int i = 0; i < n; ++i) rows[i + 1] = path[i];
    return target_rows(s, rows, n + 1, s->len - 1, NULL, logits);
}

/* fp64 softmax of fp32 logits: M = max, S = sum expf(l - M) (fp32),
 * p = exp((double)(l - M)) / S  (same formula as the GPU). */
static void softmax64(const float* l, int v, double* p) {
    float M = l[0];
    for (int i = 1; i < v; ++i)
        if (l[i] > M) M = l[i];
    float S = 0.f;
    for (int i = 0; i < v; ++i) S += expf(l[i] - M);
    for (int i = 0; i < v; ++i) p[i] = exp((double)(l[i] - M)) / (double)S;
}

int orc_drafter_row(orc_seq* s, const int32_t* path, int n, double* probs, float* logits_out) {
    if (s->len < 1 || ensure_drafter(s)) return -1;
    orc_model* m = s->m;
    const int d = m->c.hidden;
    int base = s->len - 1;
    /* root row: (f_{base-1}, e(x_base)) */
    uint16_t* pf = base > 0 ? s->feat + (size_t)(base - 1) * d : NULL;
    float* lg = s->logits;
    int32_t tok = s->tokens[base];
    if (drafter_rows(s, pf, &tok, 1, base, s->dfeat, n == 0 ? lg : NULL)) return -1;
    for (int i = 0; i < n; ++i) {
        if (drafter_rows(s, s->dfeat + (size_t)i * d, &path[i], 1, base + 1 + i, s->dfeat + (size_t)(i + 1) * d,
                         i == n - 1 ? lg : NULL))
            return -1;
    }
    if (logits_out) memcpy(logits_out, lg, sizeof(float) * (size_t)m->c.vocab);
    if (probs) softmax64(lg, m->c.vocab, probs);
    return 0;
}

int orc_seq_features(orc_seq* s, int from, int n, uint16_t* out) {
    if (from < 0 || n < 0 || ensure_target(s) || from + n > s->tgt_kv_len) return -1;
    const size_t d = (size_t)s->m->c.hidden;
    memcpy(out, s->feat + (size_t)from * d, sizeof(uint16_t) * (size_t)n * d);
    return 0;
}

int orc_seq_truncate(orc_seq* s, int len) {
    if (len < 0 || len > s->len) return -1;
    s->len = len;
    if (s->tgt_kv_len > len - 1) s->tgt_kv_len = len > 0 ? len - 1 : 0;
    if (s->drf_kv_len > len - 1) s->drf_kv_len = len > 0 ? len - 1 : 0;
    return 0;
}

/* ---------------------------------------------------- SD generation ---- */
static int drafter_cb(void* user, const int32_t* path, int n, double* out) {
    return orc_drafter_row((orc_seq*)user, path, n, out, NULL);
}
static int32_t target_argmax_cb(void* user, const int32_t* path, int n) {
    orc_seq* s = (orc_seq*)user;
    if (orc_target_logits_path(s, path, n, s->logits)) return -1;
    int v = s->m->c.vocab, best = 0;
    for (int i = 1; i < v; ++i)
        if (s->logits[i] > s->logits[best]) best = i;
    return best;
}

int orc_neural_spec_generate(orc_model* m, const int32_t* prompt, int prompt_len, int max_len,
                             const orc_strategy* st, int32_t* out_tokens, int* out_len, int32_t* accept_lens,
                             orc_node* trees, int32_t* tree_sizes, int max_steps) {
    orc_seq* s = orc_seq_create(m);
    if (!s || orc_seq_append(s, prompt, prompt_len)) return -1;
    int T = st->tokens_to_verify, gen = 0, steps = 0, rc = 0;
    orc_node* tree = (orc_node*)malloc(sizeof(orc_node) * (size_t)T);
    while (gen < max_len && steps < max_steps) { /* spec_decode.hpp:357 */
        int n = orc_build_draft_tree(drafter_cb, s, m->c.vocab, st, tree);
        if (n < 0) {
            rc = -1;
            break;
        }
        orc_accept res;
        if (orc_verify_greedy(target_argmax_cb, s, tree, n, &res)) {
            rc = -1;
            break;
        }
        if (trees) memcpy(trees + (size_t)steps * T, tree, sizeof(orc_node) * (size_t)n);
        if (tree_sizes) tree_sizes[steps] = n;
        accept_lens[steps++] = res.accept_length;
        int done = 0;
        for (int i = 0; i <= res.accept_length && !done; ++i) { /* :366-377 */
            int32_t t = i < res.accept_length ? res.accepted[i] : res.bonus;
            out_tokens[gen++] = t;
            orc_seq_append(s, &t, 1);
            if (t == TLT_EOS_TOKEN_ORC || gen >= max_len) done = 1;
        }
        if (done) break;
    }
    *out_len = gen;
    free(tree);
    orc_seq_destroy(s);
    return rc ? rc : steps;
}

/* Stochastic-path rows: same as softmax64 but the normalizer is a double sum
 * (rows sum to 1 within 1e-15, matching the GPU stochastic kernels). */
static void softmax64d(const float* l, int v, double* p) {
    float M = l[0];
    for (int i = 1; i < v; ++i)
        if (l[i] > M) M = l[i];
    double S = 0.0;
    for (int i = 0; i < v; ++i) {
        p[i] = exp((double)(l[i] - M));
        S += p[i];
    }
    for (int i = 0; i < v; ++i) p[i] /= S;
}
static int drafter_d_cb(void* user, const int32_t* path, int n, double* out) {
    orc_seq* s = (orc_seq*)user;
    if (orc_drafter_row(s, path, n, NULL, s->logits)) return -1;
    softmax64d(s->logits, s->m->c.vocab, out);
    return 0;
}
static int target_raw_cb(void* user, const int32_t* path, int n, double* out) {
    orc_seq* s = (orc_seq*)user;
    if (orc_target_logits_path(s, path, n, s->logits)) return -1;
    softmax64d(s->logits, s->m->c.vocab, out);
    return 0;
}

/* Rejection-sampling SD generate (spec_generate in StochasticLinear mode,
 * spec_decode.hpp:351-380): build_sampled_chain over the EAGLE drafter,
 * verify_stochastic over the neural target, uniforms from
 * RngStream(seed, stream). Returns #steps. */
int orc_neural_spec_generate_stochastic(orc_model* m, const int32_t* prompt, int prompt_len, int max_len, int depth,
                                        double temperature, uint64_t seed, uint64_t stream, int32_t* out_tokens,
                                        int* out_len, int32_t* accept_lens, int max_steps) {
    orc_seq* s = orc_seq_create(m);
    if (!s || orc_seq_append(s, prompt, prompt_len)) return -1;
    orc_rng r;
    orc_rng_init(&r, seed, stream);
    orc_usrc u = {&r, NULL, 0, 0};
    const int V = m->c.vocab;
    orc_node* chain = (orc_node*)malloc(sizeof(orc_node) * (size_t)depth);
    double* dd = (double*)malloc(sizeof(double) * (size_t)depth * (size_t)V);
    int gen = 0, steps = 0, rc = 0;
    while (gen < max_len && steps < max_steps) {
        if (orc_build_sampled_chain(drafter_d_cb, s, V, depth, &u, chain, dd) != depth) {
            rc = -1;
            break;
        }
        orc_accept res;
        if (orc_verify_stochastic(target_raw_cb, s, V, temperature, chain, depth, dd, &u, &res)) {
            rc = -1;
            break;
        }
        accept_lens[steps++] = res.accept_length;
        int done = 0;
        for (int i = 0; i <= res.accept_length && !done; ++i) {
            int32_t t = i < res.accept_length ? res.accepted[i] : res.bonus;
            out_tokens[gen++] = t;
            orc_seq_append(s, &t, 1);
            if (t == TLT_EOS_TOKEN_ORC || gen >= max_len) done = 1;
        }
        if (done) break;
    }
    *out_len = gen;
    free(chain);
    free(dd);
    orc_seq_destroy(s);
    return rc ? rc : steps;
}

int orc_neural_generate_ar(orc_model* m, const int32_t* prompt, int prompt_len, int max_len, int32_t* out_tokens) {
    orc_seq* s = orc_seq_create(m);
    if (!s || orc_seq_append(s, prompt, prompt_len)) return -1;
    int gen = 0;
    while (gen < max_len) { /* token_model.hpp:195-201 at temperature 0 */
        int32_t t = target_argmax_cb(s, NULL, 0);
        if (t < 0) break;
        out_tokens[gen++] = t;
        orc_seq_append(s, &t, 1);
        if (t == TLT_EOS_TOKEN_ORC) break;
    }
    orc_seq_destroy(s);
    return gen;
}
