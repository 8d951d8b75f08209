/*
 * Exact synthetic-weight element init (TEST INFRASTRUCTURE). Compiled with
 * -ffp-contract=off so every fp32 op of include/tlt_init.h rounds once,
 * matching the GPU init kernel bit for bit.
 */
#include "../include/tlt_init.h"
#include "tlt_oracle.h"

void orc_init_range(const tlt_init_params* p, uint16_t* dst, int tensor, int layer, int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i) dst[i] = tlt_init_elem(p, tensor, layer, i);
}

uint16_t orc_init_value(const orc_init_cfg* init, const orc_model_cfg* c, int tensor, int layer, int64_t idx) {
    tlt_init_params p = {init->seed, init->layer_scale, init->lm_gain, init->lm_alt, init->lm_noise, init->fc_noise,
                         c->vocab,   c->hidden,         c->heads,     c->kv_heads,    c->head_dim, c->ffn};
    return tlt_init_elem(&p, tensor, layer, idx);
}
