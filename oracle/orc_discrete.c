/*
 * Discrete semantics of the reference hot path, restated in C (TEST
 * INFRASTRUCTURE — the checker, never the product). Citations are to
 * /root/reference/proj/include/specsim/<file>:<line>.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "tlt_oracle.h"

/* ================================================================ RNG ==== */
/* rng.hpp:14-20 */
static uint64_t splitmix64(uint64_t* x) {
    *x += 0x9e3779b97f4a7c15ULL;
    uint64_t z = *x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
/* rng.hpp:22-26: returns the advanced state, not the splitmix output. */
static uint64_t mix_label(uint64_t state, uint64_t label) {
    uint64_t x = state ^ (0x9e3779b97f4a7c15ULL + label);
    (void)splitmix64(&x);
    return x;
}

/* std::mt19937_64 (C++ [rand.eng.mers] parameters). */
#define MT_N 312
#define MT_M 156
static void mt_seed(orc_rng* r, uint64_t s) {
    r->mt[0] = s;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = MT_N;
}
static void mt_twist(orc_rng* r) {
    const uint64_t UPPER = 0xFFFFFFFF80000000ULL, LOWER = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
    for (int i = 0; i < MT_N; ++i) {
        uint64_t x = (r->mt[i] & UPPER) | (r->mt[(i + 1) % MT_N] & LOWER);
        uint64_t xa = x >> 1;
        if (x & 1ULL) xa ^= A;
        r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
    }
    r->mti = 0;
}
uint64_t orc_rng_next_u64(orc_rng* r) {
    if (r->mti >= MT_N) mt_twist(r);
    uint64_t x = r->mt[r->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}
/* rng.hpp:37-41 */
void orc_rng_init(orc_rng* r, uint64_t seed, uint64_t stream_id) {
    r->seed = seed;
    r->stream_id = stream_id;
    uint64_t x = seed ^ mix_label(0x5bf03635d0d0183dULL, stream_id);
    mt_seed(r, splitmix64(&x));
}
/* rng.hpp:47-49 */
void orc_rng_fork(const orc_rng* r, uint64_t label, orc_rng* out) {
    orc_rng_init(out, r->seed, mix_label(r->stream_id + 0x9e3779b97f4a7c15ULL, label));
}
/* rng.hpp:54-56 */
double orc_rng_uniform01(orc_rng* r) { return (double)(orc_rng_next_u64(r) >> 11) * 0x1.0p-53; }
/* rng.hpp:59-61 */
uint64_t orc_rng_uniform_int(orc_rng* r, uint64_t n) { return orc_rng_next_u64(r) % n; }
/* rng.hpp:64-69 */
double orc_rng_normal(orc_rng* r) {
    double u1 = orc_rng_uniform01(r);
    double u2 = orc_rng_uniform01(r);
    return sqrt(-2.0 * log1p(-u1)) * cos(6.283185307179586477 * u2);
}
size_t orc_rng_sizeof(void) { return sizeof(orc_rng); }

double orc_usrc_next(orc_usrc* s) {
    if (s->rng) return orc_rng_uniform01(s->rng);
    if (s->cursor >= s->n) return 2.0; /* exhausted: never accepts, picks the last token */
    return s->buf[s->cursor++];
}

/* ====================================================== distributions ==== */
/* token_model.hpp:44-50: strict '>' keeps the lowest id on ties. */
int32_t orc_argmax(const double* p, int v) {
    int best = 0;
    for (int i = 1; i < v; ++i)
        if (p[i] > p[best]) best = i;
    return best;
}
/* token_model.hpp:83-91: min{t : u < CDF(t)}, sequential double sum. */
int32_t orc_inverse_cdf_pick(const double* p, int v, double u) {
    double cum = 0.0;
    int last = v - 1;
    for (int t = 0; t < last; ++t) {
        cum += p[t];
        if (u < cum) return t;
    }
    return last;
}
/* token_model.hpp:62-70 */
static void normalize(double* p, int v) {
    double sum = 0.0;
    for (int i = 0; i < v; ++i) sum += p[i];
    if (sum <= 0.0) {
        for (int i = 0; i < v; ++i) p[i] = 1.0 / (double)v;
        return;
    }
    for (int i = 0; i < v; ++i) p[i] /= sum;
}
/* token_model.hpp:161-173 */
void orc_temper(const double* raw, int v, double t, double* out) {
    if (t == 1.0) {
        memcpy(out, raw, sizeof(double) * (size_t)v);
        return;
    }
    if (t == 0.0) {
        int a = orc_argmax(raw, v);
        memset(out, 0, sizeof(double) * (size_t)v);
        out[a] = 1.0;
        return;
    }
    double inv = 1.0 / t;
    for (int i = 0; i < v; ++i) out[i] = raw[i] > 0.0 ? pow(raw[i], inv) : 0.0;
    normalize(out, v);
}

/* ========================================================== strategy ==== */
/* spec_decode.hpp:25-34 */
int64_t orc_max_tree_nodes(const orc_strategy* s) {
    int64_t total = 0, level = 1;
    const int64_t cap = 1LL << 40;
    for (int d = 0; d < s->draft_depth; ++d) {
        int64_t k = s->top_k > 1 ? s->top_k : 1;
        if (level > cap / k) return cap;
        level *= s->top_k;
        total += level;
        if (total > cap) return cap;
    }
    return total;
}
/* spec_decode.hpp:36-42 */
int orc_strategy_validate(const orc_strategy* s, const char** field) {
    const char* f = NULL;
    if (s->draft_depth < 1)
        f = "draft_depth";
    else if (s->top_k < 1)
        f = "top_k";
    else if (s->tokens_to_verify < 1)
        f = "tokens_to_verify";
    else if ((int64_t)s->tokens_to_verify > orc_max_tree_nodes(s))
        f = "tokens_to_verify";
    if (field) *field = f;
    return f ? -1 : 0;
}

/* ============================================================== tree ==== */
typedef struct {
    int32_t token, parent, depth;
    double prob, path_prob;
    int64_t birth;
} cand; /* spec_decode.hpp:84-91 */

/* spec_decode.hpp:96-101 */
static int rank_before(const cand* a, const cand* b) {
    if (a->path_prob != b->path_prob) return a->path_prob > b->path_prob;
    if (a->depth != b->depth) return a->depth < b->depth;
    if (a->token != b->token) return a->token < b->token;
    return a->birth < b->birth;
}

/* insertion sort of arena indices by rank_before (strict total order) */
static void sort_by_rank(int* idx, int n, const cand* arena) {
    for (int i = 1; i < n; ++i) {
        int x = idx[i], j = i - 1;
        while (j >= 0 && rank_before(&arena[x], &arena[idx[j]])) {
            idx[j + 1] = idx[j];
            --j;
        }
        idx[j + 1] = x;
    }
}

typedef struct {
    cand* arena;
    int n, cap;
    int32_t* path; /* scratch */
} tree_ctx;

static int arena_push(tree_ctx* t, cand c) {
    if (t->n == t->cap) {
        int nc = t->cap ? 2 * t->cap : 256;
        cand* na = (cand*)realloc(t->arena, sizeof(cand) * (size_t)nc);
        if (!na) return -1;
        t->arena = na;
        t->cap = nc;
    }
    t->arena[t->n] = c;
    return t->n++;
}

/* path tokens root->idx (spec_decode.hpp:143-151) */
static int path_of(const tree_ctx* t, int idx, int32_t* out) {
    int len = 0;
    for (int i = idx; i != -1; i = t->arena[i].parent) ++len;
    int p = len;
    for (int i = idx; i != -1; i = t->arena[i].parent) out[--p] = t->arena[i].token;
    return len;
}

/* expand (spec_decode.hpp:118-138): top_k children by (prob desc, id asc),
 * stopping at the first p <= 0. Children appended in that order. */
static int expand(tree_ctx* t, orc_row_fn f, void* user, int vocab, int top_k, int parent_idx,
                  const int32_t* path, int path_len, int depth, double parent_prob, double* row, int* created) {
    if (f(user, path, path_len, row) != 0) return -1;
    /* one pass keeping a list sorted by (p desc, id asc): an equal p is
     * inserted after the existing entries, i.e. stable over ascending id */
    int picked[64];
    int n_sel = 0;
    for (int i = 0; i < vocab; ++i) {
        double p = row[i];
        if (!(p > 0.0)) continue;
        if (n_sel == top_k && !(p > row[picked[n_sel - 1]])) continue;
        int pos = n_sel < top_k ? n_sel : top_k - 1;
        while (pos > 0 && p > row[picked[pos - 1]]) {
            picked[pos] = picked[pos - 1];
            --pos;
        }
        picked[pos] = i;
        if (n_sel < top_k) ++n_sel;
    }
    int taken = 0;
    for (int j = 0; j < n_sel; ++j) {
        int best = picked[j];
        cand c = {best, parent_idx, depth, row[best], parent_prob * row[best], (int64_t)t->n};
        int at = arena_push(t, c);
        if (at < 0) return -1;
        created[taken++] = at;
    }
    return taken;
}

/* build_draft_tree (spec_decode.hpp:111-197) */
int orc_build_draft_tree(orc_row_fn f, void* user, int vocab, const orc_strategy* s, orc_node* out) {
    if (orc_strategy_validate(s, NULL) != 0 || s->top_k > 64) return -1;
    tree_ctx t = {0};
    const int T = s->tokens_to_verify, k = s->top_k;
    double* row = (double*)malloc(sizeof(double) * (size_t)vocab);
    int32_t* path = (int32_t*)malloc(sizeof(int32_t) * (size_t)(s->draft_depth + 1));
    int* frontier = (int*)malloc(sizeof(int) * (size_t)(T * k + k));
    int* next = (int*)malloc(sizeof(int) * (size_t)(T * k + k));
    int n_front = 0, rc = -1;
    if (!row || !path || !frontier || !next) goto done;

    n_front = expand(&t, f, user, vocab, k, -1, path, 0, 1, 1.0, row, frontier); /* :140-141 */
    if (n_front < 0) goto done;
    for (int depth = 2; depth <= s->draft_depth; ++depth) { /* :153-169 */
        sort_by_rank(frontier, n_front, t.arena);
        if (n_front > T) n_front = T;
        int n_next = 0;
        for (int i = 0; i < n_front; ++i) {
            int idx = frontier[i];
            int plen = path_of(&t, idx, path);
            int got = expand(&t, f, user, vocab, k, idx, path, plen, depth, t.arena[idx].path_prob, row,
                             next + n_next);
            if (got < 0) goto done;
            n_next += got;
        }
        if (n_next == 0) break;
        memcpy(frontier, next, sizeof(int) * (size_t)n_next);
        n_front = n_next;
    }
    {
        /* :171-196 final selection and remap into rank order */
        int* keep = (int*)malloc(sizeof(int) * (size_t)t.n);
        int* to_tree = (int*)malloc(sizeof(int) * (size_t)t.n);
        if (!keep || !to_tree) {
            free(keep);
            free(to_tree);
            goto done;
        }
        for (int i = 0; i < t.n; ++i) {
            keep[i] = i;
            to_tree[i] = -1;
        }
        /* rank sort of the whole arena: merge-friendly insertion sort is fine at oracle sizes */
        sort_by_rank(keep, t.n, t.arena);
        int nk = t.n < T ? t.n : T;
        for (int i = 0; i < nk; ++i) {
            const cand* c = &t.arena[keep[i]];
            out[i].token = c->token;
            out[i].parent = c->parent == -1 ? -1 : to_tree[c->parent];
            out[i].depth = c->depth;
            out[i].prob = c->prob;
            out[i].path_prob = c->path_prob;
            to_tree[keep[i]] = i;
        }
        rc = nk;
        free(keep);
        free(to_tree);
    }
done:
    free(t.arena);
    free(row);
    free(path);
    free(frontier);
    free(next);
    return rc;
}

/* verify_greedy (spec_decode.hpp:245-268) */
int orc_verify_greedy(orc_argmax_fn f, void* user, const orc_node* tree, int n_nodes, orc_accept* out) {
    int32_t path[256];
    int node = -1, len = 0;
    out->accept_length = 0;
    for (;;) {
        int32_t want = f(user, path, len);
        if (want < 0) return -1;
        int next = -1;
        for (int i = 0; i < n_nodes; ++i) {
            if (tree[i].parent == node && tree[i].token == want) {
                next = i;
                break;
            }
        }
        if (next == -1) {
            out->bonus = want;
            return 0;
        }
        if (len >= 255) return -1;
        out->accepted[len] = want;
        out->nodes[len] = next;
        path[len++] = want;
        out->accept_length = len;
        node = next;
    }
}

/* build_sampled_chain (spec_decode.hpp:202-223) */
int orc_build_sampled_chain(orc_row_fn f, void* user, int vocab, int depth, orc_usrc* u, orc_node* out,
                            double* draft_dists) {
    int32_t path[256];
    double pp = 1.0;
    if (depth > 255) return -1;
    for (int i = 0; i < depth; ++i) {
        double* d = draft_dists + (size_t)i * (size_t)vocab;
        if (f(user, path, i, d) != 0) return -1;
        int32_t t = orc_inverse_cdf_pick(d, vocab, orc_usrc_next(u));
        out[i].token = t;
        out[i].parent = i - 1;
        out[i].depth = i + 1;
        out[i].prob = d[t];
        pp *= out[i].prob;
        out[i].path_prob = pp;
        path[i] = t;
    }
    return depth;
}

/* verify_stochastic (spec_decode.hpp:275-313) */
int orc_verify_stochastic(orc_row_fn target_fn, void* user, int vocab, double t, const orc_node* chain,
                          int n, const double* draft_dists, orc_usrc* u, orc_accept* out) {
    int32_t path[256];
    double* raw = (double*)malloc(sizeof(double) * (size_t)vocab);
    double* p = (double*)malloc(sizeof(double) * (size_t)vocab);
    int rc = -1;
    if (!raw || !p || n > 255) goto done;
    out->accept_length = 0;
    for (int i = 0; i < n; ++i) {
        if (target_fn(user, path, i, raw) != 0) goto done;
        orc_temper(raw, vocab, t, p); /* target_next_dist :281 */
        const double* dd = draft_dists ? draft_dists + (size_t)i * (size_t)vocab : NULL;
        int32_t x = chain[i].token;
        double q = dd ? dd[x] : 1.0;
        double px = p[x];
        double accept_prob = q > 0.0 ? (px / q < 1.0 ? px / q : 1.0) : 0.0;
        if (orc_usrc_next(u) < accept_prob) { /* :285 */
            out->accepted[i] = x;
            out->nodes[i] = i;
            path[i] = x;
            out->accept_length = i + 1;
            continue;
        }
        /* residual (p - q)^+ (:291-307) */
        double sum = 0.0;
        for (int j = 0; j < vocab; ++j) {
            double qj = dd ? dd[j] : (j == x ? 1.0 : 0.0);
            double diff = p[j] - qj;
            raw[j] = diff > 0.0 ? diff : 0.0;
            if (diff > 0.0) sum += diff;
        }
        if (sum <= 0.0) {
            memcpy(raw, p, sizeof(double) * (size_t)vocab);
        } else {
            for (int j = 0; j < vocab; ++j) raw[j] /= sum;
        }
        out->bonus = orc_inverse_cdf_pick(raw, vocab, orc_usrc_next(u)); /* :308 */
        rc = 0;
        goto done;
    }
    if (target_fn(user, path, n, raw) != 0) goto done; /* :311 full accept: bonus from p */
    orc_temper(raw, vocab, t, p);
    out->bonus = orc_inverse_cdf_pick(p, vocab, orc_usrc_next(u));
    rc = 0;
done:
    free(raw);
    free(p);
    return rc;
}

/* ============================================================ BEG-MAB ==== */
size_t orc_mab_sizeof(void) { return sizeof(orc_mab); }

static int cmp_double(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}
/* beg_mab.hpp:47-54: empty -> +inf; even -> mean of the middle pair */
double orc_median(const double* v, int n) {
    if (n == 0) return INFINITY;
    double tmp[ORC_MAB_MAX_WIN];
    memcpy(tmp, v, sizeof(double) * (size_t)n);
    qsort(tmp, (size_t)n, sizeof(double), cmp_double);
    int mid = n / 2;
    if (n % 2 == 1) return tmp[mid];
    return 0.5 * (tmp[mid - 1] + tmp[mid]);
}

/* beg_initialize (beg_mab.hpp:74-106) */
int orc_mab_init(orc_mab* m, const orc_strategy* s, int n, const int* thr, int n_thr, double eps, int window) {
    memset(m, 0, sizeof(*m));
    if (n < 1 || n > ORC_MAB_MAX_ARMS) return -1;
    if (eps < 0.0 || eps > 1.0) return -1;
    if (window < 1 || window > ORC_MAB_MAX_WIN) return -1;
    if (n_thr < 1 || n_thr > 32) return -1;
    for (int i = 0; i + 1 < n_thr; ++i)
        if (thr[i] >= thr[i + 1]) return -1;
    m->epsilon = eps;
    m->window = window;
    m->n_thr = n_thr;
    for (int i = 0; i < n_thr; ++i) m->thresholds[i] = thr[i];
    for (int i = 0; i < n; ++i) {
        if (orc_strategy_validate(&s[i], NULL) != 0) return -1;
        m->arms[i].strategy = s[i];
    }
    m->n_arms = n;
    /* groups by tokens_to_verify descending (std::map<int,..., greater>),
     * members in declaration order */
    int done[ORC_MAB_MAX_ARMS] = {0};
    int g = 0;
    for (;;) {
        int best = -1;
        for (int i = 0; i < n; ++i)
            if (!done[i] && (best < 0 || s[i].tokens_to_verify > s[best].tokens_to_verify)) best = i;
        if (best < 0) break;
        int tv = s[best].tokens_to_verify;
        if (g >= 32) return -1;
        m->group_size[g] = 0;
        for (int i = 0; i < n; ++i)
            if (!done[i] && s[i].tokens_to_verify == tv) {
                m->groups[g][m->group_size[g]++] = i;
                done[i] = 1;
            }
        ++g;
    }
    if (g != n_thr) return -1;
    return 0;
}

static int strategy_eq(const orc_strategy* a, const orc_strategy* b) {
    return a->draft_depth == b->draft_depth && a->top_k == b->top_k && a->tokens_to_verify == b->tokens_to_verify;
}

/* beg_record (beg_mab.hpp:111-134) */
int orc_mab_record(orc_mab* m, const orc_strategy* s, double elapsed, const int32_t* accept_lens, int batch) {
    if (batch < 1) return -1;
    if (!(elapsed > 0.0)) return -1;
    for (int a = 0; a < m->n_arms; ++a) {
        orc_arm* arm = &m->arms[a];
        if (!strategy_eq(&arm->strategy, s)) continue;
        double sum = 0.0;
        for (int i = 0; i < batch; ++i) sum += accept_lens[i];
        double a_bar = sum / (double)batch + 1.0;
        double reward = a_bar * (double)batch / elapsed;
        if (arm->n == m->window) { /* pop_front */
            memmove(arm->rewards, arm->rewards + 1, sizeof(double) * (size_t)(arm->n - 1));
            memmove(arm->accept_lens, arm->accept_lens + 1, sizeof(double) * (size_t)(arm->n - 1));
            arm->n -= 1;
        }
        arm->rewards[arm->n] = reward;
        arm->accept_lens[arm->n] = a_bar;
        arm->n += 1;
        return 0;
    }
    return -1;
}

/* beg_select (beg_mab.hpp:140-170) */
int orc_mab_select(orc_mab* m, int batch, orc_rng* rng) {
    if (m->n_thr == 0 || batch < m->thresholds[0]) return -2;
    int bucket = m->n_thr - 1;
    for (int i = 0; i + 1 < m->n_thr; ++i) {
        if (batch >= m->thresholds[i] && batch < m->thresholds[i + 1]) {
            bucket = i;
            break;
        }
    }
    const int* cands = m->groups[bucket];
    int nc = m->group_size[bucket];
    int pick;
    if (nc == 1) {
        pick = cands[0];
    } else if (orc_rng_uniform01(rng) < m->epsilon) {
        pick = cands[orc_rng_uniform_int(rng, (uint64_t)nc)];
    } else {
        pick = cands[0];
        double best = orc_median(m->arms[pick].rewards, m->arms[pick].n);
        for (int i = 1; i < nc; ++i) {
            double med = orc_median(m->arms[cands[i]].rewards, m->arms[cands[i]].n);
            if (med > best) {
                best = med;
                pick = cands[i];
            }
        }
    }
    m->arms[pick].selections += 1;
    return pick;
}

/* ======================================================= capture plan ==== */
/* capture_plan.hpp:51-54 */
static double unit_memory(const orc_capture* e) {
    int width = e->side == 0 ? e->tokens_to_verify : e->top_k;
    return (double)e->bucket_hi * (double)width;
}

/* capture_plan.hpp:58-73 */
static int bucket_ranges(const int* thr, int n_thr, int max_batch, int* lo, int* hi) {
    if (n_thr < 1) return -1;
    for (int i = 0; i + 1 < n_thr; ++i)
        if (thr[i] >= thr[i + 1]) return -1;
    if (max_batch < thr[n_thr - 1]) return -1;
    for (int i = 0; i < n_thr; ++i) {
        lo[i] = thr[i];
        hi[i] = i + 1 < n_thr ? thr[i + 1] - 1 : max_batch;
    }
    return 0;
}

static int add_entry(orc_capture* out, int* n, int max_out, orc_capture e, double* total) {
    e.memory_units = unit_memory(&e);
    *total += e.memory_units;
    if (*n >= max_out) return -1;
    out[(*n)++] = e;
    return 0;
}

/* plan_captures (capture_plan.hpp:87-126) / plan_captures_vanilla (:130-155) */
int orc_plan_captures(const orc_strategy* s, int n, const int* thr, int n_thr, int max_batch, int vanilla,
                      orc_capture* out, int max_out, double* total_units) {
    int lo[32], hi[32];
    if (n_thr > 32 || bucket_ranges(thr, n_thr, max_batch, lo, hi) != 0) return -1;
    for (int i = 0; i < n; ++i)
        if (orc_strategy_validate(&s[i], NULL) != 0) return -1;
    int cnt = 0;
    double total = 0.0;
    if (vanilla) {
        for (int i = 0; i < n; ++i)
            for (int b = 0; b < n_thr; ++b) {
                orc_capture t = {0, lo[b], hi[b], s[i].tokens_to_verify, 0, 0, 0.0};
                if (add_entry(out, &cnt, max_out, t, &total)) return -1;
                orc_capture d = {1, lo[b], hi[b], 0, s[i].top_k, s[i].draft_depth, 0.0};
                if (add_entry(out, &cnt, max_out, d, &total)) return -1;
            }
    } else {
        /* groups: tokens_to_verify descending, members in declaration order */
        int done[256] = {0};
        int bucket = 0;
        if (n > 256) return -1;
        for (;;) {
            int best = -1;
            for (int i = 0; i < n; ++i)
                if (!done[i] && (best < 0 || s[i].tokens_to_verify > s[best].tokens_to_verify)) best = i;
            if (best < 0) break;
            if (bucket >= n_thr) return -1;
            int tv = s[best].tokens_to_verify;
            orc_capture t = {0, lo[bucket], hi[bucket], tv, 0, 0, 0.0};
            if (add_entry(out, &cnt, max_out, t, &total)) return -1;
            int seen_k[256], seen_d[256], ns = 0;
            for (int i = 0; i < n; ++i) {
                if (done[i] || s[i].tokens_to_verify != tv) continue;
                done[i] = 1;
                int dup = 0;
                for (int j = 0; j < ns; ++j)
                    if (seen_k[j] == s[i].top_k && seen_d[j] == s[i].draft_depth) dup = 1;
                if (dup) continue;
                seen_k[ns] = s[i].top_k;
                seen_d[ns++] = s[i].draft_depth;
                orc_capture d = {1, lo[bucket], hi[bucket], 0, s[i].top_k, s[i].draft_depth, 0.0};
                if (add_entry(out, &cnt, max_out, d, &total)) return -1;
            }
            ++bucket;
        }
        if (bucket != n_thr) return -1;
    }
    if (total_units) *total_units = total;
    return cnt;
}

/* ======================================================= rollout bits ==== */
/* rollout.hpp:54-57 */
int orc_should_enable_sd(int active, int threshold) {
    if (threshold < 1) return -1;
    return active < threshold;
}
/* cost_model.hpp:38-48 with the default CostModelParams (:16-33) */
double orc_step_latency(int batch, int tokens_per_request, const orc_strategy* sd) {
    const double t_launch = 0.05, model_bytes = 1.0, mem_bw = 1.0, flops_per_token = 1.0, peak = 377.0,
                 drafter_step = 0.046;
    int tokens = sd ? sd->tokens_to_verify : tokens_per_request;
    double mem_t = model_bytes / mem_bw;
    double comp_t = (double)batch * (double)tokens * flops_per_token / peak;
    double t = t_launch + (mem_t > comp_t ? mem_t : comp_t);
    if (sd) t += (double)sd->draft_depth * drafter_step;
    return t;
}

double orc_now(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* ===================================================== pinning rows ==== */
static uint64_t hash64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x;
}
int orc_test_row(void* user, const int32_t* path, int path_len, double* out) {
    const orc_test_rows* c = (const orc_test_rows*)user;
    uint64_t h = hash64(c->seed ^ 0x1234567ULL);
    for (int i = 0; i < path_len; ++i) h = hash64(h ^ ((uint64_t)(uint32_t)path[i] + 0x9e3779b97f4a7c15ULL));
    double sum = 0.0;
    for (int i = 0; i < c->vocab; ++i) {
        uint64_t r = hash64(h + (uint64_t)i * 0x632be59bd9b4e019ULL);
        double u = (double)(r >> 11) * 0x1.0p-53;
        if (c->levels > 0) u = floor(u * c->levels) + 1.0; /* quantized: many exact ties */
        if ((int)((r >> 3) % 100) < c->zero_pct) u = 0.0;
        out[i] = u;
        sum += u;
    }
    if (sum <= 0.0) {
        for (int i = 0; i < c->vocab; ++i) out[i] = 1.0 / c->vocab;
        return 0;
    }
    for (int i = 0; i < c->vocab; ++i) out[i] /= sum;
    return 0;
}
int32_t orc_test_argmax(void* user, const int32_t* path, int path_len) {
    const orc_test_rows* c = (const orc_test_rows*)user;
    double* row = (double*)malloc(sizeof(double) * (size_t)c->vocab);
    if (!row) return -1;
    orc_test_row(user, path, path_len, row);
    int32_t a = orc_argmax(row, c->vocab);
    free(row);
    return a;
}

/* Arm statistics accessor (mirrors the fields beg_state_to_json dumps,
 * beg_mab.hpp:174-193). */
int orc_mab_arm_stats(const orc_mab* m, int arm, double* median_reward, int64_t* selections, int* n,
                      double* last_reward, double* last_accept) {
    if (arm < 0 || arm >= m->n_arms) return -1;
    const orc_arm* a = &m->arms[arm];
    *median_reward = orc_median(a->rewards, a->n);
    *selections = a->selections;
    *n = a->n;
    *last_reward = a->n ? a->rewards[a->n - 1] : 0.0;
    *last_accept = a->n ? a->accept_lens[a->n - 1] : 0.0;
    return 0;
}
