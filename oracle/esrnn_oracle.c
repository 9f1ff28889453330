/*
 * esrnn_oracle.c — TEST INFRASTRUCTURE ONLY (parity oracle, never shipped or measured
 * as the product).  A plain-C, fp64, single-threaded restatement of the reference's
 * ES-RNN training / forecasting hot path, exposing the engine's C-ABI
 * (include/esrnn_b200.h) so tests can diff the CUDA engine against it call by call.
 *
 * Pinned against: the reference built from its own headers (oracle/_ref, recipe in
 * oracle/Makefile) through tests/test_oracle.py, and the committed golden fixtures in
 * tests/golden/ (generated from oracle/_ref by tests/golden/make_golden.py).
 *
 * Each function cites the reference lines it restates (paths relative to
 * /root/reference/proj/include/esrnn/ unless noted).
 */
#include <math.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>

#include "esrnn_b200.h"

/* ---------------------------------------------------------------- mt19937_64 */
/* matrix.hpp:173-213 wraps std::mt19937_64; this is the published MT19937-64. */
#define MT_N 312
#define MT_M 156
typedef struct {
    uint64_t mt[MT_N];
    int mti;
    int have_spare;
    double spare;
} rng_t;

static void rng_seed(rng_t* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = MT_N;
    r->have_spare = 0;
    r->spare = 0.0;
}

static uint64_t rng_next(rng_t* r) {
    static const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (r->mti >= MT_N) {
        int i;
        uint64_t x;
        for (i = 0; i < MT_N - MT_M; ++i) {
            x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
            r->mt[i] = r->mt[i + MT_M] ^ (x >> 1) ^ mag01[x & 1ULL];
        }
        for (; i < MT_N - 1; ++i) {
            x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
            r->mt[i] = r->mt[i + (MT_M - MT_N)] ^ (x >> 1) ^ mag01[x & 1ULL];
        }
        x = (r->mt[MT_N - 1] & UM) | (r->mt[0] & LM);
        r->mt[MT_N - 1] = r->mt[MT_M - 1] ^ (x >> 1) ^ mag01[x & 1ULL];
        r->mti = 0;
    }
    uint64_t x = r->mt[r->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

/* matrix.hpp:178-180 */
static double rng_uniform01(rng_t* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }
static double rng_uniform(rng_t* r, double lo, double hi) { return lo + (hi - lo) * rng_uniform01(r); }
/* matrix.hpp:183-195 Box-Muller with a cached spare */
static double rng_normal(rng_t* r) {
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    double u1 = rng_uniform01(r), u2 = rng_uniform01(r);
    while (u1 <= 1e-300) u1 = rng_uniform01(r);
    const double rad = sqrt(-2.0 * log(u1));
    const double theta = 2.0 * 3.14159265358979323846 * u2;
    r->spare = rad * sin(theta);
    r->have_spare = 1;
    return rad * cos(theta);
}
/* matrix.hpp:198-200 (128-bit multiply-high) */
static uint64_t rng_below(rng_t* r, uint64_t n) {
    return (uint64_t)(((unsigned __int128)rng_next(r) * n) >> 64);
}

/* ---------------------------------------------------------------- fastmath */
/* fastmath.hpp:17-41 */
static double fm_exp(double x) {
    const double kLog2E = 1.4426950408889634073599;
    const double kC1 = 6.93145751953125e-1, kC2 = 1.42860682030941723212e-6;
    const double kP0 = 1.26177193074810590878e-4, kP1 = 3.02994407707441961300e-2,
                 kP2 = 9.99999999999999999910e-1;
    const double kQ0 = 3.00198505138664455042e-6, kQ1 = 2.52448340349684104192e-3,
                 kQ2 = 2.27265548208155028766e-1, kQ3 = 2.00000000000000000005e0;
    x = x > 709.4 ? 709.4 : x;
    x = x < -708.0 ? -708.0 : x;
    const double pn = floor(kLog2E * x + 0.5);
    const int64_t n = (int64_t)pn;
    x -= pn * kC1;
    x -= pn * kC2;
    const double xx = x * x;
    const double px = x * (kP2 + xx * (kP1 + xx * kP0));
    const double qx = kQ3 + xx * (kQ2 + xx * (kQ1 + xx * kQ0));
    const double e = 1.0 + 2.0 * (px / (qx - px));
    uint64_t bits = (uint64_t)(n + 1023) << 52;
    double scale;
    memcpy(&scale, &bits, sizeof scale);
    return e * scale;
}
/* fastmath.hpp:45-67 */
static double fm_tanh(double x) {
    const double kP0 = -9.64399179425052238628e-1, kP1 = -9.92877231001918586564e1,
                 kP2 = -1.61468768441708447952e3;
    const double kQ0 = 1.12811678491632931402e2, kQ1 = 2.23548839060100448583e3,
                 kQ2 = 4.84406305325125486048e3;
    const double ax = fabs(x);
    if (ax < 0.625) {
        const double z = x * x;
        const double p = kP2 + z * (kP1 + z * kP0);
        const double q = kQ2 + z * (kQ1 + z * (kQ0 + z));
        return x + x * z * (p / q);
    } else if (ax < 19.0) {
        const double s = 1.0 - 2.0 / (fm_exp(2.0 * ax) + 1.0);
        return x < 0.0 ? -s : s;
    }
    return x < 0.0 ? -1.0 : 1.0;
}
/* fastmath.hpp:70-75 */
static double fm_logistic(double x) {
    const double y = 1.0 / (1.0 + fm_exp(-x));
    const double lo = DBL_MIN, hi = 1.0 - DBL_EPSILON / 2.0;
    return y < lo ? lo : (y > hi ? hi : y);
}

/* ---------------------------------------------------------------- trainer state */
#define MAXL ESRNN_MAX_LAYERS

struct esrnn_trainer {
    esrnn_profile prof;
    esrnn_train_config cfg;
    int N, LEN, T, S, I, O, H, L, in0, nb;
    int blen[ESRNN_MAX_BLOCKS];
    int layer_in[MAXL];                 /* input width of each layer */
    int64_t off_win[MAXL], off_wrec[MAXL], off_bias[MAXL];
    int64_t off_nlw, off_nlb, off_outw, off_outb, P;
    double* vals;                       /* N x LEN */
    int* cat;                           /* N, already defaulted to Other */
    double *a_raw, *g_raw, *s_raw;      /* N, N, N x S */
    double *m_a, *v_a, *m_g, *v_g, *m_s, *v_s;
    long* steps;
    double* W;                          /* P, for_each_param order */
    double *mW, *vW;
    long net_step;
    rng_t rng;
    char err[512];
    double last_ms;
    int32_t *last_wr, *last_wa;   /* window order of the last train_epoch */
    int64_t last_nw;
};

static char g_create_err[512];

static esrnn_status fail(char* buf, esrnn_status st, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, 512, fmt, ap);
    va_end(ap);
    return st;
}

const char* esrnn_version(void) { return "oracle (plain-C fp64 restatement)"; }
int32_t esrnn_abi_version(void) { return ESRNN_ABI_VERSION; }
const char* esrnn_last_error(const esrnn_trainer* t) { return t ? t->err : g_create_err; }

static void* xcalloc(size_t n, size_t sz) {
    void* p = calloc(n ? n : 1, sz);
    if (!p) abort();
    return p;
}

/* data.hpp:101-114 FrequencyProfile::validate, trainer.hpp:34-43 TrainConfig::validate */
static esrnn_status validate_config(const esrnn_profile* p, const esrnn_train_config* c, char* err) {
    if (p->seasonality_length < 1) return fail(err, ESRNN_CONFIG_ERROR, "profile: seasonality must be >= 1");
    if (p->horizon < 1) return fail(err, ESRNN_CONFIG_ERROR, "profile: horizon must be >= 1");
    if (p->input_window < p->seasonality_length)
        return fail(err, ESRNN_CONFIG_ERROR, "profile: input_window must cover at least one season");
    if (p->n_blocks < 1) return fail(err, ESRNN_CONFIG_ERROR, "profile: dilation blocks must be non-empty");
    if (p->n_blocks > ESRNN_MAX_BLOCKS) return fail(err, ESRNN_CONFIG_ERROR, "profile: too many blocks");
    int layer = 0;
    for (int b = 0; b < p->n_blocks; ++b) {
        if (p->block_len[b] < 1) return fail(err, ESRNN_CONFIG_ERROR, "profile: empty dilation block");
        for (int j = 0; j < p->block_len[b]; ++j, ++layer) {
            if (layer >= MAXL) return fail(err, ESRNN_CONFIG_ERROR, "profile: too many layers");
            if (p->dilations[layer] < 1)
                return fail(err, ESRNN_CONFIG_ERROR, "profile: dilations must be strictly positive");
        }
    }
    if (p->hidden_size < 1) return fail(err, ESRNN_CONFIG_ERROR, "profile: hidden_size must be >= 1");
    if (p->min_length < 1) return fail(err, ESRNN_CONFIG_ERROR, "profile: min_length must be >= 1");
    if (c->epochs < 0) return fail(err, ESRNN_CONFIG_ERROR, "train: epochs must be >= 0");
    /* trainer.hpp:36-37 caps the batch at 2048; the ABI's max_batch_size extension lifts the
     * cap for the large-batch sweep, where this restatement is the only CPU checker */
    const int cap = c->max_batch_size > 0 ? c->max_batch_size : 2048;
    if (c->batch_size < 1 || c->batch_size > cap)
        return fail(err, ESRNN_CONFIG_ERROR, "train: batch_size must be in [1, %d]", cap);
    if (!(c->tau > 0.0 && c->tau < 1.0)) return fail(err, ESRNN_CONFIG_ERROR, "train: tau must be in (0, 1)");
    if (c->learning_rate_network < 0.0 || c->learning_rate_per_series < 0.0)
        return fail(err, ESRNN_CONFIG_ERROR, "train: learning rates must be non-negative");
    if (c->has_gradient_clip && c->gradient_clip <= 0.0)
        return fail(err, ESRNN_CONFIG_ERROR, "train: gradient_clip must be positive");
    if (!(c->level_variability_penalty >= 0.0) || !isfinite(c->level_variability_penalty))
        return fail(err, ESRNN_CONFIG_ERROR, "train: level_variability_penalty must be finite and >= 0");
    return ESRNN_OK;
}

/* trainer.hpp:159-200 (ctor) + network.hpp:89-116 (init_stack_weights) */
esrnn_status esrnn_trainer_create(const esrnn_profile* profile, const esrnn_train_config* cfg,
                                  int64_t n_series, int32_t length, const double* values,
                                  const int32_t* category, const esrnn_dist* dist,
                                  esrnn_trainer** out) {
    *out = NULL;
    if (dist && dist->world_size > 1)
        return fail(g_create_err, ESRNN_CONFIG_ERROR, "oracle: no sharded mode");
    esrnn_status st = validate_config(profile, cfg, g_create_err);
    if (st) return st;
    if (n_series <= 0) return fail(g_create_err, ESRNN_CONTRACT_ERROR, "trainer: no series");
    const int O = profile->horizon, S = profile->seasonality_length, I = profile->input_window;
    /* data.hpp:128-140 split_train_val_test */
    if (length < 2 * O + 1)
        return fail(g_create_err, ESRNN_INSUFFICIENT_LENGTH, "split: need at least %d values, got %d",
                    2 * O + 1, length);
    const int T = length - 2 * O;
    if (T < I + O)
        return fail(g_create_err, ESRNN_INSUFFICIENT_LENGTH,
                    "trainer: train segment of %d cannot hold an input window plus horizon", T);
    if (T < S) return fail(g_create_err, ESRNN_INSUFFICIENT_LENGTH, "trainer: train segment shorter than one season");

    esrnn_trainer* t = (esrnn_trainer*)xcalloc(1, sizeof *t);
    t->prof = *profile;
    t->cfg = *cfg;
    t->N = (int)n_series;
    t->LEN = length;
    t->T = T;
    t->S = S;
    t->I = I;
    t->O = O;
    t->H = profile->hidden_size;
    t->nb = profile->n_blocks;
    t->L = 0;
    for (int b = 0; b < t->nb; ++b) {
        t->blen[b] = profile->block_len[b];
        t->L += t->blen[b];
    }
    t->in0 = I + ESRNN_NUM_CATEGORIES;
    const int H = t->H;
    int64_t off = 0;
    for (int l = 0; l < t->L; ++l) {
        t->layer_in[l] = l == 0 ? t->in0 : H;
        t->off_win[l] = off;
        off += (int64_t)t->layer_in[l] * 4 * H;
        t->off_wrec[l] = off;
        off += (int64_t)H * 4 * H;
        t->off_bias[l] = off;
        off += 4 * H;
    }
    t->off_nlw = off;
    off += (int64_t)H * H;
    t->off_nlb = off;
    off += H;
    t->off_outw = off;
    off += (int64_t)H * O;
    t->off_outb = off;
    off += O;
    t->P = off;

    t->vals = (double*)xcalloc((size_t)t->N * length, sizeof(double));
    memcpy(t->vals, values, sizeof(double) * (size_t)t->N * length);
    t->cat = (int*)xcalloc(t->N, sizeof(int));
    for (int i = 0; i < t->N; ++i) t->cat[i] = (category && category[i] >= 0) ? category[i] : 5;
    t->a_raw = (double*)xcalloc(t->N, sizeof(double));
    t->g_raw = (double*)xcalloc(t->N, sizeof(double));
    t->s_raw = (double*)xcalloc((size_t)t->N * S, sizeof(double));
    t->m_a = (double*)xcalloc(t->N, sizeof(double));
    t->v_a = (double*)xcalloc(t->N, sizeof(double));
    t->m_g = (double*)xcalloc(t->N, sizeof(double));
    t->v_g = (double*)xcalloc(t->N, sizeof(double));
    t->m_s = (double*)xcalloc((size_t)t->N * S, sizeof(double));
    t->v_s = (double*)xcalloc((size_t)t->N * S, sizeof(double));
    t->steps = (long*)xcalloc(t->N, sizeof(long));
    t->W = (double*)xcalloc(t->P, sizeof(double));
    t->mW = (double*)xcalloc(t->P, sizeof(double));
    t->vW = (double*)xcalloc(t->P, sizeof(double));

    /* network.hpp:89-116: U(-1/sqrt(H), 1/sqrt(H)) for w_input then w_recur per layer,
     * then nl_w, then out_w; forget-gate bias 1 */
    rng_seed(&t->rng, cfg->seed);
    const double bound = 1.0 / sqrt((double)H);
    for (int l = 0; l < t->L; ++l) {
        for (int64_t e = 0; e < (int64_t)t->layer_in[l] * 4 * H; ++e)
            t->W[t->off_win[l] + e] = rng_uniform(&t->rng, -bound, bound);
        for (int64_t e = 0; e < (int64_t)H * 4 * H; ++e)
            t->W[t->off_wrec[l] + e] = rng_uniform(&t->rng, -bound, bound);
        for (int c = H; c < 2 * H; ++c) t->W[t->off_bias[l] + c] = 1.0;
    }
    for (int64_t e = 0; e < (int64_t)H * H; ++e) t->W[t->off_nlw + e] = rng_uniform(&t->rng, -bound, bound);
    for (int64_t e = 0; e < (int64_t)H * O; ++e) t->W[t->off_outw + e] = rng_uniform(&t->rng, -bound, bound);
    *out = t;
    return ESRNN_OK;
}

void esrnn_trainer_destroy(esrnn_trainer* t) {
    if (!t) return;
    free(t->vals); free(t->cat); free(t->a_raw); free(t->g_raw); free(t->s_raw);
    free(t->m_a); free(t->v_a); free(t->m_g); free(t->v_g); free(t->m_s); free(t->v_s);
    free(t->steps); free(t->W); free(t->mW); free(t->vW); free(t->last_wr); free(t->last_wa);
    free(t);
}

esrnn_status esrnn_trainer_shard(const esrnn_trainer* t, int64_t* b, int64_t* e) {
    *b = 0;
    *e = t->N;
    return ESRNN_OK;
}

esrnn_status esrnn_trainer_param_count(const esrnn_trainer* t, int32_t* n_arrays, int64_t* n_values) {
    *n_arrays = 3 * t->L + 4;
    *n_values = t->P;
    return ESRNN_OK;
}

/* network.hpp:62-74 for_each_param order and names */
esrnn_status esrnn_trainer_param_info(const esrnn_trainer* t, int32_t idx, esrnn_param_info* o) {
    memset(o, 0, sizeof *o);
    const int H = t->H;
    if (idx < 0 || idx >= 3 * t->L + 4) return ESRNN_SHAPE_ERROR;
    if (idx < 3 * t->L) {
        const int l = idx / 3, k = idx % 3;
        if (k == 0) { snprintf(o->name, 32, "lstm%d.w_input", l); o->rows = t->layer_in[l]; o->cols = 4 * H; o->offset = t->off_win[l]; }
        if (k == 1) { snprintf(o->name, 32, "lstm%d.w_recur", l); o->rows = H; o->cols = 4 * H; o->offset = t->off_wrec[l]; }
        if (k == 2) { snprintf(o->name, 32, "lstm%d.bias", l); o->rows = 1; o->cols = 4 * H; o->offset = t->off_bias[l]; }
        return ESRNN_OK;
    }
    switch (idx - 3 * t->L) {
        case 0: snprintf(o->name, 32, "head.nl_w"); o->rows = H; o->cols = H; o->offset = t->off_nlw; break;
        case 1: snprintf(o->name, 32, "head.nl_b"); o->rows = 1; o->cols = H; o->offset = t->off_nlb; break;
        case 2: snprintf(o->name, 32, "head.out_w"); o->rows = H; o->cols = t->O; o->offset = t->off_outw; break;
        default: snprintf(o->name, 32, "head.out_b"); o->rows = 1; o->cols = t->O; o->offset = t->off_outb; break;
    }
    return ESRNN_OK;
}

esrnn_status esrnn_trainer_get_weights(esrnn_trainer* t, double* flat, int64_t count) {
    if (count != t->P) return fail(t->err, ESRNN_SHAPE_ERROR, "get_weights: count %lld != %lld", (long long)count, (long long)t->P);
    memcpy(flat, t->W, sizeof(double) * t->P);
    return ESRNN_OK;
}

/* trainer.hpp:415-432 */
esrnn_status esrnn_trainer_set_weights(esrnn_trainer* t, const double* flat, int64_t count) {
    if (count != t->P)
        return fail(t->err, ESRNN_CHECKPOINT_ERROR, "checkpoint network shapes incompatible with configuration");
    memcpy(t->W, flat, sizeof(double) * t->P);
    return ESRNN_OK;
}

esrnn_status esrnn_trainer_get_per_series(esrnn_trainer* t, int64_t r0, int64_t n, double* a,
                                          double* g, double* s) {
    if (r0 < 0 || r0 + n > t->N) return fail(t->err, ESRNN_SHAPE_ERROR, "per_series: rows out of range");
    for (int64_t i = 0; i < n; ++i) {
        if (a) a[i] = t->a_raw[r0 + i];
        if (g) g[i] = t->g_raw[r0 + i];
        if (s) memcpy(s + i * t->S, t->s_raw + (r0 + i) * t->S, sizeof(double) * t->S);
    }
    return ESRNN_OK;
}

esrnn_status esrnn_trainer_set_per_series(esrnn_trainer* t, int64_t r0, int64_t n, const double* a,
                                          const double* g, const double* s) {
    if (r0 < 0 || r0 + n > t->N) return fail(t->err, ESRNN_SHAPE_ERROR, "per_series: rows out of range");
    for (int64_t i = 0; i < n; ++i) {
        if (a) t->a_raw[r0 + i] = a[i];
        if (g) t->g_raw[r0 + i] = g[i];
        if (s) memcpy(t->s_raw + (r0 + i) * t->S, s + i * t->S, sizeof(double) * t->S);
    }
    return ESRNN_OK;
}

/* ---------------------------------------------------------------- the step */
/* matrix.hpp:103-139: out(m x n) = a(m x k) * b(k x n), each element accumulated
 * in k order starting from zero. */
static void matmul(double* out, const double* a, const double* b, int m, int kk, int n, int ldb) {
    for (int i = 0; i < m; ++i) {
        double* c = out + (size_t)i * n;
        for (int j = 0; j < n; ++j) c[j] = 0.0;
        for (int k = 0; k < kk; ++k) {
            const double f = a[(size_t)i * kk + k];
            const double* br = b + (size_t)k * ldb;
            for (int j = 0; j < n; ++j) c[j] += f * br[j];
        }
    }
}

typedef struct {
    /* workspace of one build_graph + backward, sized for B windows and k slots */
    int B, k;
    int *slot_of_row, *slot_series, *wslot;
    double *y, *alpha, *gamma, *lev, *seas;           /* k, k, k, k x T, k x (T+S) */
    double *x, *tgt, *den_in, *den_out, *lvl;         /* B x in0, B x O, B x I, B x O, B */
    double* u[MAXL];                                  /* layer inputs, B x in_l */
    double *gi[MAXL], *gg[MAXL], *go[MAXL], *tc[MAXL], *h[MAXL];  /* B x H */
    double *cur, *z, *pred;                           /* B x H, B x H, B x O */
} work_t;

static void work_free(work_t* w, int L) {
    free(w->slot_of_row); free(w->slot_series); free(w->wslot);
    free(w->y); free(w->alpha); free(w->gamma); free(w->lev); free(w->seas);
    free(w->x); free(w->tgt); free(w->den_in); free(w->den_out); free(w->lvl);
    for (int l = 0; l < L; ++l) { free(w->u[l]); free(w->gi[l]); free(w->gg[l]); free(w->go[l]); free(w->tc[l]); free(w->h[l]); }
    free(w->cur); free(w->z); free(w->pred);
}

/* holt_winters.hpp:236-283 (hybrid_primer_tape forward) and trainer.hpp:493-566
 * (slot dedupe, window gathers, normalisation), then network.hpp:190-210
 * (forward_stack at sequence length 1) — the forward half of build_graph. */
static esrnn_status forward_batch(esrnn_trainer* t, work_t* w, int B, const int32_t* rows,
                                  const int32_t* anchors) {
    const int T = t->T, S = t->S, I = t->I, O = t->O, H = t->H, in0 = t->in0;
    memset(w, 0, sizeof *w);
    w->B = B;
    w->slot_of_row = (int*)xcalloc(t->N, sizeof(int));
    w->slot_series = (int*)xcalloc(B, sizeof(int));
    w->wslot = (int*)xcalloc(B, sizeof(int));
    for (int i = 0; i < t->N; ++i) w->slot_of_row[i] = -1;
    for (int b = 0; b < B; ++b) {
        if (rows[b] < 0 || rows[b] >= t->N)
            return fail(t->err, ESRNN_SHAPE_ERROR, "batch: series row %d out of range", rows[b]);
        if (w->slot_of_row[rows[b]] < 0) {
            w->slot_of_row[rows[b]] = w->k;
            w->slot_series[w->k++] = rows[b];
        }
        w->wslot[b] = w->slot_of_row[rows[b]];
    }
    const int k = w->k;
    w->y = (double*)xcalloc((size_t)k * T, sizeof(double));
    w->alpha = (double*)xcalloc(k, sizeof(double));
    w->gamma = (double*)xcalloc(k, sizeof(double));
    w->lev = (double*)xcalloc((size_t)k * T, sizeof(double));
    w->seas = (double*)xcalloc((size_t)k * (T + S), sizeof(double));
    for (int s = 0; s < k; ++s) {
        const int row = w->slot_series[s];
        memcpy(w->y + (size_t)s * T, t->vals + (size_t)row * t->LEN, sizeof(double) * T);
        w->alpha[s] = fm_logistic(t->a_raw[row]);
        w->gamma[s] = fm_logistic(t->g_raw[row]);
        for (int j = 0; j < S; ++j) w->seas[(size_t)s * (T + S) + j] = fm_exp(t->s_raw[(size_t)row * S + j]);
    }
    /* t-major like the tape so the first failing t is reported (holt_winters.hpp:270-273) */
    double* lp = (double*)xcalloc(k, sizeof(double));
    for (int s = 0; s < k; ++s) {
        double acc = 0.0;
        for (int j = 0; j < S; ++j) acc += w->y[(size_t)s * T + j];
        lp[s] = acc / (double)S;
    }
    for (int tt = 0; tt < T; ++tt) {
        int bad = 0;
        for (int s = 0; s < k; ++s) {
            const double yt = w->y[(size_t)s * T + tt];
            double* se = w->seas + (size_t)s * (T + S);
            const double a = w->alpha[s], g = w->gamma[s];
            const double lvl = a * (yt / se[tt]) + (1.0 - a) * lp[s];
            if (!(lvl > 0.0) || !isfinite(lvl)) bad = 1;
            se[tt + S] = g * (yt / lp[s]) + (1.0 - g) * se[tt];
            w->lev[(size_t)s * T + tt] = lvl;
            lp[s] = lvl;
        }
        if (bad) {
            free(lp);
            return fail(t->err, ESRNN_NUMERIC_DOMAIN_ERROR, "hybrid_primer_tape: non-positive level at t=%d", tt);
        }
    }
    free(lp);

    /* windows (trainer.hpp:532-566) */
    w->x = (double*)xcalloc((size_t)B * in0, sizeof(double));
    w->tgt = (double*)xcalloc((size_t)B * O, sizeof(double));
    w->den_in = (double*)xcalloc((size_t)B * I, sizeof(double));
    w->den_out = (double*)xcalloc((size_t)B * O, sizeof(double));
    w->lvl = (double*)xcalloc(B, sizeof(double));
    for (int b = 0; b < B; ++b) {
        const int s = w->wslot[b], a = anchors[b], row = rows[b];
        if (a < I - 1 || a > T - O - 1)
            return fail(t->err, ESRNN_SHAPE_ERROR, "batch: anchor %d out of range", a);
        const double* se = w->seas + (size_t)s * (T + S);
        const double lvl = w->lev[(size_t)s * T + a];
        w->lvl[b] = lvl;
        for (int j = 0; j < I; ++j) {
            const int idx = a - I + 1 + j;
            const double den = se[idx] * lvl;
            w->den_in[(size_t)b * I + j] = den;
            w->x[(size_t)b * in0 + j] = t->vals[(size_t)row * t->LEN + idx] / den;
        }
        for (int c = 0; c < ESRNN_NUM_CATEGORIES; ++c) w->x[(size_t)b * in0 + I + c] = (t->cat[row] == c) ? 1.0 : 0.0;
        for (int j = 0; j < O; ++j) {
            const int idx = a + 1 + j;
            const double den = se[idx] * lvl;
            w->den_out[(size_t)b * O + j] = den;
            w->tgt[(size_t)b * O + j] = t->vals[(size_t)row * t->LEN + idx] / den;
        }
    }

    /* stack (network.hpp:148-163, 190-210) with no recurrent state */
    double* pre = (double*)xcalloc((size_t)B * 4 * H, sizeof(double));
    const double* in = w->x;
    int in_w = in0, layer = 0;
    double* block_in = NULL;
    for (int bl = 0; bl < t->nb; ++bl) {
        block_in = (double*)in;
        for (int j = 0; j < t->blen[bl]; ++j, ++layer) {
            const int l = layer;
            w->u[l] = (double*)xcalloc((size_t)B * in_w, sizeof(double));
            memcpy(w->u[l], in, sizeof(double) * (size_t)B * in_w);
            matmul(pre, in, t->W + t->off_win[l], B, in_w, 4 * H, 4 * H);
            const double* bias = t->W + t->off_bias[l];
            w->gi[l] = (double*)xcalloc((size_t)B * H, sizeof(double));
            w->gg[l] = (double*)xcalloc((size_t)B * H, sizeof(double));
            w->go[l] = (double*)xcalloc((size_t)B * H, sizeof(double));
            w->tc[l] = (double*)xcalloc((size_t)B * H, sizeof(double));
            w->h[l] = (double*)xcalloc((size_t)B * H, sizeof(double));
            for (int r = 0; r < B; ++r) {
                const double* p = pre + (size_t)r * 4 * H;
                for (int hh = 0; hh < H; ++hh) {
                    const double i = fm_logistic(p[hh] + bias[hh]);
                    const double g = fm_tanh(p[2 * H + hh] + bias[2 * H + hh]);
                    const double o = fm_logistic(p[3 * H + hh] + bias[3 * H + hh]);
                    const double c = i * g;
                    const double tcv = fm_tanh(c);
                    const size_t e = (size_t)r * H + hh;
                    w->gi[l][e] = i;
                    w->gg[l][e] = g;
                    w->go[l][e] = o;
                    w->tc[l][e] = tcv;
                    w->h[l][e] = o * tcv;
                }
            }
            in = w->h[l];
            in_w = H;
        }
        if (bl > 0) {
            /* residual: current += block_in (network.hpp:204-205); store in the last h */
            double* hl = w->h[layer - 1];
            for (size_t e = 0; e < (size_t)B * H; ++e) hl[e] = hl[e] + block_in[e];
        }
    }
    free(pre);
    /* head (network.hpp:207-209) */
    w->cur = (double*)xcalloc((size_t)B * H, sizeof(double));
    memcpy(w->cur, in, sizeof(double) * (size_t)B * H);
    w->z = (double*)xcalloc((size_t)B * H, sizeof(double));
    w->pred = (double*)xcalloc((size_t)B * O, sizeof(double));
    matmul(w->z, w->cur, t->W + t->off_nlw, B, H, H, H);
    for (int r = 0; r < B; ++r)
        for (int c = 0; c < H; ++c) w->z[(size_t)r * H + c] = fm_tanh(w->z[(size_t)r * H + c] + t->W[t->off_nlb + c]);
    matmul(w->pred, w->z, t->W + t->off_outw, B, H, O, O);
    for (int r = 0; r < B; ++r)
        for (int c = 0; c < O; ++c) w->pred[(size_t)r * O + c] += t->W[t->off_outb + c];
    return ESRNN_OK;
}

/* out(kk x n) += a(m x kk)^T * g(m x n), summed over rows in order (matrix.hpp:164-168) */
static void matmul_tn_acc(double* out, const double* a, const double* g, int m, int kk, int n) {
    for (int k = 0; k < kk; ++k)
        for (int j = 0; j < n; ++j) {
            double acc = out[(size_t)k * n + j];
            for (int r = 0; r < m; ++r) acc += a[(size_t)r * kk + k] * g[(size_t)r * n + j];
            out[(size_t)k * n + j] = acc;
        }
}

/* Level-variability penalty (B200 extension; NOT in the reference, whose loss is pinball
 * only, trainer.hpp:581).  Smyl's M4 ES-RNN penalises the wiggliness of a series' levels
 * ("penalizing dramatic changes in the level"): with u_t = log l_t over
 * the train segment and e_t = u_t - 2 u_{t-1} + u_{t-2} (t = 2..T-1),
 *     P(series) = mean_t e_t^2,
 * and a batch adds  lambda * O / M * sum over its windows of P(window's series)  to the
 * masked-mean pinball (M = unmasked target count; O / M = 1 / B without a mask), i.e. c_s *
 * P(s) per distinct series with c_s = lambda * O * n_s / M.  Returns c * P; with lb != NULL
 * adds d(c * P)/d l_t to the level adjoints. */
static double lvp_series(const double* lv, int T, double c, double* lb) {
    if (T < 3) return 0.0;
    const double inv = 1.0 / (double)(T - 2);
    double acc = 0.0;
    for (int tt = 2; tt < T; ++tt) {
        const double e = log(lv[tt]) - 2.0 * log(lv[tt - 1]) + log(lv[tt - 2]);
        acc += e * e;
        if (lb) {
            const double q = c * 2.0 * inv * e;
            lb[tt] += q / lv[tt];
            lb[tt - 1] -= 2.0 * q / lv[tt - 1];
            lb[tt - 2] += q / lv[tt - 2];
        }
    }
    return c * acc * inv;
}

/* c_s = lambda * O * n_s / M for each slot (n_s = the slot's windows in the batch) */
static double* lvp_weights(const esrnn_trainer* t, const work_t* w, double count) {
    double* c = (double*)xcalloc(w->k, sizeof(double));
    for (int b = 0; b < w->B; ++b) c[w->wslot[b]] += 1.0;
    for (int s = 0; s < w->k; ++s) c[s] = t->cfg.level_variability_penalty * (double)t->O * c[s] / count;
    return c;
}

/* Reverse sweep (autodiff.hpp:397-631) specialised to build_graph's graph: pinball
 * adjoint (:611-628), head/stack adjoints (MatMul :476-482, Logistic :483, Tanh :492,
 * Mul :450, Add :428, SliceCols :544, BroadcastRow :569), window gathers/normalisation
 * (Gather :603, Div :463, BroadcastCol :576), the HW recursion (holt_winters.hpp:266-277)
 * and the leaf squashes (Logistic, Exp :501). */
static void backward_batch(esrnn_trainer* t, work_t* w, const int32_t* anchors, const double* mask,
                           double count, double* gnet, double* gps) {
    const int T = t->T, S = t->S, I = t->I, O = t->O, H = t->H, in0 = t->in0, L = t->L, B = w->B;
    const double tau = t->cfg.tau;
    memset(gnet, 0, sizeof(double) * t->P);
    double* pbar = (double*)xcalloc((size_t)B * O, sizeof(double));
    double* tbar = (double*)xcalloc((size_t)B * O, sizeof(double));
    const double gscale = 1.0 / count;
    for (size_t e = 0; e < (size_t)B * O; ++e) {
        if (mask && mask[e] == 0.0) continue;
        const int under = w->tgt[e] >= w->pred[e];
        pbar[e] = gscale * (under ? -tau : (1.0 - tau));
        tbar[e] = gscale * (under ? tau : -(1.0 - tau));
    }
    /* head: out = z*out_w + out_b ; z = tanh(cur*nl_w + nl_b) */
    double* gob = gnet + t->off_outb;
    for (int r = 0; r < B; ++r)
        for (int c = 0; c < O; ++c) gob[c] += pbar[(size_t)r * O + c];
    matmul_tn_acc(gnet + t->off_outw, w->z, pbar, B, H, O);
    double* zbar = (double*)xcalloc((size_t)B * H, sizeof(double));
    const double* ow = t->W + t->off_outw;
    for (int r = 0; r < B; ++r)
        for (int kk = 0; kk < H; ++kk) {
            double acc = 0.0;
            for (int c = 0; c < O; ++c) acc += pbar[(size_t)r * O + c] * ow[(size_t)kk * O + c];
            const double zz = w->z[(size_t)r * H + kk];
            zbar[(size_t)r * H + kk] = acc * (1.0 - zz * zz);
        }
    double* gnb = gnet + t->off_nlb;
    for (int r = 0; r < B; ++r)
        for (int c = 0; c < H; ++c) gnb[c] += zbar[(size_t)r * H + c];
    matmul_tn_acc(gnet + t->off_nlw, w->cur, zbar, B, H, H);
    double* hbar = (double*)xcalloc((size_t)B * H, sizeof(double));
    const double* nw = t->W + t->off_nlw;
    for (int r = 0; r < B; ++r)
        for (int kk = 0; kk < H; ++kk) {
            double acc = 0.0;
            for (int c = 0; c < H; ++c) acc += zbar[(size_t)r * H + c] * nw[(size_t)kk * H + c];
            hbar[(size_t)r * H + kk] = acc;
        }
    free(zbar);

    /* layers in reverse; the residual of block b>0 adds the block output adjoint to block_in */
    double* pre_bar = (double*)xcalloc((size_t)B * 4 * H, sizeof(double));
    double* xbar = (double*)xcalloc((size_t)B * in0, sizeof(double));
    int layer = L;
    double* resid = (double*)xcalloc((size_t)B * H, sizeof(double));
    for (int bl = t->nb - 1; bl >= 0; --bl) {
        if (bl > 0) memcpy(resid, hbar, sizeof(double) * (size_t)B * H);
        for (int j = t->blen[bl] - 1; j >= 0; --j) {
            const int l = --layer;
            const int in_w = t->layer_in[l];
            memset(pre_bar, 0, sizeof(double) * (size_t)B * 4 * H);
            for (int r = 0; r < B; ++r)
                for (int hh = 0; hh < H; ++hh) {
                    const size_t e = (size_t)r * H + hh;
                    const double hb = hbar[e];
                    const double i = w->gi[l][e], g = w->gg[l][e], o = w->go[l][e], tcv = w->tc[l][e];
                    const double ob = hb * tcv;
                    const double cb = (hb * o) * (1.0 - tcv * tcv);
                    const double ib = cb * g, gb = cb * i;
                    double* pb = pre_bar + (size_t)r * 4 * H;
                    pb[hh] = ib * i * (1.0 - i);
                    pb[2 * H + hh] = gb * (1.0 - g * g);
                    pb[3 * H + hh] = ob * o * (1.0 - o);
                }
            double* gb_ = gnet + t->off_bias[l];
            for (int r = 0; r < B; ++r)
                for (int c = 0; c < 4 * H; ++c) gb_[c] += pre_bar[(size_t)r * 4 * H + c];
            matmul_tn_acc(gnet + t->off_win[l], w->u[l], pre_bar, B, in_w, 4 * H);
            /* input adjoint u_bar = pre_bar * W_in^T */
            double* ubar = (l == 0) ? xbar : hbar;
            const double* Wl = t->W + t->off_win[l];
            double* tmp = (double*)xcalloc((size_t)B * in_w, sizeof(double));
            for (int r = 0; r < B; ++r)
                for (int kk = 0; kk < in_w; ++kk) {
                    double acc = 0.0;
                    for (int c = 0; c < 4 * H; ++c) acc += pre_bar[(size_t)r * 4 * H + c] * Wl[(size_t)kk * 4 * H + c];
                    tmp[(size_t)r * in_w + kk] = acc;
                }
            memcpy(ubar, tmp, sizeof(double) * (size_t)B * in_w);
            free(tmp);
        }
        if (bl > 0)
            for (size_t e = 0; e < (size_t)B * H; ++e) hbar[e] += resid[e];
    }
    free(resid);
    free(pre_bar);
    free(hbar);

    if (gps && t->cfg.attach_es_state) {
        const int k = w->k;
        double* lbar = (double*)xcalloc((size_t)k * T, sizeof(double));
        double* sbar = (double*)xcalloc((size_t)k * (T + S), sizeof(double));
        double* lg = (double*)xcalloc(B, sizeof(double));
        double* sout = (double*)xcalloc((size_t)B * O, sizeof(double));
        double* sin_ = (double*)xcalloc((size_t)B * I, sizeof(double));
        for (int b = 0; b < B; ++b) {
            /* targets = y_out / (seas_out * level): Div, Mul, BroadcastCol adjoints */
            double acc_o = 0.0;
            for (int j = 0; j < O; ++j) {
                const size_t e = (size_t)b * O + j;
                const double denb = -(tbar[e] * w->tgt[e] / w->den_out[e]);
                sout[e] = denb * w->lvl[b];
                const int idx = anchors[b] + 1 + j;
                acc_o += denb * w->seas[(size_t)w->wslot[b] * (T + S) + idx];
            }
            double acc_i = 0.0;
            for (int j = 0; j < I; ++j) {
                const size_t e = (size_t)b * I + j;
                const double xv = w->x[(size_t)b * in0 + j];
                const double denb = -(xbar[(size_t)b * in0 + j] * xv / w->den_in[e]);
                sin_[e] = denb * w->lvl[b];
                const int idx = anchors[b] - I + 1 + j;
                acc_i += denb * w->seas[(size_t)w->wslot[b] * (T + S) + idx];
            }
            lg[b] = acc_o;
            lg[b] += acc_i;
        }
        /* gather adjoints scatter in creation-reverse order: level, seas_out, seas_in */
        for (int b = 0; b < B; ++b) lbar[(size_t)w->wslot[b] * T + anchors[b]] += lg[b];
        for (int b = 0; b < B; ++b)
            for (int j = 0; j < O; ++j)
                sbar[(size_t)w->wslot[b] * (T + S) + anchors[b] + 1 + j] += sout[(size_t)b * O + j];
        for (int b = 0; b < B; ++b)
            for (int j = 0; j < I; ++j)
                sbar[(size_t)w->wslot[b] * (T + S) + anchors[b] - I + 1 + j] += sin_[(size_t)b * I + j];
        free(lg); free(sout); free(sin_);
        if (t->cfg.level_variability_penalty > 0.0) {
            double* c = lvp_weights(t, w, count);
            for (int s = 0; s < k; ++s) lvp_series(w->lev + (size_t)s * T, T, c[s], lbar + (size_t)s * T);
            free(c);
        }

        /* reverse HW scan per slot (holt_winters.hpp:266-277 adjoints) */
        for (int s = 0; s < k; ++s) {
            const double* y = w->y + (size_t)s * T;
            const double* lv = w->lev + (size_t)s * T;
            const double* se = w->seas + (size_t)s * (T + S);
            double* lb = lbar + (size_t)s * T;
            double* sb = sbar + (size_t)s * (T + S);
            const double a = w->alpha[s], g = w->gamma[s];
            double l0 = 0.0;
            for (int j = 0; j < S; ++j) l0 += y[j];
            l0 /= (double)S;
            double abar = 0.0, gbar = 0.0, omabar = 0.0, omgbar = 0.0;
            for (int tt = T - 1; tt >= 0; --tt) {
                const double lp = tt > 0 ? lv[tt - 1] : l0;
                const double Sb = sb[tt + S];
                /* s_{t+S} = gamma*(y/lp) + (1-gamma)*s_t */
                omgbar += Sb * se[tt];
                sb[tt] += Sb * (1.0 - g);
                const double d2 = y[tt] / lp;
                gbar += Sb * d2;
                const double d2b = Sb * g;
                if (tt > 0) lb[tt - 1] -= d2b * d2 / lp;
                /* l_t = alpha*(y/s_t) + (1-alpha)*lp */
                const double Lb = lb[tt];
                omabar += Lb * lp;
                if (tt > 0) lb[tt - 1] += Lb * (1.0 - a);
                const double d1 = y[tt] / se[tt];
                abar += Lb * d1;
                const double d1b = Lb * a;
                sb[tt] -= d1b * d1 / se[tt];
            }
            abar -= omabar;
            gbar -= omgbar;
            double* o = gps + (size_t)s * (2 + S);
            o[0] = abar * a * (1.0 - a);
            o[1] = gbar * g * (1.0 - g);
            for (int j = 0; j < S; ++j) o[2 + j] = sb[j] * se[j];
        }
        free(lbar);
        free(sbar);
    }
    free(xbar);
    free(pbar);
    free(tbar);
}

/* trainer.hpp:602-655 apply_updates */
static void apply_updates(esrnn_trainer* t, work_t* w, const double* gnet, const double* gps) {
    const int S = t->S;
    double sq = 0.0;
    for (int64_t p = 0; p < t->P; ++p) sq += gnet[p] * gnet[p];
    if (t->cfg.attach_es_state) {
        for (int s = 0; s < w->k; ++s) sq += gps[(size_t)s * (2 + S)] * gps[(size_t)s * (2 + S)];
        for (int s = 0; s < w->k; ++s) sq += gps[(size_t)s * (2 + S) + 1] * gps[(size_t)s * (2 + S) + 1];
        for (int s = 0; s < w->k; ++s)
            for (int j = 0; j < S; ++j) sq += gps[(size_t)s * (2 + S) + 2 + j] * gps[(size_t)s * (2 + S) + 2 + j];
    }
    double scale = 1.0;
    if (t->cfg.has_gradient_clip) {
        const double norm = sqrt(sq);
        if (norm > t->cfg.gradient_clip) scale = t->cfg.gradient_clip / norm;
    }
    t->net_step += 1;
    const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
    const double bc1 = 1.0 - pow(b1, (double)t->net_step), bc2 = 1.0 - pow(b2, (double)t->net_step);
    const double lr = t->cfg.learning_rate_network;
    for (int64_t p = 0; p < t->P; ++p) {
        const double g = gnet[p] * scale;
        t->mW[p] = b1 * t->mW[p] + (1.0 - b1) * g;
        t->vW[p] = b2 * t->vW[p] + (1.0 - b2) * g * g;
        t->W[p] -= lr * (t->mW[p] / bc1) / (sqrt(t->vW[p] / bc2) + eps);
    }
    if (!t->cfg.attach_es_state) return;
    const double lrs = t->cfg.learning_rate_per_series;
    for (int s = 0; s < w->k; ++s) {
        const int row = w->slot_series[s];
        t->steps[row] += 1;
        const double sc1 = 1.0 - pow(b1, (double)t->steps[row]), sc2 = 1.0 - pow(b2, (double)t->steps[row]);
#define ADAM(param, m, v, gin)                                                 \
    do {                                                                       \
        const double gg_ = (gin) * scale;                                      \
        (m) = b1 * (m) + (1.0 - b1) * gg_;                                     \
        (v) = b2 * (v) + (1.0 - b2) * gg_ * gg_;                               \
        (param) -= lrs * ((m) / sc1) / (sqrt((v) / sc2) + eps);                \
    } while (0)
        const double* gs = gps + (size_t)s * (2 + S);
        ADAM(t->a_raw[row], t->m_a[row], t->v_a[row], gs[0]);
        ADAM(t->g_raw[row], t->m_g[row], t->v_g[row], gs[1]);
        for (int j = 0; j < S; ++j)
            ADAM(t->s_raw[(size_t)row * S + j], t->m_s[(size_t)row * S + j], t->v_s[(size_t)row * S + j], gs[2 + j]);
#undef ADAM
    }
}

/* build_graph + backward + apply_updates for one caller batch (trainer.hpp:308-342, 593-600) */
static esrnn_status run_batch_impl(esrnn_trainer* t, int32_t B, const int32_t* rows,
                                   const int32_t* anchors, const double* mask, int32_t flags,
                                   double* loss, double* mask_count, double* inputs, double* targets,
                                   double* seas_out, double* levels, double* net_grads,
                                   int32_t* n_slots, int32_t* slot_rows, double* ps_grads) {
    const int O = t->O, S = t->S, I = t->I, T = t->T, in0 = t->in0;
    if (B <= 0) return fail(t->err, ESRNN_CONTRACT_ERROR, "batch: empty");
    work_t w;
    esrnn_status st = forward_batch(t, &w, B, rows, anchors);
    if (st) {
        work_free(&w, t->L);
        return st;
    }
    /* autodiff.hpp:370-395 masked-mean pinball */
    double count = 0.0, acc = 0.0;
    for (size_t e = 0; e < (size_t)B * O; ++e) count += (!mask || mask[e] != 0.0) ? 1.0 : 0.0;
    if (count == 0.0) {
        work_free(&w, t->L);
        return fail(t->err, ESRNN_CONTRACT_ERROR, "pinball: all-zero mask, mean undefined");
    }
    for (size_t e = 0; e < (size_t)B * O; ++e) {
        if (mask && mask[e] == 0.0) continue;
        const double d = w.tgt[e] - w.pred[e];
        acc += (d >= 0.0) ? t->cfg.tau * d : (t->cfg.tau - 1.0) * d;
    }
    double l = acc / count;
    if (t->cfg.level_variability_penalty > 0.0 && t->cfg.attach_es_state) {
        double* c = lvp_weights(t, &w, count);
        for (int s = 0; s < w.k; ++s) l += lvp_series(w.lev + (size_t)s * T, T, c[s], NULL);
        free(c);
    }
    if (loss) *loss = l;
    if (mask_count) *mask_count = count;
    if (inputs) memcpy(inputs, w.x, sizeof(double) * (size_t)B * in0);
    if (targets) memcpy(targets, w.tgt, sizeof(double) * (size_t)B * O);
    if (seas_out)
        for (int b = 0; b < B; ++b)
            for (int j = 0; j < O; ++j)
                seas_out[(size_t)b * O + j] = w.seas[(size_t)w.wslot[b] * (T + S) + anchors[b] + 1 + j];
    if (levels) memcpy(levels, w.lvl, sizeof(double) * B);
    if (n_slots) *n_slots = w.k;
    if (slot_rows) memcpy(slot_rows, w.slot_series, sizeof(int32_t) * w.k);
    (void)I;
    if (flags & ESRNN_BATCH_GRADS) {
        double* gnet = (double*)xcalloc(t->P, sizeof(double));
        double* gps = (double*)xcalloc((size_t)w.k * (2 + S), sizeof(double));
        backward_batch(t, &w, anchors, mask, count, gnet, gps);
        if (net_grads) memcpy(net_grads, gnet, sizeof(double) * t->P);
        if (ps_grads && t->cfg.attach_es_state) memcpy(ps_grads, gps, sizeof(double) * (size_t)w.k * (2 + S));
        if (flags & ESRNN_BATCH_UPDATE) apply_updates(t, &w, gnet, gps);
        free(gnet);
        free(gps);
    }
    work_free(&w, t->L);
    return ESRNN_OK;
}

esrnn_status esrnn_trainer_run_batch(esrnn_trainer* t, int32_t B, const int32_t* rows,
                                     const int32_t* anchors, const double* mask, int32_t flags,
                                     double* loss, double* mask_count, double* inputs,
                                     double* targets, double* seasonality_slices,
                                     double* anchor_levels, double* net_grads, int32_t* n_slots,
                                     int32_t* slot_rows, double* ps_grads) {
    return run_batch_impl(t, B, rows, anchors, mask, flags, loss, mask_count, inputs, targets,
                          seasonality_slices, anchor_levels, net_grads, n_slots, slot_rows, ps_grads);
}

/* trainer.hpp:214-223 all_windows, :82-102 make_batches, :234-243 train_epoch */
esrnn_status esrnn_trainer_train_epoch(esrnn_trainer* t, double* mean_loss) {
    const int I = t->I, O = t->O, T = t->T;
    const int per = T - O - I + 1;
    const int64_t nw = (int64_t)t->N * per;
    if (nw <= 0) return fail(t->err, ESRNN_CONTRACT_ERROR, "make_batches: no windows");
    int32_t* wr = (int32_t*)xcalloc(nw, sizeof(int32_t));
    int32_t* wa = (int32_t*)xcalloc(nw, sizeof(int32_t));
    int64_t n = 0;
    for (int r = 0; r < t->N; ++r)
        for (int a = I - 1; a <= T - O - 1; ++a) {
            wr[n] = r;
            wa[n] = a;
            ++n;
        }
    for (int64_t i = nw; i > 1; --i) {   /* matrix.hpp:203-205 */
        const int64_t j = (int64_t)rng_below(&t->rng, (uint64_t)i);
        int32_t tr = wr[i - 1], ta = wa[i - 1];
        wr[i - 1] = wr[j]; wa[i - 1] = wa[j];
        wr[j] = tr; wa[j] = ta;
    }
    double acc = 0.0, weight = 0.0;
    esrnn_status st = ESRNN_OK;
    for (int64_t start = 0; start < nw; start += t->cfg.batch_size) {
        const int64_t stop = start + t->cfg.batch_size < nw ? start + t->cfg.batch_size : nw;
        double l = 0.0, mc = 0.0;
        st = run_batch_impl(t, (int32_t)(stop - start), wr + start, wa + start, NULL,
                            ESRNN_BATCH_GRADS | ESRNN_BATCH_UPDATE, &l, &mc, NULL, NULL, NULL, NULL,
                            NULL, NULL, NULL, NULL);
        if (st) break;
        acc += l * mc;
        weight += mc;
    }
    free(t->last_wr);
    free(t->last_wa);
    t->last_wr = wr;
    t->last_wa = wa;
    t->last_nw = nw;
    if (st) return st;
    *mean_loss = acc / weight;
    return ESRNN_OK;
}

/* trainer.hpp:248-288 forecast_at with the plain primer (holt_winters.hpp:66-97),
 * deseasonalize_normalize (:153-166), plain::forward_stack (network.hpp:268-287),
 * reseasonalize_denormalize (:169-181) and HWState::seasonal_at (:55-59). */
esrnn_status esrnn_trainer_forecast(esrnn_trainer* t, int64_t drop_tail, double* out) {
    const int I = t->I, O = t->O, S = t->S, H = t->H, in0 = t->in0, N = t->N;
    if ((int64_t)t->LEN < drop_tail + I)
        return fail(t->err, ESRNN_INSUFFICIENT_LENGTH, "forecast_at: not enough in-sample data");
    const int tins = (int)(t->LEN - drop_tail);
    if (tins < S)
        return fail(t->err, ESRNN_INSUFFICIENT_LENGTH, "hybrid_primer: series length %d shorter than season length %d", tins, S);
    double* X = (double*)xcalloc((size_t)N * in0, sizeof(double));
    double* lvl_last = (double*)xcalloc(N, sizeof(double));
    double* seas_o = (double*)xcalloc((size_t)N * O, sizeof(double));
    double* se = (double*)xcalloc((size_t)tins + S, sizeof(double));
    esrnn_status st = ESRNN_OK;
    for (int r = 0; r < N && !st; ++r) {
        const double* v = t->vals + (size_t)r * t->LEN;
        for (int tt = 0; tt < tins; ++tt)
            if (!(v[tt] > 0.0)) {
                st = fail(t->err, ESRNN_NUMERIC_DOMAIN_ERROR, "hybrid_primer: non-positive observation at t=%d", tt);
                break;
            }
        if (st) break;
        for (int j = 0; j < S; ++j) se[j] = fm_exp(t->s_raw[(size_t)r * S + j]);
        const double a = fm_logistic(t->a_raw[r]), g = fm_logistic(t->g_raw[r]);
        double lp = 0.0;
        for (int j = 0; j < S; ++j) lp += v[j];
        lp /= (double)S;
        for (int tt = 0; tt < tins; ++tt) {
            const double lvl = a * (v[tt] / se[tt]) + (1.0 - a) * lp;
            if (!(lvl > 0.0) || !isfinite(lvl)) {
                st = fail(t->err, ESRNN_NUMERIC_DOMAIN_ERROR, "hybrid_primer: non-positive level at t=%d", tt);
                break;
            }
            se[tt + S] = g * (v[tt] / lp) + (1.0 - g) * se[tt];
            lp = lvl;
        }
        if (st) break;
        const double level = lp;
        lvl_last[r] = level;
        for (int j = 0; j < I; ++j) {
            const double sv = se[tins - I + j];
            if (!(sv > 0.0)) {
                st = fail(t->err, ESRNN_NUMERIC_DOMAIN_ERROR, "deseasonalize_normalize: non-positive seasonality");
                break;
            }
            X[(size_t)r * in0 + j] = v[tins - I + j] / (level * sv);
        }
        const int c = t->cat[r];
        X[(size_t)r * in0 + I + c] = 1.0;
        for (int j = 0; j < O; ++j) {
            size_t idx = (size_t)tins + j;
            while (idx >= (size_t)tins + S) idx -= S;
            seas_o[(size_t)r * O + j] = se[idx];
        }
    }
    free(se);
    if (!st) {
        /* plain stack forward on all rows */
        double* pre = (double*)xcalloc((size_t)N * 4 * H, sizeof(double));
        double* hbuf = (double*)xcalloc((size_t)N * H, sizeof(double));
        double* cur = (double*)xcalloc((size_t)N * H, sizeof(double));
        double* blk = (double*)xcalloc((size_t)N * H, sizeof(double));
        const double* in = X;
        int in_w = in0, layer = 0;
        for (int bl = 0; bl < t->nb; ++bl) {
            if (bl > 0) memcpy(blk, cur, sizeof(double) * (size_t)N * H);
            for (int j = 0; j < t->blen[bl]; ++j, ++layer) {
                matmul(pre, in, t->W + t->off_win[layer], N, in_w, 4 * H, 4 * H);
                const double* bias = t->W + t->off_bias[layer];
                for (int r = 0; r < N; ++r)
                    for (int hh = 0; hh < H; ++hh) {
                        const double* p = pre + (size_t)r * 4 * H;
                        const double i = fm_logistic(p[hh] + bias[hh]);
                        const double g = fm_tanh(p[2 * H + hh] + bias[2 * H + hh]);
                        const double o = fm_logistic(p[3 * H + hh] + bias[3 * H + hh]);
                        const double cc = 0.0 + i * g;
                        hbuf[(size_t)r * H + hh] = o * fm_tanh(cc);
                    }
                memcpy(cur, hbuf, sizeof(double) * (size_t)N * H);
                in = cur;
                in_w = H;
            }
            if (bl > 0)
                for (size_t e = 0; e < (size_t)N * H; ++e) cur[e] = cur[e] + blk[e];
        }
        double* z = (double*)xcalloc((size_t)N * H, sizeof(double));
        matmul(z, cur, t->W + t->off_nlw, N, H, H, H);
        for (int r = 0; r < N; ++r)
            for (int c = 0; c < H; ++c) z[(size_t)r * H + c] = fm_tanh(z[(size_t)r * H + c] + t->W[t->off_nlb + c]);
        matmul(out, z, t->W + t->off_outw, N, H, O, O);
        for (int r = 0; r < N; ++r) {
            if (!(lvl_last[r] > 0.0)) {
                st = fail(t->err, ESRNN_NUMERIC_DOMAIN_ERROR, "reseasonalize_denormalize: level must be positive");
                break;
            }
            for (int c = 0; c < O; ++c) {
                const double pr = out[(size_t)r * O + c] + t->W[t->off_outb + c];
                out[(size_t)r * O + c] = pr * lvl_last[r] * seas_o[(size_t)r * O + c];
            }
        }
        free(z); free(pre); free(hbuf); free(cur); free(blk);
    }
    free(X);
    free(lvl_last);
    free(seas_o);
    return st;
}

/* metrics.hpp:17-28 sMAPE */
static double smape(const double* a, const double* f, int n) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) {
        const double den = fabs(a[i]) + fabs(f[i]);
        if (den > 0.0) acc += fabs(a[i] - f[i]) / den;
    }
    return 200.0 * acc / (double)n;
}

/* trainer.hpp:292-305 validate */
esrnn_status esrnn_trainer_validate(esrnn_trainer* t, double* forecasts, double* smape_per_series,
                                    double* mean_smape) {
    const int O = t->O, N = t->N;
    double* fc = (double*)xcalloc((size_t)N * O, sizeof(double));
    esrnn_status st = esrnn_trainer_forecast(t, 2 * O, fc);
    if (!st) {
        double acc = 0.0;
        for (int r = 0; r < N; ++r) {
            const double s = smape(t->vals + (size_t)r * t->LEN + t->T, fc + (size_t)r * O, O);
            if (smape_per_series) smape_per_series[r] = s;
            acc += s;
        }
        if (mean_smape) *mean_smape = acc / (double)N;
        if (forecasts) memcpy(forecasts, fc, sizeof(double) * (size_t)N * O);
    }
    free(fc);
    return st;
}

/* network.hpp:148-210 forward_stack over a general sequence (full LSTM cells with forget
 * gates, recurrent matrices and (h, c) from step t-d), and the adjoints of Tape::backward
 * for an upstream out_bar (autodiff.hpp:428-610: MatMul / Add / Mul / Logistic / Tanh). */
esrnn_status esrnn_trainer_forward_stack(esrnn_trainer* t, int32_t T, int32_t B, const double* X, double* out,
                                         const double* obar, double* wbar, double* xbar) {
    if (T < 1) return fail(t->err, ESRNN_CONTRACT_ERROR, "forward_stack: empty sequence");
    if (B < 1) return fail(t->err, ESRNN_SHAPE_ERROR, "forward_stack: empty batch");
    const int L = t->L, H = t->H, O = t->O, in0 = t->in0, G = 4 * H;
    int dil[MAXL], res_src[MAXL];
    for (int l = 0, b = 0, first = 0; b < t->nb; first += t->blen[b], ++b)
        for (int j = 0; j < t->blen[b]; ++j, ++l) {
            dil[l] = t->prof.dilations[l];
            res_src[l] = (b > 0 && j == t->blen[b] - 1) ? first - 1 : -1;
        }
    const size_t LTB = (size_t)L * T * B;
    double* gates = (double*)xcalloc(LTB * G, sizeof(double));
    double* cs = (double*)xcalloc(LTB * H, sizeof(double));
    double* hr = (double*)xcalloc(LTB * H, sizeof(double));
    double* cur = (double*)xcalloc(LTB * H, sizeof(double));
    double* z = (double*)xcalloc((size_t)B * H, sizeof(double));
#define SI(l, tt, r) ((((size_t)(l) * T + (tt)) * B + (r)))
    const double* W = t->W;
    for (int l = 0; l < L; ++l) {
        const int K = t->layer_in[l], d = dil[l];
        for (int tt = 0; tt < T; ++tt)
            for (int r = 0; r < B; ++r) {
                const double* x = l == 0 ? X + ((size_t)tt * B + r) * in0 : cur + SI(l - 1, tt, r) * H;
                double* g = gates + SI(l, tt, r) * G;
                for (int j = 0; j < G; ++j) {
                    double a = 0.0;
                    for (int k = 0; k < K; ++k) a += x[k] * W[t->off_win[l] + (int64_t)k * G + j];
                    if (tt >= d) {
                        const double* hp = hr + SI(l, tt - d, r) * H;
                        double a2 = 0.0;
                        for (int k = 0; k < H; ++k) a2 += hp[k] * W[t->off_wrec[l] + (int64_t)k * G + j];
                        a += a2;
                    }
                    a += W[t->off_bias[l] + j];
                    g[j] = (j >= 2 * H && j < 3 * H) ? fm_tanh(a) : fm_logistic(a);
                }
                for (int j = 0; j < H; ++j) {
                    const double c = (tt >= d ? g[H + j] * cs[SI(l, tt - d, r) * H + j] : 0.0) + g[j] * g[2 * H + j];
                    const double h = g[3 * H + j] * fm_tanh(c);
                    cs[SI(l, tt, r) * H + j] = c;
                    hr[SI(l, tt, r) * H + j] = h;
                    cur[SI(l, tt, r) * H + j] = res_src[l] >= 0 ? h + cur[SI(res_src[l], tt, r) * H + j] : h;
                }
            }
    }
    for (int r = 0; r < B; ++r) {
        const double* last = cur + SI(L - 1, T - 1, r) * H;
        for (int j = 0; j < H; ++j) {
            double a = 0.0;
            for (int k = 0; k < H; ++k) a += last[k] * W[t->off_nlw + (int64_t)k * H + j];
            z[(size_t)r * H + j] = fm_tanh(a + W[t->off_nlb + j]);
        }
        for (int o = 0; o < O; ++o) {
            double a = 0.0;
            for (int k = 0; k < H; ++k) a += z[(size_t)r * H + k] * W[t->off_outw + (int64_t)k * O + o];
            if (out) out[(size_t)r * O + o] = a + W[t->off_outb + o];
        }
    }
    if (obar) {
        double* wb = (double*)xcalloc((size_t)t->P, sizeof(double));
        double* dcur = (double*)xcalloc(LTB * H, sizeof(double));
        double* dhr = (double*)xcalloc((size_t)T * B * H, sizeof(double));
        double* dcr = (double*)xcalloc((size_t)T * B * H, sizeof(double));
        double* dpre = (double*)xcalloc((size_t)T * B * G, sizeof(double));
        double* dzp = (double*)xcalloc((size_t)B * H, sizeof(double));
        for (int r = 0; r < B; ++r) {
            const double* ob = obar + (size_t)r * O;
            const double* last = cur + SI(L - 1, T - 1, r) * H;
            for (int o = 0; o < O; ++o) wb[t->off_outb + o] += ob[o];
            for (int k = 0; k < H; ++k) {
                double dz = 0.0;
                for (int o = 0; o < O; ++o) {
                    wb[t->off_outw + (int64_t)k * O + o] += z[(size_t)r * H + k] * ob[o];
                    dz += ob[o] * W[t->off_outw + (int64_t)k * O + o];
                }
                dzp[(size_t)r * H + k] = dz * (1.0 - z[(size_t)r * H + k] * z[(size_t)r * H + k]);
            }
            for (int j = 0; j < H; ++j) wb[t->off_nlb + j] += dzp[(size_t)r * H + j];
            for (int k = 0; k < H; ++k) {
                double a = 0.0;
                for (int j = 0; j < H; ++j) {
                    wb[t->off_nlw + (int64_t)k * H + j] += last[k] * dzp[(size_t)r * H + j];
                    a += dzp[(size_t)r * H + j] * W[t->off_nlw + (int64_t)k * H + j];
                }
                dcur[SI(L - 1, T - 1, r) * H + k] = a;
            }
        }
        for (int l = L - 1; l >= 0; --l) {
            const int K = t->layer_in[l], d = dil[l];
            if (res_src[l] >= 0)
                for (size_t e = 0; e < (size_t)T * B * H; ++e) {
                    const size_t tt = e / ((size_t)B * H), rj = e % ((size_t)B * H);
                    dcur[SI(res_src[l], tt, 0) * H + rj] += dcur[SI(l, tt, 0) * H + rj];
                }
            memset(dhr, 0, sizeof(double) * (size_t)T * B * H);
            memset(dcr, 0, sizeof(double) * (size_t)T * B * H);
            for (int tt = T - 1; tt >= 0; --tt)
                for (int r = 0; r < B; ++r) {
                    const double* g = gates + SI(l, tt, r) * G;
                    double* dp = dpre + ((size_t)tt * B + r) * G;
                    for (int j = 0; j < H; ++j) {
                        const double i = g[j], f = g[H + j], gg = g[2 * H + j], o = g[3 * H + j];
                        const double tc = fm_tanh(cs[SI(l, tt, r) * H + j]);
                        const size_t q = ((size_t)tt * B + r) * H + j;
                        const double dh = dcur[SI(l, tt, r) * H + j] + dhr[q];
                        const double dc = dcr[q] + dh * o * (1.0 - tc * tc);
                        double df = 0.0;
                        if (tt >= d) {
                            df = dc * cs[SI(l, tt - d, r) * H + j];
                            dcr[((size_t)(tt - d) * B + r) * H + j] += dc * f;
                        }
                        dp[j] = dc * gg * i * (1.0 - i);
                        dp[H + j] = df * f * (1.0 - f);
                        dp[2 * H + j] = dc * i * (1.0 - gg * gg);
                        dp[3 * H + j] = dh * tc * o * (1.0 - o);
                    }
                    for (int k = 0; k < K; ++k) {
                        double a = 0.0;
                        for (int j = 0; j < G; ++j) a += dp[j] * W[t->off_win[l] + (int64_t)k * G + j];
                        if (l > 0) dcur[SI(l - 1, tt, r) * H + k] += a;
                        else if (xbar) xbar[((size_t)tt * B + r) * in0 + k] = a;
                    }
                    if (tt >= d)
                        for (int k = 0; k < H; ++k) {
                            double a = 0.0;
                            for (int j = 0; j < G; ++j) a += dp[j] * W[t->off_wrec[l] + (int64_t)k * G + j];
                            dhr[((size_t)(tt - d) * B + r) * H + k] += a;
                        }
                    const double* x = l == 0 ? X + ((size_t)tt * B + r) * in0 : cur + SI(l - 1, tt, r) * H;
                    for (int j = 0; j < G; ++j) {
                        for (int k = 0; k < K; ++k) wb[t->off_win[l] + (int64_t)k * G + j] += x[k] * dp[j];
                        if (tt >= d)
                            for (int k = 0; k < H; ++k)
                                wb[t->off_wrec[l] + (int64_t)k * G + j] += hr[SI(l, tt - d, r) * H + k] * dp[j];
                        wb[t->off_bias[l] + j] += dp[j];
                    }
                }
        }
        if (wbar) memcpy(wbar, wb, sizeof(double) * (size_t)t->P);
        free(wb), free(dcur), free(dhr), free(dcr), free(dpre), free(dzp);
    }
#undef SI
    free(gates), free(cs), free(hr), free(cur), free(z);
    return ESRNN_OK;
}

/* Exact-resume training state (B200 extension of the ABI): the Adam moments / steps of
 * apply_updates (trainer.hpp:602-655) and the trainer RNG in std::mt19937_64's text form
 * (the 312 state words, then the position), which this MT19937-64 restatement shares. */
esrnn_status esrnn_trainer_get_train_state(esrnn_trainer* t, double* adam_m, double* adam_v, int64_t n_values,
                                           int64_t row_begin, int64_t n, double* ps_m, double* ps_v,
                                           int64_t* ps_steps, int64_t* net_step, char* rng_text, int64_t rng_cap) {
    const int S = t->S;
    if ((adam_m || adam_v) && n_values != t->P)
        return fail(t->err, ESRNN_CHECKPOINT_ERROR, "train state: %lld network values, expected %lld", (long long)n_values, (long long)t->P);
    if (n < 0 || row_begin < 0 || row_begin + n > t->N) return fail(t->err, ESRNN_SHAPE_ERROR, "train state: rows out of range");
    if (adam_m) memcpy(adam_m, t->mW, sizeof(double) * (size_t)t->P);
    if (adam_v) memcpy(adam_v, t->vW, sizeof(double) * (size_t)t->P);
    for (int64_t i = 0; i < n; ++i) {
        const int64_t r = row_begin + i;
        if (ps_m) {
            ps_m[i * (2 + S)] = t->m_a[r];
            ps_m[i * (2 + S) + 1] = t->m_g[r];
            for (int j = 0; j < S; ++j) ps_m[i * (2 + S) + 2 + j] = t->m_s[(size_t)r * S + j];
        }
        if (ps_v) {
            ps_v[i * (2 + S)] = t->v_a[r];
            ps_v[i * (2 + S) + 1] = t->v_g[r];
            for (int j = 0; j < S; ++j) ps_v[i * (2 + S) + 2 + j] = t->v_s[(size_t)r * S + j];
        }
        if (ps_steps) ps_steps[i] = t->steps[r];
    }
    if (net_step) *net_step = t->net_step;
    if (rng_text) {
        int64_t at = 0;
        for (int i = 0; i <= MT_N; ++i) {
            char buf[32];
            const int k = i < MT_N ? snprintf(buf, sizeof buf, "%llu ", (unsigned long long)t->rng.mt[i])
                                   : snprintf(buf, sizeof buf, "%d", t->rng.mti);
            if (at + k + 1 > rng_cap) return fail(t->err, ESRNN_SHAPE_ERROR, "train state: rng buffer too small");
            memcpy(rng_text + at, buf, (size_t)k);
            at += k;
        }
        rng_text[at] = 0;
    }
    return ESRNN_OK;
}

esrnn_status esrnn_trainer_set_train_state(esrnn_trainer* t, const double* adam_m, const double* adam_v,
                                           int64_t n_values, int64_t row_begin, int64_t n, const double* ps_m,
                                           const double* ps_v, const int64_t* ps_steps, int64_t net_step,
                                           const char* rng_text) {
    const int S = t->S;
    if ((adam_m || adam_v) && n_values != t->P)
        return fail(t->err, ESRNN_CHECKPOINT_ERROR, "train state: %lld network values, expected %lld", (long long)n_values, (long long)t->P);
    if (n < 0 || row_begin < 0 || row_begin + n > t->N) return fail(t->err, ESRNN_SHAPE_ERROR, "train state: rows out of range");
    if (net_step < 0) return fail(t->err, ESRNN_CHECKPOINT_ERROR, "train state: negative Adam step");
    rng_t g = t->rng;
    if (rng_text) {
        const char* p = rng_text;
        for (int i = 0; i <= MT_N; ++i) {
            char* end = NULL;
            const unsigned long long v = strtoull(p, &end, 10);
            if (end == p) return fail(t->err, ESRNN_CHECKPOINT_ERROR, "train state: malformed rng state");
            if (i < MT_N) g.mt[i] = (uint64_t)v;
            else g.mti = (int)v;
            p = end;
        }
    }
    if (adam_m) memcpy(t->mW, adam_m, sizeof(double) * (size_t)t->P);
    if (adam_v) memcpy(t->vW, adam_v, sizeof(double) * (size_t)t->P);
    for (int64_t i = 0; i < n; ++i) {
        const int64_t r = row_begin + i;
        if (ps_m) {
            t->m_a[r] = ps_m[i * (2 + S)];
            t->m_g[r] = ps_m[i * (2 + S) + 1];
            for (int j = 0; j < S; ++j) t->m_s[(size_t)r * S + j] = ps_m[i * (2 + S) + 2 + j];
        }
        if (ps_v) {
            t->v_a[r] = ps_v[i * (2 + S)];
            t->v_g[r] = ps_v[i * (2 + S) + 1];
            for (int j = 0; j < S; ++j) t->v_s[(size_t)r * S + j] = ps_v[i * (2 + S) + 2 + j];
        }
        if (ps_steps) t->steps[r] = (long)ps_steps[i];
    }
    t->net_step = (long)net_step;
    t->rng = g;
    return ESRNN_OK;
}

/* metrics.hpp:33-49 mase: forecast MAE over the in-sample seasonal-naive MAE; returns NAN for
 * the reference's std::nullopt (zero denominator) */
static double mase(const double* ins, int n_ins, const double* a, const double* f, int n, int S) {
    double den = 0.0;
    for (int t = S; t < n_ins; ++t) den += fabs(ins[t] - ins[t - S]);
    den /= (double)(n_ins - S);
    if (den == 0.0) return NAN;
    double num = 0.0;
    for (int i = 0; i < n; ++i) num += fabs(a[i] - f[i]);
    num /= (double)n;
    return num / den;
}

/* commands.hpp:285-338 score_forecasts / cmd_evaluate with metrics.hpp:52-59 seasonal_naive */
esrnn_status esrnn_trainer_evaluate(esrnn_trainer* t, int32_t against_test, double* forecasts, double* smape_o,
                                    double* mase_o, double* naive_smape, double* naive_mase, double* totals) {
    const int O = t->O, N = t->N, S = t->S;
    const int t_ins = against_test ? t->T + O : t->T;
    if (t_ins <= S) return fail(t->err, ESRNN_INSUFFICIENT_LENGTH, "mase: in-sample length must exceed season length");
    double* fc = (double*)xcalloc((size_t)N * O, sizeof(double));
    double* nv = (double*)xcalloc((size_t)O, sizeof(double));
    esrnn_status st = esrnn_trainer_forecast(t, against_test ? O : 2 * O, fc);
    if (!st) {
        double tot[8] = {0, 0, 0, 0, 0, 0, (double)N, 0};
        for (int r = 0; r < N; ++r) {
            const double* v = t->vals + (size_t)r * t->LEN;
            const double* act = v + t_ins;
            const double* f = fc + (size_t)r * O;
            for (int i = 0; i < O; ++i) nv[i] = v[t_ins - S + (i % S)];
            const double s = smape(act, f, O), m = mase(v, t_ins, act, f, O, S);
            const double ns = smape(act, nv, O), nm = mase(v, t_ins, act, nv, O, S);
            if (smape_o) smape_o[r] = s;
            if (mase_o) mase_o[r] = m;
            if (naive_smape) naive_smape[r] = ns;
            if (naive_mase) naive_mase[r] = nm;
            tot[0] += s;
            if (!isnan(m)) { tot[1] += m; tot[2] += 1; }
            tot[3] += ns;
            if (!isnan(nm)) { tot[4] += nm; tot[5] += 1; }
        }
        if (forecasts) memcpy(forecasts, fc, sizeof(double) * (size_t)N * O);
        if (totals) memcpy(totals, tot, sizeof tot);
    }
    free(nv);
    free(fc);
    return st;
}

/* holt_winters.hpp:66-97 hybrid_primer on values[0:t_len] of one series */
esrnn_status esrnn_trainer_hw_state(esrnn_trainer* t, int64_t row, int64_t t_len, double* levels,
                                    double* seas) {
    const int S = t->S;
    if (row < 0 || row >= t->N) return fail(t->err, ESRNN_SHAPE_ERROR, "hw_state: row out of range");
    if (t_len < S || t_len > t->LEN)
        return fail(t->err, ESRNN_INSUFFICIENT_LENGTH, "hybrid_primer: series length %lld shorter than season length %d", (long long)t_len, S);
    const double* v = t->vals + (size_t)row * t->LEN;
    for (int64_t tt = 0; tt < t_len; ++tt)
        if (!(v[tt] > 0.0))
            return fail(t->err, ESRNN_NUMERIC_DOMAIN_ERROR, "hybrid_primer: non-positive observation at t=%lld", (long long)tt);
    for (int j = 0; j < S; ++j) seas[j] = fm_exp(t->s_raw[(size_t)row * S + j]);
    const double a = fm_logistic(t->a_raw[row]), g = fm_logistic(t->g_raw[row]);
    double lp = 0.0;
    for (int j = 0; j < S; ++j) lp += v[j];
    lp /= (double)S;
    for (int64_t tt = 0; tt < t_len; ++tt) {
        const double lvl = a * (v[tt] / seas[tt]) + (1.0 - a) * lp;
        if (!(lvl > 0.0) || !isfinite(lvl))
            return fail(t->err, ESRNN_NUMERIC_DOMAIN_ERROR, "hybrid_primer: non-positive level at t=%lld", (long long)tt);
        seas[tt + S] = g * (v[tt] / lp) + (1.0 - g) * seas[tt];
        levels[tt] = lvl;
        lp = lvl;
    }
    return ESRNN_OK;
}

esrnn_status esrnn_trainer_last_epoch_windows(const esrnn_trainer* t, int32_t* rows, int32_t* anchors, int64_t n) {
    if (n != t->last_nw || !t->last_wr) return ESRNN_SHAPE_ERROR;
    memcpy(rows, t->last_wr, sizeof(int32_t) * n);
    memcpy(anchors, t->last_wa, sizeof(int32_t) * n);
    return ESRNN_OK;
}

esrnn_status esrnn_trainer_last_device_ms(const esrnn_trainer* t, double* ms) {
    *ms = t->last_ms;
    return ESRNN_OK;
}

esrnn_status esrnn_trainer_kernel_launches(const esrnn_trainer* t, int64_t* n) {
    (void)t;
    *n = 0;
    return ESRNN_OK;
}

esrnn_status esrnn_trainer_profile_kernels(esrnn_trainer* t, int32_t enable) {
    (void)t; (void)enable;
    return ESRNN_OK;
}

esrnn_status esrnn_trainer_kernel_times(esrnn_trainer* t, double* total_ms, int64_t* launches) {
    (void)t;
    for (int i = 0; i < ESRNN_KERNEL_CLASSES; ++i) {
        if (total_ms) total_ms[i] = 0.0;
        if (launches) launches[i] = 0;
    }
    return ESRNN_OK;
}

esrnn_status esrnn_release_cached_memory(void) { return ESRNN_OK; }

/* Sharded-mode entry points (B200 extension): the oracle is single-process, unsharded. */
esrnn_status esrnn_group_create(int32_t world_size, esrnn_group** out) {
    (void)world_size;
    *out = NULL;
    snprintf(g_create_err, sizeof g_create_err, "oracle: no sharded mode");
    return ESRNN_CONFIG_ERROR;
}
void esrnn_group_destroy(esrnn_group* g) { (void)g; }
esrnn_status esrnn_trainer_gather_per_series(esrnn_trainer* t, double* a, double* g, double* s) {
    return esrnn_trainer_get_per_series(t, 0, t->N, a, g, s);
}

esrnn_status esrnn_nccl_unique_id(uint8_t out[128]) {
    (void)out;
    snprintf(g_create_err, sizeof g_create_err, "oracle: no NCCL");
    return ESRNN_NCCL_ERROR;
}

/* tests/helpers.hpp:148-172 make_multiplicative_series, consumed in order from Rng(seed) */
esrnn_status esrnn_make_synthetic(uint64_t seed, int64_t n, int32_t length, int32_t season_length,
                                  double noise_sigma, double* values, int32_t* category) {
    rng_t rng;
    rng_seed(&rng, seed);
    double* season = (double*)xcalloc(season_length, sizeof(double));
    for (int64_t i = 0; i < n; ++i) {
        category[i] = (int32_t)rng_below(&rng, 6);
        const double level = rng_uniform(&rng, 50.0, 150.0);
        const double trend = rng_uniform(&rng, 0.005, 0.02);
        double log_mean = 0.0;
        for (int j = 0; j < season_length; ++j) {
            season[j] = rng_uniform(&rng, 0.6, 1.4);
            log_mean += log(season[j]);
        }
        log_mean /= (double)season_length;
        for (int j = 0; j < season_length; ++j) season[j] = exp(log(season[j]) - log_mean);
        for (int tt = 0; tt < length; ++tt) {
            const double noise = noise_sigma > 0.0 ? exp(noise_sigma * rng_normal(&rng)) : 1.0;
            values[i * length + tt] = level * pow(1.0 + trend, (double)tt) * season[tt % season_length] * noise;
        }
    }
    free(season);
    return ESRNN_OK;
}

/* Ingestion: not restated in C -- its checker is the reference's own parser behind
 * oracle/ref_shim.cpp (data.hpp:205-290 compiled where it lies). */
struct esrnn_dataset { int unused; };
const char* esrnn_ingest_last_error(void) { return "C oracle: ingestion is checked against the reference shim"; }
esrnn_status esrnn_ingest_m4_csv(const char* train_csv, const char* info_csv, int32_t frequency,
                                 const esrnn_profile* profile, int32_t threads, esrnn_dataset** out,
                                 esrnn_ingest_stats* stats) {
    (void)train_csv; (void)info_csv; (void)frequency; (void)profile; (void)threads; (void)stats;
    *out = NULL;
    return ESRNN_ERROR;
}
esrnn_status esrnn_dataset_shape(const esrnn_dataset* d, int64_t* n, int32_t* length) {
    (void)d; *n = 0; *length = 0;
    return ESRNN_ERROR;
}
const double* esrnn_dataset_values(const esrnn_dataset* d) { (void)d; return NULL; }
const int32_t* esrnn_dataset_categories(const esrnn_dataset* d) { (void)d; return NULL; }
const char* esrnn_dataset_id(const esrnn_dataset* d, int64_t i) { (void)d; (void)i; return NULL; }
void esrnn_dataset_destroy(esrnn_dataset* d) { (void)d; }
