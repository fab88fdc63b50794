/* ORACLE / TEST INFRASTRUCTURE ONLY — CPU restatement of the reference MEFT hot path.
 * See meft_oracle.h for the contract, the parity pins and who may load this.
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj). Compiled with -ffp-contract=off (oracle/Makefile). */
#include "meft_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- rng.hpp */

uint64_t or_mix_seed(uint64_t seed, uint64_t stream) { /* rng.hpp:13-21 */
    uint64_t x = seed ^ (0x9E3779B97F4A7C15ull * (stream + 1));
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

/* std::mt19937_64 as specified by [rand.eng.mers] (the reference relies on its
 * standard-mandated raw output, rng.hpp:23-25, 30). */
typedef struct {
    uint64_t s[312];
    int i;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
    g->s[0] = seed;
    for (int k = 1; k < 312; ++k) g->s[k] = 6364136223846793005ull * (g->s[k - 1] ^ (g->s[k - 1] >> 62)) + (uint64_t)k;
    g->i = 312;
}

static uint64_t mt64_next(mt64* g) {
    if (g->i >= 312) {
        for (int k = 0; k < 312; ++k) {
            const uint64_t y = (g->s[k] & 0xFFFFFFFF80000000ull) | (g->s[(k + 1) % 312] & 0x7FFFFFFFull);
            uint64_t v = g->s[(k + 156) % 312] ^ (y >> 1);
            if (y & 1ull) v ^= 0xB5026F5AA96619E9ull;
            g->s[k] = v;
        }
        g->i = 0;
    }
    uint64_t z = g->s[g->i++];
    z ^= (z >> 29) & 0x5555555555555555ull;
    z ^= (z << 17) & 0x71D67FFFEDA60000ull;
    z ^= (z << 37) & 0xFFF7EEE000000000ull;
    z ^= z >> 43;
    return z;
}

void or_uniform_matrix(uint64_t seed, int64_t count, double lo, double hi, double* out) {
    /* rng.hpp:34-36 uniform() = (u64 >> 11) * 2^-53; uniform(lo,hi) = lo + (hi-lo)*u.
     * The compiled reference (FMA-capable -march) contracts lo + (hi-lo)*u into one fma;
     * we restate the compiled form so HostStore::init tables match bit for bit. */
    mt64* g = (mt64*)malloc(sizeof(mt64));
    mt64_seed(g, seed);
    for (int64_t i = 0; i < count; ++i) {
        const double u = (double)(mt64_next(g) >> 11) * 0x1.0p-53;
        out[i] = fma(hi - lo, u, lo);
    }
    free(g);
}

/* ------------------------------------------------------------ kernels.hpp */

double or_dot(const double* a, const double* b, int64_t d) { /* kernels.hpp:37-41 */
    double acc = 0.0;
    for (int64_t k = 0; k < d; ++k) acc += a[k] * b[k];
    return acc;
}

/* kernels.cpp:34-41 matmul_row: out[i,:] += a[i,k]*b[k,:] over ascending k, a[i,k]==0 skipped.
 * The compiled reference contracts this into an fma chain. */
void or_matmul(const double* a, const double* b, int64_t m, int64_t k, int64_t n, double* out) {
#pragma omp parallel for schedule(static) if (m * k * n > 32768)
    for (int64_t i = 0; i < m; ++i) {
        double* orow = out + i * n;
        for (int64_t j = 0; j < n; ++j) orow[j] = 0.0;
        for (int64_t kk = 0; kk < k; ++kk) {
            const double aik = a[i * k + kk];
            if (aik == 0.0) continue;
            const double* brow = b + kk * n;
            for (int64_t j = 0; j < n; ++j) orow[j] = fma(aik, brow[j], orow[j]);
        }
    }
}

static double* transpose_new(const double* a, int64_t rows, int64_t cols) {
    double* t = (double*)malloc(sizeof(double) * (size_t)(rows * cols > 0 ? rows * cols : 1));
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t j = 0; j < cols; ++j) t[j * rows + i] = a[i * cols + j];
    return t;
}

/* ------------------------------------------------------------ experts.cpp */

void or_route_scores(const double* h_token, int64_t d, const double* w_g, int64_t n, double* p) {
    for (int64_t i = 0; i < n; ++i) p[i] = or_dot(w_g + i * d, h_token, d); /* experts.cpp:21-28 */
}

/* Total order of experts.cpp:36-41 / :96-100 / adapter.cpp:67-72:
 * higher score first; equal scores (==, so -0.0 == +0.0) -> lower index first. */
static int beats(double sa, int64_t ia, double sb, int64_t ib) {
    if (sa != sb) return sa > sb;
    return ia < ib;
}

typedef struct {
    double s;
    int64_t idx;
} cand_t;

static int cand_cmp(const void* x, const void* y) {
    const cand_t* a = (const cand_t*)x;
    const cand_t* b = (const cand_t*)y;
    if (beats(a->s, a->idx, b->s, b->idx)) return -1;
    if (beats(b->s, b->idx, a->s, a->idx)) return 1;
    return 0;
}

static int i64_cmp(const void* x, const void* y) {
    const int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
    return (a > b) - (a < b);
}

/* Top-`take` of (score, idx) under the total order, written ascending by index. */
static void top_take_sorted(cand_t* c, int64_t nc, int64_t take, int64_t* out) {
    qsort(c, (size_t)nc, sizeof(cand_t), cand_cmp);
    for (int64_t i = 0; i < take; ++i) out[i] = c[i].idx;
    qsort(out, (size_t)take, sizeof(int64_t), i64_cmp);
}

int64_t or_select_experts(const double* p, int64_t n, int64_t kk, int64_t* out) {
    if (kk < 1) return -2; /* experts.cpp:31 */
    const int64_t take = kk < n ? kk : n;
    cand_t* c = (cand_t*)malloc(sizeof(cand_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) {
        c[i].s = p[i];
        c[i].idx = i;
    }
    top_take_sorted(c, n, take, out);
    free(c);
    return take;
}

static void union_of(const int64_t* per_token, int64_t tokens, int64_t take, int64_t r, int64_t* union_out,
                     int64_t* union_size) { /* experts.cpp:109-115 */
    char* mask = (char*)calloc((size_t)(r > 0 ? r : 1), 1);
    for (int64_t i = 0; i < tokens * take; ++i) mask[per_token[i]] = 1;
    int64_t u = 0;
    for (int64_t j = 0; j < r; ++j)
        if (mask[j]) union_out[u++] = j;
    *union_size = u;
    free(mask);
}

int or_ke_select(const double* h, int64_t tokens, int64_t d, const double* w_g, int64_t n_experts,
                 const double* w_a, int64_t r, int64_t kk, int64_t k, int64_t* per_token, int64_t* tau,
                 int64_t* union_out, int64_t* union_size, int64_t* take_out, int* warned) {
    if (k < 1) return 2;                                  /* experts.cpp:50 */
    if (n_experts < 1 || r < 1 || r % n_experts) return 2; /* ExpertPartition::make, experts.cpp:12-19 */
    if (kk < 1) return 2;                                 /* select_experts, experts.cpp:31 */
    const int64_t e_size = r / n_experts;
    const int64_t kk_eff = kk < n_experts ? kk : n_experts; /* :57 */
    const int64_t visible = kk_eff * e_size;
    *warned = k > visible;                                 /* :59-65 */
    const int64_t take = k < visible ? k : visible;
    *take_out = take;
    double* keys_t = transpose_new(w_a, d, r); /* :68 neuron-major copy */
    int err = 0;
#pragma omp parallel for schedule(static) if (tokens > 1)
    for (int64_t t = 0; t < tokens; ++t) {
        const double* ht = h + t * d;
        double* p = (double*)malloc(sizeof(double) * (size_t)n_experts);
        int64_t* tt = (int64_t*)malloc(sizeof(int64_t) * (size_t)kk_eff);
        or_route_scores(ht, d, w_g, n_experts, p);
        or_select_experts(p, n_experts, kk_eff, tt);
        cand_t* c = (cand_t*)malloc(sizeof(cand_t) * (size_t)visible);
        int64_t nc = 0;
        for (int64_t q = 0; q < kk_eff; ++q) { /* :83-92 tau ascending, then j ascending */
            for (int64_t j = tt[q] * e_size; j < (tt[q] + 1) * e_size; ++j) {
                c[nc].s = or_dot(ht, keys_t + j * d, d);
                c[nc].idx = j;
                ++nc;
            }
        }
        top_take_sorted(c, nc, take, per_token + t * take); /* :94-105 */
        if (tau)
            for (int64_t q = 0; q < kk_eff; ++q) tau[t * kk_eff + q] = tt[q];
        free(c);
        free(tt);
        free(p);
    }
    free(keys_t);
    union_of(per_token, tokens, take, r, union_out, union_size);
    return err;
}

/* ------------------------------------------------------------ adapter.cpp */

int or_topk_select(const double* h, int64_t tokens, int64_t d, const double* w_a, int64_t r, int64_t k,
                   int64_t* per_token, int64_t* union_out, int64_t* union_size, int64_t* take_out,
                   int* warned) {
    if (k < 1) return 2; /* adapter.cpp:43 */
    *warned = k > r;     /* :46-48 */
    const int64_t take = k < r ? k : r;
    *take_out = take;
    double* keys_t = transpose_new(w_a, d, r);
#pragma omp parallel for schedule(static) if (tokens > 1)
    for (int64_t t = 0; t < tokens; ++t) {
        cand_t* c = (cand_t*)malloc(sizeof(cand_t) * (size_t)(r > 0 ? r : 1));
        for (int64_t j = 0; j < r; ++j) {
            c[j].s = or_dot(h + t * d, keys_t + j * d, d);
            c[j].idx = j;
        }
        top_take_sorted(c, r, take, per_token + t * take);
        free(c);
    }
    free(keys_t);
    union_of(per_token, tokens, take, r, union_out, union_size);
    return 0;
}

int or_gather_adapter(const double* w_a, const double* w_b, int64_t d, int64_t r, const int64_t* s,
                      int64_t ns, double* w_a_k, double* w_b_k, int64_t* bad_index) {
    for (int64_t i = 0; i < ns; ++i) { /* adapter.cpp:89-98: range first, then strict ascent */
        if (s[i] < 0 || s[i] >= r) {
            *bad_index = s[i];
            return 3;
        }
        if (i > 0 && s[i] <= s[i - 1]) return 2;
    }
    for (int64_t i = 0; i < d; ++i)
        for (int64_t j = 0; j < ns; ++j) w_a_k[i * ns + j] = w_a[i * r + s[j]];
    for (int64_t j = 0; j < ns; ++j) memcpy(w_b_k + j * d, w_b + s[j] * d, sizeof(double) * (size_t)d);
    return 0;
}

static double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }          /* kernels.cpp:15 */
static double silu_grad(double x) {                                       /* kernels.cpp:19-22 */
    const double s = sigmoid(x);
    return s * (1.0 + x * (1.0 - s));
}

int or_ffn_forward(const double* h, int64_t tokens, int64_t d, const double* w_in, const double* w_out,
                   int64_t n, int act, const double* w_a_k, const double* w_b_k, int64_t s, double* out,
                   double* z, double* base_pre) {
    /* adapter.cpp:118-126: base = act(h w_in) w_out, then out += ReLU(h w_a_k) w_b_k */
    const size_t td = (size_t)(tokens * d);
    double* pre = (double*)malloc(sizeof(double) * (size_t)(tokens * n > 0 ? tokens * n : 1));
    or_matmul(h, w_in, tokens, d, n, pre);
    double* a = (double*)malloc(sizeof(double) * (size_t)(tokens * n > 0 ? tokens * n : 1));
    for (int64_t i = 0; i < tokens * n; ++i)
        a[i] = act == 1 ? (pre[i] > 0.0 ? pre[i] : 0.0) : pre[i] * sigmoid(pre[i]);
    or_matmul(a, w_out, tokens, n, d, out);
    if (s > 0) {
        double* zz = (double*)malloc(sizeof(double) * (size_t)(tokens * s));
        double* rz = (double*)malloc(sizeof(double) * (size_t)(tokens * s));
        double* ad = (double*)malloc(sizeof(double) * td);
        or_matmul(h, w_a_k, tokens, d, s, zz);
        for (int64_t i = 0; i < tokens * s; ++i) rz[i] = zz[i] > 0.0 ? zz[i] : 0.0;
        or_matmul(rz, w_b_k, tokens, s, d, ad);
        for (size_t i = 0; i < td; ++i) out[i] += ad[i]; /* add_inplace, kernels.cpp:136-139 */
        if (z) memcpy(z, zz, sizeof(double) * (size_t)(tokens * s));
        free(zz);
        free(rz);
        free(ad);
    }
    if (base_pre && n > 0) memcpy(base_pre, pre, sizeof(double) * (size_t)(tokens * n));
    free(pre);
    free(a);
    return 0;
}

int or_ffn_backward(const double* grad_out, const double* h, const double* z, const double* base_pre,
                    int64_t tokens, int64_t d, const double* w_in, const double* w_out, int64_t n, int act,
                    const double* w_a_k, const double* w_b_k, int64_t s, double* grad_w_a_k,
                    double* grad_w_b_k, double* grad_h) {
    const size_t tn = (size_t)(tokens * n > 0 ? tokens * n : 1);
    /* adapter.cpp:153-164 frozen-base path */
    double* w_out_t = transpose_new(w_out, n, d);
    double* d_act = (double*)malloc(sizeof(double) * tn);
    or_matmul(grad_out, w_out_t, tokens, d, n, d_act);
    for (int64_t i = 0; i < tokens * n; ++i)
        d_act[i] = act == 1 ? (base_pre[i] > 0.0 ? d_act[i] : 0.0) : d_act[i] * silu_grad(base_pre[i]);
    double* w_in_t = transpose_new(w_in, d, n);
    or_matmul(d_act, w_in_t, tokens, n, d, grad_h);
    free(w_out_t);
    free(w_in_t);
    free(d_act);
    if (s > 0) { /* adapter.cpp:166-175 */
        double* w_b_t = transpose_new(w_b_k, s, d);
        double* masked = (double*)malloc(sizeof(double) * (size_t)(tokens * s));
        or_matmul(grad_out, w_b_t, tokens, d, s, masked);
        for (int64_t i = 0; i < tokens * s; ++i)
            if (!(z[i] > 0.0)) masked[i] = 0.0;
        double* rz = (double*)malloc(sizeof(double) * (size_t)(tokens * s));
        for (int64_t i = 0; i < tokens * s; ++i) rz[i] = z[i] > 0.0 ? z[i] : 0.0;
        double* rz_t = transpose_new(rz, tokens, s);
        or_matmul(rz_t, grad_out, s, tokens, d, grad_w_b_k);
        double* h_t = transpose_new(h, tokens, d);
        or_matmul(h_t, masked, d, tokens, s, grad_w_a_k);
        double* w_a_t = transpose_new(w_a_k, d, s);
        double* gh = (double*)malloc(sizeof(double) * (size_t)(tokens * d));
        or_matmul(masked, w_a_t, tokens, s, d, gh);
        for (int64_t i = 0; i < tokens * d; ++i) grad_h[i] += gh[i];
        free(w_b_t);
        free(masked);
        free(rz);
        free(rz_t);
        free(h_t);
        free(w_a_t);
        free(gh);
    }
    return 0;
}

/* ------------------------------------------------------------ memtier.cpp */

int or_scatter_grads(int64_t d, int64_t r, double* stage_a, double* stage_b, int8_t* staged,
                     const int64_t* s, int64_t ns, const double* gwa, const double* gwb, int64_t* bad_index) {
    for (int64_t j = 0; j < ns; ++j) { /* memtier.cpp:140-150 */
        const int64_t col = s[j];
        if (col < 0 || col >= r) {
            *bad_index = col;
            return 3;
        }
        for (int64_t i = 0; i < d; ++i) stage_a[i * r + col] += gwa[i * ns + j];
        for (int64_t i = 0; i < d; ++i) stage_b[col * d + i] += gwb[j * d + i];
        staged[col] = 1;
    }
    return 0;
}

static void adam_entry(double* w, double* m, double* v, double g, double b1, double b2, double eps, double lr,
                       double c1, double c2) { /* memtier.cpp:176-185 */
    *m = b1 * *m + (1.0 - b1) * g;
    *v = b2 * *v + (1.0 - b2) * g * g;
    const double mhat = *m / c1;
    const double vhat = *v / c2;
    *w -= lr * mhat / (sqrt(vhat) + eps);
}

void or_sparse_adam(int64_t d, int64_t r, double* w_a, double* w_b, double* m_a, double* v_a, double* m_b,
                    double* v_b, double* stage_a, double* stage_b, int8_t* staged, int64_t* pair_step,
                    double beta1, double beta2, double eps, double lr) {
    for (int64_t j = 0; j < r; ++j) { /* memtier.cpp:191-210 */
        if (!staged[j]) continue;
        const int64_t t = ++pair_step[j];
        const double c1 = 1.0 - pow(beta1, (double)t);
        const double c2 = 1.0 - pow(beta2, (double)t);
        for (int64_t i = 0; i < d; ++i) {
            const int64_t q = i * r + j;
            adam_entry(&w_a[q], &m_a[q], &v_a[q], stage_a[q], beta1, beta2, eps, lr, c1, c2);
            stage_a[q] = 0.0;
        }
        for (int64_t i = 0; i < d; ++i) {
            const int64_t q = j * d + i;
            adam_entry(&w_b[q], &m_b[q], &v_b[q], stage_b[q], beta1, beta2, eps, lr, c1, c2);
            stage_b[q] = 0.0;
        }
        staged[j] = 0;
    }
}

/* Straight-through router gradient, restating trainer.cpp:140-181 (stage_router_ste; private to the reference's
 * trainer and not covered by its tests, so this restatement is its oracle). For every token t and each of its
 * routed experts e (tau row t, kk entries): y = sum over union positions c of expert e (s[c] / esz == e) with
 * z[t][c] > 0 of z[t][c] * w_b_k[c]; skipped when no such c; dldp = dot(grad_out[t], y) (kernels.hpp:37-41);
 * grad_g[e] += dldp * h[t] (accumulated in token order); touched[e] = 1. grad_g [n_experts x d] must be zeroed. */
void or_router_ste(const double* h, const double* z, const double* w_b_k, const int64_t* s, int64_t n_s,
                   const int64_t* tau, int64_t kk, const double* grad_out, int64_t tokens, int64_t d, int64_t esz,
                   double* grad_g, int8_t* touched) {
    double* y = (double*)malloc((size_t)d * sizeof(double));
    for (int64_t t = 0; t < tokens; ++t) {
        for (int64_t q = 0; q < kk; ++q) {
            const int64_t e = tau[t * kk + q];
            for (int64_t x = 0; x < d; ++x) y[x] = 0.0;
            int any = 0;
            for (int64_t c = 0; c < n_s; ++c) {
                if (s[c] / esz != e) continue;
                const double a = z[t * n_s + c];
                if (a <= 0.0) continue;
                const double* brow = w_b_k + c * d;
                for (int64_t x = 0; x < d; ++x) y[x] += a * brow[x];
                any = 1;
            }
            if (!any) continue;
            const double dldp = or_dot(grad_out + t * d, y, d);
            for (int64_t x = 0; x < d; ++x) grad_g[e * d + x] += dldp * h[t * d + x];
            touched[e] = 1;
        }
    }
    free(y);
}
