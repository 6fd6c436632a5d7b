/* TEST INFRASTRUCTURE — the parity checker, never the product.
 *
 * A plain-C restatement of the reference RES-PCA solver path
 * (/root/reference/proj/src/{solver,kmeans,matrix}.cpp).  Every function cites
 * the reference lines it follows and keeps the reference's floating-point
 * operation order (compile with -ffp-contract=off: no FMA contraction), so on
 * the same inputs its outputs are bit-identical to the reference's.  That
 * claim is pinned in tests/test_oracle.py against (a) the unmodified
 * reference compiled into oracle/_ref/librespca_ref.so and (b) the golden
 * fingerprints committed under tests/golden/ (made by tests/golden/make_golden.py
 * from the reference itself).
 *
 * The k-means++ seeding draws from std::mt19937_64 through libstdc++'s
 * uniform_int_distribution<size_t> (Lemire's nearly-divisionless method with a
 * 128-bit product, bits/uniform_int_dist.h of GCC 13) and
 * uniform_real_distribution<double> (generate_canonical: one 64-bit draw
 * divided by 2^64, clamped below 1, then `u * (b - a) + a`).  Those published
 * algorithms are restated here in orc_mt_*, orc_uniform_int, orc_canonical.
 *
 * Loaded only by tests/, __graft_entry__.smoke() and bench.py's CPU legs.
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "oracle_abi.h"

enum { OK = 0, EINVAL_ = 1, ERUNTIME = 2, EOTHER = 3 };

static __thread char g_err[256];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------ */
/* std::mt19937_64 (Matsumoto & Nishimura 2000, 64-bit parameters)           */
/* ------------------------------------------------------------------------ */
#define MT_N 312
#define MT_M 156
typedef struct {
    uint64_t s[MT_N];
    int i;
} orc_mt;

static void orc_mt_seed(orc_mt* g, uint64_t seed) {
    g->s[0] = seed;
    for (int k = 1; k < MT_N; ++k)
        g->s[k] = 6364136223846793005ULL * (g->s[k - 1] ^ (g->s[k - 1] >> 62)) + (uint64_t)k;
    g->i = MT_N;
}

static uint64_t orc_mt_next(orc_mt* g) {
    const uint64_t UPPER = 0xFFFFFFFF80000000ULL, LOWER = 0x7FFFFFFFULL;
    const uint64_t A = 0xB5026F5AA96619E9ULL;
    if (g->i >= MT_N) {
        for (int k = 0; k < MT_N; ++k) {
            uint64_t y = (g->s[k] & UPPER) | (g->s[(k + 1) % MT_N] & LOWER);
            g->s[k] = g->s[(k + MT_M) % MT_N] ^ (y >> 1) ^ ((y & 1ULL) ? A : 0ULL);
        }
        g->i = 0;
    }
    uint64_t z = g->s[g->i++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
}

/* uniform_int_distribution<size_t>(lo, hi) over a full-range 64-bit engine. */
static uint64_t orc_uniform_int_draw(orc_mt* g, uint64_t lo, uint64_t hi) {
    const uint64_t urange = hi - lo;
    if (urange == UINT64_MAX) return orc_mt_next(g) + lo; /* engine range == range */
    const uint64_t range = urange + 1;
    unsigned __int128 prod = (unsigned __int128)orc_mt_next(g) * range;
    uint64_t low = (uint64_t)prod;
    if (low < range) {
        const uint64_t threshold = (uint64_t)(-range) % range;
        while (low < threshold) {
            prod = (unsigned __int128)orc_mt_next(g) * range;
            low = (uint64_t)prod;
        }
    }
    return (uint64_t)(prod >> 64) + lo;
}

/* generate_canonical<double, 53>: k = 1 draw for a 64-bit engine. */
static double orc_canonical(orc_mt* g) {
    double r = (double)orc_mt_next(g) / 18446744073709551616.0;
    if (r >= 1.0) r = nextafter(1.0, 0.0);
    return r;
}

static double orc_uniform_real_draw(orc_mt* g, double a, double b) {
    return orc_canonical(g) * (b - a) + a;
}

int orc_uniform_int(uint64_t seed, uint64_t lo, uint64_t hi, uint64_t count, uint64_t* out) {
    orc_mt g;
    orc_mt_seed(&g, seed);
    for (uint64_t k = 0; k < count; ++k) out[k] = orc_uniform_int_draw(&g, lo, hi);
    return OK;
}

int orc_uniform_real(uint64_t seed, double a, double b, uint64_t count, double* out) {
    orc_mt g;
    orc_mt_seed(&g, seed);
    for (uint64_t k = 0; k < count; ++k) out[k] = orc_uniform_real_draw(&g, a, b);
    return OK;
}

/* ------------------------------------------------------------------------ */
/* core (matrix.cpp)                                                         */
/* ------------------------------------------------------------------------ */
static int all_finite(const double* m, uint64_t N) { /* matrix.cpp:29-34 */
    for (uint64_t k = 0; k < N; ++k)
        if (!isfinite(m[k])) return 0;
    return 1;
}

/* GroupAssignment(labels, c) validation, matrix.cpp:36-47 */
static int check_groups(const uint64_t* labels, uint64_t n, uint64_t c) {
    if (c == 0) return fail(EINVAL_, "GroupAssignment: c must be >= 1");
    char* seen = calloc(c, 1);
    for (uint64_t j = 0; j < n; ++j) {
        if (labels[j] >= c) {
            free(seen);
            return fail(EINVAL_, "GroupAssignment: label out of range");
        }
        seen[labels[j]] = 1;
    }
    for (uint64_t k = 0; k < c; ++k)
        if (!seen[k]) {
            free(seen);
            return fail(EINVAL_, "GroupAssignment: empty group");
        }
    free(seen);
    return OK;
}

/* group_indices(), matrix.cpp:49-55: ascending member lists, CSR layout. */
static void group_csr(const uint64_t* labels, uint64_t n, uint64_t c, uint64_t* off,
                      uint64_t* members) {
    memset(off, 0, (c + 1) * sizeof(uint64_t));
    for (uint64_t j = 0; j < n; ++j) off[labels[j] + 1]++;
    for (uint64_t k = 0; k < c; ++k) off[k + 1] += off[k];
    uint64_t* fill = malloc(c * sizeof(uint64_t));
    memcpy(fill, off, c * sizeof(uint64_t));
    for (uint64_t j = 0; j < n; ++j) members[fill[labels[j]]++] = j;
    free(fill);
}

/* column_mean, matrix.cpp:63-79 */
static void column_mean_raw(const double* m, uint64_t d, const uint64_t* cols, uint64_t nc,
                            double* mean) {
    for (uint64_t i = 0; i < d; ++i) mean[i] = 0.0;
    for (uint64_t t = 0; t < nc; ++t) {
        const double* col = m + cols[t] * d;
        for (uint64_t i = 0; i < d; ++i) mean[i] += col[i];
    }
    const double inv = 1.0 / (double)nc;
    for (uint64_t i = 0; i < d; ++i) mean[i] *= inv;
}

int orc_column_mean(const double* m, uint64_t d, uint64_t n, const uint64_t* cols, uint64_t nc,
                    double* out) {
    if (nc == 0) return fail(EINVAL_, "column_mean: empty column set");
    for (uint64_t t = 0; t < nc; ++t)
        if (cols[t] >= n) return fail(EINVAL_, "column_mean: column index out of range");
    column_mean_raw(m, d, cols, nc, out);
    return OK;
}

/* group_scatter, matrix.cpp:81-97 */
static double group_scatter_raw(const double* m, uint64_t d, uint64_t n, const uint64_t* labels,
                                uint64_t c) {
    uint64_t* off = malloc((c + 1) * sizeof(uint64_t));
    uint64_t* mem = malloc(n * sizeof(uint64_t));
    double* mean = malloc(d * sizeof(double));
    group_csr(labels, n, c, off, mem);
    double total = 0.0;
    for (uint64_t g = 0; g < c; ++g) {
        column_mean_raw(m, d, mem + off[g], off[g + 1] - off[g], mean);
        for (uint64_t t = off[g]; t < off[g + 1]; ++t) {
            const double* col = m + mem[t] * d;
            for (uint64_t i = 0; i < d; ++i) {
                const double dl = col[i] - mean[i];
                total += dl * dl;
            }
        }
    }
    free(off);
    free(mem);
    free(mean);
    return total;
}

int orc_group_scatter(const double* m, uint64_t d, uint64_t n, const uint64_t* labels, uint64_t c,
                      double* out) {
    int rc = check_groups(labels, n, c);
    if (rc) return rc;
    *out = group_scatter_raw(m, d, n, labels, c);
    return OK;
}

static double frob_raw(const double* m, uint64_t N) { /* matrix.cpp:99-103 */
    double sq = 0.0;
    for (uint64_t k = 0; k < N; ++k) sq += m[k] * m[k];
    return sqrt(sq);
}

int orc_frob_norm(const double* m, uint64_t d, uint64_t n, double* out) {
    *out = frob_raw(m, d * n);
    return OK;
}

static double l1_raw(const double* m, uint64_t N) { /* matrix.cpp:105-109 */
    double s = 0.0;
    for (uint64_t k = 0; k < N; ++k) s += fabs(m[k]);
    return s;
}

int orc_elementwise_l1(const double* m, uint64_t d, uint64_t n, double* out) {
    *out = l1_raw(m, d * n);
    return OK;
}

static void col_norms_raw(const double* m, uint64_t d, uint64_t n, double* out) {
    for (uint64_t j = 0; j < n; ++j) { /* matrix.cpp:117-125 */
        double sq = 0.0;
        for (uint64_t i = 0; i < d; ++i) sq += m[j * d + i] * m[j * d + i];
        out[j] = sqrt(sq);
    }
}

int orc_column_l2_norms(const double* m, uint64_t d, uint64_t n, double* out) {
    col_norms_raw(m, d, n, out);
    return OK;
}

static double l21_raw(const double* m, uint64_t d, uint64_t n) { /* matrix.cpp:111-115 */
    double* nr = malloc(n * sizeof(double));
    col_norms_raw(m, d, n, nr);
    double s = 0.0;
    for (uint64_t j = 0; j < n; ++j) s += nr[j];
    free(nr);
    return s;
}

int orc_l21_norm(const double* m, uint64_t d, uint64_t n, double* out) {
    *out = l21_raw(m, d, n);
    return OK;
}

/* ------------------------------------------------------------------------ */
/* clustering (kmeans.cpp)                                                   */
/* ------------------------------------------------------------------------ */
static double sq_dist(const double* a, const double* b, uint64_t d) { /* kmeans.cpp:12-19 */
    double s = 0.0;
    for (uint64_t i = 0; i < d; ++i) {
        const double t = a[i] - b[i];
        s += t * t;
    }
    return s;
}

/* assign_nearest, kmeans.cpp:21-37 (strict < keeps the lowest index on ties) */
static void assign_nearest(const double* m, uint64_t d, uint64_t n, const double* C, uint64_t c,
                           uint64_t* labels) {
    for (uint64_t j = 0; j < n; ++j) {
        double best = INFINITY;
        uint64_t arg = 0;
        for (uint64_t k = 0; k < c; ++k) {
            const double v = sq_dist(m + j * d, C + k * d, d);
            if (v < best) {
                best = v;
                arg = k;
            }
        }
        labels[j] = arg;
    }
}

/* repair_empty, kmeans.cpp:40-64 */
static int repair_empty(const double* m, uint64_t d, uint64_t n, const double* C, uint64_t c,
                        uint64_t* labels) {
    uint64_t* counts = calloc(c, sizeof(uint64_t));
    for (uint64_t j = 0; j < n; ++j) counts[labels[j]]++;
    for (uint64_t e = 0; e < c; ++e) {
        if (counts[e] > 0) continue;
        double worst = -1.0;
        uint64_t steal = 0;
        for (uint64_t j = 0; j < n; ++j) {
            if (counts[labels[j]] <= 1) continue;
            const double v = sq_dist(m + j * d, C + labels[j] * d, d);
            if (v > worst) {
                worst = v;
                steal = j;
            }
        }
        if (worst < 0.0) {
            free(counts);
            return fail(ERUNTIME, "kmeans: cannot repair empty cluster");
        }
        counts[labels[steal]]--;
        labels[steal] = e;
        counts[e]++;
    }
    free(counts);
    return OK;
}

/* means_of, kmeans.cpp:66-82 */
static void means_of(const double* m, uint64_t d, uint64_t n, const uint64_t* labels, uint64_t c,
                     double* C) {
    uint64_t* counts = calloc(c, sizeof(uint64_t));
    memset(C, 0, d * c * sizeof(double));
    for (uint64_t j = 0; j < n; ++j) {
        double* dst = C + labels[j] * d;
        const double* src = m + j * d;
        for (uint64_t i = 0; i < d; ++i) dst[i] += src[i];
        counts[labels[j]]++;
    }
    for (uint64_t k = 0; k < c; ++k) {
        const double inv = 1.0 / (double)counts[k];
        for (uint64_t i = 0; i < d; ++i) C[k * d + i] *= inv;
    }
    free(counts);
}

/* inertia_of, kmeans.cpp:84-91 */
static double inertia_of(const double* m, uint64_t d, uint64_t n, const uint64_t* labels,
                         const double* C) {
    double s = 0.0;
    for (uint64_t j = 0; j < n; ++j) s += sq_dist(m + j * d, C + labels[j] * d, d);
    return s;
}

/* hartigan_refine, kmeans.cpp:96-139 */
static void hartigan_refine(const double* m, uint64_t d, uint64_t n, uint64_t* labels, double* C,
                            uint64_t c) {
    uint64_t* counts = calloc(c, sizeof(uint64_t));
    for (uint64_t j = 0; j < n; ++j) counts[labels[j]]++;
    for (int pass = 0; pass < 50; ++pass) {
        int improved = 0;
        for (uint64_t j = 0; j < n; ++j) {
            const uint64_t from = labels[j];
            if (counts[from] <= 1) continue;
            const double na = (double)counts[from];
            const double gain = na / (na - 1.0) * sq_dist(m + j * d, C + from * d, d);
            double best_delta = -1e-12;
            uint64_t to = from;
            for (uint64_t k = 0; k < c; ++k) {
                if (k == from) continue;
                const double nb = (double)counts[k];
                const double cost = nb / (nb + 1.0) * sq_dist(m + j * d, C + k * d, d);
                if (cost - gain < best_delta) {
                    best_delta = cost - gain;
                    to = k;
                }
            }
            if (to == from) continue;
            double* cf = C + from * d;
            double* ct = C + to * d;
            const double* x = m + j * d;
            const double na1 = (double)(counts[from] - 1);
            const double nb1 = (double)(counts[to] + 1);
            for (uint64_t i = 0; i < d; ++i) {
                cf[i] = (cf[i] * (double)counts[from] - x[i]) / na1;
                ct[i] = (ct[i] * (double)counts[to] + x[i]) / nb1;
            }
            counts[from]--;
            counts[to]++;
            labels[j] = to;
            improved = 1;
        }
        if (!improved) break;
    }
    free(counts);
}

/* lloyd_step, kmeans.cpp:226-235 */
static int lloyd_step_raw(const double* m, uint64_t d, uint64_t n, const double* C, uint64_t c,
                          uint64_t* labels, double* next) {
    assign_nearest(m, d, n, C, c, labels);
    int rc = repair_empty(m, d, n, C, c, labels);
    if (rc) return rc;
    means_of(m, d, n, labels, c, next);
    return OK;
}

int orc_lloyd_step(const double* m, uint64_t d, uint64_t n, const double* C, uint64_t c,
                   uint64_t* labels, double* next) {
    if (c == 0) return fail(EINVAL_, "lloyd_step: bad centroid matrix");
    return lloyd_step_raw(m, d, n, C, c, labels, next);
}

/* lloyd_run, kmeans.cpp:141-168. C is updated in place to the final centroids. */
static int lloyd_run(const double* m, uint64_t d, uint64_t n, double* C, uint64_t c,
                     uint64_t max_iters, double tol, uint64_t* labels, double* inertia,
                     uint64_t* iters_run) {
    double* next = malloc(d * c * sizeof(double));
    uint64_t it = 0;
    for (; it < max_iters; ++it) {
        int rc = lloyd_step_raw(m, d, n, C, c, labels, next);
        if (rc) {
            free(next);
            return rc;
        }
        double moved = 0.0, scale = 0.0;
        for (uint64_t k = 0; k < d * c; ++k) {
            const double t = next[k] - C[k];
            moved += t * t;
            scale += C[k] * C[k];
        }
        memcpy(C, next, d * c * sizeof(double));
        const double s = sqrt(scale);
        const double floor_ = (s < 1e-300) ? 1e-300 : s;
        if (sqrt(moved) <= tol * floor_) {
            ++it;
            break;
        }
    }
    free(next);
    hartigan_refine(m, d, n, labels, C, c);
    means_of(m, d, n, labels, c, C);
    *inertia = inertia_of(m, d, n, labels, C);
    int rc = check_groups(labels, n, c);
    if (rc) return rc;
    *iters_run = it;
    return OK;
}

/* kmeans_pp_init, kmeans.cpp:172-224; returns chosen column indices. */
static int pp_init_idx(const double* m, uint64_t d, uint64_t n, uint64_t c, orc_mt* rng,
                       uint64_t* chosen) {
    if (c == 0) return fail(EINVAL_, "kmeans_pp_init: c must be >= 1");
    if (c > n) return fail(EINVAL_, "kmeans_pp_init: c exceeds column count");
    char* is_chosen = calloc(n, 1);
    double* d2 = malloc(n * sizeof(double));
    uint64_t nch = 0;
    chosen[nch++] = orc_uniform_int_draw(rng, 0, n - 1);
    is_chosen[chosen[0]] = 1;
    for (uint64_t j = 0; j < n; ++j) d2[j] = INFINITY;
    while (nch < c) {
        const uint64_t last = chosen[nch - 1];
        double total = 0.0;
        for (uint64_t j = 0; j < n; ++j) {
            const double v = sq_dist(m + j * d, m + last * d, d);
            d2[j] = (v < d2[j]) ? v : d2[j]; /* std::min(d2[j], v) */
            total += d2[j];
        }
        uint64_t pick = n;
        if (total > 0.0) {
            double r = orc_uniform_real_draw(rng, 0.0, total);
            for (uint64_t j = 0; j < n; ++j) {
                r -= d2[j];
                if (r <= 0.0 && !is_chosen[j]) {
                    pick = j;
                    break;
                }
            }
        }
        if (pick == n) {
            for (uint64_t j = 0; j < n; ++j)
                if (!is_chosen[j]) {
                    pick = j;
                    break;
                }
        }
        chosen[nch++] = pick;
        is_chosen[pick] = 1;
    }
    free(is_chosen);
    free(d2);
    return OK;
}

int orc_kmeans_pp_init(const double* m, uint64_t d, uint64_t n, uint64_t c, uint64_t seed,
                       double* C) {
    orc_mt g;
    orc_mt_seed(&g, seed);
    uint64_t* ch = malloc((c ? c : 1) * sizeof(uint64_t));
    int rc = pp_init_idx(m, d, n, c, &g, ch);
    if (!rc)
        for (uint64_t k = 0; k < c; ++k) memcpy(C + k * d, m + ch[k] * d, d * sizeof(double));
    free(ch);
    return rc;
}

/* kmeans, kmeans.cpp:237-250 */
static int kmeans_raw(const double* m, uint64_t d, uint64_t n, uint64_t c, uint64_t max_iters,
                      uint64_t n_restarts, uint64_t seed, double tol, uint64_t* labels,
                      double* C, double* inertia, uint64_t* iters_run) {
    if (c == 0) return fail(EINVAL_, "kmeans: c must be >= 1");
    if (c > n) return fail(EINVAL_, "kmeans: c exceeds column count");
    orc_mt g;
    orc_mt_seed(&g, seed);
    double best = INFINITY;
    uint64_t* ch = malloc(c * sizeof(uint64_t));
    uint64_t* lab = malloc(n * sizeof(uint64_t));
    double* cen = malloc(d * c * sizeof(double));
    int rc = OK;
    for (uint64_t r = 0; r < n_restarts; ++r) {
        rc = pp_init_idx(m, d, n, c, &g, ch);
        if (rc) break;
        for (uint64_t k = 0; k < c; ++k) memcpy(cen + k * d, m + ch[k] * d, d * sizeof(double));
        double in;
        uint64_t it;
        rc = lloyd_run(m, d, n, cen, c, max_iters, tol, lab, &in, &it);
        if (rc) break;
        if (in < best) {
            best = in;
            memcpy(labels, lab, n * sizeof(uint64_t));
            memcpy(C, cen, d * c * sizeof(double));
            *inertia = in;
            *iters_run = it;
        }
    }
    free(ch);
    free(lab);
    free(cen);
    return rc;
}

int orc_kmeans(const double* m, uint64_t d, uint64_t n, uint64_t c, uint64_t max_iters,
               uint64_t n_restarts, uint64_t seed, double tol, uint64_t* labels, double* C,
               double* inertia, uint64_t* iters_run) {
    return kmeans_raw(m, d, n, c, max_iters, n_restarts, seed, tol, labels, C, inertia,
                      iters_run);
}

/* kmeans_warm, kmeans.cpp:252-258 */
int orc_kmeans_warm(const double* m, uint64_t d, uint64_t n, uint64_t c, uint64_t max_iters,
                    double tol, const uint64_t* init, uint64_t* labels, double* C,
                    double* inertia, uint64_t* iters_run) {
    int rc = check_groups(init, n, c); /* GroupAssignment ctor, matrix.cpp:36-47 */
    if (rc) return rc;
    means_of(m, d, n, init, c, C);
    return lloyd_run(m, d, n, C, c, max_iters, tol, labels, inertia, iters_run);
}

/* ------------------------------------------------------------------------ */
/* solver (solver.cpp)                                                       */
/* ------------------------------------------------------------------------ */
static void l_update_raw(const double* D, uint64_t d, uint64_t n, const uint64_t* labels,
                         uint64_t c, double lambda, double rho, double* L) {
    /* solver.cpp:51-77 */
    const double own_w = rho / (2.0 * lambda + rho);
    uint64_t* off = malloc((c + 1) * sizeof(uint64_t));
    uint64_t* mem = malloc(n * sizeof(uint64_t));
    double* sum = malloc(d * sizeof(double));
    group_csr(labels, n, c, off, mem);
    for (uint64_t g = 0; g < c; ++g) {
        for (uint64_t i = 0; i < d; ++i) sum[i] = 0.0;
        for (uint64_t t = off[g]; t < off[g + 1]; ++t) {
            const double* col = D + mem[t] * d;
            for (uint64_t i = 0; i < d; ++i) sum[i] += col[i];
        }
        const double mean_w = 2.0 * lambda / ((double)(off[g + 1] - off[g]) * (2.0 * lambda + rho));
        for (uint64_t t = off[g]; t < off[g + 1]; ++t) {
            const double* src = D + mem[t] * d;
            double* dst = L + mem[t] * d;
            for (uint64_t i = 0; i < d; ++i) dst[i] = own_w * src[i] + mean_w * sum[i];
        }
    }
    free(off);
    free(mem);
    free(sum);
}

int orc_l_update(const double* D, uint64_t d, uint64_t n, const uint64_t* labels, uint64_t c,
                 double lambda, double rho, double* L) {
    int rc = check_groups(labels, n, c);
    if (rc) return rc;
    if (rho <= 0.0) return fail(EINVAL_, "l_update: rho must be > 0");
    if (lambda < 0.0) return fail(EINVAL_, "l_update: lambda must be >= 0");
    l_update_raw(D, d, n, labels, c, lambda, rho, L);
    return OK;
}

static void shrink_l1(const double* B, uint64_t N, double thr, double* S) {
    for (uint64_t k = 0; k < N; ++k) { /* solver.cpp:82-86 */
        const double v = B[k];
        const double mag = fabs(v) - thr;
        S[k] = mag > 0.0 ? copysign(mag, v) : 0.0;
    }
}

int orc_s_update_l1(const double* B, uint64_t d, uint64_t n, double thr, double* S) {
    if (thr < 0.0) return fail(EINVAL_, "s_update_l1: negative threshold");
    shrink_l1(B, d * n, thr, S);
    return OK;
}

static void shrink_l21(const double* B, uint64_t d, uint64_t n, double thr, double* S) {
    double* nr = malloc(n * sizeof(double)); /* solver.cpp:90-102 */
    col_norms_raw(B, d, n, nr);
    for (uint64_t j = 0; j < n; ++j) {
        if (nr[j] <= thr) {
            for (uint64_t i = 0; i < d; ++i) S[j * d + i] = 0.0;
            continue;
        }
        const double scale = 1.0 - thr / nr[j];
        for (uint64_t i = 0; i < d; ++i) S[j * d + i] = scale * B[j * d + i];
    }
    free(nr);
}

int orc_s_update_l21(const double* B, uint64_t d, uint64_t n, double thr, double* S) {
    if (thr < 0.0) return fail(EINVAL_, "s_update_l21: negative threshold");
    shrink_l21(B, d, n, thr, S);
    return OK;
}

int orc_multiplier_update(double* theta, const double* x, const double* L, const double* S,
                          uint64_t d, uint64_t n, double* rho, double kappa) {
    if (kappa <= 1.0) return fail(EINVAL_, "multiplier_update: kappa must be > 1");
    const double r = *rho; /* solver.cpp:104-111 */
    for (uint64_t k = 0; k < d * n; ++k) theta[k] += r * (x[k] - L[k] - S[k]);
    const double nr = r * kappa;
    *rho = (1e12 < nr) ? 1e12 : nr; /* std::min(rho*kappa, kRhoCap) */
    return OK;
}

static double rel_diff(const double* a, const double* b, uint64_t N, double xn) {
    double sq = 0.0; /* solver.cpp:14-21 */
    for (uint64_t k = 0; k < N; ++k) {
        const double t = a[k] - b[k];
        sq += t * t;
    }
    return sqrt(sq) / xn;
}

static double feas_residual(const double* x, const double* l, const double* s, uint64_t N,
                            double xn) {
    double sq = 0.0; /* solver.cpp:23-31 */
    for (uint64_t k = 0; k < N; ++k) {
        const double t = x[k] - l[k] - s[k];
        sq += t * t;
    }
    return sqrt(sq) / xn;
}

static double max3(double a, double b, double c) { /* std::max({a, b, c}) */
    double r = a;
    if (r < b) r = b;
    if (r < c) r = c;
    return r;
}

int orc_check_convergence(const double* x, const double* lp, const double* l, const double* sp,
                          const double* s, uint64_t d, uint64_t n, double tol, int* conv,
                          double* feas, double* dl, double* ds) {
    const uint64_t N = d * n; /* solver.cpp:113-125 */
    const double xn = frob_raw(x, N);
    if (xn == 0.0) return fail(EINVAL_, "check_convergence: all-zero X");
    *feas = feas_residual(x, l, s, N, xn);
    *dl = rel_diff(l, lp, N, xn);
    *ds = rel_diff(s, sp, N, xn);
    *conv = max3(*feas, *dl, *ds) <= tol;
    return OK;
}

static int validate_cfg(const orc_config* c) { /* solver.cpp:40-47 */
    if (c->has_lambda && c->lambda <= 0.0) return fail(EINVAL_, "lambda must be > 0");
    if (c->rho0 <= 0.0) return fail(EINVAL_, "rho0 must be > 0");
    if (c->kappa <= 1.0) return fail(EINVAL_, "kappa must be > 1");
    if (c->tol <= 0.0) return fail(EINVAL_, "tol must be > 0");
    if (c->c == 0) return fail(EINVAL_, "c must be >= 1");
    if (c->max_iter == 0) return fail(EINVAL_, "max_iter must be >= 1");
    return OK;
}

int orc_solve(const double* x, uint64_t d, uint64_t n, const orc_config* cfg, double* L,
              double* S, uint64_t* labels, double* feas, double* dl, double* ds, double* obj,
              uint64_t* iters, int* converged, double* lambda_out, double* wall) {
    /* solver.cpp:127-210 */
    int rc = validate_cfg(cfg);
    if (rc) return rc;
    if (cfg->c > n) return fail(EINVAL_, "solve: c exceeds column count");
    const uint64_t N = d * n;
    if (!all_finite(x, N)) return fail(EINVAL_, "solve: non-finite X");
    const double xn = frob_raw(x, N);
    if (xn == 0.0) return fail(EINVAL_, "solve: all-zero X");
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    const double lambda = cfg->has_lambda ? cfg->lambda : sqrt((double)(d > n ? d : n));

    double* Th = calloc(N, sizeof(double));
    double* D = malloc(N * sizeof(double));
    double* Lp = malloc(N * sizeof(double));
    double* Sp = malloc(N * sizeof(double));
    double* C = malloc(d * cfg->c * sizeof(double));
    uint64_t* lab2 = malloc(n * sizeof(uint64_t));
    memcpy(L, x, N * sizeof(double));
    memset(S, 0, N * sizeof(double));
    double rho = cfg->rho0;

    const uint64_t restarts = cfg->km_n_restarts > 5 ? cfg->km_n_restarts : 5;
    double inertia;
    uint64_t itr;
    rc = kmeans_raw(x, d, n, cfg->c, cfg->km_max_iters, restarts, cfg->km_seed, cfg->km_tol,
                    labels, C, &inertia, &itr);
    const uint64_t budget = cfg->has_fixed_iters ? cfg->fixed_iters : cfg->max_iter;
    uint64_t t = 0, done = 0;
    *converged = 0;
    for (; !rc && t < budget; ++t) {
        memcpy(Lp, L, N * sizeof(double));
        memcpy(Sp, S, N * sizeof(double));
        for (uint64_t k = 0; k < N; ++k) D[k] = x[k] - S[k] + Th[k] / rho;
        l_update_raw(D, d, n, labels, cfg->c, lambda, rho, L);
        rc = orc_kmeans_warm(L, d, n, cfg->c, cfg->km_max_iters, cfg->km_tol, labels, lab2, C,
                             &inertia, &itr);
        if (rc) break;
        memcpy(labels, lab2, n * sizeof(uint64_t));
        for (uint64_t k = 0; k < N; ++k) D[k] = x[k] - L[k] + Th[k] / rho;
        const double thr = 1.0 / rho;
        if (cfg->sparse_norm) shrink_l21(D, d, n, thr, S);
        else shrink_l1(D, N, thr, S);
        orc_multiplier_update(Th, x, L, S, d, n, &rho, cfg->kappa);
        done = t + 1;
        feas[t] = feas_residual(x, L, S, N, xn);
        dl[t] = rel_diff(L, Lp, N, xn);
        ds[t] = rel_diff(S, Sp, N, xn);
        const double sparse = cfg->sparse_norm ? l21_raw(S, d, n) : l1_raw(S, N);
        obj[t] = lambda * group_scatter_raw(L, d, n, labels, cfg->c) + sparse;
        if (!cfg->has_fixed_iters && max3(feas[t], dl[t], ds[t]) <= cfg->tol) {
            *converged = 1;
            break;
        }
    }
    free(Th);
    free(D);
    free(Lp);
    free(Sp);
    free(C);
    free(lab2);
    if (rc) return rc;
    *iters = done;
    *lambda_out = lambda;
    clock_gettime(CLOCK_MONOTONIC, &t1);
    *wall = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
    return OK;
}
