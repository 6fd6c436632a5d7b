/* Seeded synthetic inputs for the BASELINE.json configurations (host, C11 +
 * OpenMP).  Shared by bench.py and the parity tests so both solvers see the
 * same bytes; the reference ships no benchmark data set.
 *
 * Generator version "respca-synth-1".  Randomness is counter-based: every
 * draw is mix64(stream key, element index), so the output is independent of
 * the thread count.  Arithmetic is plain IEEE double with FMA contraction
 * disabled (-ffp-contract=off); normals use Box-Muller through glibc
 * log/cos/sqrt, so a given image (same glibc) reproduces the bytes exactly.
 *
 *   rpca  (C1, C2, C3, C5):  X = U·Vᵀ + S0,  U (d×r), V (n×r) i.i.d.
 *         N(0, sigma²); S0 Bernoulli(p) support, values U[lo, hi].
 *   video (C4):  240×320 frames flattened row-major, n frames; rank-3
 *         background B·Cᵀ from three Gaussian-blurred noise fields scaled so
 *         Σ_k B_k ∈ [0, 0.8]; C_jk = base_k (1 + δ_jk), base ~ U[0.9, 1.1],
 *         δ ~ U[-0.02, 0.02]; a 40×40 block of value U[0.3, 1.0] on a seeded
 *         random walk (±4 px / frame, reflecting); N(0, 0.01²) dense noise;
 *         clamp to [0, 1].
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "synth.h"

static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static inline uint64_t stream_key(uint64_t seed, uint64_t stream) {
    return mix64(seed + 0x9E3779B97F4A7C15ULL * (stream + 1));
}

static inline uint64_t draw(uint64_t key, uint64_t idx) {
    return mix64(key ^ (idx * 0xD1B54A32D192ED03ULL + 0x632BE59BD9B4E019ULL));
}

static inline double unit01(uint64_t u) { /* [0, 1) */
    return (double)(u >> 11) * (1.0 / 9007199254740992.0);
}

static inline double normal01(uint64_t key, uint64_t idx) {
    const double u1 = ((double)(draw(key, 2 * idx) >> 11) + 1.0) * (1.0 / 9007199254740992.0);
    const double u2 = unit01(draw(key, 2 * idx + 1));
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

const char* synth_version(void) { return "respca-synth-1"; }

/* the factors of synth_rpca alone: U (d×r column-major), V (n×r, row j =
 * V[j, :]) — the device assembly (respca_cu_synth_rpca) uses these */
int synth_rpca_factors(const synth_rpca_spec* sp, double* U, double* V) {
    const uint64_t d = sp->d, n = sp->n, r = sp->r;
    if (d == 0 || n == 0 || r == 0) return 1;
    const uint64_t ku = stream_key(sp->seed, 0), kv = stream_key(sp->seed, 1);
#pragma omp parallel for schedule(static)
    for (uint64_t e = 0; e < d * r; ++e) U[e] = sp->sigma * normal01(ku, e);
#pragma omp parallel for schedule(static)
    for (uint64_t e = 0; e < n * r; ++e) V[e] = sp->sigma * normal01(kv, e);
    return 0;
}

/* the S0 stream keys (support, values) of a spec */
void synth_rpca_keys(const synth_rpca_spec* sp, uint64_t* ks, uint64_t* kval) {
    *ks = stream_key(sp->seed, 2);
    *kval = stream_key(sp->seed, 3);
}

int synth_rpca(const synth_rpca_spec* sp, double* X, double* L0, double* S0) {
    const uint64_t d = sp->d, n = sp->n, r = sp->r;
    if (d == 0 || n == 0 || r == 0) return 1;
    double* U = malloc(d * r * sizeof(double)); /* column-major d×r */
    double* V = malloc(n * r * sizeof(double)); /* row j holds V[j, :] contiguous */
    if (!U || !V) {
        free(U);
        free(V);
        return 2;
    }
    const uint64_t ku = stream_key(sp->seed, 0), kv = stream_key(sp->seed, 1);
    const uint64_t ks = stream_key(sp->seed, 2), kval = stream_key(sp->seed, 3);
#pragma omp parallel for schedule(static)
    for (uint64_t e = 0; e < d * r; ++e) U[e] = sp->sigma * normal01(ku, e);
#pragma omp parallel for schedule(static)
    for (uint64_t e = 0; e < n * r; ++e) V[e] = sp->sigma * normal01(kv, e);
    const double span = sp->hi - sp->lo;
#pragma omp parallel
    {
        double* acc = malloc(d * sizeof(double));
#pragma omp for schedule(static)
        for (uint64_t j = 0; j < n; ++j) {
            for (uint64_t i = 0; i < d; ++i) acc[i] = 0.0;
            for (uint64_t k = 0; k < r; ++k) {
                const double v = V[j * r + k];
                const double* u = U + k * d;
                for (uint64_t i = 0; i < d; ++i) acc[i] += u[i] * v;
            }
            for (uint64_t i = 0; i < d; ++i) {
                const uint64_t e = j * d + i;
                double s = 0.0;
                if (unit01(draw(ks, e)) < sp->p) s = sp->lo + span * unit01(draw(kval, e));
                if (L0) L0[e] = acc[i];
                if (S0) S0[e] = s;
                X[e] = acc[i] + s;
            }
        }
        free(acc);
    }
    free(U);
    free(V);
    return 0;
}

/* separable Gaussian blur with reflecting borders, H×W row-major */
static void blur(double* f, uint64_t H, uint64_t W, double sigma) {
    const int R = (int)ceil(3.0 * sigma);
    double* w = malloc((2 * R + 1) * sizeof(double));
    double ws = 0.0;
    for (int t = -R; t <= R; ++t) ws += (w[t + R] = exp(-0.5 * (double)(t * t) / (sigma * sigma)));
    for (int t = 0; t <= 2 * R; ++t) w[t] /= ws;
    double* tmp = malloc(H * W * sizeof(double));
    for (uint64_t y = 0; y < H; ++y)
        for (uint64_t x = 0; x < W; ++x) {
            double s = 0.0;
            for (int t = -R; t <= R; ++t) {
                long xx = (long)x + t;
                while (xx < 0 || xx >= (long)W) xx = xx < 0 ? -xx - 1 : 2 * (long)W - xx - 1;
                s += w[t + R] * f[y * W + (uint64_t)xx];
            }
            tmp[y * W + x] = s;
        }
    for (uint64_t y = 0; y < H; ++y)
        for (uint64_t x = 0; x < W; ++x) {
            double s = 0.0;
            for (int t = -R; t <= R; ++t) {
                long yy = (long)y + t;
                while (yy < 0 || yy >= (long)H) yy = yy < 0 ? -yy - 1 : 2 * (long)H - yy - 1;
                s += w[t + R] * tmp[(uint64_t)yy * W + x];
            }
            f[y * W + x] = s;
        }
    free(tmp);
    free(w);
}

int synth_video(const synth_video_spec* sp, double* X, double* L0, double* S0) {
    const uint64_t H = sp->height, W = sp->width, n = sp->frames, d = H * W, B = sp->block;
    if (!H || !W || !n || B > H || B > W) return 1;
    double* F = malloc(3 * d * sizeof(double)); /* background fields B_k, d×3 col-major */
    double C[3];
    for (int k = 0; k < 3; ++k) {
        const uint64_t kf = stream_key(sp->seed, 10 + (uint64_t)k);
        double* f = F + (uint64_t)k * d;
        for (uint64_t e = 0; e < d; ++e) f[e] = normal01(kf, e);
        blur(f, H, W, sp->blur_sigma);
        double lo = f[0], hi = f[0];
        for (uint64_t e = 1; e < d; ++e) {
            lo = f[e] < lo ? f[e] : lo;
            hi = f[e] > hi ? f[e] : hi;
        }
        const double scale = (0.8 / 3.0) / (hi - lo);
        for (uint64_t e = 0; e < d; ++e) f[e] = (f[e] - lo) * scale;
        C[k] = 0.9 + 0.2 * unit01(draw(stream_key(sp->seed, 20), (uint64_t)k));
    }
    /* block random walk (sequential, cheap) */
    uint64_t* by = malloc(n * sizeof(uint64_t));
    uint64_t* bx = malloc(n * sizeof(uint64_t));
    const uint64_t kw = stream_key(sp->seed, 22);
    long y = (long)(draw(kw, 0) % (H - B + 1)), x = (long)(draw(kw, 1) % (W - B + 1));
    for (uint64_t j = 0; j < n; ++j) {
        if (j) {
            y += (long)(draw(kw, 2 + 2 * j) % 9) - 4;
            x += (long)(draw(kw, 3 + 2 * j) % 9) - 4;
            if (y < 0) y = -y;
            if (x < 0) x = -x;
            if (y > (long)(H - B)) y = 2 * (long)(H - B) - y;
            if (x > (long)(W - B)) x = 2 * (long)(W - B) - x;
        }
        by[j] = (uint64_t)y;
        bx[j] = (uint64_t)x;
    }
    const uint64_t kd = stream_key(sp->seed, 21), kv = stream_key(sp->seed, 23);
    const uint64_t kn = stream_key(sp->seed, 24);
#pragma omp parallel for schedule(static)
    for (uint64_t j = 0; j < n; ++j) {
        double cj[3];
        for (int k = 0; k < 3; ++k)
            cj[k] = C[k] * (1.0 + (-0.02 + 0.04 * unit01(draw(kd, j * 3 + (uint64_t)k))));
        const double v = 0.3 + 0.7 * unit01(draw(kv, j));
        for (uint64_t p = 0; p < d; ++p) {
            const uint64_t e = j * d + p;
            double l = 0.0;
            for (int k = 0; k < 3; ++k) l += F[(uint64_t)k * d + p] * cj[k];
            const uint64_t py = p / W, px = p % W;
            const int in = py >= by[j] && py < by[j] + B && px >= bx[j] && px < bx[j] + B;
            const double clean = in ? v : l;
            double xv = clean + sp->noise_sigma * normal01(kn, e);
            xv = xv < 0.0 ? 0.0 : (xv > 1.0 ? 1.0 : xv);
            if (L0) L0[e] = l;
            if (S0) S0[e] = clean - l;
            X[e] = xv;
        }
    }
    free(F);
    free(by);
    free(bx);
    return 0;
}

void synth_to_f32(const double* src, float* dst, uint64_t count) {
#pragma omp parallel for schedule(static)
    for (uint64_t e = 0; e < count; ++e) dst[e] = (float)src[e];
}
