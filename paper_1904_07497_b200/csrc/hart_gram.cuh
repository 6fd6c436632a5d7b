// Exact sequential Hartigan refinement (kmeans.cpp:96-139) on the Gram matrix.
//
// hartigan_refine visits columns j = 0..n−1 pass after pass and applies every
// improving single-point move at once, so each decision sees the centroids
// and counts left by all earlier moves.  The persistent kernel of
// hartigan.cuh keeps that order with distance intervals refreshed from the
// d-long centroid rows (O(d·n·c) per pass).  Here the same decisions are made
// from quantities that a move changes in O(n) work, independent of d:
//
//   G = MᵀM (n×n, FP64 tensor cores, once per kmeans(X), shared by every
//   restart), and per restart, for every centroid k with members Σ_k:
//     S_k[j] = x_j·Σ_k          (n values; a move m: f→t subtracts / adds G[:,m])
//     Q_k    = ‖Σ_k‖²            (O(1) per move)
//     ‖x_j − μ_k‖² = G_jj − 2·S_k[j]/n_k + Q_k/n_k²     (μ_k = Σ_k/n_k)
//
// The reference's centroids are not the exact means μ_k but running values
// c_k (means_of rounding, then the incremental update of kmeans.cpp:128-129
// per move), and its distance is the sequential chain of rounded squares.
// Every source of difference is bounded rigorously and carried per centroid:
//   |Ŝ_k[j] − x_j·Σ_k| ≤ ‖x_j‖·ES_k       |Q̂_k − ‖Σ_k‖²| ≤ EQ_k
//   ‖c_k − μ_k‖ ≤ Δ_k                      |Ĝ_jm − x_j·x_m| ≤ γ_G‖x_j‖‖x_m‖
//   |chain − ‖x − c‖²| ≤ γ_c‖x − c‖²       (γ_c = (d+3)u·1.02, hart_widen)
// so each (j, k) pair gets an interval that provably holds the reference's
// sq_dist value; a decision is taken only when it is the same for every value
// in the intervals (monotone IEEE rounding of the weights, as in
// hartigan.cuh).  Undecidable columns replay the logged moves onto the
// centroids with the reference's own formula and decide on the reference's
// chain.  Labels are therefore bit-identical to the reference's.
//
// One thread-block cluster per restart (k_hart_gram below): a window of
// 8·CL columns is decided by all warps of the cluster (lanes over centroids),
// the first column that is not provably "no move" is settled, its O(n) update
// is applied by every CTA to the columns it owns, and the scan resumes at the
// next column — no grid barrier per move.
#pragma once

#include "km.cuh"
#include "tc_screen.cuh"  // mbarrier helpers
#include "hartigan.cuh"   // bulk_g2s

namespace respca_dev {

// ---------------------------------------------------------------------------
// G = MᵀM: lower-triangle 128×128 tiles (mirrored on store), m16n8k8 DMMA,
// 3-stage cp.async ring over K-chunks of 32 rows.  8 warps, warp tile 64×32.
// ---------------------------------------------------------------------------
constexpr int GR_T = 128, GR_KC = 32, GR_AS = GR_KC + 4, GR_ST = 3;

template <typename T>
size_t gram_smem() {
    return (size_t)2 * GR_ST * GR_T * GR_AS * sizeof(T);
}

template <typename T>
__global__ void __launch_bounds__(256, 1) k_gram(const T* __restrict__ M, int64_t d, int n,
                                                 double* __restrict__ G, long long ntiles, long long t0 = 0) {
    extern __shared__ __align__(16) unsigned char sm[];
    T* As = reinterpret_cast<T*>(sm);        // [ST][128][AS]  columns i0.. (rows of A)
    T* Bs = As + GR_ST * GR_T * GR_AS;       // [ST][128][AS]  columns j0..
    constexpr int EPV = 16 / sizeof(T);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int wr = warp >> 2, wc = warp & 3;
    // a grid smaller than the tile count loops over tiles (G can then share
    // the GPU with the restarts' seeding and Lloyd steps)
    // tiles [t0, ntiles) of the row-major lower triangle (a band of block rows
    // when G is computed while X is still arriving)
    for (long long tix = t0 + blockIdx.x; tix < ntiles; tix += gridDim.x) {
    __syncthreads();  // the previous tile's stages are free
    int bi = (int)((sqrt(8.0 * (double)tix + 1.0) - 1.0) * 0.5);
    while ((long long)(bi + 1) * (bi + 2) / 2 <= tix) ++bi;
    while ((long long)bi * (bi + 1) / 2 > tix) --bi;
    const int bj = (int)(tix - (long long)bi * (bi + 1) / 2);
    const int i0 = bi * GR_T, j0 = bj * GR_T;
    const int nch = (int)((d + GR_KC - 1) / GR_KC);
    const bool vec = (d % EPV) == 0 && ((uintptr_t)M % 16) == 0;

    auto load = [&](int ch, int buf) {
        const int64_t k0 = (int64_t)ch * GR_KC;
        T* ad = As + (size_t)buf * GR_T * GR_AS;
        T* bd = Bs + (size_t)buf * GR_T * GR_AS;
        if (vec) {
            constexpr int VPC = GR_KC / EPV;  // vectors per column chunk
            for (int e = tid; e < 2 * GR_T * VPC; e += 256) {
                const int half = e / (GR_T * VPC), r = (e / VPC) % GR_T, v = e % VPC;
                const int col = (half ? j0 : i0) + r;
                const int64_t k = k0 + v * EPV;
                int bytes = 0;
                if (col < n && k < d) bytes = (int)(sizeof(T) * (d - k < EPV ? d - k : EPV));
                T* dst = (half ? bd : ad) + r * GR_AS + v * EPV;
                cp_async16(dst, bytes ? M + (int64_t)col * d + k : M, bytes);
            }
        } else {
            for (int e = tid; e < 2 * GR_T * GR_KC; e += 256) {
                const int half = e / (GR_T * GR_KC), r = (e / GR_KC) % GR_T, kk = e % GR_KC;
                const int col = (half ? j0 : i0) + r;
                const int64_t k = k0 + kk;
                const bool p = col < n && k < d;
                T* dst = (half ? bd : ad) + r * GR_AS + kk;
                if (sizeof(T) == 8) cp_async8(dst, p ? M + (int64_t)col * d + k : M, p);
                else cp_async4(dst, p ? M + (int64_t)col * d + k : M, p);
            }
        }
        cp_commit();
    };

    double acc[4][4][4];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y)
#pragma unroll
            for (int z = 0; z < 4; ++z) acc[x][y][z] = 0.0;

    for (int s = 0; s < GR_ST - 1; ++s) {
        if (s < nch) load(s, s);
        else cp_commit();
    }
    for (int ch = 0; ch < nch; ++ch) {
        cp_wait<GR_ST - 2>();
        __syncthreads();
        // refill the stage consumed two chunks ago
        if (ch + GR_ST - 1 < nch) load(ch + GR_ST - 1, (ch + GR_ST - 1) % GR_ST);
        else cp_commit();
        const T* as = As + (size_t)(ch % GR_ST) * GR_T * GR_AS + (wr * 64 + g) * GR_AS + t4;
        const T* bs = Bs + (size_t)(ch % GR_ST) * GR_T * GR_AS + (wc * 32 + g) * GR_AS + t4;
#pragma unroll
        for (int kk = 0; kk < GR_KC; kk += 8) {
            double a[4][4], b[4][2];
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                a[x][0] = (double)as[(x * 16) * GR_AS + kk];
                a[x][1] = (double)as[(x * 16 + 8) * GR_AS + kk];
                a[x][2] = (double)as[(x * 16) * GR_AS + kk + 4];
                a[x][3] = (double)as[(x * 16 + 8) * GR_AS + kk + 4];
            }
#pragma unroll
            for (int y = 0; y < 4; ++y) {
                b[y][0] = (double)bs[(y * 8) * GR_AS + kk];
                b[y][1] = (double)bs[(y * 8) * GR_AS + kk + 4];
            }
#pragma unroll
            for (int x = 0; x < 4; ++x)
#pragma unroll
                for (int y = 0; y < 4; ++y)
                    dmma1688(acc[x][y][0], acc[x][y][1], acc[x][y][2], acc[x][y][3], a[x][0], a[x][1],
                             a[x][2], a[x][3], b[y][0], b[y][1]);
        }
    }
    cp_wait<0>();
    // epilogue: (r, q) with r ≥ q stored at G[q·n + r] and G[r·n + q]
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y)
#pragma unroll
            for (int z = 0; z < 4; ++z) {
                const int r = i0 + wr * 64 + x * 16 + g + (z >= 2 ? 8 : 0);
                const int q = j0 + wc * 32 + y * 8 + 2 * t4 + (z & 1);
                if (r < n && q < n && r >= q) {
                    __stcg(G + (int64_t)q * n + r, acc[x][y][z]);
                    __stcg(G + (int64_t)r * n + q, acc[x][y][z]);
                }
            }
    }
}

// diagonal: xx = Ĝ_jj, xn ≥ ‖x_j‖ ≥ xl (|Ĝ_jj − ‖x_j‖²| ≤ γ_G‖x_j‖²)
__global__ void k_gram_diag(const double* __restrict__ G, int n, double gamG, double* __restrict__ xx,
                            double* __restrict__ xn, double* __restrict__ xl) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const double v = fmax(G[(int64_t)j * n + j], 0.0);
    xx[j] = v;
    xn[j] = __dsqrt_ru(__dmul_ru(v, __dadd_ru(1.0, 2.0 * gamG)));
    xl[j] = __dsqrt_rd(fmax(__dmul_rd(v, __dsub_rd(1.0, 2.0 * gamG)), 0.0));
}

// k-means++ d² (kmeans.cpp:188-191) of R restarts from G: one row of G per
// restart and pick instead of a pass over the d×n columns.
//   d̃(j, m) = max((Ĝ_jj + Ĝ_mm) − 2Ĝ_jm, 0)
//   |d̃(j, m) − sq_dist(x_j, x_m)| ≤ (γ_G + γ_c + 8u)·(‖x_j‖ + ‖x_m‖)²
// (γ_G: any DMMA accumulation order; γ_c: the reference's chain of rounded
// squares; 8u: the three FP64 operations here).  The host turns the d̃ values
// into the pick with this bound and falls back to the exact chains when the
// draw lands inside it (KMeansEngine::pp_joint).
template <int R>
__global__ void __launch_bounds__(256) k_pp_gram(const double* __restrict__ G, const double* __restrict__ xx, int n,
                                                 PPLast last, double* __restrict__ d2) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const double xj = xx[j];
    double g[R], xm[R], o[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int m = last.v[r];
        g[r] = __ldg(G + (int64_t)m * n + j);
        xm[r] = __ldg(xx + m);
        o[r] = d2[(int64_t)r * n + j];
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const double v = fmax((xj + xm[r]) - 2.0 * g[r], 0.0);
        d2[(int64_t)r * n + j] = fmin(o[r], v);
    }
}

// per-centroid state of the Gram refinement
struct GramScal {
    double Q, A, ES, EQ, Dl;  // Q̂_k, Σ‖x_m‖ (upper), S error / ‖x_j‖, Q error, ‖c_k − μ_k‖
};

RESPCA_DEV double gam_n(double m) {  // γ_m = m·u/(1 − m·u), bounded with slack
    return m * kU * 1.01;
}

// initial scalars from S⁰ and the start centroids C = means_of (kmeans.cpp:66-82);
// one block per centroid (the bounds below hold for any summation order)
__global__ void __launch_bounds__(256) k_gram_scal(const double* __restrict__ S, const double* __restrict__ xn,
                                                   const int* __restrict__ goff, const int* __restrict__ members,
                                                   int n, int c, double gamG, GramScal* __restrict__ out) {
    __shared__ double ra[32], rq[32];
    const int k = blockIdx.x;
    if (k >= c) return;
    const int p0 = goff[k], p1 = goff[k + 1];
    const double nk = (double)(p1 - p0);
    double A = 0.0, Q = 0.0;
    for (int p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
        const int m = __ldg(members + p);
        A = __dadd_ru(A, __ldg(xn + m));
        Q += __ldcg(S + (int64_t)k * n + m);
    }
    for (int o = 16; o > 0; o >>= 1) {
        A = __dadd_ru(A, __shfl_xor_sync(0xffffffffu, A, o));
        Q += __shfl_xor_sync(0xffffffffu, Q, o);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 0) {
        ra[warp] = A;
        rq[warp] = Q;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    A = 0.0;
    Q = 0.0;
    for (int w = 0; w < nw; ++w) {
        A = __dadd_ru(A, ra[w]);
        Q += rq[w];
    }
    const double gn = gam_n(nk);
    GramScal s;
    s.A = A;
    s.Q = Q;
    // Ŝ⁰ = Σ_m Ĝ[m][j] (any order): summation error γ_nk·Σ|Ĝ| plus the Ĝ errors
    s.ES = __dmul_ru(__dadd_ru(__dmul_ru(gn, 1.0 + gamG), gamG), __dmul_ru(A, 1.01));
    // Q̂⁰ = Σ_m Ŝ⁰_k[m] (any order): Σ_m xn_m·ES + γ_nk·Σ_m xn_m (A + ES)
    s.EQ = __dmul_ru(__dadd_ru(__dmul_ru(A, s.ES), __dmul_ru(gn, __dmul_ru(A, __dadd_ru(A, s.ES)))), 1.01);
    // start centroid = fl(fl(Σ x_m) · fl(1/n_k)): ‖c − μ‖ ≤ γ_nk·A/n_k·(1+3u) + 2.01u·‖μ‖
    const double mn = __dsqrt_ru(fmax(__ddiv_ru(__dadd_ru(Q, s.EQ), nk * nk), 0.0));
    s.Dl = __dmul_ru(__dadd_ru(__dmul_ru(__ddiv_ru(__dmul_ru(gn, A), nk), 1.0 + 4.0 * kU),
                               __dmul_ru(2.02 * kU, mn)),
                     1.01);
    out[k] = s;
}

struct GramArgs {
    const double* G;   // [n][n] Ĝ (column m contiguous)
    const double* xx;  // [n] Ĝ_jj
    const double* xn;  // [n] ≥ ‖x_j‖
    const double* xl;  // [n] ≤ ‖x_j‖
    double* S;         // [c][n] Ŝ_k[j]
    const GramScal* scal0;  // [c] initial scalars
    int* labels;       // [n] in/out
    int* counts;       // [c] in: start counts, out: final counts
    double* Cs;        // [c][d] stored centroids (in: start centroids; replayed on demand)
    int* log;          // [max_pass·n][5] moves (m, from, to, n_from, n_to)
    unsigned long long* stats;  // [8] moves, passes, windows, exact fallbacks, replayed rows·moves
    const void* M;     // the data (T), for the exact fallback
    int64_t d;
    int n, c, max_pass;
    int force_exact;   // tests: every candidate goes through the exact fallback
    int timing;        // RESPCA_TRACE: per-phase SM cycle counters in stats[5..12]
    double gamG, gamc;
};

// per-centroid decision coefficients (shared memory)
struct GramCoef {
    double wa, wb;   // n/(n−1), n/(n+1) as the reference rounds them (kmeans.cpp:107, 114)
    double a2, bq;   // fl(2/n), fl(Q̂/n²)
    double E0, E1;   // interval half-width = E0 + E1·‖x_j‖ + γ_G‖x_j‖² + 5.1u(Ĝ_jj + |t| + bq)
    double mn;       // ≥ ‖μ_k‖
};

// Bounds below are evaluated in round-to-nearest: every one is a chain of at
// most a few dozen positive terms, so a final factor (1 + 64u) covers the
// roundings (each op contributes at most a relative u).
constexpr double kSlack = 1.0 + 64.0 * kU;

RESPCA_DEV void gram_coef(const GramScal& s, int cnt, GramCoef& o) {
    const double nk = (double)cnt;
    o.wa = nk / (nk - 1.0);  // the reference's correctly rounded weights
    o.wb = nk / (nk + 1.0);
    const double rn = 1.0 / nk;
    o.a2 = 2.0 * rn;           // |a2 − 2/n| ≤ u·a2
    o.bq = (s.Q * rn) * rn;    // |bq − Q̂/n²| ≤ 3.01u·|bq|
    const double r2 = rn * rn * kSlack;
    o.mn = sqrt(fmax((s.Q + s.EQ) * r2, 0.0)) * kSlack;
    // ‖x − c‖² vs ‖x − μ‖²: 2(‖x‖ + ‖μ‖)Δ + Δ²
    o.E0 = ((s.EQ * r2 + 2.0 * o.mn * s.Dl) + s.Dl * s.Dl) * kSlack;
    o.E1 = (2.0 * s.ES * rn + 2.0 * s.Dl) * kSlack;
}

// interval [lo, hi] ∋ the reference's sq_dist(x_j, c_k); mid for the argmin
struct GramCol {
    double gjj, xnj, gq;
};
RESPCA_DEV void gram_iv(const GramCol& col, const GramCoef& cf, double s, double gamc, double& lo, double& hi,
                        double& mid) {
    const double t = cf.a2 * s;
    mid = (col.gjj - t) + cf.bq;
    const double e =
        ((cf.E0 + cf.E1 * col.xnj) + (col.gq + 7.1 * kU * (fabs(t) + cf.bq))) * (1.0 + 16.0 * kU);
    lo = fmax(mid - e, 0.0) * ((1.0 - gamc) * (1.0 - 8.0 * kU));
    hi = (mid + e) * ((1.0 + gamc) * (1.0 + 8.0 * kU));
    if (!(lo <= hi)) {  // non-finite: never decides
        lo = 0.0;
        hi = INFINITY;
    }
}

// One warp decides column `from` on per-lane intervals (k = lane + 32q):
// 0 = provably no move, 1 = provably moves to `to`, 2 = undecidable.
// Same decision logic as hart_decide_warp_w (hartigan.cuh).
template <int KPL>
RESPCA_DEV int gram_decide(int from, int c, const GramCoef* cf, const int* cnt, const double (&lo)[KPL],
                           const double (&hi)[KPL], const double (&mid)[KPL], int& to) {
    const int lane = threadIdx.x & 31;
    if (cnt[from] <= 1) return 0;  // kmeans.cpp:105
    const int fq = from >> 5, fl_ = from & 31;
    // the common verdict first, on a branch-free path: "provably no move" needs only
    // the own centroid's upper end and the others' lower ends
    double fhi = 0;
#pragma unroll
    for (int q = 0; q < KPL; ++q)
        if (q == fq) fhi = __shfl_sync(0xffffffffu, hi[q], fl_);
    const double w_a = cf[from].wa;
    const double g_hi = w_a * fhi;
    double wbq[KPL];
    bool none = true;
#pragma unroll
    for (int q = 0; q < KPL; ++q) {
        const int k = lane + 32 * q;
        const bool valid = k < c && k != from;
        wbq[q] = cf[valid ? k : from].wb;
        none &= !valid || !(wbq[q] * lo[q] - g_hi < -1e-12);  // kmeans.cpp:116, best_delta = −1e-12
    }
    none = __all_sync(0xffffffffu, none);
    if (none) return 0;
    double flo = 0, fmid = 0;
#pragma unroll
    for (int q = 0; q < KPL; ++q)
        if (q == fq) {
            flo = __shfl_sync(0xffffffffu, lo[q], fl_);
            fmid = __shfl_sync(0xffffffffu, mid[q], fl_);
        }
    const double g_lo = w_a * flo, g_mid = w_a * fmid;
    double bd = INFINITY;
    int bk = 0x7fffffff;
#pragma unroll
    for (int q = 0; q < KPL; ++q) {
        const int k = lane + 32 * q;
        if (k >= c || k == from) continue;
        const double dmid = wbq[q] * mid[q] - g_mid;
        if (dmid < bd) {
            bd = dmid;
            bk = k;
        }
    }
    warp_argmin(bd, bk);
    if (bk >= c) return 2;
    const int bq_ = bk >> 5, bl = bk & 31;
    double bhi = 0;
#pragma unroll
    for (int q = 0; q < KPL; ++q)
        if (q == bq_) bhi = __shfl_sync(0xffffffffu, hi[q], bl);
    const double dhi_k = cf[bk].wb * bhi - g_lo;
    bool ok = dhi_k < -1e-12;
#pragma unroll
    for (int q = 0; q < KPL; ++q) {
        const int k = lane + 32 * q;
        if (k >= c || k == from || k == bk) continue;
        const double dlo = cf[k].wb * lo[q] - g_hi;
        if (k < bk) ok &= dhi_k < dlo;  // an earlier k must lose strictly
        else ok &= dhi_k <= dlo;        // a later k never replaces an equal delta
    }
    ok = __all_sync(0xffffffffu, ok);
    if (!ok) return 2;
    to = bk;
    return 1;
}

constexpr unsigned long long kHartWaitNs = 30000000000ULL;  // mbarrier waits of the refinement: 30 s
constexpr int GRAM_THREADS = 256;
constexpr int GRAM_WARPS = GRAM_THREADS / 32;

// The move m: from → to (kmeans.cpp:122-135) on one side's scalars (side 0 =
// from, 1 = to): Q, A, ES, EQ, Δ and the decision coefficients.  sv = Ŝ_k[m]
// before the move.
RESPCA_DEV void gram_side(int side, GramScal& S, GramCoef& cf, int& cnt, double sv, double gmm, double xnm,
                          double xlm, double gamG) {
    const double nk = (double)cnt;
    const double g2 = gamG * xnm * xnm;
    const double gx = gamG * xnm;
    // Q: ‖Σ ∓ x_m‖² = Q ∓ 2x_m·Σ + ‖x_m‖²  (two rounded adds: ≤ 2.01u of the magnitudes)
    const double q = side ? (S.Q + 2.0 * sv) + gmm : (S.Q - 2.0 * sv) + gmm;
    const double eq = ((S.EQ + 2.0 * xnm * S.ES) + (g2 + 2.02 * kU * (fabs(S.Q) + 2.0 * fabs(sv) + gmm))) * kSlack;
    // A stays an upper bound of Σ‖x_m‖ over the members
    const double A = side ? (S.A + xnm) * kSlack : fmax(S.A - xlm * (1.0 - 4.0 * kU), 0.0) * kSlack;
    // S: one rounded ∓ Ĝ[j][m] per entry; |Ŝ′| ≤ ‖x_j‖(A′ + ES + γ_G‖x_m‖)
    const double es = ((S.ES + gx) + kU * 1.01 * ((A + S.ES) + gx)) * kSlack;
    // Δ: c′ − μ′ = n(c − μ)/(n ∓ 1) + ρ, ‖ρ‖ ≤ 3.01u(n‖c‖ + ‖x_m‖)/(n ∓ 1), ‖c‖ ≤ ‖μ‖ + Δ
    const double dl = ((S.Dl * nk + 3.02 * kU * (nk * (cf.mn + S.Dl) + xnm)) / (side ? nk + 1.0 : nk - 1.0)) * kSlack;
    S.Q = q;
    S.EQ = eq;
    S.A = A;
    S.ES = es;
    S.Dl = dl;
    cnt = side ? cnt + 1 : cnt - 1;
    gram_coef(S, cnt, cf);
}

// ---- thread-block cluster helpers (DSMEM + cluster barrier)
RESPCA_DEV uint32_t gcl_smem(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
RESPCA_DEV uint32_t gcl_map(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(gcl_smem(p)), "r"(rank));
    return r;
}
RESPCA_DEV int gcl_ld_i32(uint32_t a) {
    int v;
    asm volatile("ld.shared::cluster.b32 %0, [%1];\n" : "=r"(v) : "r"(a) : "memory");
    return v;
}
RESPCA_DEV double gcl_ld_f64(uint32_t a) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];\n" : "=d"(v) : "r"(a) : "memory");
    return v;
}
RESPCA_DEV void gcl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
RESPCA_DEV uint32_t gcl_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
RESPCA_DEV uint32_t gcl_size() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;\n" : "=r"(r));
    return r;
}
constexpr int GRAM_MAXCL = 16;

RESPCA_DEV void gcl_st_i32(uint32_t a, int v) {
    asm volatile("st.shared::cluster.b32 [%0], %1;\n" ::"r"(a), "r"(v) : "memory");
}
RESPCA_DEV double gcl_ld_w(uint32_t a) { return gcl_ld_f64(a); }
RESPCA_DEV void gcl_st_f64(uint32_t a, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(a), "d"(v) : "memory");
}

// ---------------------------------------------------------------------------
// k_hart_gram: one thread-block cluster per restart, the window's data resident
// on chip.  Every CTA keeps a replica of the per-centroid state; a window of
// W = GRAM_WARPS·CL consecutive columns is decided by all warps of the cluster.
//
// (Round 1 staged every window's Ŝ block from L2 — columns moved between CTAs
// as the window start moved — so each window paid an L2 round trip before it
// could decide, and every CTA's global Ŝ stores had to be fenced cluster-wide
// under a cluster barrier per window: 3.6 µs per window, 78 ms per restart at
// C3; this kernel: 3.1 µs, 68 ms.)  Column ownership is fixed: columns are dealt to the CTAs in
// groups of GW = GRAM_WARPS (group g → CTA g mod CL), so ANY window of
// W = GW·CL consecutive columns holds exactly GW columns of every CTA (one
// whole group, or the two partial groups of the CTA straddling the window
// start).  Each CTA keeps, in shared memory, for its current and next group:
//   * Ŝ_k[j] of the group's columns for every centroid k,
//   * the Ĝ row segments Ĝ[j][J0 − 2W .. J0 + W + GW) of its columns — every
//     column that can move while the group is cached,
//   * label, Ĝ_jj and the norm bounds,
// loaded with cp.async one group-stride (≈ five windows) ahead.  The elected
// move is applied to the cached groups from shared memory (Ŝ_from −= Ĝ[j][m],
// Ŝ_to += Ĝ[j][m], one rounded operation each — the arithmetic of k_hart_gram)
// and to the CTA's other columns in global memory, which only this CTA ever
// reads or writes — so no cluster-wide fence is needed.  A window is then:
// patch (shared memory) → decide → every CTA pushes its first candidate
// (verdict, column, the move's five inputs) into every CTA's shared memory with
// st.async, each store completing bytes on the receiver's mbarrier → wait on the
// local mbarrier → elect the lowest column; the far stores and the block change
// ride behind the push.  No load from L2, no cluster barrier and no fence sit on
// that path.  The decisions are made on the rigorous intervals above; an
// undecidable column replays the logged moves and decides on the reference's
// own chain (CTA 0, cluster barriers on that rare path only).
// ---------------------------------------------------------------------------
// asynchronous store into another CTA's shared memory that completes bytes on
// that CTA's mbarrier: the receiver's mbarrier wait orders the data, no
// cluster-wide fence or barrier is involved
RESPCA_DEV void gcl_st_async_b64(uint32_t remote_addr, uint64_t v, uint32_t remote_bar) {
    asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n" ::"r"(remote_addr),
                 "l"(v), "r"(remote_bar)
                 : "memory");
}

template <typename T, int KPL>
__global__ void __launch_bounds__(GRAM_THREADS, 1) k_hart_gram(GramArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int c = a.c, n = a.n;
    const int64_t d = a.d;
    constexpr int GW = GRAM_WARPS;
    constexpr int MVW = 5;  // a move's inputs: Ŝ_from[j], Ŝ_to[j], Ĝ_jj, ‖x_j‖ upper / lower bound
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int rank = (int)gcl_rank(), CL = (int)gcl_size();
    const int W = GW * CL;
    const int LCL = __ffs(CL) - 1, LW = LCL + 3;  // CL is a power of two (host): divisions by CL, W are shifts
    static_assert(GW == 8, "LW = log2(GW·CL)");
    constexpr int NSL = 3;      // cached groups per CTA: the blocks of the window and the next one
    const int GL = 4 * W;       // cached Ĝ row segment of block m's group: columns (m − 2)W .. (m + 2)W − 1
    const int CS = (c + 1) & ~1;
    GramCoef* cf = reinterpret_cast<GramCoef*>(sm);
    GramScal* sc = reinterpret_cast<GramScal*>(cf + c);
    double* dist = reinterpret_cast<double*>(sc + c);  // [c] exact chains (fallback)
    int* cnt = reinterpret_cast<int*>(dist + c);
    // 16-byte aligned behind cnt (offset arithmetic, so the pointer stays a shared-memory one)
    const size_t sc_off = ((size_t)c * (sizeof(GramCoef) + sizeof(GramScal) + sizeof(double)) +
                           sizeof(int) * (size_t)((c + 1) & ~1) + 15) & ~(size_t)15;
    double* scache = reinterpret_cast<double*>(sm + sc_off);  // [NSL][GW][CS]
    double* gseg = scache + (size_t)NSL * GW * CS;                                   // [NSL][GW][GL]
    __shared__ int clab[NSL][GW];
    __shared__ double cxx[NSL][GW], cxn[NSL][GW], cxl[NSL][GW];
    __shared__ int s_loc[GW];                  // this CTA's verdicts: status | to << 2 | from << 17
    __shared__ double s_sv[GW][MVW];           // this CTA's candidates' move inputs
    // every CTA's first candidate of the window: word 0 = verdict | column << 32,
    // words 1..5 = the move's inputs; written by st.async from every CTA, each
    // store completing 8 bytes on this CTA's mbarrier xbar[parity]
    constexpr int XW = 1 + MVW;
    __shared__ __align__(16) unsigned long long s_xch[2][GRAM_MAXCL][XW];
    __shared__ __align__(8) uint64_t xbar[2];
    __shared__ __align__(8) uint64_t gbar;  // the Ĝ row segments of a group load (bulk copies)
    __shared__ int s_xres;        // exact fallback verdict (CTA 0)
    __shared__ double s_xsv[MVW];  // ... and the move's inputs (the column's owner)
    const T* M = static_cast<const T*>(a.M);
    const double gamG = a.gamG, gamc = a.gamc;
    // this CTA's groups: m = 0 .. NG − 1, group m = columns J0(m) .. J0(m) + GW − 1 of
    // block m = columns mW .. (m + 1)W − 1.  Cached: the groups of blocks cur, cur + 1
    // (any window starting in block cur lies inside them) and cur + 2 (loaded one
    // block ahead); every CTA rotates in the same window, when the cursor enters the
    // next block, so no CTA waits at the cluster barrier for another's rotation
    const int ngroups = (n + GW - 1) / GW;
    const int NG = rank < ngroups ? (ngroups - rank + CL - 1) / CL : 0;
    auto J0 = [&](int m) { return (m * CL + rank) * GW; };
    constexpr int UPT = 3;  // far columns per thread held across the window

    for (int k = tid; k < c; k += blockDim.x) {
        const int ck = a.counts[k];
        cnt[k] = ck;
        sc[k] = a.scal0[k];
        gram_coef(sc[k], ck, cf[k]);
    }
    if (tid == 0) {
        mbar_init(&xbar[0], 1);  // one arrival per window: this CTA's expect_tx
        mbar_init(&xbar[1], 1);
        mbar_init(&gbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    gcl_sync();  // every replica and mbarrier initialised before remote stores land
    unsigned xph[2] = {0, 0};  // completed phases of xbar[0], xbar[1]
    unsigned gph = 0;          // completed phases of gbar
    const bool gbulk = (n & 1) == 0 && (reinterpret_cast<uintptr_t>(a.G) & 15) == 0;  // 16-byte aligned rows

    unsigned long long moves = 0, windows = 0, fallbacks = 0, replay_work = 0;
    unsigned long long tph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    unsigned long long tmk = clock64();
    const bool timing = a.timing != 0;
    auto lap = [&](int slot) {
        if (timing && tid == 0) {
            const unsigned long long t = clock64();
            tph[slot] += t - tmk;
            tmk = t;
        }
    };
    uint32_t gbytes = 0;  // thread 0: bytes of the bulk copies issued since the last commit
    // group m's Ŝ columns, Ĝ row segments and per-column scalars → shared memory (cp.async / bulk copies)
    auto load_group = [&](int m) {
        if (m >= NG) return;
        const int slot = m % NSL, j0 = J0(m);
        for (int e = tid; e < c * GW; e += GRAM_THREADS) {
            const int k = e / GW, col = e - k * GW;
            const bool ok = j0 + col < n;
            cp_async8(&scache[(size_t)(slot * GW + col) * CS + k], ok ? a.S + (int64_t)k * n + j0 + col : a.S, ok);
        }
        const int base = (m - 2) * W;
        if (gbulk) {  // one bulk copy per column (thread 0 issues them; gbar counts the bytes)
            if (tid == 0) {
                const int q0 = base < 0 ? -base : 0, q1 = base + GL > n ? n - base : GL;  // even: W, n even
                for (int col = 0; col < GW; ++col)
                    if (j0 + col < n && q1 > q0) {
                        bulk_g2s(&gseg[(size_t)(slot * GW + col) * GL + q0], a.G + (int64_t)(j0 + col) * n + base + q0,
                                 (uint32_t)(q1 - q0) * 8u, &gbar);
                        gbytes += (uint32_t)(q1 - q0) * 8u;
                    }
            }
        } else {
            for (int e = tid; e < GW * GL; e += GRAM_THREADS) {
                const int col = e / GL, q = e - col * GL;
                const int jq = base + q;
                const bool ok = j0 + col < n && jq >= 0 && jq < n;
                cp_async8(&gseg[(size_t)(slot * GW + col) * GL + q], ok ? a.G + (int64_t)(j0 + col) * n + jq : a.G, ok);
            }
        }
        if (tid < GW) {  // per-column scalars, asynchronously too (a plain load would stall this warp for an L2 round trip)
            const int j = j0 + tid;
            const bool ok = j < n;
            cp_async4(&clab[slot][tid], ok ? a.labels + j : a.labels, ok);
            cp_async8(&cxx[slot][tid], ok ? a.xx + j : a.xx, ok);
            cp_async8(&cxn[slot][tid], ok ? a.xn + j : a.xn, ok);
            cp_async8(&cxl[slot][tid], ok ? a.xl + j : a.xl, ok);
        }
    };
    auto writeback_group = [&](int m) {
        if (m >= NG) return;
        const int slot = m % NSL, j0 = J0(m);
        for (int e = tid; e < c * GW; e += GRAM_THREADS) {
            const int k = e / GW, col = e - k * GW;
            if (j0 + col < n) __stcg(a.S + (int64_t)k * n + j0 + col, scache[(size_t)(slot * GW + col) * CS + k]);
        }
    };
    // the pending move on the cached groups (one thread per cached column); the
    // replicas took it when it was elected
    auto patch_cached = [&](int cur, int pj, int pf, int pt, const double (&pmv)[5]) {
        const int pt_ = tid - (GRAM_THREADS - 64);  // the last warp but one (the last one carries the replica update)
        if (pt_ >= 0 && pt_ < NSL * GW) {
            const int gi = pt_ / GW, col = pt_ - gi * GW, m = cur + gi;
            if (m < NG && J0(m) + col < n) {
                const int slot = m % NSL;
                const double g = gseg[(slot * GW + col) * GL + (pj - (m - 2) * W)];
                double* sv = scache + (slot * GW + col) * CS;
                sv[pf] = sv[pf] - g;
                sv[pt] = sv[pt] + g;
                if (J0(m) + col == pj) clab[slot][col] = pt;
            }
        }
    };
    // e-th far column of this CTA (its columns outside the cached groups cur .. cur + 2), or −1
    auto far_col = [&](int e, int cur) -> int {
        const int gi = e / GW;
        if (gi >= NG || (gi >= cur && gi <= cur + 2)) return -1;
        const int q = J0(gi) + (e - gi * GW);
        return q < n ? q : -1;
    };

    bool loading = false;  // a group load is outstanding
    auto commit_load = [&]() {
        cp_commit();
        if (gbulk && tid == 0) {
            if (gbytes) mbar_expect_tx_cta(&gbar, gbytes);
            else mbar_arrive(&gbar);
            gbytes = 0;
        }
        loading = true;
    };
    auto finish_load = [&]() {  // all threads: the outstanding group load has landed
        cp_wait<0>();
        if (gbulk) {
            if (!mbar_wait(&gbar, gph & 1u, kHartWaitNs)) asm volatile("trap;\n");
            ++gph;
        }
        __syncthreads();
        loading = false;
    };
    int nlog = 0, replayed = 0, pass = 0, par = 0;
    int pj = -1, pf = 0, pt = 0;  // the pending move (uniform over the cluster)
    double pmv[5] = {0, 0, 0, 0, 0};
    int cur = -1;           // current block (−1: nothing cached)
    for (;;) {
        // ---- pass start: drain the pending move, write the cached groups back, cache groups 0, 1, 2
        {
            if (loading) finish_load();  // never two group loads outstanding
            if (pj >= 0) {
                for (int e = tid; e < NG * GW; e += GRAM_THREADS) {
                    const int q = far_col(e, cur);
                    if (q >= 0) {
                        const double g = __ldcg(a.G + (int64_t)pj * n + q);
                        const double f0 = __ldcg(a.S + (int64_t)pf * n + q), t0 = __ldcg(a.S + (int64_t)pt * n + q);
                        __stcg(a.S + (int64_t)pf * n + q, f0 - g);
                        __stcg(a.S + (int64_t)pt * n + q, t0 + g);
                    }
                }
                patch_cached(cur, pj, pf, pt, pmv);
                ++nlog;
                pj = -1;
            }
            __syncthreads();
            if (cur >= 0) {
                writeback_group(cur);
                writeback_group(cur + 1);
                writeback_group(cur + 2);
            }
            __syncthreads();
            cur = 0;
            load_group(0);
            load_group(1);
            load_group(2);
            commit_load();
            finish_load();
        }
        int improved = 0;
        int cursor = 0;
        while (cursor < n) {
            const bool mv = pj >= 0;
            const int fcur = cur;
            if (loading) finish_load();  // the group loaded at the last block change (a window ago at least)
            // ---- (1) the pending move: far columns loaded, cached columns patched in shared memory
            double ug[UPT], uf[UPT], ut[UPT];
            int uq[UPT];
            const double* Gp = a.G + (int64_t)(mv ? pj : 0) * n;  // the pending move's rows
            double* Sf = a.S + (int64_t)pf * n;
            double* St = a.S + (int64_t)pt * n;
            if (mv) {
                patch_cached(cur, pj, pf, pt, pmv);
#pragma unroll
                for (int e = 0; e < UPT; ++e) {
                    uq[e] = far_col(tid + e * GRAM_THREADS, cur);
                    if (uq[e] >= 0) {
                        ug[e] = __ldcg(Gp + uq[e]);
                        uf[e] = __ldcg(Sf + uq[e]);
                        ut[e] = __ldcg(St + uq[e]);
                    }
                }
                ++nlog;
            }
            lap(2);
            __syncthreads();
            // ---- (3) this warp's column of the window: the warp-th of this CTA's columns in it
            int j = n;
            {
                const int g0 = cursor / GW, o = cursor - g0 * GW;
                const int dg = (rank - g0) & (CL - 1);
                if (dg == 0 && o > 0) j = warp < GW - o ? cursor + warp : (g0 + CL) * GW + (warp - (GW - o));
                else j = (g0 + dg) * GW + warp;
                if (j >= n) j = n;
            }
            const int jm = j < n ? j >> LW : cur;  // the column's block: cur or cur + 1, both landed
            int st = 0, to = -1, from = 0;
            if (j < n) {
                const int slot = jm % NSL, col = j - (j / GW) * GW;
                from = clab[slot][col];
                const double gjj = cxx[slot][col], xnj = cxn[slot][col];
                const double* svp = scache + (slot * GW + col) * CS;
                double sv[KPL];
#pragma unroll
                for (int q = 0; q < KPL; ++q) {
                    const int k = lane + 32 * q;
                    sv[q] = k < c ? svp[k] : 0.0;
                }
                if (cnt[from] > 1) {
                    GramCol colv;
                    colv.gjj = gjj;
                    colv.xnj = xnj;
                    colv.gq = gamG * xnj * xnj * (1.0 + 4.0 * kU) + 7.1 * kU * gjj;
                    double lo[KPL], hi[KPL], mid[KPL];
#pragma unroll
                    for (int q = 0; q < KPL; ++q) {  // branch-free: lanes past c compute on centroid 0 and discard
                        const int k = lane + 32 * q;
                        gram_iv(colv, cf[k < c ? k : 0], sv[q], gamc, lo[q], hi[q], mid[q]);
                        if (k >= c) lo[q] = hi[q] = mid[q] = INFINITY;
                    }
                    st = gram_decide<KPL>(from, c, cf, cnt, lo, hi, mid, to);
                    if (a.force_exact && st == 1) st = 2;
                    if (st != 0 && lane == 0) {
                        // a candidate: its Ĝ row (every CTA's far update) to L2
                        const uintptr_t b0 = reinterpret_cast<uintptr_t>(a.G + (int64_t)j * n);
                        const uintptr_t s0 = b0 & ~(uintptr_t)15;
                        const unsigned bytes = (unsigned)((b0 + (uintptr_t)n * 8 - s0 + 15) & ~(uintptr_t)15);
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(s0), "r"(bytes) : "memory");
                    }
                    if (st == 1 && lane == 0) {  // the move's inputs
                        s_sv[warp][0] = svp[from];
                        s_sv[warp][1] = svp[to];
                        s_sv[warp][2] = gjj;
                        s_sv[warp][3] = xnj;
                        s_sv[warp][4] = cxl[slot][col];
                    }
                }
            }
            lap(4);
            // ---- (4) this warp's verdict; the CTA's first candidate → every CTA
            if (lane == 0) s_loc[warp] = st | ((to < 0 ? 0 : to) << 2) | (from << 17);
            __syncthreads();
            {
                const int v = lane < GW ? s_loc[lane] : 0;
                const unsigned bal = __ballot_sync(0xffffffffu, (v & 3) != 0);
                const int fw = bal ? __ffs(bal) - 1 : 0;  // warps are in column order
                if (warp == fw) {
                    const int fv = __shfl_sync(0xffffffffu, v, fw);
                    const unsigned long long vw =
                        (unsigned long long)(unsigned)(bal ? fv : 0) | ((unsigned long long)(unsigned)j << 32);
                    // CL·XW words, always all of them (every CTA expects CL·XW·8 bytes per
                    // window), spread over the warp's lanes: word q of receiver r
                    for (int e = lane; e < CL * XW; e += 32) {
                        const int r = e / XW, q = e - r * XW;
                        const unsigned long long word =
                            q == 0 ? vw
                                   : ((fv & 3) == 1 ? (unsigned long long)__double_as_longlong(s_sv[fw][q - 1]) : 0ull);
                        gcl_st_async_b64(gcl_map(&s_xch[par][rank][q], (uint32_t)r), word,
                                         gcl_map(&xbar[par], (uint32_t)r));
                    }
                }
                if (tid == 0) mbar_expect_tx_cta(&xbar[par], (uint32_t)(CL * XW * 8));
            }
            lap(5);
            // the far stores and the block change ride in the shadow of the exchange
            // ---- (3b) far stores: their loads were issued at the window's start and have
            //      landed behind the decide; nothing below waits for them (no fence)
            if (mv) {
#pragma unroll
                for (int e = 0; e < UPT; ++e)
                    if (uq[e] >= 0) {
                        __stcg(Sf + uq[e], uf[e] - ug[e]);
                        __stcg(St + uq[e], ut[e] + ug[e]);
                    }
                if (NG * GW > UPT * GRAM_THREADS)
                    for (int e = tid + UPT * GRAM_THREADS; e < NG * GW; e += GRAM_THREADS) {
                        const int q = far_col(e, fcur);
                        if (q >= 0) {
                            const double g = __ldcg(Gp + q);
                            const double f0 = __ldcg(Sf + q), t0 = __ldcg(St + q);
                            __stcg(Sf + q, f0 - g);
                            __stcg(St + q, t0 + g);
                        }
                    }
                pj = -1;
            }
            lap(1);
            // ---- (3c) the cursor entered the next block (every CTA in this same window): the
            //      old block's group goes back to global memory, its slot takes block cur + 3's
            //      group — after the far stores above, under which it was still a far group
            if ((cursor >> LW) > cur) {
                writeback_group(cur);
                __syncthreads();  // far stores and write-back issued; the slot's readers are done
                ++cur;
                load_group(cur + 2);
                commit_load();
            }
            lap(3);
            // a lost exchange aborts the kernel instead of hanging the GPU; the limit is
            // generous so that a time-sliced or preempted context does not trip it
            if (!mbar_wait(&xbar[par], xph[par] & 1u, kHartWaitNs)) asm volatile("trap;\n");
            ++xph[par];
            lap(6);
            // ---- (5) every warp: the window's first candidate = the lowest column
            int pr = -1, jj = 0x7fffffff, w = 0;
            {
                const unsigned long long vw = lane < CL ? s_xch[par][lane][0] : 0ull;
                const int v = (int)(unsigned)(vw & 0xffffffffull);
                const int jc = lane < CL && (v & 3) != 0 ? (int)(unsigned)(vw >> 32) : 0x7fffffff;
                int bj = jc, br = lane;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const int oj = __shfl_xor_sync(0xffffffffu, bj, o), orr = __shfl_xor_sync(0xffffffffu, br, o);
                    if (oj < bj) {
                        bj = oj;
                        br = orr;
                    }
                }
                if (bj != 0x7fffffff) {
                    pr = br;
                    jj = bj;
                    w = (int)(unsigned)(s_xch[par][pr][0] & 0xffffffffull);
                }
            }
            ++windows;
            lap(0);
            if (pr < 0) {
                cursor += W;
                par ^= 1;
                continue;
            }
            cursor = jj + 1;
            const int mfrom = w >> 17;
            int mst = w & 3, mto = (w >> 2) & 0x7fff;
            double mvin[MVW];
            if (mst == 1) {
#pragma unroll
                for (int q = 0; q < MVW; ++q) mvin[q] = __longlong_as_double((long long)s_xch[par][pr][1 + q]);
            } else {
                // ---- near-tie (CTA 0): the reference's own chain on the reference's
                //      centroids (logged moves replayed, kmeans.cpp:128-129)
                ++fallbacks;
                if (rank == 0) {
                    for (int64_t i = tid; i < d; i += blockDim.x) {
                        for (int e = replayed; e < nlog; ++e) {
                            const int* lg = a.log + 5 * (int64_t)e;
                            const int m = __ldcg(lg), f = __ldcg(lg + 1), t = __ldcg(lg + 2);
                            const double nf = (double)__ldcg(lg + 3), nt = (double)__ldcg(lg + 4);
                            const double x = (double)M[(int64_t)m * d + i];
                            double* cfp = a.Cs + (int64_t)f * d + i;
                            double* ctp = a.Cs + (int64_t)t * d + i;
                            *cfp = (*cfp * nf - x) / (nf - 1.0);
                            *ctp = (*ctp * nt + x) / (nt + 1.0);
                        }
                    }
                    __syncthreads();
                    for (int k = tid; k < c; k += blockDim.x) {  // kmeans.cpp:12-19
                        const T* x = M + (int64_t)jj * d;
                        const double* ck = a.Cs + (int64_t)k * d;
                        double s = 0.0;
                        for (int64_t i = 0; i < d; ++i) {
                            const double t = (double)x[i] - ck[i];
                            s += t * t;
                        }
                        dist[k] = s;
                    }
                    __syncthreads();
                    if (warp == 0) {
                        double lo[KPL], hi[KPL], mid[KPL];
#pragma unroll
                        for (int q = 0; q < KPL; ++q) {
                            const int k = lane + 32 * q;
                            lo[q] = hi[q] = mid[q] = k < c ? dist[k] : INFINITY;
                        }
                        int t2 = -1;
                        const int s2 = gram_decide<KPL>(mfrom, c, cf, cnt, lo, hi, mid, t2);
                        if (lane == 0) s_xres = s2 == 1 ? (1 | (t2 << 2)) : 0;  // exact: 2 only for NaN
                    }
                }
                replay_work += (unsigned long long)(nlog - replayed);
                replayed = nlog;
                gcl_sync();
                const int xr = gcl_ld_i32(gcl_map(&s_xres, 0));
                mst = xr & 3;
                mto = xr >> 2;
                // the move's inputs live in the column owner's cache
                const int orank = (jj >> 3) & (CL - 1);
                if (mst == 1 && rank == orank && tid == 0) {
                    const int jm2 = jj >> LW, slot = jm2 % NSL, col = jj - (jj / GW) * GW;
                    const double* svp = &scache[(size_t)(slot * GW + col) * CS];
                    s_xsv[0] = svp[mfrom];
                    s_xsv[1] = svp[mto];
                    s_xsv[2] = cxx[slot][col];
                    s_xsv[3] = cxn[slot][col];
                    s_xsv[4] = cxl[slot][col];
                }
                gcl_sync();
                if (mst == 1)
#pragma unroll
                    for (int q = 0; q < MVW; ++q) mvin[q] = gcl_ld_f64(gcl_map(&s_xsv[q], (uint32_t)orank));
                gcl_sync();  // s_xsv / s_xres read before a later fallback rewrites them
                lap(1);
            }
            if (mst == 1) {
                // the last warp: the log (the counts before the move), then the replicas'
                // per-centroid state — two lanes, identical inputs in every CTA → identical
                // replicas — while the other warps go on to the next window's far loads and
                // cache patch; nothing reads cf / cnt before the next window's first barrier
                if (warp == GRAM_WARPS - 1) {
                    if (lane == 0 && rank == 0) {
                        int* lg = a.log + 5 * (int64_t)(nlog + (pj >= 0 ? 1 : 0));
                        lg[0] = jj;
                        lg[1] = mfrom;
                        lg[2] = mto;
                        lg[3] = cnt[mfrom];
                        lg[4] = cnt[mto];
                    }
                    __syncwarp();
                    if (lane < 2) {
                        const int kk = lane ? mto : mfrom;
                        gram_side(lane, sc[kk], cf[kk], cnt[kk], lane ? mvin[1] : mvin[0], mvin[2], mvin[3], mvin[4], gamG);
                    }
                }
                if (tid == 0 && rank == ((jj >> 3) & (CL - 1))) __stcg(a.labels + jj, mto);
#pragma unroll
                for (int q = 0; q < MVW; ++q) pmv[q] = mvin[q];
                lap(7);
                pj = jj;
                pf = mfrom;
                pt = mto;
                ++moves;
                improved = 1;
            }
            par ^= 1;
        }
        ++pass;
        if (!improved || pass >= a.max_pass) break;
    }
    // the last move's label and counts were taken when it was elected (its Ŝ
    // update is no longer needed)
    if (loading) finish_load();
    __syncthreads();
    if (rank == 0) {
        for (int k = tid; k < c; k += blockDim.x) a.counts[k] = cnt[k];
        if (tid == 0) {
            a.stats[0] = moves;
            a.stats[1] = (unsigned long long)pass;
            a.stats[2] = windows;
            a.stats[3] = fallbacks;
            a.stats[4] = replay_work;
            for (int q = 0; q < 8; ++q) a.stats[5 + q] = tph[q];
        }
    }
    gcl_sync();  // no CTA leaves while another may still read its shared memory
}

}  // namespace respca_dev
