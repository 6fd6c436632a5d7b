// Exact sequential Hartigan refinement (kmeans.cpp:96-139) on the device.
//
// The reference visits columns j = 0..n−1 in order, pass after pass (≤ 50),
// and applies each improving single-point move at once (incremental centroid
// update, kmeans.cpp:122-135), so every later decision sees the updated
// centroids and counts.  The device keeps exactly that order with ONE
// persistent cooperative kernel for the whole refinement (all passes):
//
//  * every CTA owns `cpb` columns of the current block of B = G·cpb columns,
//    cached in shared memory with their interval rows [a − e, a + e] (a
//    screened sq_dist that provably contains the reference's value, km.cuh);
//  * interval rows live in HBM between visits with a per-entry stamp: entry
//    (j, k) is valid while centroid k has not moved since it was computed.  On
//    entering a block a CTA recomputes only its stale entries (lazy refresh:
//    late passes, with few moves, refresh almost nothing);
//  * a round: (1a) every CTA writes one row slice of the previous move's two
//    updated centroids (the reference's exact formula, into the other slot of
//    a double-buffered store) plus the slice's ‖c′‖² partial; grid barrier;
//    (1b) the owned columns still to visit refresh their two stale entries;
//    (2) one warp per owned column decides it on the intervals and the
//    smallest column that is not provably "no move" is elected (atomicMin);
//    grid barrier; (3) every CTA settles the elected column identically — a
//    provable move is applied to the replicated counts, an undecidable
//    near-tie is resolved with the reference's own sequential chain.
//
// Labels, counts and centroids are therefore bit-identical to the reference.
#pragma once

#include "km.cuh"
#include "tc_screen.cuh"

namespace respca_dev {

RESPCA_DEV unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Hartigan decision of one column on intervals (one warp), with the weights
// wa[k] = n_k/(n_k−1), wb[k] = n_k/(n_k+1) (the reference's correctly-rounded
// divisions, kmeans.cpp:107, 114):
//   0 = provably no move, 1 = provably moves to `to`, 2 = undecidable
template <typename IV>
RESPCA_DEV int hart_decide_warp_w(int from, int c, const int* cnt, const double* wa,
                                  const double* wb, const IV& iv, int& to) {
    const int lane = threadIdx.x & 31;
    if (cnt[from] <= 1) return 0;  // kmeans.cpp:105
    double flo, fhi, fmid;
    iv(from, flo, fhi, fmid);
    const double w_a = wa[from];
    const double g_lo = w_a * flo, g_hi = w_a * fhi, g_mid = w_a * fmid;
    double bd = INFINITY;
    int bk = 0x7fffffff;
    bool none = true;
    for (int k = lane; k < c; k += 32) {
        if (k == from) continue;
        double lo, hi, mid;
        iv(k, lo, hi, mid);
        const double w_b = wb[k];
        none &= !(w_b * lo - g_hi < -1e-12);  // kmeans.cpp:116, best_delta = -1e-12
        const double dmid = w_b * mid - g_mid;
        if (dmid < bd) {
            bd = dmid;
            bk = k;
        }
    }
    none = __all_sync(0xffffffffu, none);
    if (none) return 0;
    warp_argmin(bd, bk);
    if (bk >= c) return 2;
    double blo, bhi, bmid;
    iv(bk, blo, bhi, bmid);
    const double dhi_k = wb[bk] * bhi - g_lo;
    bool ok = dhi_k < -1e-12;
    for (int k = lane; k < c; k += 32) {
        if (k == from || k == bk) continue;
        double lo, hi, mid;
        iv(k, lo, hi, mid);
        const double dlo = wb[k] * lo - g_hi;
        if (k < bk) ok &= dhi_k < dlo;  // an earlier k must lose strictly
        else ok &= dhi_k <= dlo;        // a later k never replaces an equal delta
    }
    ok = __all_sync(0xffffffffu, ok);
    if (!ok) return 2;
    to = bk;
    return 1;
}

// Hartigan intervals [mid − e, mid + e] contain BOTH the reference's computed
// sq_dist (sequential chain) and the real ‖x − c‖² to the stored centroid:
// |ref − real| ≤ γ·real for a chain of d positive rounded squares, γ = (d+3)u·1.02.
// The real value is what the exact move identities below transform.
RESPCA_DEV double hart_widen(double mid, double e, double gam) {
    return __dadd_ru(e, __dmul_ru(gam, __dadd_ru(fabs(mid), e)));
}

// intervals of every (column, centroid) pair from a full screen (start state)
__global__ void k_hart_fill(Screen sc, double* __restrict__ A, double* __restrict__ E,
                            double* __restrict__ xx, int n, int c, double gam) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)n * c) return;
    const int j = (int)(e / c), k = (int)(e % c);
    const double xxj = sc.xx(j);
    double lo, hi, mid;
    sc.get(j, k, xxj, sqrt(fabs(xxj)), lo, hi, mid);
    A[e] = mid;
    E[e] = isfinite(hi - mid) ? hart_widen(mid, hi - mid, gam) : INFINITY;
    if (k == 0) xx[j] = xxj;
}

// copy centroids living in slot 1 back to slot 0, reset the slot map
__global__ void k_hart_consolidate(double* __restrict__ Cs, const int* __restrict__ ver, int64_t d,
                                   int c) {
    for (int k = blockIdx.y; k < c; k += gridDim.y) {
        if (ver[k] == 0) continue;
        const double* src = Cs + ((int64_t)c + k) * d;
        double* dst = Cs + (int64_t)k * d;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d;
             i += (int64_t)gridDim.x * blockDim.x)
            dst[i] = src[i];
    }
}

struct HartGlobal {
    // each hot word on its own 128-byte line: the barrier spin, the barrier
    // arrivals and the per-round election slots must not share L2 lines
    alignas(128) unsigned bar_count;
    alignas(128) unsigned bar_gen;
    alignas(128) unsigned long long first[3][16];  // per-round election slots, round r uses r % 3
    alignas(128) unsigned long long xres;          // exact-fallback verdict broadcast
    alignas(128) unsigned long long moves, exact_fallbacks, rounds, passes, blocks, refreshed;
    unsigned long long t_kernel, t_load, t_cols;  // globaltimer (CTA 0): whole kernel, block loads, column fills
    unsigned long long stale_sum, heavy_blocks;   // CTA 0: stale centroids over all block entries, entries with > 8
    unsigned long long tsub1, tsub2, redos, act_cycles, act_rounds, dq_cycles;
    unsigned long long hist[9];  // diagnostics: no-move margins below 1e-1..1e-8, total
    unsigned long long tm[8];  // CTA 0 phase sums: 1, entry tiles, entry barrier, entry reduce, decide, barrier, settle
};

RESPCA_DEV void grid_barrier(HartGlobal* g) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = &g->bar_gen;
        const unsigned my = *gen;
        __threadfence();
        if (atomicAdd(&g->bar_count, 1u) == gridDim.x - 1) {
            g->bar_count = 0;
            __threadfence();
            atomicAdd(&g->bar_gen, 1u);
        } else {
            while (*gen == my) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

// (j, status, from, to) → 64 bits, ordered by j first
RESPCA_DEV unsigned long long pack4(int j, int st, int from, int to) {
    return ((unsigned long long)(unsigned)j << 32) | ((unsigned long long)(st & 3) << 30) |
           ((unsigned long long)(from & 0x7fff) << 15) | (unsigned long long)(to & 0x7fff);
}

__global__ void k_hart_first_reset(HartGlobal* g) {
    g->first[0][0] = g->first[1][0] = g->first[2][0] = ~0ULL;
}

// bulk global→shared copy (async proxy), completion counted on `bar`
RESPCA_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
RESPCA_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
RESPCA_DEV void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}

struct HartArgs {
    HartGlobal* g;
    int* labels;          // [n]   (device copy, written by CTA 0)
    int* counts;          // [c]   in: start counts, out: final counts
    double* Cs;           // [2][c][d] centroid slots; slot 0 holds the start centroids
    int* ver;             // [c]   out: slot of each final centroid
    double* A;            // [n][c] interval mid-points
    double* E;            // [n][c] interval half-widths
    int* ebuf;            // [blocks] move count at the last entry of each block (0)
    double* part;         // [G][B][c] row-slice partial dots of the block refresh
    const double* xx;     // [n]   ‖x_j‖² (screen)
    const double* cc0;    // [c]   ‖c_k‖² of the start centroids (screen)
    double* scratch;      // [c]   exact distances of one column (near-tie)
    double* cand;         // [n][4] a candidate column's (mid, e) to its from / to centroid
    double* ccp;          // [c][G] row-slice partials of ‖c‖² (block refresh)
    int64_t d;
    int n, c, cpb, cache_cols, max_pass, stage_rows, stages, diag;
    double kappa_d;       // screen bound factor (km.cuh) + the reciprocal-update term
    double gam;           // (d+3)u·1.02: reference chain vs real distance (hart_widen)
};

constexpr int HART_RED = 32 * 24;  // block_sum scratch (≤ 24 sums)
constexpr int HART_MAXG = 160;     // max CTAs of the Hartigan kernel (partials per entry)

RESPCA_DEV void cp_wait_dyn(int pending) {
    switch (pending) {
        case 0: cp_wait<0>(); break;
        case 1: cp_wait<1>(); break;
        case 2: cp_wait<2>(); break;
        default: cp_wait<3>(); break;
    }
}

// Block refresh partials of one CTA on the FP64 tensor cores (DMMA m8n8k4):
// its row slice [s0, s1) of x_jb · c_stale[t] for every block column jb < nb
// and stale centroid t.  Operands are staged i-contiguous ([col][row], row
// stride R + 4: conflict-free fragment loads, as in km.cuh), in chunks of R
// rows (a power of two ≥ 8) through a.stages cp.async stages, zero-padded to
// whole 16×16 warp tiles (2×2 DMMA tiles: each fragment feeds two MMAs).
// A warp owns up to TPW warp tiles per round.  Output: part[(jb·c + t)·G + CTA].
template <typename T, int TPW>
RESPCA_DEV void hart_entry_dmma(const T* __restrict__ M, const HartArgs& a, const int* vs,
                                const int* stale, int nstale, int b0, int nb, int64_t s0, int64_t s1,
                                int R, T* stc, double* sce, unsigned long long* tacc, double* ccacc) {
    const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, lane = tid & 31;
    const int nwarps = nt >> 5;
    const int c = a.c, G = gridDim.x, NS = a.stages;
    const int64_t d = a.d;
    const double* __restrict__ Cs = a.Cs;
    const int MP = (nb + 15) & ~15, NP = (nstale + 15) & ~15, RS = R + 4;
    const int wtn = NP >> 4, nwt = (MP >> 4) * wtn;  // 16×16 warp tiles
    const int lgR = 31 - __clz(R);
    const size_t sstc = (size_t)MP * RS, ssce = (size_t)NP * RS;
    const int nch = s1 > s0 ? (int)((s1 - s0 + R - 1) / R) : 0;
    const int g = lane >> 2, t4 = lane & 3;
    unsigned long long tq0 = tid == 0 ? (unsigned long long)clock64() : 0;
    auto lapt = [&](int slot) {
        if (tid == 0) {
            const unsigned long long t = (unsigned long long)clock64();
            tacc[slot] += t - tq0;
            tq0 = t;
        }
    };
    auto issue = [&](int ch) {
        const int64_t c0 = s0 + (int64_t)ch * R;
        const int rows = (int)(s1 - c0 < R ? s1 - c0 : R);
        T* sb = stc + (size_t)(ch % NS) * sstc;
        double* cb = sce + (size_t)(ch % NS) * ssce;
        for (int e = tid; e < (MP << lgR); e += nt) {
            const int jb = e >> lgR, rr = e & (R - 1);
            const bool ok = jb < nb && rr < rows;
            const T* src = M + (int64_t)(b0 + (ok ? jb : 0)) * d + c0 + (ok ? rr : 0);
            if (sizeof(T) == 8) cp_async8(sb + jb * RS + rr, src, ok);
            else cp_async4(sb + jb * RS + rr, src, ok);
        }
        for (int e = tid; e < (NP << lgR); e += nt) {
            const int t = e >> lgR, rr = e & (R - 1);
            const bool ok = t < nstale && rr < rows;
            const int k = stale[t < nstale ? t : 0];
            cp_async8(cb + t * RS + rr, Cs + ((int64_t)vs[k] * c + k) * d + c0 + (ok ? rr : 0), ok);
        }
        cp_commit();
    };
    for (int tr0 = 0; tr0 < nwt; tr0 += nwarps * TPW) {
        double acc[TPW][2][2][2];  // [warp tile][m half][n half][fragment]
        int wm[TPW], wn[TPW];
#pragma unroll
        for (int i = 0; i < TPW; ++i) {
            const int wt = tr0 + warp + i * nwarps;
            wm[i] = wt < nwt ? wt / wtn : -1;
            wn[i] = wt < nwt ? wt - (wt / wtn) * wtn : 0;
#pragma unroll
            for (int x = 0; x < 2; ++x)
#pragma unroll
                for (int y = 0; y < 2; ++y) acc[i][x][y][0] = acc[i][x][y][1] = 0.0;
        }
        const bool norms = tr0 == 0;  // ‖c‖² slice partials, once
        if (norms)
            for (int t = tid; t < nstale; t += nt) ccacc[t] = 0.0;
        __syncthreads();  // stage buffers free
        int issued = 0;
        for (; issued < nch && issued < NS - 1; ++issued) issue(issued);
        for (int ch = 0; ch < nch; ++ch) {
            lapt(2);
            if (issued < nch) issue(issued++);  // refills the stage chunk ch−1 used
            lapt(0);
            cp_wait_dyn(issued - ch - 1);
            __syncthreads();
            lapt(1);
            const T* sb = stc + (size_t)(ch % NS) * sstc;
            const double* cb = sce + (size_t)(ch % NS) * ssce;
            if (norms) {  // thread per stale centroid, on the warps without tiles if any
                const int w0 = nwt < nwarps ? nwt : 0, nw0 = nwarps - w0;
                if (warp >= w0)
                    for (int t = (warp - w0) * 32 + lane; t < nstale; t += nw0 * 32) {
                        double v = ccacc[t];
                        for (int rr = 0; rr < R; ++rr) v = __fma_rn(cb[t * RS + rr], cb[t * RS + rr], v);
                        ccacc[t] = v;
                    }
            }
#pragma unroll
            for (int i = 0; i < TPW; ++i) {
                if (wm[i] < 0) continue;
                const T* ap = sb + (wm[i] * 16 + g) * RS + t4;
                const double* bp = cb + (wn[i] * 16 + g) * RS + t4;
                for (int k0 = 0; k0 < R; k0 += 4) {
                    const double a0 = (double)ap[k0], a1 = (double)ap[8 * RS + k0];
                    const double bv0 = bp[k0], bv1 = bp[8 * RS + k0];
                    dmma884(acc[i][0][0][0], acc[i][0][0][1], a0, bv0);
                    dmma884(acc[i][0][1][0], acc[i][0][1][1], a0, bv1);
                    dmma884(acc[i][1][0][0], acc[i][1][0][1], a1, bv0);
                    dmma884(acc[i][1][1][0], acc[i][1][1][1], a1, bv1);
                }
            }
            __syncthreads();  // chunk consumed before its stage is refilled
        }
#pragma unroll
        for (int i = 0; i < TPW; ++i)
            if (wm[i] >= 0)
#pragma unroll
                for (int x = 0; x < 2; ++x) {
                    const int jb = wm[i] * 16 + x * 8 + g;
#pragma unroll
                    for (int y = 0; y < 2; ++y)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int t = wn[i] * 16 + y * 8 + 2 * t4 + h;
                            if (jb < nb && t < nstale)
                                __stcg(a.part + ((size_t)jb * c + t) * G + blockIdx.x, acc[i][x][y][h]);
                        }
                }
    }
    __syncthreads();
    for (int t = tid; t < nstale; t += nt) __stcg(a.ccp + (size_t)t * G + blockIdx.x, ccacc[t]);
}

template <typename T, int MAXQ>
__global__ void __launch_bounds__(512, 1) k_hart_all(const T* __restrict__ M, HartArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int64_t d = a.d;
    const int c = a.c, n = a.n, cpb = a.cpb, cache_cols = a.cache_cols;
    HartGlobal* hg = a.g;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nwarps = blockDim.x >> 5;
    const int G = gridDim.x, B = G * cpb, R = a.stage_rows;
    // ---- shared memory carve-up
    T* colc = reinterpret_cast<T*>(sm);
    size_t off = cache_cols ? (size_t)cpb * d * sizeof(T) : 0;
    off = (off + 15) & ~(size_t)15;
    double* As = reinterpret_cast<double*>(sm + off);
    off += sizeof(double) * cpb * c;
    double* Es = reinterpret_cast<double*>(sm + off);
    off += sizeof(double) * cpb * c;
    double* wa = reinterpret_cast<double*>(sm + off);
    off += sizeof(double) * c;
    double* wb = reinterpret_cast<double*>(sm + off);
    off += sizeof(double) * c;
    double* ccs = reinterpret_cast<double*>(sm + off);
    off += sizeof(double) * c;
    double* red = reinterpret_cast<double*>(sm + off);
    off += sizeof(double) * HART_RED;
    T* stc = reinterpret_cast<T*>(sm + off);  // [stages][B↑16][R+4] block-column row chunks
    off += (size_t)a.stages * sizeof(double) * (size_t)(R + 4) * ((B + 15) & ~15);
    double* sce = reinterpret_cast<double*>(sm + off);  // [stages][c↑16][R+4] stale-centroid row chunks
    off += (size_t)a.stages * sizeof(double) * (size_t)(R + 4) * ((c + 15) & ~15);
    double* ccacc = reinterpret_cast<double*>(sm + off);  // [c] ‖c‖² slice partials
    off += sizeof(double) * c;
    int* stale = reinterpret_cast<int*>(sm + off);
    off += sizeof(int) * c;
    int* cnt = reinterpret_cast<int*>(sm + off);
    off += sizeof(int) * c;
    int* vs = reinterpret_cast<int*>(sm + off);
    off += sizeof(int) * c;
    int* mv = reinterpret_cast<int*>(sm + off);
    __shared__ double s_xx[MAXQ];
    __shared__ int s_lab[MAXQ];
    __shared__ int s_nstale;
    __shared__ __align__(8) uint64_t s_bar;  // column fills (bulk copies)


    const uint32_t col_bytes = (uint32_t)(d * (int64_t)sizeof(T));
    const bool bulk = cache_cols && (col_bytes % 16 == 0) && ((uintptr_t)M % 16 == 0);
    uint32_t bar_phase = 0;
    if (tid == 0) {
        mbar_init(&s_bar, 1);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    }
    // ---- replicated sequential state
    for (int k = tid; k < c; k += blockDim.x) {
        const int ck = __ldcg(a.counts + k);
        cnt[k] = ck;
        const double nk = (double)ck;
        wa[k] = nk / (nk - 1.0);  // kmeans.cpp:107
        wb[k] = nk / (nk + 1.0);  // kmeans.cpp:114
        vs[k] = 0;
        mv[k] = 0;
        ccs[k] = __ldcg(a.cc0 + k);
    }
    __syncthreads();
    auto colv = [&](int jo, int q, int64_t i) -> double {
        return cache_cols ? (double)colc[(int64_t)q * d + i] : (double)__ldg(M + (int64_t)(jo + q) * d + i);
    };

    int pass = 0, improved = 0;
    int b0 = -1, bend = 0, cursor = 0, jown = 0, nown = 0;
    int pf = -1, pt = -1, pm = -1, pnf = 0, pnt = 0;
    int mvcount = 0;  // move counter (thread 0 stamps the replicated versions)
    // this CTA's row slice: it alone stores those rows of every updated centroid
    const int64_t slice = (d + G - 1) / G;
    const int64_t s0 = (int64_t)blockIdx.x * slice < d ? (int64_t)blockIdx.x * slice : d;
    const int64_t s1 = s0 + slice < d ? s0 + slice : d;
    unsigned long long rounds = 0, blocks = 0, refreshed = 0, t_load = 0, t_cols = 0;
    unsigned long long stale_sum = 0, heavy = 0, redos = 0, act_cycles = 0, act_rounds = 0, dq_cycles = 0;
    unsigned long long tm[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    unsigned long long tsub[3] = {0, 0, 0};  // entry tiles: issue, wait, compute+sync
    unsigned long long tmark = (unsigned long long)clock64();  // SM cycles
    auto lap = [&](int slot) {
        if (tid == 0) {
            const unsigned long long t = (unsigned long long)clock64();
            tm[slot] += t - tmark;
            tmark = t;
        }
    };
    const unsigned long long tk0 = gtimer();

    for (int r = 0;; ++r) {
        lap(7);
        // ---- phase 1: the pending move (kmeans.cpp:126-131).
        //  (a) this CTA's row slice of both updated centroids, with the
        //      reference's exact formula, to the other slot (other CTAs read a
        //      slot's slices only after the next grid barrier);
        //  (b) the owned columns still to visit get their from/to intervals by
        //      the exact move identities (real distances; e = exact update)
        //        ‖x−e_f‖² = (n·D_xf − D_xm)/(n−1) + n·D_fm/(n−1)²
        //        ‖x−e_t‖² = (n·D_xt + D_xm)/(n+1) − n·D_tm/(n+1)²
        //      evaluated in directed rounding from the old intervals, the
        //      moved column's own (broadcast by its owner) and D_xm = ‖x − x_m‖²
        //      (one pass over x_m), plus the stored-vs-exact centroid rounding
        //      and the chain-vs-real slack; when that interval has grown too
        //      wide the CTA recomputes its entries from the new centroid values.
        if (pf >= 0) {
            const double* of = a.Cs + ((int64_t)vs[pf] * c + pf) * d;
            const double* ot = a.Cs + ((int64_t)vs[pt] * c + pt) * d;
            double* nfp = a.Cs + ((int64_t)(1 - vs[pf]) * c + pf) * d;
            double* ntp = a.Cs + ((int64_t)(1 - vs[pt]) * c + pt) * d;
            const T* xm = M + (int64_t)pm * d;
            const double dcf = (double)pnf, dct = (double)pnt;
            const double na1 = (double)(pnf - 1), nb1 = (double)(pnt + 1);
            for (int64_t i = s0 + tid; i < s1; i += blockDim.x) {
                const double x = (double)__ldg(xm + i);
                __stcg(nfp + i, (__ldcg(of + i) * dcf - x) / na1);  // kmeans.cpp:128-129 operation order
                __stcg(ntp + i, (__ldcg(ot + i) * dct + x) / nb1);
            }
            int nact = 0;
            for (int q = 0; q < nown; ++q) nact += (jown + q >= cursor);
            const int q0 = nown - nact;  // active owned columns: the suffix q0..nown-1
            const double mf = __ldcg(a.cand + 4 * (int64_t)pm), ef = __ldcg(a.cand + 4 * (int64_t)pm + 1);
            const double mt = __ldcg(a.cand + 4 * (int64_t)pm + 2), et = __ldcg(a.cand + 4 * (int64_t)pm + 3);
            const double xxm = __ldcg(a.xx + pm);
            bool redo = false;
            double nmid = 0.0, ne = INFINITY;
            const unsigned long long ta0 = clock64();
            if (nact) {  // block-uniform
                double dq[MAXQ];
#pragma unroll
                for (int q = 0; q < MAXQ; ++q) dq[q] = 0.0;
                auto rowq = [&](int64_t i, double x) {
#pragma unroll
                    for (int q = 0; q < MAXQ; ++q)
                        if (q < nact) {
                            const double t = colv(jown, q0 + q, i) - x;
                            dq[q] = __fma_rn(t, t, dq[q]);
                        }
                };
                const int64_t step = blockDim.x;
                if (sizeof(T) == 8 && (d & 1) == 0) {
                    const double2* x2 = reinterpret_cast<const double2*>(xm);
                    const int64_t dh = d >> 1;
                    int64_t i = tid;
                    for (; i + 7 * step < dh; i += 8 * step) {
                        double2 xv[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) xv[u] = __ldg(x2 + i + u * step);
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            rowq(2 * (i + u * step), xv[u].x);
                            rowq(2 * (i + u * step) + 1, xv[u].y);
                        }
                    }
                    if (i + 3 * step < dh) {
                        double2 xv[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) xv[u] = __ldg(x2 + i + u * step);
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            rowq(2 * (i + u * step), xv[u].x);
                            rowq(2 * (i + u * step) + 1, xv[u].y);
                        }
                        i += 4 * step;
                    }
                    for (; i < dh; i += step) {
                        const double2 xv = __ldg(x2 + i);
                        rowq(2 * i, xv.x);
                        rowq(2 * i + 1, xv.y);
                    }
                } else {
                    for (int64_t i = tid; i < d; i += step) rowq(i, (double)__ldg(xm + i));
                }
                block_sum<MAXQ>(dq, red);
                if (tid == 0) dq_cycles += clock64() - ta0;
                bool wide = false;
                if (tid < 2 * nact) {
                    const int qa = tid >> 1, which = tid & 1, q = q0 + qa;
                    const int k = which ? pt : pf;
                    double dqm = 0.0;
#pragma unroll
                    for (int e = 0; e < MAXQ; ++e)
                        if (e == qa) dqm = dq[e];
                    // D_xm interval (positive-term chain): [dqm(1−γ), dqm(1+2γ)]
                    const double dlo = dqm * (1.0 - 1.01 * a.gam), dhi = dqm * (1.0 + 2.02 * a.gam);
                    const double om = As[q * c + k], oe = Es[q * c + k];
                    const double lo = fmax(om - oe, 0.0), hi = om + oe;
                    // identities in round-to-nearest with reciprocal multiplies;
                    // every term is ≥ 0, so 16u of their magnitude sum covers the
                    // roundings (≤ 8 operations per chain)
                    double flo, fhi, nn, dn;
                    if (!which) {  // from: n = pnf, n−1 = na1
                        nn = dcf;
                        dn = na1;
                        const double r1 = 1.0 / dn, r2 = r1 * r1;
                        const double m1 = fmax(mf - ef, 0.0), m2 = mf + ef;
                        flo = (nn * lo - dhi) * r1 + nn * m1 * r2;
                        fhi = (nn * hi - dlo) * r1 + nn * m2 * r2;
                        const double sl = 16.0 * kU * ((nn * hi + dhi) * r1 + nn * m2 * r2);
                        flo -= sl;
                        fhi += sl;
                    } else {  // to: n = pnt, n+1 = nb1
                        nn = dct;
                        dn = nb1;
                        const double r1 = 1.0 / dn, r2 = r1 * r1;
                        const double m1 = fmax(mt - et, 0.0), m2 = mt + et;
                        flo = (nn * lo + dlo) * r1 - nn * m2 * r2;
                        fhi = (nn * hi + dhi) * r1 - nn * m1 * r2;
                        const double sl = 16.0 * kU * ((nn * hi + dhi) * r1 + nn * m2 * r2);
                        flo -= sl;
                        fhi += sl;
                    }
                    flo = fmax(flo, 0.0);
                    // stored centroid vs the exact update: |δ_i| ≤ 3u(n|c_i| + |x_i|)/dn
                    const double del = 3.03 * kU * (nn * sqrt(fabs(ccs[k])) + sqrt(fabs(xxm))) / dn;
                    const double sh = sqrt(fmax(fhi, 0.0));
                    const double rlo = fmax(flo - 2.0 * sh * del * 1.01, 0.0);
                    const double rhi = fhi + (2.0 * sh * del + del * del) * 1.01;
                    // union with the reference's chain value
                    const double ulo = rlo * (1.0 - 1.01 * a.gam), uhi = rhi * (1.0 + 1.01 * a.gam);
                    nmid = 0.5 * (ulo + uhi);
                    ne = (0.5 * (uhi - ulo)) * (1.0 + 8.0 * kU) + 4.0 * kU * uhi;
                    const double fresh = screen_err(a.kappa_d, sqrt(fabs(s_xx[q])), sqrt(fabs(ccs[k])), nmid);
                    wide = !(isfinite(nmid) && isfinite(ne) && ne <= 64.0 * fresh);
                }
                redo = __syncthreads_or(wide) != 0;
                if (tid == 0) {
                    act_cycles += clock64() - ta0;
                    ++act_rounds;
                }
            }
            if (!redo) {
                if (tid < 2 * nact) {
                    const int qa = tid >> 1, which = tid & 1, q = q0 + qa;
                    const int k = which ? pt : pf;
                    As[q * c + k] = nmid;
                    Es[q * c + k] = ne;
                }
            } else {
                // recompute from the new values over all rows (reciprocal multiply
                // inside the bound, kappa_d)
                const double rf = 1.0 / na1, rt = 1.0 / nb1;
                double acc[2 + 2 * MAXQ];
#pragma unroll
                for (int e = 0; e < 2 + 2 * MAXQ; ++e) acc[e] = 0.0;
                for (int64_t i = tid; i < d; i += blockDim.x) {
                    const double x = (double)__ldg(xm + i);
                    const double cf = (__ldcg(of + i) * dcf - x) * rf, ct = (__ldcg(ot + i) * dct + x) * rt;
                    acc[0] = __fma_rn(cf, cf, acc[0]);
                    acc[1] = __fma_rn(ct, ct, acc[1]);
#pragma unroll
                    for (int q = 0; q < MAXQ; ++q)
                        if (q < nact) {
                            const double xq = colv(jown, q0 + q, i);
                            acc[2 + 2 * q] = __fma_rn(xq, cf, acc[2 + 2 * q]);
                            acc[3 + 2 * q] = __fma_rn(xq, ct, acc[3 + 2 * q]);
                        }
                }
                block_sum<2 + 2 * MAXQ>(acc, red);
                if (tid < 2 * nact) {
                    const int qa = tid >> 1, which = tid & 1, q = q0 + qa;
                    double dot = 0.0;
#pragma unroll
                    for (int e = 0; e < 2 * MAXQ; ++e)
                        if (e == tid) dot = acc[2 + e];
                    const double cck = which ? acc[1] : acc[0];
                    const double xxj = s_xx[q];
                    const double mid = (xxj + cck) - 2.0 * dot;
                    const double e = screen_err(a.kappa_d, sqrt(fabs(xxj)), sqrt(fabs(cck)), mid);
                    const int k = which ? pt : pf;
                    As[q * c + k] = mid;
                    Es[q * c + k] = isfinite(mid) && isfinite(e) ? hart_widen(mid, e, a.gam) : INFINITY;
                }
                if (tid == 0) ++redos;
            }
            __syncthreads();
            if (tid == 0) {
                // ‖c′‖² by the same identities (only the bound's scale uses it
                // between block entries, which recompute it from the slices)
                ccs[pf] = fmax((dcf * ccs[pf] - xxm) / na1 + dcf * mf / (na1 * na1), 0.0);
                ccs[pt] = fmax((dct * ccs[pt] + xxm) / nb1 - dct * mt / (nb1 * nb1), 0.0);
                vs[pf] ^= 1;  // this CTA's slices of the new values are stored
                vs[pt] ^= 1;
            }
            __syncthreads();
            pf = -1;
        }
        lap(0);

        if (cursor >= bend) {
            // ---- leave the block: its interval rows go back to HBM
            for (int e = tid; e < nown * c; e += blockDim.x) {
                const int64_t idx = (int64_t)jown * c + e;
                __stcg(a.A + idx, As[e]);
                __stcg(a.E + idx, Es[e]);
            }
            int nb0 = b0 < 0 ? 0 : bend;
            if (nb0 >= n) {  // end of a pass (kmeans.cpp:137)
                ++pass;
                if (!improved || pass >= a.max_pass) break;
                improved = 0;
                nb0 = 0;
            }
            const unsigned long long tl0 = gtimer();
            b0 = nb0;
            bend = b0 + B < n ? b0 + B : n;
            const int nb = bend - b0, blk = b0 / B;
            cursor = b0;
            jown = b0 + blockIdx.x * cpb;
            nown = bend - jown;
            nown = nown < 0 ? 0 : (nown > cpb ? cpb : nown);
            ++blocks;
            __syncthreads();
            // ---- enter the block: owned columns (bulk copies when aligned),
            //      interval rows, labels; the next block's columns go to L2
            if (bulk) {
                if (tid == 0 && nown > 0) {
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    mbar_expect_tx(&s_bar, col_bytes * (uint32_t)nown);
                    for (int q = 0; q < nown; ++q) {
                        const unsigned char* src = reinterpret_cast<const unsigned char*>(M + (int64_t)(jown + q) * d);
                        unsigned char* dst = reinterpret_cast<unsigned char*>(colc + (int64_t)q * d);
                        for (uint32_t o = 0; o < col_bytes; o += 65536u) {
                            const uint32_t len = col_bytes - o < 65536u ? col_bytes - o : 65536u;
                            bulk_g2s(dst + o, src + o, len, &s_bar);
                        }
                    }
                }
                if (tid == 32) {
                    const int nj = (bend < n ? bend : 0) + blockIdx.x * cpb;
                    for (int q = 0; q < cpb && nj + q < n; ++q) {
                        const unsigned char* src = reinterpret_cast<const unsigned char*>(M + (int64_t)(nj + q) * d);
                        for (uint32_t o = 0; o < col_bytes; o += 65536u)
                            bulk_prefetch_l2(src + o, col_bytes - o < 65536u ? col_bytes - o : 65536u);
                    }
                }
            } else if (cache_cols) {
                for (int q = 0; q < nown; ++q)
                    for (int64_t i = tid; i < d; i += blockDim.x)
                        colc[(int64_t)q * d + i] = __ldg(M + (int64_t)(jown + q) * d + i);
            }
            for (int e = tid; e < nown * c; e += blockDim.x) {
                const int64_t idx = (int64_t)jown * c + e;
                As[e] = __ldcg(a.A + idx);
                Es[e] = __ldcg(a.E + idx);
            }
            if (tid < nown) {
                s_xx[tid] = __ldcg(a.xx + jown + tid);
                s_lab[tid] = __ldcg(a.labels + jown + tid);
            }
            // centroids moved since this block's last entry (every column's
            // entries are valid as of then), ascending
            const int eb = __ldcg(a.ebuf + blk);
            if (warp == 0) {
                int cv = 0;
                for (int k0 = 0; k0 < c; k0 += 32) {
                    const int k = k0 + lane;
                    const bool sk = k < c && mv[k] > eb;
                    const unsigned bal = __ballot_sync(0xffffffffu, sk);
                    if (sk) stale[cv + __popc(bal & ((1u << lane) - 1u))] = k;
                    cv += __popc(bal);
                }
                if (lane == 0) s_nstale = cv;
            }
            __syncthreads();
            const int nstale = s_nstale;
            if (tid == 0) {
                stale_sum += nstale;
                heavy += nstale > 8;
            }
            if (nstale > 0) {
                // ---- block refresh, split over rows: this CTA's row slice of
                //      (every block column) · (every stale centroid) → HBM
                //      partials; then each owned column sums its G partials
                {
                    const int nwt = ((nb + 15) >> 4) * ((nstale + 15) >> 4), nw = (int)(blockDim.x >> 5);
                    if (nwt <= nw)
                        hart_entry_dmma<T, 1>(M, a, vs, stale, nstale, b0, nb, s0, s1, R, stc, sce, tsub, ccacc);
                    else
                        hart_entry_dmma<T, 2>(M, a, vs, stale, nstale, b0, nb, s0, s1, R, stc, sce, tsub, ccacc);
                }
                lap(1);
                grid_barrier(hg);
                lap(2);
                // ---- ‖c‖² of the stale centroids (slice partials, fixed order)
                for (int t = warp; t < nstale; t += nwarps) {
                    double v = 0.0;
                    for (int g2 = lane; g2 < G; g2 += 32) v += __ldcg(a.ccp + (size_t)t * G + g2);
                    v = warp_sum(v);
                    if (lane == 0) ccs[stale[t]] = v;
                }
                __syncthreads();
                // ---- owned columns: the G slice partials (contiguous) in fixed
                //      order; two pairs per warp in flight
                const int npairs = nown * nstale;
                for (int p0 = warp; p0 < npairs; p0 += 2 * nwarps) {
                    double v[2][HART_MAXG / 32];
#pragma unroll
                    for (int m = 0; m < 2; ++m) {
                        const int p = p0 + m * nwarps;
                        const int q = p / nstale, t = p - (p / nstale) * nstale;
                        const double* base = a.part + ((size_t)(jown - b0 + q) * c + t) * G;
#pragma unroll
                        for (int u = 0; u < HART_MAXG / 32; ++u) {
                            const int g2 = lane + 32 * u;
                            v[m][u] = (p < npairs && g2 < G) ? __ldcg(base + g2) : 0.0;
                        }
                    }
#pragma unroll
                    for (int m = 0; m < 2; ++m) {
                        const int p = p0 + m * nwarps;
                        double sdot = 0.0;
#pragma unroll
                        for (int u = 0; u < HART_MAXG / 32; ++u) sdot += v[m][u];
                        sdot = warp_sum(sdot);
                        if (lane == 0 && p < npairs) {
                            const int q = p / nstale, t = p - (p / nstale) * nstale;
                            const int k = stale[t];
                            const double cck = ccs[k], xxj = s_xx[q];
                            const double mid = (xxj + cck) - 2.0 * sdot;
                            const double e = screen_err(a.kappa_d, sqrt(fabs(xxj)), sqrt(fabs(cck)), mid);
                            As[q * c + k] = mid;
                            Es[q * c + k] = isfinite(mid) && isfinite(e) ? hart_widen(mid, e, a.gam) : INFINITY;
                            ++refreshed;
                        }
                    }
                }
            }
            lap(3);
            if (blockIdx.x == 0 && tid == 0) __stcg(a.ebuf + blk, mvcount);
            if (bulk && nown > 0) {
                if (!mbar_wait(&s_bar, bar_phase)) __trap();
                bar_phase ^= 1;
            }
            __syncthreads();
            if (tid == 0) t_load += gtimer() - tl0;
        }

        // ---- phase 2: decide owned columns (warp per column), elect the first
        if (warp < nown) {
            const int j = jown + warp;
            if (j >= cursor) {
                const int from = s_lab[warp];
                int to = -1;
                auto iv = [&](int k, double& lo, double& hi, double& mid) {
                    mid = As[warp * c + k];
                    const double e = Es[warp * c + k];
                    lo = mid - e;
                    hi = mid + e;
                };
                const int st = hart_decide_warp_w(from, c, cnt, wa, wb, iv, to);
                if (st != 0 && lane == 0) {
                    // this column's intervals to its from / to centroid, for the
                    // identities of phase 1 should it be the elected move
                    double* cd = a.cand + 4 * (int64_t)j;
                    __stcg(cd, As[warp * c + from]);
                    __stcg(cd + 1, Es[warp * c + from]);
                    __stcg(cd + 2, to >= 0 ? As[warp * c + to] : 0.0);
                    __stcg(cd + 3, to >= 0 ? Es[warp * c + to] : INFINITY);
                    __threadfence();
                    atomicMin(&hg->first[r % 3][0], pack4(j, st, from, to));
                }
                if (a.diag && st == 0 && cnt[from] > 1) {
                    // diagnostics: relative margin of a "no move" decision
                    double mn = INFINITY;
                    for (int k = lane; k < c; k += 32)
                        if (k != from) mn = fmin(mn, wb[k] * As[warp * c + k]);
                    for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
                    if (lane == 0) {
                        const double sc = sqrt(fabs(s_xx[warp])) + sqrt(fabs(ccs[from]));
                        const double m = (mn - wa[from] * As[warp * c + from]) / (sc * sc);
                        double th = 1e-1;
                        for (int b = 0; b < 8; ++b, th *= 0.1)
                            if (m < th) atomicAdd(&hg->hist[b], 1ULL);
                        atomicAdd(&hg->hist[8], 1ULL);
                    }
                }
            }
        }
        // slot (r+1)%3 is next written after this barrier and last read before
        // barrier r-1 completed, so resetting it here cannot race
        if (blockIdx.x == 0 && tid == 0) hg->first[(r + 1) % 3][0] = ~0ULL;
        lap(4);
        grid_barrier(hg);
        lap(5);

        // ---- phase 3: settle (identically in every CTA)
        ++rounds;
        const unsigned long long f = __ldcg(&hg->first[r % 3][0]);
        if (f == ~0ULL) {
            cursor = bend;
        } else {
            const int j = (int)(f >> 32);
            int st = (int)((f >> 30) & 3);
            const int from = (int)((f >> 15) & 0x7fff);
            int to = (int)(f & 0x7fff);
            if (st == 2) {
                // near-tie: the owner resolves it with the reference's chain
                // (kmeans.cpp:12-19) and broadcasts the verdict
                const int owner = (j - b0) / cpb;
                if ((int)blockIdx.x == owner) {
                    const int q = j - jown;
                    for (int k = tid; k < c; k += blockDim.x) {
                        const double* cv = a.Cs + ((int64_t)vs[k] * c + k) * d;
                        double s = 0.0;
                        for (int64_t i = 0; i < d; ++i) {
                            const double t = colv(jown, q, i) - __ldcg(cv + i);
                            s += t * t;
                        }
                        a.scratch[k] = s;
                    }
                    __syncthreads();
                    if (warp == 0) {
                        int t2 = -1;
                        auto iv = [&](int k, double& lo, double& hi, double& mid) {
                            mid = __ldcg(a.scratch + k);
                            lo = hi = mid;
                        };
                        const int s2 = hart_decide_warp_w(from, c, cnt, wa, wb, iv, t2);
                        if (lane == 0) {
                            if (s2 == 1) {  // the reference's own values (chain): ± γ covers the real ones
                                const double vf = __ldcg(a.scratch + from), vt = __ldcg(a.scratch + t2);
                                double* cd = a.cand + 4 * (int64_t)j;
                                __stcg(cd, vf);
                                __stcg(cd + 1, hart_widen(vf, 0.0, a.gam));
                                __stcg(cd + 2, vt);
                                __stcg(cd + 3, hart_widen(vt, 0.0, a.gam));
                            }
                            hg->xres = pack4(j, s2, from, t2);
                            hg->exact_fallbacks += 1;
                        }
                    }
                }
                grid_barrier(hg);
                const unsigned long long x = __ldcg(&hg->xres);
                st = (int)((x >> 30) & 3);
                to = (int)(x & 0x7fff);
            }
            if (st == 1) {  // kmeans.cpp:122-135
                const int nf = cnt[from], nt = cnt[to];
                __syncthreads();
                if (tid == 0) {
                    cnt[from] = nf - 1;
                    cnt[to] = nt + 1;
                    const double fa = (double)(nf - 1), fb = (double)(nt + 1);
                    wa[from] = fa / (fa - 1.0);
                    wb[from] = fa / (fa + 1.0);
                    wa[to] = fb / (fb - 1.0);
                    wb[to] = fb / (fb + 1.0);
                    mv[from] = mv[to] = ++mvcount;
                    if (j >= jown && j < jown + nown) s_lab[j - jown] = to;
                }
                if (blockIdx.x == 0 && tid == 0) {
                    __stcg(a.labels + j, to);
                    hg->moves += 1;
                }
                improved = 1;
                pf = from;
                pt = to;
                pm = j;
                pnf = nf;
                pnt = nt;
            }
            cursor = j + 1;
        }
        __syncthreads();
    }

    // ---- publish (CTA 0): final counts and slot map.  The last move's slices
    //      were stored in this round; the kernel boundary publishes them.
    if (blockIdx.x == 0) {
        for (int k = tid; k < c; k += blockDim.x) {
            a.counts[k] = cnt[k];
            a.ver[k] = vs[k];
        }
        if (tid == 0) {
            hg->rounds = rounds;
            hg->passes = (unsigned long long)pass;
            hg->blocks = blocks;
            hg->t_kernel = gtimer() - tk0;
            hg->t_load = t_load;
            hg->t_cols = t_cols;
            hg->stale_sum = stale_sum;
            hg->heavy_blocks = heavy;
            hg->redos = redos;
            hg->act_cycles = act_cycles;
            hg->act_rounds = act_rounds;
            hg->dq_cycles = dq_cycles;
            for (int q = 0; q < 8; ++q) hg->tm[q] = tm[q];
            hg->tm[6] = tsub[0]; hg->tsub1 = tsub[1]; hg->tsub2 = tsub[2];
        }
    }
    if (lane == 0 && refreshed) atomicAdd(&hg->refreshed, refreshed);
}

}  // namespace respca_dev
