// Warp-specialised persistent Hartigan (kmeans.cpp:96-139): the same exact
// sequential semantics as k_hart_all (hartigan.cuh), with the block refresh
// taken off the critical path.
//
//   warps 0-7  (group R): the rounds — move update, decisions, election,
//               settle — and the block transitions;
//   warps 8-15 (group P): while group R plays block b's rounds, the row-split
//               FP64 tensor-core partials of block b+1's columns against a
//               SNAPSHOT of the centroids taken when block b was entered.
//
// On entering block b+1, group R sums the partials (after one grid barrier),
// then recomputes only the centroids that moved since the snapshot (≈ 2 moves
// per block at C3) with full-length dots against the owned columns.  A
// snapshot slot can be overwritten only by a centroid's second move after the
// snapshot, and every moved centroid is recomputed, so a torn read there is
// never used.  Partials are double-buffered by block parity: a CTA's group P
// starts block b+2 only after the grid barrier of block b+1's entry, which
// every CTA reaches after summing block b.
#pragma once

#include "hartigan.cuh"

namespace respca_dev {

constexpr int WS_R = 256, WS_P = 256;                    // threads per group
constexpr int BAR_R = 1, BAR_P = 2, BAR_GO = 3, BAR_DONE = 4;

RESPCA_DEV void nbar(int id, int count) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory"); }

// fixed-order reduction of NV doubles over the nw warps of one group
template <int NV>
RESPCA_DEV void gsum(double (&v)[NV], double* red, int bar, int lt, int nw) {
    const int lane = lt & 31, w = lt >> 5;
#pragma unroll
    for (int q = 0; q < NV; ++q) v[q] = warp_sum(v[q]);
    nbar(bar, nw * 32);
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < NV; ++q) red[q * 32 + w] = v[q];
    nbar(bar, nw * 32);
#pragma unroll
    for (int q = 0; q < NV; ++q) v[q] = warp_sum(lane < nw ? red[q * 32 + lane] : 0.0);
    nbar(bar, nw * 32);
}

// grid barrier among the R groups (thread 0 of every CTA is in group R)
RESPCA_DEV void grid_barrier_r(HartGlobal* g) {
    nbar(BAR_R, WS_R);
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
    nbar(BAR_R, WS_R);
}

struct HartWsArgs {
    HartGlobal* g;
    int* labels;       // [n]
    int* counts;       // [c]  in: start counts, out: final counts
    double* Cs;        // [2][c][d] centroid slots; slot 0 holds the start centroids
    int* ver;          // [c]  out: slot of each final centroid
    double* part;      // [2][B][c][G] row-slice partial dots (block parity)
    double* ccp;       // [2][c][G]    row-slice partials of ‖c‖²
    double* cand;      // [n][4] a candidate column's (mid, e) to its from / to centroid
    double* scratch;   // [c]   exact distances of one column (near-tie)
    int64_t d;
    int n, c, cpb, cache_cols, max_pass, stage_rows, stages;
    double kappa_d;    // screen bound factor + the reciprocal-update term
    double gam;        // (d+3)u·1.02 (hart_widen)
};

// Group P: partials of block [b0, b0+nb) × all c centroids over this CTA's row
// slice, centroids read from the snapshot slots vsnap; DMMA m8n8k4 with 2×2
// warp tiles and `stages` cp.async stages of R rows ([col][R+4] layout).
template <typename T, int TPW>
RESPCA_DEV void ws_partials(const T* __restrict__ M, const HartWsArgs& a, const int* vsnap, int b0, int nb,
                            int64_t s0, int64_t s1, int R, T* stc, double* sce, double* ccacc, int buf) {
    const int lt = threadIdx.x - WS_R, nt = WS_P, warp = lt >> 5, lane = lt & 31, nwarps = WS_P / 32;
    const int c = a.c, G = gridDim.x, NS = a.stages;
    const int64_t d = a.d;
    const double* __restrict__ Cs = a.Cs;
    const int MP = (nb + 15) & ~15, NP = (c + 15) & ~15, RS = R + 4;
    const int wtn = NP >> 4, nwt = (MP >> 4) * wtn;
    const int lgR = 31 - __clz(R);
    const size_t sstc = (size_t)MP * RS, ssce = (size_t)NP * RS;
    const int nch = s1 > s0 ? (int)((s1 - s0 + R - 1) / R) : 0;
    const int g = lane >> 2, t4 = lane & 3;
    const int B = gridDim.x * a.cpb;
    double* part = a.part + (size_t)buf * B * c * G;
    double* ccp = a.ccp + (size_t)buf * c * G;
    auto issue = [&](int ch) {
        const int64_t c0 = s0 + (int64_t)ch * R;
        const int rows = (int)(s1 - c0 < R ? s1 - c0 : R);
        T* sb = stc + (size_t)(ch % NS) * sstc;
        double* cb = sce + (size_t)(ch % NS) * ssce;
        for (int e = lt; e < (MP << lgR); e += nt) {
            const int jb = e >> lgR, rr = e & (R - 1);
            const bool ok = jb < nb && rr < rows;
            const T* src = M + (int64_t)(b0 + (ok ? jb : 0)) * d + c0 + (ok ? rr : 0);
            if (sizeof(T) == 8) cp_async8(sb + jb * RS + rr, src, ok);
            else cp_async4(sb + jb * RS + rr, src, ok);
        }
        for (int e = lt; e < (NP << lgR); e += nt) {
            const int k = e >> lgR, rr = e & (R - 1);
            const bool ok = k < c && rr < rows;
            const int kk = k < c ? k : 0;
            cp_async8(cb + k * RS + rr, Cs + ((int64_t)vsnap[kk] * c + kk) * d + c0 + (ok ? rr : 0), ok);
        }
        cp_commit();
    };
    for (int tr0 = 0; tr0 < nwt; tr0 += nwarps * TPW) {
        double acc[TPW][2][2][2];
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
        const bool norms = tr0 == 0;
        if (norms)
            for (int k = lt; k < c; k += nt) ccacc[k] = 0.0;
        nbar(BAR_P, WS_P);
        int issued = 0;
        for (; issued < nch && issued < NS - 1; ++issued) issue(issued);
        for (int ch = 0; ch < nch; ++ch) {
            if (issued < nch) issue(issued++);
            cp_wait_dyn(issued - ch - 1);
            nbar(BAR_P, WS_P);
            const T* sb = stc + (size_t)(ch % NS) * sstc;
            const double* cb = sce + (size_t)(ch % NS) * ssce;
            if (norms) {  // ‖c_k‖² slice partials on the warps without tiles (else all)
                const int w0 = nwt < nwarps ? nwt : 0, nw0 = nwarps - w0;
                if (warp >= w0)
                    for (int k = (warp - w0) * 32 + lane; k < c; k += nw0 * 32) {
                        double v = ccacc[k];
                        for (int rr = 0; rr < R; ++rr) v = __fma_rn(cb[k * RS + rr], cb[k * RS + rr], v);
                        ccacc[k] = v;
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
            nbar(BAR_P, WS_P);
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
                            const int k = wn[i] * 16 + y * 8 + 2 * t4 + h;
                            if (jb < nb && k < c)
                                __stcg(part + ((size_t)jb * c + k) * G + blockIdx.x, acc[i][x][y][h]);
                        }
                }
    }
    nbar(BAR_P, WS_P);
    for (int k = lt; k < c; k += nt) __stcg(ccp + (size_t)k * G + blockIdx.x, ccacc[k]);
}

// Σ_g p[g] in fixed order, eight loads in flight
RESPCA_DEV double ws_sum_g(const double* __restrict__ p, int G) {
    double s = 0.0;
    int g = 0;
    for (; g + 8 <= G; g += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(p + g + u);
#pragma unroll
        for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; g < G; ++g) s += __ldcg(p + g);
    return s;
}

template <typename T, int MAXQ>
__global__ void __launch_bounds__(512, 1) k_hart_ws(const T* __restrict__ M, HartWsArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int64_t d = a.d;
    const int c = a.c, n = a.n, cpb = a.cpb, cache_cols = a.cache_cols;
    HartGlobal* hg = a.g;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
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
    double* red = reinterpret_cast<double*>(sm + off);  // group R sums
    off += sizeof(double) * HART_RED;
    T* stc = reinterpret_cast<T*>(sm + off);  // group P stages [stages][B↑16][R+4]
    off += (size_t)a.stages * sizeof(double) * (size_t)(R + 4) * ((B + 15) & ~15);
    double* sce = reinterpret_cast<double*>(sm + off);  // [stages][c↑16][R+4]
    off += (size_t)a.stages * sizeof(double) * (size_t)(R + 4) * ((c + 15) & ~15);
    double* ccacc = reinterpret_cast<double*>(sm + off);  // group P ‖c‖² slice sums
    off += sizeof(double) * c;
    int* vsnap = reinterpret_cast<int*>(sm + off);  // slot map at the snapshot
    off += sizeof(int) * c;
    int* stale = reinterpret_cast<int*>(sm + off);
    off += sizeof(int) * c;
    int* cnt = reinterpret_cast<int*>(sm + off);
    off += sizeof(int) * c;
    int* vs = reinterpret_cast<int*>(sm + off);
    off += sizeof(int) * c;
    int* mv = reinterpret_cast<int*>(sm + off);
    __shared__ double s_xx[MAXQ];
    __shared__ int s_lab[MAXQ];
    __shared__ int s_nstale, s_exit, s_next_b0, s_next_buf, s_mv_snap;
    __shared__ __align__(8) uint64_t s_bar;  // column fills (bulk copies)

    const uint32_t col_bytes = (uint32_t)(d * (int64_t)sizeof(T));
    const bool bulk = cache_cols && (col_bytes % 16 == 0) && ((uintptr_t)M % 16 == 0);
    if (tid == 0) {
        mbar_init(&s_bar, 1);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    }
    for (int k = tid; k < c; k += blockDim.x) {
        const int ck = __ldcg(a.counts + k);
        cnt[k] = ck;
        const double nk = (double)ck;
        wa[k] = nk / (nk - 1.0);  // kmeans.cpp:107
        wb[k] = nk / (nk + 1.0);  // kmeans.cpp:114
        vs[k] = 0;
        vsnap[k] = 0;
        mv[k] = 0;
    }
    if (tid == 0) {
        s_exit = 0;
        s_next_b0 = 0;
        s_next_buf = 0;
        s_mv_snap = 0;
    }
    __syncthreads();
    // this CTA's row slice: it alone stores those rows of every updated centroid
    const int64_t slice = (d + G - 1) / G;
    const int64_t s0 = (int64_t)blockIdx.x * slice < d ? (int64_t)blockIdx.x * slice : d;
    const int64_t s1 = s0 + slice < d ? s0 + slice : d;

    if (tid >= WS_R) {
        // ======================= group P =======================
        for (;;) {
            nbar(BAR_GO, 512);
            if (s_exit) return;
            const int nb0 = s_next_b0, buf = s_next_buf;
            const int nbn = (nb0 + B < n ? nb0 + B : n) - nb0;
            const int nwt = ((nbn + 15) >> 4) * ((c + 15) >> 4);
            if (nwt <= 8)
                ws_partials<T, 1>(M, a, vsnap, nb0, nbn, s0, s1, R, stc, sce, ccacc, buf);
            else
                ws_partials<T, 2>(M, a, vsnap, nb0, nbn, s0, s1, R, stc, sce, ccacc, buf);
            nbar(BAR_DONE, 512);
        }
    }

    // ========================= group R =========================
    auto colv = [&](int jo, int q, int64_t i) -> double {
        return cache_cols ? (double)colc[(int64_t)q * d + i] : (double)__ldg(M + (int64_t)(jo + q) * d + i);
    };
    int pass = 0, improved = 0;
    int b0 = -1, bend = 0, cursor = 0, jown = 0, nown = 0, blk = 0;
    int pf = -1, pt = -1, pm = -1, pnf = 0, pnt = 0;
    int mvcount = 0;  // thread 0's move counter
    uint32_t bar_phase = 0;
    unsigned long long rounds = 0, blocks = 0, refreshed = 0, redos = 0;
    const unsigned long long tk0 = gtimer();
    unsigned long long t_entry = 0, t_wait = 0;
    nbar(BAR_GO, 512);  // group P: partials of block 0 against the start centroids

    for (int r = 0;; ++r) {
        // ---- phase 1: the pending move (kmeans.cpp:126-131), as k_hart_all
        if (pf >= 0) {
            const double* of = a.Cs + ((int64_t)vs[pf] * c + pf) * d;
            const double* ot = a.Cs + ((int64_t)vs[pt] * c + pt) * d;
            double* nfp = a.Cs + ((int64_t)(1 - vs[pf]) * c + pf) * d;
            double* ntp = a.Cs + ((int64_t)(1 - vs[pt]) * c + pt) * d;
            const T* xm = M + (int64_t)pm * d;
            const double dcf = (double)pnf, dct = (double)pnt;
            const double na1 = (double)(pnf - 1), nb1 = (double)(pnt + 1);
            for (int64_t i = s0 + tid; i < s1; i += WS_R) {
                const double x = (double)__ldg(xm + i);
                __stcg(nfp + i, (__ldcg(of + i) * dcf - x) / na1);  // kmeans.cpp:128-129 operation order
                __stcg(ntp + i, (__ldcg(ot + i) * dct + x) / nb1);
            }
            int nact = 0;
            for (int q = 0; q < nown; ++q) nact += (jown + q >= cursor);
            const int q0 = nown - nact;
            const double mf = __ldcg(a.cand + 4 * (int64_t)pm), ef = __ldcg(a.cand + 4 * (int64_t)pm + 1);
            const double mt = __ldcg(a.cand + 4 * (int64_t)pm + 2), et = __ldcg(a.cand + 4 * (int64_t)pm + 3);
            double xxm = 0.0;
            bool redo = false;
            double nmid = 0.0, ne = INFINITY;
            if (nact) {  // group-uniform
                double dq[MAXQ + 1];
#pragma unroll
                for (int q = 0; q <= MAXQ; ++q) dq[q] = 0.0;
                auto rowq = [&](int64_t i, double x) {
                    dq[MAXQ] = __fma_rn(x, x, dq[MAXQ]);  // ‖x_m‖² (bound scale only)
#pragma unroll
                    for (int q = 0; q < MAXQ; ++q)
                        if (q < nact) {
                            const double t = colv(jown, q0 + q, i) - x;
                            dq[q] = __fma_rn(t, t, dq[q]);
                        }
                };
                const int64_t step = WS_R;
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
                    for (; i < dh; i += step) {
                        const double2 xv = __ldg(x2 + i);
                        rowq(2 * i, xv.x);
                        rowq(2 * i + 1, xv.y);
                    }
                } else {
                    for (int64_t i = tid; i < d; i += step) rowq(i, (double)__ldg(xm + i));
                }
                gsum<MAXQ + 1>(dq, red, BAR_R, tid, WS_R / 32);
                xxm = dq[MAXQ];
                bool wide = false;
                if (tid < 2 * nact) {
                    const int qa = tid >> 1, which = tid & 1, q = q0 + qa;
                    const int k = which ? pt : pf;
                    double dqm = 0.0;
#pragma unroll
                    for (int e = 0; e < MAXQ; ++e)
                        if (e == qa) dqm = dq[e];
                    const double dlo = dqm * (1.0 - 1.01 * a.gam), dhi = dqm * (1.0 + 2.02 * a.gam);
                    const double om = As[q * c + k], oe = Es[q * c + k];
                    const double lo = fmax(om - oe, 0.0), hi = om + oe;
                    double flo, fhi, nn, dn;
                    if (!which) {  // ‖x−e_f‖² = (n·D_xf − D_xm)/(n−1) + n·D_fm/(n−1)²
                        nn = dcf;
                        dn = na1;
                        const double r1 = 1.0 / dn, r2 = r1 * r1;
                        const double m1 = fmax(mf - ef, 0.0), m2 = mf + ef;
                        flo = (nn * lo - dhi) * r1 + nn * m1 * r2;
                        fhi = (nn * hi - dlo) * r1 + nn * m2 * r2;
                        const double sl = 16.0 * kU * ((nn * hi + dhi) * r1 + nn * m2 * r2);
                        flo -= sl;
                        fhi += sl;
                    } else {  // ‖x−e_t‖² = (n·D_xt + D_xm)/(n+1) − n·D_tm/(n+1)²
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
                    const double del = 3.03 * kU * (nn * sqrt(fabs(ccs[k])) + sqrt(fabs(xxm))) / dn;
                    const double sh = sqrt(fmax(fhi, 0.0));
                    const double rlo = fmax(flo - 2.0 * sh * del * 1.01, 0.0);
                    const double rhi = fhi + (2.0 * sh * del + del * del) * 1.01;
                    const double ulo = rlo * (1.0 - 1.01 * a.gam), uhi = rhi * (1.0 + 1.01 * a.gam);
                    nmid = 0.5 * (ulo + uhi);
                    ne = (0.5 * (uhi - ulo)) * (1.0 + 8.0 * kU) + 4.0 * kU * uhi;
                    const double fresh = screen_err(a.kappa_d, sqrt(fabs(s_xx[q])), sqrt(fabs(ccs[k])), nmid);
                    wide = !(isfinite(nmid) && isfinite(ne) && ne <= 64.0 * fresh);
                }
                // group-uniform "any wide": through the group reduction
                double wv[1] = {wide ? 1.0 : 0.0};
                gsum<1>(wv, red, BAR_R, tid, WS_R / 32);
                redo = wv[0] > 0.0;
            }
            if (!redo) {
                if (tid < 2 * nact) {
                    const int qa = tid >> 1, which = tid & 1, q = q0 + qa;
                    const int k = which ? pt : pf;
                    As[q * c + k] = nmid;
                    Es[q * c + k] = ne;
                }
            } else {  // recompute from the new values over all rows
                const double rf = 1.0 / na1, rt = 1.0 / nb1;
                double acc[2 + 2 * MAXQ];
#pragma unroll
                for (int e = 0; e < 2 + 2 * MAXQ; ++e) acc[e] = 0.0;
                for (int64_t i = tid; i < d; i += WS_R) {
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
                gsum<2 + 2 * MAXQ>(acc, red, BAR_R, tid, WS_R / 32);
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
            nbar(BAR_R, WS_R);
            if (tid == 0) {
                // ‖c′‖² by the same identities: only the bound's scale uses it
                // until the next block entry recomputes it
                if (nact) {
                    ccs[pf] = fmax((dcf * ccs[pf] - xxm) / na1 + dcf * mf / (na1 * na1), 0.0);
                    ccs[pt] = fmax((dct * ccs[pt] + xxm) / nb1 - dct * mt / (nb1 * nb1), 0.0);
                }
                vs[pf] ^= 1;  // this CTA's slices of the new values are stored
                vs[pt] ^= 1;
            }
            nbar(BAR_R, WS_R);
            pf = -1;
        }

        if (cursor >= bend) {
            // ---- block transition
            int nb0 = b0 < 0 ? 0 : bend;
            bool finish = false;
            if (nb0 >= n) {  // end of a pass (kmeans.cpp:137)
                ++pass;
                if (!improved || pass >= a.max_pass) finish = true;
                improved = 0;
                nb0 = 0;
            }
            const unsigned long long te0 = gtimer();
            if (finish) {
                nbar(BAR_DONE, 512);  // group P's speculative partials are done
                if (tid == 0) s_exit = 1;
                nbar(BAR_R, WS_R);
                nbar(BAR_GO, 512);  // release group P
                break;
            }
            b0 = nb0;
            bend = b0 + B < n ? b0 + B : n;
            cursor = b0;
            jown = b0 + blockIdx.x * cpb;
            nown = bend - jown;
            nown = nown < 0 ? 0 : (nown > cpb ? cpb : nown);
            ++blocks;
            // owned columns (bulk copies when aligned), labels — in flight
            // while group P finishes
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
            } else if (cache_cols) {
                for (int q = 0; q < nown; ++q)
                    for (int64_t i = tid; i < d; i += WS_R)
                        colc[(int64_t)q * d + i] = __ldg(M + (int64_t)(jown + q) * d + i);
            }
            if (tid < nown) s_lab[tid] = __ldcg(a.labels + jown + tid);
            nbar(BAR_DONE, 512);  // group P: partials of this block are written
            if (tid == 0) t_wait += gtimer() - te0;
            // every CTA's partials of this block complete; phase 1 of this
            // round (new centroid slices) complete everywhere
            grid_barrier_r(hg);
            // ‖c_k‖² at the snapshot (slice partials, fixed order)
            const double* ccp = a.ccp + (size_t)(blk & 1) * c * G;
            const double* part = a.part + (size_t)(blk & 1) * B * c * G;
            for (int k = tid; k < c; k += WS_R) ccs[k] = ws_sum_g(ccp + (size_t)k * G, G);
            if (bulk && nown > 0) {
                if (!mbar_wait(&s_bar, bar_phase)) __trap();
                bar_phase ^= 1;
            }
            nbar(BAR_R, WS_R);
            // ‖x_j‖² of the owned columns
            for (int q = 0; q < nown; ++q) {
                double v[1] = {0.0};
                for (int64_t i = tid; i < d; i += WS_R) {
                    const double x = colv(jown, q, i);
                    v[0] = __fma_rn(x, x, v[0]);
                }
                gsum<1>(v, red, BAR_R, tid, WS_R / 32);
                if (tid == 0) s_xx[q] = v[0];
            }
            nbar(BAR_R, WS_R);
            // intervals of the owned columns against every centroid at the snapshot
            for (int p = tid; p < nown * c; p += WS_R) {
                const int q = p / c, k = p - (p / c) * c;
                const double sdot = ws_sum_g(part + ((size_t)(jown - b0 + q) * c + k) * G, G);
                {
                    const double cck = ccs[k], xxj = s_xx[q];
                    const double mid = (xxj + cck) - 2.0 * sdot;
                    const double e = screen_err(a.kappa_d, sqrt(fabs(xxj)), sqrt(fabs(cck)), mid);
                    As[q * c + k] = mid;
                    Es[q * c + k] = isfinite(mid) && isfinite(e) ? hart_widen(mid, e, a.gam) : INFINITY;
                }
            }
            // centroids moved since the snapshot: full-length dots with the
            // owned columns against their current values (ascending k, two at a time)
            if (warp == 0) {
                int cv = 0;
                for (int k0 = 0; k0 < c; k0 += 32) {
                    const int k = k0 + lane;
                    const bool sk = k < c && mv[k] > s_mv_snap;
                    const unsigned bal = __ballot_sync(0xffffffffu, sk);
                    if (sk) stale[cv + __popc(bal & ((1u << lane) - 1u))] = k;
                    cv += __popc(bal);
                }
                if (lane == 0) s_nstale = cv;
            }
            nbar(BAR_R, WS_R);
            const int nst = s_nstale;
            for (int t0 = 0; t0 < nst; t0 += 2) {
                const int k1 = stale[t0], k2 = t0 + 1 < nst ? stale[t0 + 1] : stale[t0];
                const double* c1 = a.Cs + ((int64_t)vs[k1] * c + k1) * d;
                const double* c2 = a.Cs + ((int64_t)vs[k2] * c + k2) * d;
                double v[2 + 2 * MAXQ];
#pragma unroll
                for (int e = 0; e < 2 + 2 * MAXQ; ++e) v[e] = 0.0;
                for (int64_t i = tid; i < d; i += WS_R) {
                    const double u1 = __ldcg(c1 + i), u2 = __ldcg(c2 + i);
                    v[0] = __fma_rn(u1, u1, v[0]);
                    v[1] = __fma_rn(u2, u2, v[1]);
#pragma unroll
                    for (int q = 0; q < MAXQ; ++q)
                        if (q < nown) {
                            const double xq = colv(jown, q, i);
                            v[2 + 2 * q] = __fma_rn(xq, u1, v[2 + 2 * q]);
                            v[3 + 2 * q] = __fma_rn(xq, u2, v[3 + 2 * q]);
                        }
                }
                gsum<2 + 2 * MAXQ>(v, red, BAR_R, tid, WS_R / 32);
                if (tid < 2 * nown) {
                    const int q = tid >> 1, which = tid & 1;
                    const int k = which ? k2 : k1;
                    double dot = 0.0;
#pragma unroll
                    for (int e = 0; e < 2 * MAXQ; ++e)
                        if (e == tid) dot = v[2 + e];
                    const double cck = which ? v[1] : v[0], xxj = s_xx[q];
                    const double mid = (xxj + cck) - 2.0 * dot;
                    const double e = screen_err(a.kappa_d, sqrt(fabs(xxj)), sqrt(fabs(cck)), mid);
                    As[q * c + k] = mid;
                    Es[q * c + k] = isfinite(mid) && isfinite(e) ? hart_widen(mid, e, a.gam) : INFINITY;
                }
                if (tid == 0) {
                    ccs[k1] = v[0];
                    ccs[k2] = v[1];
                }
                nbar(BAR_R, WS_R);
            }
            refreshed += nst;
            // group P: the next block's partials against the centroids now
            {
                const int nxt = bend < n ? bend : 0;
                for (int k = tid; k < c; k += WS_R) vsnap[k] = vs[k];
                if (tid == 0) {
                    s_next_b0 = nxt;
                    s_next_buf = (blk + 1) & 1;
                    s_mv_snap = mvcount;
                }
                nbar(BAR_GO, 512);
            }
            ++blk;
            if (tid == 0) t_entry += gtimer() - te0;
        }

        // ---- decide owned columns (warp per column), elect the first
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
                    double* cd = a.cand + 4 * (int64_t)j;
                    __stcg(cd, As[warp * c + from]);
                    __stcg(cd + 1, Es[warp * c + from]);
                    __stcg(cd + 2, to >= 0 ? As[warp * c + to] : 0.0);
                    __stcg(cd + 3, to >= 0 ? Es[warp * c + to] : INFINITY);
                    __threadfence();
                    atomicMin(&hg->first[r % 3][0], pack4(j, st, from, to));
                }
            }
        }
        if (blockIdx.x == 0 && tid == 0) hg->first[(r + 1) % 3][0] = ~0ULL;
        grid_barrier_r(hg);

        // ---- settle (identically in every CTA)
        ++rounds;
        const unsigned long long f = __ldcg(&hg->first[r % 3][0]);
        if (f == ~0ULL) {
            cursor = bend;
        } else {
            const int j = (int)(f >> 32);
            int st = (int)((f >> 30) & 3);
            const int from = (int)((f >> 15) & 0x7fff);
            int to = (int)(f & 0x7fff);
            if (st == 2) {  // near-tie: the owner resolves it with the reference's chain
                const int owner = (j - b0) / cpb;
                if ((int)blockIdx.x == owner) {
                    const int q = j - jown;
                    for (int k = tid; k < c; k += WS_R) {
                        const double* cvp = a.Cs + ((int64_t)vs[k] * c + k) * d;
                        double s = 0.0;
                        for (int64_t i = 0; i < d; ++i) {
                            const double t = colv(jown, q, i) - __ldcg(cvp + i);
                            s += t * t;  // kmeans.cpp:12-19
                        }
                        a.scratch[k] = s;
                    }
                    nbar(BAR_R, WS_R);
                    if (warp == 0) {
                        int t2 = -1;
                        auto iv = [&](int k, double& lo, double& hi, double& mid) {
                            mid = __ldcg(a.scratch + k);
                            lo = hi = mid;
                        };
                        const int s2 = hart_decide_warp_w(from, c, cnt, wa, wb, iv, t2);
                        if (lane == 0) {
                            if (s2 == 1) {
                                const double vf = __ldcg(a.scratch + from), vt = __ldcg(a.scratch + t2);
                                double* cd = a.cand + 4 * (int64_t)j;
                                __stcg(cd, vf);
                                __stcg(cd + 1, hart_widen(vf, 0.0, a.gam));
                                __stcg(cd + 2, vt);
                                __stcg(cd + 3, hart_widen(vt, 0.0, a.gam));
                            }
                            hg->xres = pack4(j, s2, from, t2);
                            atomicAdd(&hg->exact_fallbacks, 1ULL);
                        }
                    }
                }
                grid_barrier_r(hg);
                const unsigned long long x = __ldcg(&hg->xres);
                st = (int)((x >> 30) & 3);
                to = (int)(x & 0x7fff);
            }
            if (st == 1) {  // kmeans.cpp:122-135
                const int nf = cnt[from], nt = cnt[to];
                nbar(BAR_R, WS_R);
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
        nbar(BAR_R, WS_R);
    }

    if (blockIdx.x == 0) {
        for (int k = tid; k < c; k += WS_R) {
            a.counts[k] = cnt[k];
            a.ver[k] = vs[k];
        }
        if (tid == 0) {
            hg->rounds = rounds;
            hg->passes = (unsigned long long)pass;
            hg->blocks = blocks;
            hg->t_kernel = gtimer() - tk0;
            hg->t_load = t_entry;
            hg->t_cols = t_wait;
            hg->refreshed = refreshed;
            hg->redos = redos;
        }
    }
}

}  // namespace respca_dev
