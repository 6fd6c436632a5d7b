// Exact sequential Hartigan refinement (kmeans.cpp:96-139) on the device.
//
// The reference visits columns j = 0..n−1 in order and applies each improving
// single-point move at once (incremental centroid update, kmeans.cpp:122-135),
// so every later decision sees the updated centroids and counts.  The device
// keeps exactly that order:
//
//  * columns are processed in blocks of B.  At block start, the screened
//    distance of every (block column, centroid) pair is computed by the DMMA
//    screen (km.cuh) — an interval [a − e, a + e] that provably contains the
//    reference's sq_dist;
//  * a round (one kernel, CTA per 8 block columns) first refreshes the two
//    entries of every remaining column that the previous move made stale (its
//    `from` and `to` centroids), computing the moved centroids' new values on
//    the fly with the reference's exact update formula (and writing them to
//    the other slot of a double-buffered centroid store); then one warp per
//    column decides it on the intervals; the last CTA to finish takes the
//    FIRST column that is not provably "no move" (all columns before it
//    provably do not move in the sequential order): a provable move is applied,
//    an undecidable near-tie is resolved with the exact sequential chain.
//
// Labels, counts and centroids are therefore bit-identical to the reference.
// Rounds run as a CUDA-graph WHILE loop; blocks and passes are stream-ordered
// and the host only synchronises once per pass.
#pragma once

#include "km.cuh"

namespace respca_dev {

struct HartState {
    int cursor;        // next column to visit
    int bend;          // end of the current block
    int pass;          // 0..49
    int improved;      // a move happened in this pass
    int block_done;
    int pending_from;  // centroid update of the last move, applied next round (-1: none)
    int pending_to, pending_j, pending_nf, pending_nt;
    int act_j;         // column the last CTA acts on
    unsigned arrive;   // last-CTA election
    unsigned long long first;  // packed (j, status, to) of the first non-trivial column
    unsigned long long moves, exact_fallbacks, rounds;
    unsigned long long t0, tsum;  // globaltimer: earliest CTA start of a round, summed round spans
    unsigned long long tp1, tp2, sp1, sp2, sp3s;  // phase-end stamps (max over CTAs) and sums
};

RESPCA_DEV unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

struct HartArrays {
    double* A;       // [n][c] screened distance
    double* E;       // [n][c] its half-width
    double* xx;      // [n]    ‖x_j‖² (screen input)
    int* labels;
    int* counts;
    double* C;       // [2][c][d] centroid slots (slot 0 = the caller's centroids)
    int* ver;        // [c] current slot of centroid k
    double* scratch; // [c] exact distances of one column
    double kappa_d;  // screen bound factor (km.cuh)
};

RESPCA_DEV double* cslot(const HartArrays& h, int c, int64_t d, int k, int s) {
    return h.C + ((int64_t)s * c + k) * d;
}

// Hartigan decision of column j on intervals (one warp):
//   0 = provably no move, 1 = provably moves to `to`, 2 = undecidable
template <typename IV>
RESPCA_DEV int hart_decide_warp(int j, int c, const int* __restrict__ labels,
                                const int* __restrict__ counts, const IV& iv, int& to) {
    const int lane = threadIdx.x & 31;
    const int from = labels[j];
    const int cf = counts[from];
    if (cf <= 1) return 0;  // kmeans.cpp:105
    double flo, fhi, fmid;
    iv(from, flo, fhi, fmid);
    const double na = (double)cf;
    const double wa = na / (na - 1.0);  // kmeans.cpp:107-108
    const double g_lo = wa * flo, g_hi = wa * fhi, g_mid = wa * fmid;
    double bd = INFINITY;
    int bk = 0x7fffffff;
    bool none = true;
    for (int k = lane; k < c; k += 32) {
        if (k == from) continue;
        double lo, hi, mid;
        iv(k, lo, hi, mid);
        const double nb = (double)counts[k];
        const double wb = nb / (nb + 1.0);  // kmeans.cpp:113-115
        none &= !(wb * lo - g_hi < -1e-12);
        const double dmid = wb * mid - g_mid;
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
    const double nbk = (double)counts[bk];
    const double dhi_k = (nbk / (nbk + 1.0)) * bhi - g_lo;
    bool ok = dhi_k < -1e-12;  // kmeans.cpp:116 with best_delta = -1e-12
    for (int k = lane; k < c; k += 32) {
        if (k == from || k == bk) continue;
        double lo, hi, mid;
        iv(k, lo, hi, mid);
        const double nb = (double)counts[k];
        const double dlo = (nb / (nb + 1.0)) * lo - g_hi;
        if (k < bk) ok &= dhi_k < dlo;  // an earlier k must lose strictly
        else ok &= dhi_k <= dlo;        // a later k never replaces an equal delta
    }
    ok = __all_sync(0xffffffffu, ok);
    if (!ok) return 2;
    to = bk;
    return 1;
}

// same decision with precomputed weights wa[k] = n_k/(n_k−1), wb[k] = n_k/(n_k+1)
// (the identical correctly-rounded divisions) and per-CTA counts
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
        none &= !(w_b * lo - g_hi < -1e-12);
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
        if (k < bk) ok &= dhi_k < dlo;
        else ok &= dhi_k <= dlo;
    }
    ok = __all_sync(0xffffffffu, ok);
    if (!ok) return 2;
    to = bk;
    return 1;
}

RESPCA_DEV unsigned long long pack_first(int j, int status, int to) {
    return ((unsigned long long)(unsigned)j << 32) | ((unsigned long long)status << 24) |
           (unsigned long long)(unsigned)(to & 0xffffff);
}

template <typename T, int CPB>
__global__ void __launch_bounds__(512) k_hart_round(const T* __restrict__ M,
                                                    HartState* __restrict__ hs, HartArrays h,
                                                    int64_t d, int n, int c,
                                                    cudaGraphConditionalHandle cond) {
    constexpr int NV = 2 + 2 * CPB;
    __shared__ double red[32 * NV];
    __shared__ bool s_last;
    __shared__ int s_st, s_to;
    const bool has_cond = cond != 0;
    if (hs->block_done) {
        if (blockIdx.x == 0 && threadIdx.x == 0 && has_cond) cudaGraphSetConditional(cond, 0u);
        return;
    }
    if (threadIdx.x == 0) atomicMin(&hs->t0, gtimer());
    const int cursor = hs->cursor, bend = hs->bend;
    const int jb = cursor + blockIdx.x * CPB;  // first column of this CTA
    const int pf = hs->pending_from;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // ---- phase 1: apply the pending move's centroid update (kmeans.cpp:126-131)
    //      and refresh the (column, from/to) entries of this CTA's columns
    if (pf >= 0) {
        const int pt = hs->pending_to, pm = hs->pending_j;
        const double dcf = (double)hs->pending_nf, dct = (double)hs->pending_nt;
        const double na1 = (double)(hs->pending_nf - 1), nb1 = (double)(hs->pending_nt + 1);
        const int vf = h.ver[pf], vt = h.ver[pt];
        const double* of = cslot(h, c, d, pf, vf);
        const double* ot = cslot(h, c, d, pt, vt);
        double* nf_ = cslot(h, c, d, pf, 1 - vf);
        double* nt_ = cslot(h, c, d, pt, 1 - vt);
        const T* xm = M + (int64_t)pm * d;
        const int64_t slice = (d + gridDim.x - 1) / gridDim.x;
        const int64_t s0 = (int64_t)blockIdx.x * slice, s1 = s0 + slice;
        bool active = false;
        for (int q = 0; q < CPB; ++q) active |= (jb + q < bend);
        double v[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) v[q] = 0.0;
        const int64_t ibeg = active ? 0 : s0, iend = active ? d : (s1 < d ? s1 : d);
#pragma unroll 4
        for (int64_t i = ibeg + threadIdx.x; i < iend; i += blockDim.x) {
            const double x = (double)xm[i];
            const double cf = (of[i] * dcf - x) / na1;
            const double ct = (ot[i] * dct + x) / nb1;
            if (i >= s0 && i < s1) {
                nf_[i] = cf;
                nt_[i] = ct;
            }
            if (active) {
                v[0] = __fma_rn(cf, cf, v[0]);
                v[1] = __fma_rn(ct, ct, v[1]);
#pragma unroll
                for (int q = 0; q < CPB; ++q) {
                    const int j = jb + q;
                    if (j < bend) {
                        const double xj = (double)__ldg(M + (int64_t)j * d + i);
                        v[2 + 2 * q] = __fma_rn(xj, cf, v[2 + 2 * q]);
                        v[3 + 2 * q] = __fma_rn(xj, ct, v[3 + 2 * q]);
                    }
                }
            }
        }
        if (active) {  // block-uniform
            block_sum<NV>(v, red);
            if (threadIdx.x < 2 * CPB) {
                const int q = threadIdx.x >> 1, which = threadIdx.x & 1;
                const int j = jb + q;
                if (j < bend) {
                    const int k = which ? pt : pf;
                    double dot = 0.0;
#pragma unroll
                    for (int r = 0; r < 2 * CPB; ++r)
                        if (r == (int)threadIdx.x) dot = v[2 + r];
                    const double cck = which ? v[1] : v[0];
                    const double xxj = h.xx[j];
                    const double mid = (xxj + cck) - 2.0 * dot;
                    const double e = screen_err(h.kappa_d, sqrt(fabs(xxj)), sqrt(fabs(cck)), mid);
                    const int64_t idx = (int64_t)j * c + k;
                    h.A[idx] = mid;
                    h.E[idx] = isfinite(mid) && isfinite(e) ? e : INFINITY;
                }
            }
        }
        __syncthreads();
    }

    if (threadIdx.x == 0) atomicMax(&hs->tp1, gtimer());
    // ---- phase 2: decide this CTA's columns (warp per column)
    if (warp < CPB) {
        const int j = jb + warp;
        if (j < bend) {
            int to = -1;
            auto iv = [&](int k, double& lo, double& hi, double& mid) {
                const int64_t idx = (int64_t)j * c + k;
                mid = h.A[idx];
                const double e = h.E[idx];
                lo = mid - e;
                hi = mid + e;
            };
            const int st = hart_decide_warp(j, c, h.labels, h.counts, iv, to);
            if (st != 0 && lane == 0) atomicMin(&hs->first, pack_first(j, st, to));
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicMax(&hs->tp2, gtimer());
        __threadfence();
        s_last = atomicAdd(&hs->arrive, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;

    // ---- phase 3 (last CTA): settle the round
    __threadfence();
    if (threadIdx.x == 0) {
        const unsigned long long t3 = gtimer();
        hs->sp1 += hs->tp1 - hs->t0;
        hs->sp2 += hs->tp2 - hs->t0;
        hs->sp3s += t3 - hs->t0;
        hs->tp1 = 0;
        hs->tp2 = 0;
        hs->arrive = 0;
        hs->rounds += 1;
        if (pf >= 0) {  // the new centroid values are complete: switch slots
            h.ver[pf] ^= 1;
            h.ver[hs->pending_to] ^= 1;
            hs->pending_from = -1;
        }
        const unsigned long long f = hs->first;
        hs->first = ~0ULL;
        if (f == ~0ULL) {
            s_st = -1;
            hs->cursor = bend;
        } else {
            s_st = (int)((f >> 24) & 0xff);
            s_to = (int)(f & 0xffffff);
            hs->act_j = (int)(f >> 32);
        }
        __threadfence();
    }
    __syncthreads();
    if (s_st == 2) {  // near-tie: the reference's own sequential chain (kmeans.cpp:12-19)
        const int j = hs->act_j;
        const T* x = M + (int64_t)j * d;
        for (int k = threadIdx.x; k < c; k += blockDim.x) {
            const double* cv = cslot(h, c, d, k, h.ver[k]);
            double s = 0.0;
            for (int64_t i = 0; i < d; ++i) {
                const double t = (double)x[i] - cv[i];
                s += t * t;
            }
            h.scratch[k] = s;
        }
        __syncthreads();
        if (warp == 0) {
            int to = -1;
            auto iv = [&](int k, double& lo, double& hi, double& mid) {
                mid = h.scratch[k];
                lo = hi = mid;
            };
            const int st = hart_decide_warp(j, c, h.labels, h.counts, iv, to);
            if (lane == 0) {
                s_st = st;
                s_to = to;
                hs->exact_fallbacks += 1;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (s_st == 0) {
            hs->cursor = hs->act_j + 1;
        } else if (s_st == 1) {  // bookkeeping of the move (kmeans.cpp:132-135)
            const int j = hs->act_j, from = h.labels[j], to = s_to;
            const int nf = h.counts[from], nt = h.counts[to];
            h.counts[from] = nf - 1;
            h.counts[to] = nt + 1;
            h.labels[j] = to;
            hs->pending_j = j;
            hs->pending_from = from;
            hs->pending_to = to;
            hs->pending_nf = nf;
            hs->pending_nt = nt;
            hs->improved = 1;
            hs->moves += 1;
            hs->cursor = j + 1;
        }
        const int done = hs->cursor >= bend && hs->pending_from < 0;
        hs->block_done = done;
        hs->tsum += gtimer() - hs->t0;
        hs->t0 = ~0ULL;
        __threadfence();
        if (has_cond) cudaGraphSetConditional(cond, done ? 0u : 1u);
    }
}

// block start: intervals of every (block column, centroid) pair from the screen
__global__ void k_hart_fill(Screen sc, HartArrays h, int j0, int nb, int c) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)nb * c) return;
    const int jl = (int)(e / c), k = (int)(e % c);
    const double xxj = sc.xx(jl);
    double lo, hi, mid;
    sc.get(jl, k, xxj, sqrt(fabs(xxj)), lo, hi, mid);
    const int64_t idx = (int64_t)(j0 + jl) * c + k;
    h.A[idx] = mid;
    h.E[idx] = isfinite(hi - mid) ? hi - mid : INFINITY;
    if (k == 0) h.xx[j0 + jl] = xxj;
}

__global__ void k_hart_block_begin(HartState* hs, int b0, int bend) {
    hs->cursor = b0;
    hs->bend = bend;
    hs->block_done = 0;
    hs->first = ~0ULL;
    hs->arrive = 0;
    hs->t0 = ~0ULL;
}

// copy centroids living in slot 1 back to slot 0 (the screen reads slot 0)
__global__ void k_hart_consolidate(HartArrays h, int64_t d, int c) {
    for (int k = blockIdx.y; k < c; k += gridDim.y) {
        if (h.ver[k] == 0) continue;
        const double* src = h.C + ((int64_t)c + k) * d;
        double* dst = h.C + (int64_t)k * d;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d;
             i += (int64_t)gridDim.x * blockDim.x)
            dst[i] = src[i];
    }
}
__global__ void k_hart_ver_reset(HartArrays h, int c) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < c; k += gridDim.x * blockDim.x)
        h.ver[k] = 0;
}

}  // namespace respca_dev

namespace respca_dev {

// ---------------------------------------------------------------------------
// Persistent cooperative variant: one launch per block of columns, every CTA
// resident (cudaLaunchCooperativeKernel), rounds separated by ONE grid barrier.
// Each CTA owns up to `cpb` block columns, caches them in shared memory, keeps
// their interval rows in shared memory, and replicates the small sequential
// state (counts, Hartigan weights, slot versions, cursor, pending move) so
// that every CTA settles a round identically from the elected first column.
// ---------------------------------------------------------------------------
struct HartGlobal {
    // each hot word on its own 128-byte line: the barrier spin, the barrier
    // arrivals and the per-round election slots must not share L2 lines
    alignas(128) unsigned bar_count;
    alignas(128) unsigned bar_gen;
    alignas(128) unsigned long long first[3][16];  // per-round election slots, round r uses r % 3
    alignas(128) unsigned long long xres;          // exact-fallback verdict broadcast
    alignas(128) int cursor, improved;
    unsigned long long moves, exact_fallbacks, rounds;
    unsigned long long t_kernel, t_phase1, t_phase2;  // globaltimer sums (CTA 0)
    unsigned long long t_phase1_max;                  // max over CTAs of summed phase-1 time
    unsigned long long tmax[6];  // per-CTA sums, max over CTAs: 1a, barrier A, 1b, decide, barrier B, settle
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
__global__ void k_hart_improved_reset(HartGlobal* g) { g->improved = 0; }

// v[2q], v[2q+1] += Σ_i x_{q0+q}[i]·f[i], x·t[i] for the NQ active owned columns
// (thread-strided rows, FMA chains; only ever used inside the screen bound)
template <typename T, int NQ>
RESPCA_DEV void hart_dots(double* v, const double* __restrict__ f, const double* __restrict__ t,
                          const T* colc, const T* __restrict__ M, int jown, int q0, int nact,
                          int64_t d, int cache_cols) {
    // v[2q], v[2q+1] = Σ_i x_{q0+q}[i]·f[i], ·t[i] for the nact (≤ NQ) active owned
    // columns (FMA chains; only ever used inside the screen bound)
    double acc[2 * NQ];
#pragma unroll
    for (int q = 0; q < 2 * NQ; ++q) acc[q] = 0.0;
    const T* base[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int qq = q < nact ? q0 + q : q0;
        base[q] = cache_cols ? colc + (int64_t)qq * d : M + (int64_t)(jown + qq) * d;
    }
    constexpr int UR = 4;
    const int64_t step = (int64_t)blockDim.x;
    int64_t i = threadIdx.x;
    for (; i + (UR - 1) * step < d; i += UR * step) {
        double fb[UR], tb[UR];
#pragma unroll
        for (int u = 0; u < UR; ++u) {
            fb[u] = __ldcg(f + i + u * step);
            tb[u] = __ldcg(t + i + u * step);
        }
#pragma unroll
        for (int u = 0; u < UR; ++u)
#pragma unroll
            for (int q = 0; q < NQ; ++q)
                if (q < nact) {
                    const double x = (double)base[q][i + u * step];
                    acc[2 * q] = __fma_rn(x, fb[u], acc[2 * q]);
                    acc[2 * q + 1] = __fma_rn(x, tb[u], acc[2 * q + 1]);
                }
    }
    for (; i < d; i += step) {
        const double fv = __ldcg(f + i), tv = __ldcg(t + i);
#pragma unroll
        for (int q = 0; q < NQ; ++q)
            if (q < nact) {
                const double x = (double)base[q][i];
                acc[2 * q] = __fma_rn(x, fv, acc[2 * q]);
                acc[2 * q + 1] = __fma_rn(x, tv, acc[2 * q + 1]);
            }
    }
#pragma unroll
    for (int q = 0; q < 2 * NQ; ++q) v[q] = acc[q];
}

template <typename T, int MAXQ>
__global__ void __launch_bounds__(512, 1) k_hart_block(
    const T* __restrict__ M, HartGlobal* __restrict__ hg, int* __restrict__ labels,
    int* __restrict__ counts, double* __restrict__ Cs, int* __restrict__ ver,
    Screen scr, double* __restrict__ scratch, double* __restrict__ ccpart, int64_t d, int c, int b0,
    int bend, int cpb, int cache_cols, double kappa_d, int dbg) {
    extern __shared__ __align__(16) unsigned char sm[];
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
    double* red = reinterpret_cast<double*>(sm + off);
    off += sizeof(double) * 32 * (2 * MAXQ);
    int* cnt = reinterpret_cast<int*>(sm + off);
    off += sizeof(int) * c;
    int* vs = reinterpret_cast<int*>(sm + off);
    __shared__ double s_xx[MAXQ];
    __shared__ int s_lab[MAXQ];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int jown = b0 + blockIdx.x * cpb;  // first owned column
    int nown = bend - jown;
    nown = nown < 0 ? 0 : (nown > cpb ? cpb : nown);

    // ---- load owned columns, interval rows, replicated state
    if (cache_cols)
        for (int q = 0; q < nown; ++q)
            for (int64_t i = tid; i < d; i += blockDim.x)
                colc[(int64_t)q * d + i] = M[(int64_t)(jown + q) * d + i];
    // intervals of the owned columns from the block's screen (split-K partials
    // summed in fixed order; km.cuh bound)
    for (int e = tid; e < nown * c; e += blockDim.x) {
        const int q = e / c, k = e - (e / c) * c;
        const int jl = jown - b0 + q;
        const double xxj = scr.xx(jl);
        double lo, hi, mid;
        scr.get(jl, k, xxj, sqrt(fabs(xxj)), lo, hi, mid);
        As[e] = mid;
        Es[e] = isfinite(hi - mid) ? hi - mid : INFINITY;
    }
    for (int k = tid; k < c; k += blockDim.x) {
        const int ck = __ldcg(counts + k);
        cnt[k] = ck;
        const double nk = (double)ck;
        wa[k] = nk / (nk - 1.0);  // kmeans.cpp:107
        wb[k] = nk / (nk + 1.0);  // kmeans.cpp:114
        vs[k] = __ldcg(ver + k);
    }
    if (tid < nown) {
        s_xx[tid] = scr.xx(jown - b0 + tid);
        s_lab[tid] = __ldcg(labels + jown + tid);
    }
    __syncthreads();
    auto colv = [&](int q, int64_t i) -> double {
        return cache_cols ? (double)colc[(int64_t)q * d + i] : (double)__ldg(M + (int64_t)(jown + q) * d + i);
    };

    int cursor = b0;
    int pf = -1, pt = -1, pm = -1, pnf = 0, pnt = 0;
    const int64_t slice = (d + gridDim.x - 1) / gridDim.x;
    const int64_t s0 = (int64_t)blockIdx.x * slice;
    const int64_t s1 = s0 + slice < d ? s0 + slice : d;
    unsigned long long rounds = 0;

    const unsigned long long tk0 = gtimer();
    unsigned long long tph1 = 0, tph2 = 0;
    unsigned long long ts[6] = {0, 0, 0, 0, 0, 0};
    unsigned long long act_rounds = 0;
    for (int r = 0;; ++r) {
        const unsigned long long tr0 = gtimer();
        // ---- phase 1a: the pending move's centroid update (kmeans.cpp:126-131),
        //      each CTA computing ONE row slice (exact division), plus that
        //      slice's partial ‖c'‖² sums
        if (pf >= 0) {
            const double* of = Cs + ((int64_t)vs[pf] * c + pf) * d;
            const double* ot = Cs + ((int64_t)vs[pt] * c + pt) * d;
            double* nfp = Cs + ((int64_t)(1 - vs[pf]) * c + pf) * d;
            double* ntp = Cs + ((int64_t)(1 - vs[pt]) * c + pt) * d;
            const T* xm = M + (int64_t)pm * d;
            const double dcf = (double)pnf, dct = (double)pnt;
            const double na1 = (double)(pnf - 1), nb1 = (double)(pnt + 1);
            double v2[2] = {0.0, 0.0};
            for (int64_t i = s0 + tid; i < s1; i += blockDim.x) {
                const double x = (double)__ldg(xm + i);
                const double cf = (__ldcg(of + i) * dcf - x) / na1;
                const double ct = (__ldcg(ot + i) * dct + x) / nb1;
                __stcg(nfp + i, cf);
                __stcg(ntp + i, ct);
                v2[0] = __fma_rn(cf, cf, v2[0]);
                v2[1] = __fma_rn(ct, ct, v2[1]);
            }
            block_sum<2>(v2, red);
            if (tid == 0) {
                __stcg(ccpart + 2 * blockIdx.x, v2[0]);
                __stcg(ccpart + 2 * blockIdx.x + 1, v2[1]);
            }
            const unsigned long long ta = gtimer();
            ts[0] += ta - tr0;
            grid_barrier(hg);
            const unsigned long long tb = gtimer();
            ts[1] += tb - ta;
            // ---- phase 1b: refresh the (column, from/to) intervals of the owned
            //      columns still to be decided, reading the new slots (L2)
            int nact = 0;
            for (int q = 0; q < nown; ++q) nact += (jown + q >= cursor);
            if (nact && !(dbg & 1)) {
                act_rounds++;
                // slice partials of ‖c'‖²: one load per thread, fixed-order tree
                double cc2[2] = {0.0, 0.0};
                for (unsigned b = tid; b < gridDim.x; b += blockDim.x) {
                    cc2[0] += __ldcg(ccpart + 2 * b);
                    cc2[1] += __ldcg(ccpart + 2 * b + 1);
                }
                block_sum<2>(cc2, red);
                const double ccf = cc2[0], cct = cc2[1];
                double v[2 * MAXQ];
#pragma unroll
                for (int q = 0; q < 2 * MAXQ; ++q) v[q] = 0.0;
                // active owned columns are the suffix q0..nown-1 of the owned range
                const int q0 = nown - nact;
                hart_dots<T, MAXQ>(v, nfp, ntp, colc, M, jown, q0, nact, d, cache_cols);
                block_sum<2 * MAXQ>(v, red);
                if (tid < 2 * nown) {
                    const int q = tid >> 1, which = tid & 1;
                    if (jown + q >= cursor) {
                        const int idx = 2 * (q - q0) + which;  // hart_dots packs actives first
                        double dot = 0.0;
#pragma unroll
                        for (int rr = 0; rr < 2 * MAXQ; ++rr)
                            if (rr == idx) dot = v[rr];
                        const double cck = which ? cct : ccf;
                        const double xxj = s_xx[q];
                        const double mid = (xxj + cck) - 2.0 * dot;
                        const double e = screen_err(kappa_d, sqrt(fabs(xxj)), sqrt(fabs(cck)), mid);
                        const int k = which ? pt : pf;
                        As[q * c + k] = mid;
                        Es[q * c + k] = isfinite(mid) && isfinite(e) ? e : INFINITY;
                    }
                }
            }
            __syncthreads();
        }
        const unsigned long long tr1 = gtimer();
        tph1 += tr1 - tr0;
        if (pf >= 0) ts[2] += tr1 - (tr0 + 0);
        // ---- phase 2: decide owned columns (warp per column)
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
                if (st != 0 && lane == 0) atomicMin(&hg->first[r % 3][0], pack4(j, st, from, to));
            }
        }
        // slot (r+1)%3 is next written after this barrier and last read before
        // barrier r-1 completed, so resetting it here cannot race
        if (blockIdx.x == 0 && tid == 0) hg->first[(r + 1) % 3][0] = ~0ULL;
        const unsigned long long td = gtimer();
        tph2 += td - tr1;
        ts[3] += td - tr1;
        grid_barrier(hg);
        const unsigned long long te = gtimer();
        ts[4] += te - td;
        // ---- settle (identically in every CTA)
        ++rounds;
        const unsigned long long f = __ldcg(&hg->first[r % 3][0]);
        if (pf >= 0) {
            if (tid == 0) {
                vs[pf] ^= 1;
                vs[pt] ^= 1;
            }
            pf = -1;
        }
        __syncthreads();
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
                        const double* cv = Cs + ((int64_t)vs[k] * c + k) * d;
                        double s = 0.0;
                        for (int64_t i = 0; i < d; ++i) {
                            const double t = colv(q, i) - __ldcg(cv + i);
                            s += t * t;
                        }
                        scratch[k] = s;
                    }
                    __syncthreads();
                    if (warp == 0) {
                        int t2 = -1;
                        auto iv = [&](int k, double& lo, double& hi, double& mid) {
                            mid = __ldcg(scratch + k);
                            lo = hi = mid;
                        };
                        const int s2 = hart_decide_warp_w(from, c, cnt, wa, wb, iv, t2);
                        if (lane == 0) {
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
                    const double a = (double)(nf - 1), b = (double)(nt + 1);
                    wa[from] = a / (a - 1.0);
                    wb[from] = a / (a + 1.0);
                    wa[to] = b / (b - 1.0);
                    wb[to] = b / (b + 1.0);
                    if (j >= jown && j < jown + nown) s_lab[j - jown] = to;
                }
                if (blockIdx.x == 0 && tid == 0) {
                    labels[j] = to;
                    hg->moves += 1;
                    hg->improved = 1;
                }
                pf = from;
                pt = to;
                pm = j;
                pnf = nf;
                pnt = nt;
            }
            cursor = j + 1;
        }
        __syncthreads();
        ts[5] += gtimer() - te;
        if (cursor >= bend && pf < 0) break;
        if (cursor >= bend) cursor = bend;  // one more round applies the pending update
    }
    if (tid == 0) {
        atomicMax(&hg->t_phase1_max, tph1);
        for (int q = 0; q < 6; ++q) atomicAdd(&hg->tmax[q], ts[q]);  // summed over CTAs
    }
    // every CTA is past its last read of the election slots: reset them for
    // the next block launch
    grid_barrier(hg);
    if (blockIdx.x == 0 && tid == 0)
        hg->first[0][0] = hg->first[1][0] = hg->first[2][0] = ~0ULL;
    // publish the replicated state
    if (blockIdx.x == 0) {
        for (int k = tid; k < c; k += blockDim.x) {
            counts[k] = cnt[k];
            ver[k] = vs[k];
        }
        if (tid == 0) {
            hg->cursor = cursor;
            hg->rounds += rounds;
            hg->t_kernel += gtimer() - tk0;
            hg->t_phase1 += tph1;
            hg->t_phase2 += tph2;
        }
    }
}

}  // namespace respca_dev
