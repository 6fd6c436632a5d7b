// ALM-loop kernels: the fused elementwise pass ("Pass F"), group sums, the
// per-iteration finalize, and the standalone building blocks.
//
// Data layout (HBM): X, L, S, Θ are column-major d×n of T (double or float),
// leading dimension d — the reference's DenseMatrix (matrix.hpp:26-31).
// Groups are held as a CSR member list (goff[c+1], members[n]) with members in
// ascending column order, i.e. GroupAssignment::group_indices()
// (matrix.cpp:49-55).  Per-group d-vectors (group sums G, centroids C) are
// d×c column-major doubles.
//
// Thread mapping of every ordered group reduction: one thread owns R
// consecutive rows of ONE group and walks that group's member columns in
// ascending order, so each (row, group) sum is accumulated in exactly the
// reference's order (solver.cpp:61-65, kmeans.cpp:70-75) while a warp reads a
// contiguous 32·R-element slice of each member column (coalesced, 128-bit for
// R=2 doubles).
#pragma once

#include <cuda_bf16.h>

#include "common.cuh"
#include "km.cuh"  // cp.async helpers

namespace respca_dev {

template <typename T, int R>
struct Vec;
template <>
struct Vec<double, 1> {
    double v[1];
    RESPCA_DEV void load(const double* p) { v[0] = __ldg(p); }
    RESPCA_DEV void load_cs(const double* p) { v[0] = __ldcs(p); }
    RESPCA_DEV static void store(double* p, const double (&a)[1]) { __stcs(p, a[0]); }
};
template <>
struct Vec<double, 2> {
    double v[2];
    RESPCA_DEV void load(const double* p) {
        double2 t = __ldg(reinterpret_cast<const double2*>(p));
        v[0] = t.x;
        v[1] = t.y;
    }
    RESPCA_DEV void load_cs(const double* p) {
        double2 t = __ldcs(reinterpret_cast<const double2*>(p));
        v[0] = t.x;
        v[1] = t.y;
    }
    RESPCA_DEV static void store(double* p, const double (&a)[2]) {
        __stcs(reinterpret_cast<double2*>(p), make_double2(a[0], a[1]));
    }
};
template <>
struct Vec<float, 1> {
    double v[1];
    RESPCA_DEV void load(const float* p) { v[0] = (double)__ldg(p); }
    RESPCA_DEV void load_cs(const float* p) { v[0] = (double)__ldcs(p); }
    RESPCA_DEV static void store(float* p, const double (&a)[1]) { __stcs(p, (float)a[0]); }
};
template <>
struct Vec<float, 2> {
    double v[2];
    RESPCA_DEV void load(const float* p) {
        float2 t = __ldg(reinterpret_cast<const float2*>(p));
        v[0] = t.x;
        v[1] = t.y;
    }
    RESPCA_DEV void load_cs(const float* p) {
        float2 t = __ldcs(reinterpret_cast<const float2*>(p));
        v[0] = t.x;
        v[1] = t.y;
    }
    RESPCA_DEV static void store(float* p, const double (&a)[2]) {
        __stcs(reinterpret_cast<float2*>(p), make_float2((float)a[0], (float)a[1]));
    }
};
template <>
struct Vec<float, 4> {
    double v[4];
    RESPCA_DEV void load(const float* p) {
        float4 t = __ldg(reinterpret_cast<const float4*>(p));
        v[0] = t.x;
        v[1] = t.y;
        v[2] = t.z;
        v[3] = t.w;
    }
    RESPCA_DEV void load_cs(const float* p) {
        float4 t = __ldcs(reinterpret_cast<const float4*>(p));
        v[0] = t.x;
        v[1] = t.y;
        v[2] = t.z;
        v[3] = t.w;
    }
    RESPCA_DEV static void store(float* p, const double (&a)[4]) {
        __stcs(reinterpret_cast<float4*>(p),
               make_float4((float)a[0], (float)a[1], (float)a[2], (float)a[3]));
    }
};

// ---------------------------------------------------------------------------
// Pass F: one fused HBM pass per ALM iteration (steady state).
//
// For every element of group g (labels_t), in the reference's op order:
//   q   = θ/ρ_t
//   D   = (x − s) + q                         solver.cpp:163-164
//   L'  = own_w·D + mean_w_g·G_t[i,g]         solver.cpp:72 (G_t = Σ_{j∈g} D_j)
//   B   = (x − L') + q                        solver.cpp:172-173
//   S'  = |B|−1/ρ > 0 ? copysign(|B|−1/ρ, B) : 0     solver.cpp:83-85
//   Θ'  = θ + ρ_t((x − L') − S')              solver.cpp:107-108
// and, in the same walk,
//   Cw[i,g]    = (Σ_{j∈g} L'_j)·(1/n_g)       = means_of(L', labels_t), the
//                                               kmeans_warm start (kmeans.cpp:257, 66-82)
//   Gnext[i,g] = Σ_{j∈g} ((x − S') + Θ'/ρ_{t+1})  = G_{t+1} if labels stay
//   partials   : Σ((x−L')−S')², Σ(L'−L_t)², Σ(S'−S_t)², Σ|S'|, Σ(L'−m̃_g)²
// Traffic: reads X, S, Θ, L_t; writes L', S', Θ' — 7·d·n·sizeof(T).
// L, S, Θ are updated in place (each element is owned by one thread).
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// Pass F for few groups (c·⌈d/512⌉ CTAs would not fill the GPU, e.g. c = 1):
// the same per-element work and member-order sums as k_pass_f, one thread per
// row, 64-thread CTAs, and each thread streams its row of the next U members'
// X, S, Θ, L through a private cp.async ring in shared memory — the member
// walk (sequential per row: the reference's summation order) keeps U·4
// elements in flight per thread instead of the few a register batch holds.
// ---------------------------------------------------------------------------
constexpr int PFR_T = 64;  // default CTA rows
constexpr int PFR_MC = 1024; // member indices staged in shared memory
RESPCA_DEV double abs_a(double v) { return fabs(v); }
RESPCA_DEV float abs_a(float v) { return fabsf(v); }
RESPCA_DEV double copysign_a(double m, double s) { return copysign(m, s); }
RESPCA_DEV float copysign_a(float m, float s) { return copysignf(m, s); }
RESPCA_DEV double min_a(double a, double b) { return fmin(a, b); }
RESPCA_DEV float min_a(float a, float b) { return fminf(a, b); }
template <typename T, int RW, typename A>
RESPCA_DEV void store_row(T* p, const A (&a)[RW]) {
    if constexpr (sizeof(T) == 8) {
        if constexpr (RW == 2) __stcs(reinterpret_cast<double2*>(p), make_double2(a[0], a[1]));
        else __stcs(p, (double)a[0]);
    } else {
        if constexpr (RW == 4) __stcs(reinterpret_cast<float4*>(p), make_float4((float)a[0], (float)a[1], (float)a[2], (float)a[3]));
        else if constexpr (RW == 2) __stcs(reinterpret_cast<float2*>(p), make_float2((float)a[0], (float)a[1]));
        else __stcs(p, (float)a[0]);
    }
}
// F32A (fp32 storage only): the element chain in FP32 arithmetic — fp32 mode's
// tolerance is 1e-4 of the fp64 reference and every stored value is rounded to
// FP32 anyway; the ordered group sums (Cw, G_{t+1}) and the residual partials
// still accumulate in FP64 (one widening per term / per batch).  Without it
// the kernel spends its issue slots on F2F conversions and FP64 operations
// (ncu: fp64 30 %, xu 30 % busy at 29 % occupancy) and stays at 0.69 of HBM.
template <typename T, int U, int NT = PFR_T, int B = 1, int RW = 1, bool F32A = false>
__global__ void __launch_bounds__(NT) k_pass_f_ring(
    const T* __restrict__ X, T* __restrict__ L, T* __restrict__ S, T* __restrict__ Th,
    const int* __restrict__ goff, const int* __restrict__ members, const double* G0, const double* G1,
    double* Gn0, double* Gn1, double* __restrict__ Cw, const double* __restrict__ mean_w,
    const Ctl* __restrict__ ctl, double* __restrict__ partials, int64_t d, int rowblocks,
    __nv_bfloat16* __restrict__ Lb, int64_t dpad) {
    static_assert(!F32A || sizeof(T) == 4, "FP32 arithmetic is for fp32 storage");
    using A = std::conditional_t<F32A, float, double>;  // arithmetic type of the element chain
    // RW rows per thread (RW = 2 needs d even): one 2·sizeof(T)-byte copy per
    // array and member, so a warp moves 32·RW·sizeof(T) contiguous bytes
    __shared__ double red[32 * 5];
    // the group's first PFR_MC member indices staged once per CTA: the walk's
    // addresses then come from shared memory instead of a dependent global load
    // per member (ncu: long_scoreboard was the top stall of the fp32 walk)
    // (kept to the four-row fp32 walk: C4 0.824 → 0.874 of HBM, C3-f32 +1 %; the fp64
    // walks lose 1–7 % to the extra barrier and branch)
    constexpr bool STAGE_M = F32A && RW == 4;
    __shared__ int mcol[STAGE_M ? PFR_MC : 1];
    extern __shared__ __align__(16) unsigned char pfr_sm[];
    auto ring = reinterpret_cast<T(*)[4][NT * RW]>(pfr_sm);  // [stage][X, S, Θ, L][row]
    pdl_enter();
    if (ctl->done) return;
    const int g = blockIdx.x / rowblocks;
    const int rb = blockIdx.x - g * rowblocks;
    const int tid = threadIdx.x;
    const int64_t i = ((int64_t)rb * NT + tid) * RW;
    const bool active = i < d;
    const int par = ctl->parity;
    const double* Gc = par ? G1 : G0;
    double* Gn = par ? Gn0 : Gn1;
    const double rho = ctl->rho, rho_n = ctl->rho_next, own_w = ctl->own_w, thr = ctl->thr;
    // fp32 storage only (its tolerance is 1e-4 of the fp64 reference): the two
    // FP64 divisions per element become multiplies by the reciprocals
    const double irn = sizeof(T) == 8 ? 0.0 : 1.0 / rho_n;
    const A rho_a = (A)rho, own_a = (A)own_w, thr_a = (A)thr, irn_a = (A)irn;
    const double mw = mean_w[g];
    const int beg = goff[g], end = goff[g + 1];
    const double ng = (double)(end - beg);
    const double mscale = own_w / ng + mw;
    if constexpr (STAGE_M) {
        for (int t = tid; t < PFR_MC && beg + t < end; t += NT) mcol[t] = __ldg(members + beg + t);
        __syncthreads();
    }
    auto member = [&](int t) -> int {
        if constexpr (STAGE_M) return t - beg < PFR_MC ? mcol[t - beg] : __ldg(members + t);
        else return __ldg(members + t);
    };
    double pf = 0.0, pl = 0.0, ps = 0.0, p1 = 0.0, psc = 0.0, smin = INFINITY;
    if (active) {
        double cacc[RW], gacc[RW];
        A gterm[RW], mt[RW];  // mean_w·G_t[i,g] (solver.cpp:72), m̃_g[i]
#pragma unroll
        for (int w = 0; w < RW; ++w) {
            const double Gi = Gc[(int64_t)g * d + i + w];
            gterm[w] = (A)(mw * Gi);
            mt[w] = (A)(Gi * mscale);
            cacc[w] = 0.0;
            gacc[w] = 0.0;
        }
        auto cp = [&](T* dst, const T* src, bool ok) {
            if (RW * sizeof(T) == 16) cp_async16(dst, ok ? src : X, ok ? 16 : 0);
            else if (RW * sizeof(T) == 8) cp_async8(dst, ok ? src : X, ok);
            else cp_async4(dst, ok ? src : X, ok);
        };
        auto issue = [&](int t) {
            const int slot = (t - beg) % U;
            const bool ok = t < end;
            const int64_t off = ok ? (int64_t)member(t) * d + i : 0;
            cp(&ring[slot][0][tid * RW], X + off, ok);
            cp(&ring[slot][1][tid * RW], S + off, ok);
            cp(&ring[slot][2][tid * RW], Th + off, ok);
            cp(&ring[slot][3][tid * RW], L + off, ok);
            cp_commit();
        };
        // batches of B members: their element chains are independent (ILP),
        // the sums take them in member order afterwards
        static_assert(U % B == 0 && U >= 2 * B, "ring");
        for (int t = beg; t < beg + U; ++t) issue(t);
        for (int t0 = beg; t0 < end; t0 += B) {
            cp_wait<U - B>();
            A xs[B][RW], ss[B][RW], ts[B][RW], lo[B][RW];
#pragma unroll
            for (int u = 0; u < B; ++u) {
                const int slot = (t0 + u - beg) % U;
#pragma unroll
                for (int w = 0; w < RW; ++w) {
                    xs[u][w] = (A)ring[slot][0][tid * RW + w];
                    ss[u][w] = (A)ring[slot][1][tid * RW + w];
                    ts[u][w] = (A)ring[slot][2][tid * RW + w];
                    lo[u][w] = (A)ring[slot][3][tid * RW + w];
                }
            }
            // this thread's reads of the B slots are done before they refill
#pragma unroll
            for (int u = 0; u < B; ++u) issue(t0 + U + u);
            A ln[B][RW], sn[B][RW], tn[B][RW], rr[B][RW], sm[B][RW], mg[B][RW];
#pragma unroll
            for (int u = 0; u < B; ++u)
#pragma unroll
                for (int w = 0; w < RW; ++w) {
                    // solver.cpp:163-164, 72, 172-173, 83-85, 107-108 (the reference's op order)
                    const A x = xs[u][w], s = ss[u][w], th = ts[u][w];
                    A q;
                    if constexpr (sizeof(T) == 8) q = th / rho;
                    else q = th * thr_a;  // fp32 storage: reciprocal (1e-4 tolerance)
                    const A dv = (x - s) + q;
                    ln[u][w] = own_a * dv + gterm[w];
                    const A xl = x - ln[u][w];
                    const A b = xl + q;
                    const A mag = abs_a(b) - thr_a;
                    mg[u][w] = abs_a(mag);
                    sn[u][w] = mag > (A)0 ? copysign_a(mag, b) : (A)0;
                    rr[u][w] = xl - sn[u][w];
                    tn[u][w] = th + rho_a * rr[u][w];
                    if constexpr (sizeof(T) == 8) sm[u][w] = (x - sn[u][w]) + tn[u][w] / rho_n;
                    else sm[u][w] = (x - sn[u][w]) + tn[u][w] * irn_a;
                }
            // residual partials of the batch in the arithmetic type, widened once per batch
            A bf = (A)0, bl = (A)0, bs = (A)0, b1 = (A)0, bsc = (A)0, bmin = (A)INFINITY;
#pragma unroll
            for (int u = 0; u < B; ++u) {
                if (t0 + u >= end) break;
                const int col = member(t0 + u);
                const int64_t off = (int64_t)col * d + i;
#pragma unroll
                for (int w = 0; w < RW; ++w) {
                    cacc[w] += (double)ln[u][w];  // ascending member order (solver.cpp:64, kmeans.cpp:73)
                    gacc[w] += (double)sm[u][w];
                    const A dl = ln[u][w] - lo[u][w];
                    const A ds = sn[u][w] - ss[u][w];
                    const A dm = ln[u][w] - mt[w];
                    if constexpr (F32A) {
                        bf += rr[u][w] * rr[u][w];
                        bl += dl * dl;
                        bs += ds * ds;
                        b1 += abs_a(sn[u][w]);
                        bsc += dm * dm;
                        bmin = min_a(bmin, mg[u][w]);
                    } else {
                        pf += rr[u][w] * rr[u][w];
                        pl += dl * dl;
                        ps += ds * ds;
                        p1 += abs_a(sn[u][w]);
                        psc += dm * dm;
                        smin = fmin(smin, mg[u][w]);
                    }
                }
                store_row<T, RW, A>(L + off, ln[u]);
                store_row<T, RW, A>(S + off, sn[u]);
                store_row<T, RW, A>(Th + off, tn[u]);
                if (Lb) {
                    __nv_bfloat16* lb = Lb + (int64_t)col * dpad + i;
                    if (RW >= 2) {
#pragma unroll
                        for (int w = 0; w + 1 < RW; w += 2) {
                            __nv_bfloat162 b2;
                            if constexpr (F32A) {
                                b2 = __floats2bfloat162_rn(ln[u][w], ln[u][w + 1]);
                            } else {
                                b2.x = __double2bfloat16(ln[u][w]);
                                b2.y = __double2bfloat16(ln[u][w + 1]);
                            }
                            *reinterpret_cast<__nv_bfloat162*>(lb + w) = b2;
                        }
                    } else {
                        if constexpr (F32A) lb[0] = __float2bfloat16(ln[u][0]);
                        else lb[0] = __double2bfloat16(ln[u][0]);
                    }
                }
            }
            if constexpr (F32A) {
                pf += (double)bf;
                pl += (double)bl;
                ps += (double)bs;
                p1 += (double)b1;
                psc += (double)bsc;
                smin = fmin(smin, (double)bmin);
            }
        }
        cp_wait<0>();
#pragma unroll
        for (int w = 0; w < RW; ++w) {
            Cw[(int64_t)g * d + i + w] = cacc[w] * (1.0 / ng);  // kmeans.cpp:78-79
            Gn[(int64_t)g * d + i + w] = gacc[w];
        }
    }
    double v[5] = {pf, pl, ps, p1, psc};
    block_sum<5>(v, red);
    const double mn = block_min(smin, red);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < 5; ++q) partials[(int64_t)blockIdx.x * PF_STRIDE + q] = v[q];
        partials[(int64_t)blockIdx.x * PF_STRIDE + 5] = mn;
    }
}

template <typename T>
RESPCA_DEV void store_vec16(T* p, const double* a);
template <>
RESPCA_DEV void store_vec16<double>(double* p, const double* a) {
    __stcs(reinterpret_cast<double2*>(p), make_double2(a[0], a[1]));
}
template <>
RESPCA_DEV void store_vec16<float>(float* p, const double* a) {
    __stcs(reinterpret_cast<float4*>(p), make_float4((float)a[0], (float)a[1], (float)a[2], (float)a[3]));
}

// ---------------------------------------------------------------------------
// Pass F as streams: one CTA per (group g, block of rb rows) walks g's members
// in ascending order, so each row's two running sums stay inside one CTA (no
// cross-CTA hand-off), while the element work of a stage of mps members is
// spread over all 256 threads (a thread owns K 16-byte chunks = K·VEC rows of
// one member each) — what the one-thread-per-row walk of k_pass_f_ring lacks
// when d is small relative to the GPU (C3-c1: 10⁴ rows for 148 SMs).
//
// rb is a runtime multiple of VEC (16-byte aligned segments since d % VEC == 0),
// chosen by the host so that the c·⌈d/rb⌉ streams fill whole waves of the
// resident CTAs (c = 1: one wave, every stream runs the whole time).
//
// Pipeline: NS stages of X, S, Θ, L [mps][rb] staged by cp.async, NS − 1 in
// flight while one is computed.  A thread loads and later reads only its own
// chunks of every stage (fixed chunk positions), so the stages need no
// barrier.  The two summands of each element go to a double-buffered shared
// array; after one __syncthreads per stage, warp 0 adds them in member order
// (lane = row, RPL rows per lane) while the other warps go on to the next
// stage.  Member indices are staged one stage ahead (a register prefetch
// plus a per-thread shared slot), so no address waits on a global load.
// ---------------------------------------------------------------------------
template <typename T, int K, int NS, int RBMAX>
struct StreamCfg {
    static constexpr int VEC = 16 / (int)sizeof(T);
    static constexpr int CPS = 256 * K;  // 16-byte chunks per stage (all arrays count once)
    static constexpr int RPL = RBMAX / 32;
    static constexpr int SMEM = NS * 4 * CPS * 16 + 2 * 2 * CPS * VEC * 8 + NS * CPS * 4;
};

RESPCA_DEV void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }
RESPCA_DEV void named_bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }

// the stream kernel's chain warp (RP rows per lane): per stage, wait for the
// element warps' summands (FULL), add them in member order, release (EMPTY)
template <int RP>
RESPCA_DEV void stream_chain(const double* summ, int half, int rb_rows, int nst, int m, int mps, int lane,
                             int64_t r0, int64_t d, int g, double ng, double* __restrict__ Cw,
                             double* __restrict__ Gn) {
    constexpr int BAR_FULL = 1, BAR_EMPTY = 3, NT = 288;
    double a[RP], b[RP];
    int rl[RP];
#pragma unroll
    for (int q = 0; q < RP; ++q) {
        a[q] = b[q] = 0.0;
        rl[q] = (lane + 32 * q) < rb_rows ? lane + 32 * q : 0;
    }
    for (int s = 0; s < nst; ++s) {
        named_bar_sync(BAR_FULL + (s & 1), NT);
        const double* y0 = summ + (size_t)(s & 1) * 2 * half;
        const double* y1 = y0 + half;
        const int cnt = m - s * mps < mps ? m - s * mps : mps;
#pragma unroll 4
        for (int u = 0; u < cnt; ++u)
#pragma unroll
            for (int q = 0; q < RP; ++q) {
                a[q] += y0[u * rb_rows + rl[q]];  // ascending member order (solver.cpp:64, kmeans.cpp:73)
                b[q] += y1[u * rb_rows + rl[q]];
            }
        if (s + 2 < nst) named_bar_arrive(BAR_EMPTY + (s & 1), NT);
    }
#pragma unroll
    for (int q = 0; q < RP; ++q) {
        const int r_ = lane + 32 * q;
        if (r_ < rb_rows && r0 + r_ < d) {
            Cw[(int64_t)g * d + r0 + r_] = a[q] * (1.0 / ng);  // kmeans.cpp:78-79
            Gn[(int64_t)g * d + r0 + r_] = b[q];
        }
    }
}

constexpr int PFS_THREADS = 288;  // 8 element warps + 1 chain warp
template <typename T, int K, int NS, int RBMAX>
__global__ void __launch_bounds__(PFS_THREADS, NS <= 3 ? 3 : 2) k_pass_f_stream(
    const T* __restrict__ X, T* __restrict__ L, T* __restrict__ S, T* __restrict__ Th,
    const int* __restrict__ goff, const int* __restrict__ members, const int* __restrict__ gorder,
    const double* G0, const double* G1, double* Gn0, double* Gn1, double* __restrict__ Cw,
    const double* __restrict__ mean_w, const Ctl* __restrict__ ctl, double* __restrict__ partials,
    int64_t d, int rb_rows, int nrb, __nv_bfloat16* __restrict__ Lb, int64_t dpad, int ident) {
    // ident: every group's members are consecutive columns (c = 1: the one group
    // is 0..n−1), so a member index is gb + position and needs no load
    using C = StreamCfg<T, K, NS, RBMAX>;
    constexpr int VEC = C::VEC, CPS = C::CPS, RPL = C::RPL;
    static_assert(RBMAX % 32 == 0 && RBMAX / VEC <= CPS, "stream tile");
    // named barriers: FULL[b] (element warps → chain warp), EMPTY[b] (back)
    constexpr int BAR_FULL = 1, BAR_EMPTY = 3;
    extern __shared__ __align__(16) unsigned char pfs_sm[];
    // stage s, array a, chunk k: 16 bytes at ((s·4 + a)·CPS + k)·16
    unsigned char* stg = pfs_sm;
    double* summ = reinterpret_cast<double*>(pfs_sm + NS * 4 * CPS * 16);  // [2 bufs][2][CPS·VEC]
    int* scol = reinterpret_cast<int*>(pfs_sm + NS * 4 * CPS * 16 + 2 * 2 * CPS * VEC * 8);  // [NS][CPS]
    __shared__ double red[32 * 5];
    pdl_enter();
    if (ctl->done) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gi = blockIdx.x / nrb;
    const int rbi = blockIdx.x - gi * nrb;
    const int g = gorder ? __ldg(gorder + gi) : gi;  // longest member walks first
    const int lpc = rb_rows / VEC;                    // chunks per member segment
    const int mps = CPS / lpc;                        // members per stage
    const int64_t r0 = (int64_t)rbi * rb_rows;
    const int par = ctl->parity;
    const double* Gc = par ? G1 : G0;
    double* Gn = par ? Gn0 : Gn1;
    const double rho = ctl->rho, rho_n = ctl->rho_next, own_w = ctl->own_w, thr = ctl->thr;
    const double irn = sizeof(T) == 8 ? 0.0 : 1.0 / rho_n;  // fp32 storage: reciprocal multiplies
    const double mw = mean_w[g];
    const int gb = __ldg(goff + g), ge = __ldg(goff + g + 1);
    const int m = ge - gb;
    const int nst = (m + mps - 1) / mps;
    const double ng = (double)m;
    double pf = 0.0, pl = 0.0, ps = 0.0, p1 = 0.0, psc = 0.0, smin = INFINITY;
    if (warp < 8) {
        // ================= element warps =================
        const double mscale = own_w / ng + mw;
        // this thread's chunks (the same positions in every stage)
        int cmem[K], csub[K];
        bool crow[K];
        double Gi[K][VEC], mt[K][VEC];
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const int k = tid + 256 * j;
            cmem[j] = k / lpc;
            csub[j] = k - cmem[j] * lpc;
            crow[j] = cmem[j] < mps && r0 + csub[j] * VEC < d;
            const int64_t row = r0 + csub[j] * VEC;
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
                Gi[j][v] = crow[j] ? Gc[(int64_t)g * d + row + v] : 0.0;
                mt[j][v] = Gi[j][v] * mscale;
            }
        }
        // member index of chunk j in stage s (−1: none)
        auto member_of = [&](int s, int j) -> int {
            const int c_ = s * mps + cmem[j];
            return (s < nst && crow[j] && c_ < m) ? (ident ? gb + c_ : __ldg(members + gb + c_)) : -1;
        };
        auto issue = [&](int s, const int (&col)[K]) {
            if (s < nst) {
#pragma unroll
                for (int j = 0; j < K; ++j) {
                    const int k = tid + 256 * j;
                    const bool ok = col[j] >= 0;
                    const int64_t off = ok ? (int64_t)col[j] * d + r0 + csub[j] * VEC : 0;
                    const int nb = ok ? 16 : 0;
                    unsigned char* base = stg + (size_t)(s % NS) * 4 * CPS * 16 + (size_t)k * 16;
                    cp_async16(base, X + off, nb);
                    cp_async16(base + CPS * 16, S + off, nb);
                    cp_async16(base + 2 * CPS * 16, Th + off, nb);
                    cp_async16(base + 3 * CPS * 16, L + off, nb);
                    scol[(s % NS) * CPS + k] = col[j];
                }
            }
            cp_commit();  // one group per stage, empty past the end
        };
        int nxt[K];
#pragma unroll
        for (int s = 0; s < NS - 1; ++s) {
            int col[K];
#pragma unroll
            for (int j = 0; j < K; ++j) col[j] = member_of(s, j);
            issue(s, col);
        }
#pragma unroll
        for (int j = 0; j < K; ++j) nxt[j] = member_of(NS - 1, j);
        for (int s = 0; s < nst; ++s) {
            issue(s + NS - 1, nxt);
#pragma unroll
            for (int j = 0; j < K; ++j) nxt[j] = member_of(s + NS, j);  // consumed next stage
            cp_wait<NS - 1>();  // this thread's chunks of stage s have landed
            if (s >= 2) named_bar_sync(BAR_EMPTY + (s & 1), PFS_THREADS);  // chain of stage s − 2 done
            double* sm_ = summ + (size_t)(s & 1) * 2 * CPS * VEC;
#pragma unroll
            for (int j = 0; j < K; ++j) {
                // a chunk past the stage's members (mps·lpc < CPS), or of rows past d in the
                // last, partial row block: nothing to compute.  (Computing on their
                // zero-filled tiles sent both divisions down the IEEE slow path — 0/ρ — so
                // that one stream ran ≈1.5× longer than the others and, every stream
                // lasting the whole kernel, so did the launch: C3-c1 rb = 32 0.48 of HBM,
                // against 0.75 at rb = 40 with d % rb = 0.)
                if (!crow[j]) continue;
                const int k = tid + 256 * j;
                const unsigned char* base = stg + (size_t)(s % NS) * 4 * CPS * 16 + (size_t)k * 16;
                const T* xs = reinterpret_cast<const T*>(base);
                const T* ss = reinterpret_cast<const T*>(base + CPS * 16);
                const T* ts = reinterpret_cast<const T*>(base + 2 * CPS * 16);
                const T* ls = reinterpret_cast<const T*>(base + 3 * CPS * 16);
                const int col = scol[(s % NS) * CPS + k];
                const bool ok = col >= 0;
                double lo_[VEC], so_[VEC], to_[VEC], gs_[VEC];
#pragma unroll
                for (int v = 0; v < VEC; ++v) {
                    // solver.cpp:163-164, 72, 172-173, 83-85, 107-108 (op order as k_pass_f)
                    const double x = (double)xs[v], sv = (double)ss[v], th = (double)ts[v], lp = (double)ls[v];
                    const double qq = sizeof(T) == 8 ? th / rho : th * thr;  // fp32 storage: reciprocal
                    const double dv = (x - sv) + qq;
                    const double ln = own_w * dv + mw * Gi[j][v];
                    const double xl = x - ln;
                    const double bb = xl + qq;
                    const double mag = fabs(bb) - thr;
                    const double sn = mag > 0.0 ? copysign(mag, bb) : 0.0;
                    const double r = xl - sn;
                    const double tn = th + rho * r;
                    if (ok) smin = fmin(smin, fabs(mag));
                    gs_[v] = (x - sn) + (sizeof(T) == 8 ? tn / rho_n : tn * irn);
                    lo_[v] = ln;
                    so_[v] = sn;
                    to_[v] = tn;
                    if (ok) {
                        pf += r * r;
                        const double dl = ln - lp;
                        pl += dl * dl;
                        const double ds = sn - sv;
                        ps += ds * ds;
                        p1 += fabs(sn);
                        const double dm = ln - mt[j][v];
                        psc += dm * dm;
                    }
                }
                {   // summand layout [2][member][row of the block]; 16-byte stores (rb_rows % VEC == 0)
                    const int e = cmem[j] * rb_rows + csub[j] * VEC;
#pragma unroll
                    for (int v = 0; v < VEC; v += 2) {
                        *reinterpret_cast<double2*>(sm_ + e + v) = make_double2(lo_[v], lo_[v + 1]);
                        *reinterpret_cast<double2*>(sm_ + CPS * VEC + e + v) = make_double2(gs_[v], gs_[v + 1]);
                    }
                }
                if (ok) {
                    const int64_t off = (int64_t)col * d + r0 + csub[j] * VEC;
                    store_vec16<T>(L + off, lo_);
                    store_vec16<T>(S + off, so_);
                    store_vec16<T>(Th + off, to_);
                    if (Lb) {
                        __nv_bfloat16* lb = Lb + (int64_t)col * dpad + r0 + csub[j] * VEC;
#pragma unroll
                        for (int v = 0; v < VEC; v += 2) {
                            __nv_bfloat162 b2;
                            b2.x = __double2bfloat16(lo_[v]);
                            b2.y = __double2bfloat16(lo_[v + 1]);
                            *reinterpret_cast<__nv_bfloat162*>(lb + v) = b2;
                        }
                    }
                }
            }
            named_bar_arrive(BAR_FULL + (s & 1), PFS_THREADS);  // stage s's summands are in place
        }
        cp_wait<0>();
    } else {
        // ================= the chain warp: each row's two sums in member order =================
        // (instantiated for the rows per lane this stream needs: no idle chains)
        const int rpl = (rb_rows + 31) / 32;
        auto run = [&](auto rplc) {
            constexpr int RP = decltype(rplc)::value;
            stream_chain<RP>(summ, CPS * VEC, rb_rows, nst, m, mps, lane, r0, d, g, ng, Cw, Gn);
        };
        if (rpl <= 1) run(std::integral_constant<int, 1>{});
        else if (rpl == 2) run(std::integral_constant<int, 2>{});
        else if (rpl <= 4 || RPL <= 4) run(std::integral_constant<int, (RPL < 4 ? RPL : 4)>{});
        else run(std::integral_constant<int, RPL>{});
    }
    double pv[5] = {pf, pl, ps, p1, psc};
    block_sum<5>(pv, red);
    const double mn = block_min(smin, red);
    if (tid == 0) {
#pragma unroll
        for (int q = 0; q < 5; ++q) partials[(int64_t)blockIdx.x * PF_STRIDE + q] = pv[q];
        partials[(int64_t)blockIdx.x * PF_STRIDE + 5] = mn;
    }
}

// ---------------------------------------------------------------------------
// ℓ2,1 variant of the iteration (sparse_norm = L21, solver.cpp:90-102), split
// around the column norms of B that the shrinkage needs:
//   F1: D-form, L' (+ Cw sums, dL and scatter partials)          reads 4N, writes 1N
//   column norms ‖B_j‖ = sqrt(Σ_i B_ij²), B = (x − L') + θ/ρ, sequential over i
//   F2: S' = ‖B_j‖ <= 1/ρ ? 0 : (1 − (1/ρ)/‖B_j‖)·B_j, Θ', G_{t+1}, feas/dS partials
// ---------------------------------------------------------------------------
template <typename T, int R>
__global__ void __launch_bounds__(256) k_pass_f1(
    const T* __restrict__ X, T* __restrict__ L, const T* __restrict__ S, const T* __restrict__ Th,
    const int* __restrict__ goff, const int* __restrict__ members, const double* G0,
    const double* G1, double* __restrict__ Cw, const double* __restrict__ mean_w,
    const Ctl* __restrict__ ctl, double* __restrict__ partials, int64_t d, int rowblocks) {
    __shared__ double red[32 * 5];
    if (ctl->done) return;
    const int g = blockIdx.x / rowblocks;
    const int rb = blockIdx.x - g * rowblocks;
    const int64_t i0 = ((int64_t)rb * blockDim.x + threadIdx.x) * R;
    const bool active = i0 < d;
    const double* Gc = ctl->parity ? G1 : G0;
    const double rho = ctl->rho, own_w = ctl->own_w, mw = mean_w[g];
    const int beg = goff[g], end = goff[g + 1];
    const double ng = (double)(end - beg);
    const double mscale = own_w / ng + mw;
    double pl = 0.0, psc = 0.0;
    if (active) {
        double G[R], cacc[R], mt[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            G[r] = Gc[(int64_t)g * d + i0 + r];
            mt[r] = G[r] * mscale;
            cacc[r] = 0.0;
        }
        for (int t = beg; t < end; ++t) {
            const int64_t off = (int64_t)__ldg(members + t) * d + i0;
            Vec<T, R> xv, sv, tv, lv;
            xv.load(X + off);
            sv.load(S + off);
            tv.load(Th + off);
            lv.load_cs(L + off);
            double lo[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double dv = (xv.v[r] - sv.v[r]) + tv.v[r] / rho;   // solver.cpp:163-164
                const double ln = own_w * dv + mw * G[r];                   // solver.cpp:72
                cacc[r] += ln;
                const double dl = ln - lv.v[r];
                pl += dl * dl;
                const double dm = ln - mt[r];
                psc += dm * dm;
                lo[r] = ln;
            }
            Vec<T, R>::store(L + off, lo);
        }
        const double inv = 1.0 / ng;
#pragma unroll
        for (int r = 0; r < R; ++r) Cw[(int64_t)g * d + i0 + r] = cacc[r] * inv;
    }
    double v[5] = {0.0, pl, 0.0, 0.0, psc};
    block_sum<5>(v, red);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < 5; ++q) partials[(int64_t)blockIdx.x * PF_STRIDE + q] = v[q];
        partials[(int64_t)blockIdx.x * PF_STRIDE + 5] = INFINITY;  // ℓ2,1: k_l21_term's column margin
    }
}

// ‖B_j‖ for the ℓ2,1 shrinkage: exact sequential chain per column, warp-
// transposed tiles (lane = column), ρ read from the control block
template <typename T>
__global__ void __launch_bounds__(128) k_bnorms(const T* __restrict__ X, const T* __restrict__ L,
                                                const T* __restrict__ Th,
                                                const Ctl* __restrict__ ctl, int64_t d, int64_t n,
                                                double* __restrict__ out) {
    __shared__ double tile[4][32][33];
    if (ctl->done) return;
    const double rho = ctl->rho;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t j0 = ((int64_t)blockIdx.x * 4 + w) * 32;
    if (j0 >= n) return;
    double acc = 0.0;
    for (int64_t i0 = 0; i0 < d; i0 += 32) {
        const int64_t i = i0 + lane;
        for (int cc = 0; cc < 32; ++cc) {
            const int64_t j = j0 + cc;
            double v = 0.0;
            if (j < n && i < d) {
                const int64_t e = j * d + i;
                v = (ld(X + e) - ld(L + e)) + ld(Th + e) / rho;  // solver.cpp:172-173
            }
            tile[w][cc][lane] = v;
        }
        __syncwarp();
        const int lim = (int)((d - i0) < 32 ? (d - i0) : 32);
        for (int r = 0; r < lim; ++r) {
            const double v = tile[w][lane][r];
            acc += v * v;  // column_l2_norms, matrix.cpp:117-125
        }
        __syncwarp();
    }
    if (j0 + lane < n) out[j0 + lane] = sqrt(acc);
}

template <typename T, int R>
__global__ void __launch_bounds__(256) k_pass_f2(
    const T* __restrict__ X, const T* __restrict__ L, T* __restrict__ S, T* __restrict__ Th,
    const int* __restrict__ goff, const int* __restrict__ members, const double* __restrict__ bn,
    double* Gn0, double* Gn1, const Ctl* __restrict__ ctl, double* __restrict__ partials,
    int64_t d, int rowblocks) {
    __shared__ double red[32 * 5];
    if (ctl->done) return;
    const int g = blockIdx.x / rowblocks;
    const int rb = blockIdx.x - g * rowblocks;
    const int64_t i0 = ((int64_t)rb * blockDim.x + threadIdx.x) * R;
    const bool active = i0 < d;
    double* Gn = ctl->parity ? Gn0 : Gn1;
    const double rho = ctl->rho, rho_n = ctl->rho_next, thr = ctl->thr;
    const int beg = goff[g], end = goff[g + 1];
    double pf = 0.0, ps = 0.0;
    if (active) {
        double gacc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) gacc[r] = 0.0;
        for (int t = beg; t < end; ++t) {
            const int jm = __ldg(members + t);
            const int64_t off = (int64_t)jm * d + i0;
            const double nrm = __ldg(bn + jm);
            const bool zero = nrm <= thr;                        // solver.cpp:95
            const double scale = zero ? 0.0 : 1.0 - thr / nrm;   // solver.cpp:96
            Vec<T, R> xv, lv, sv, tv;
            xv.load(X + off);
            lv.load(L + off);
            sv.load_cs(S + off);
            tv.load_cs(Th + off);
            double so[R], to[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double x = xv.v[r], th = tv.v[r];
                const double xl = x - lv.v[r];
                const double b = xl + th / rho;
                const double sn = zero ? 0.0 : scale * b;        // solver.cpp:99
                const double rr = xl - sn;
                const double tn = th + rho * rr;                 // solver.cpp:107-108
                gacc[r] += (x - sn) + tn / rho_n;
                pf += rr * rr;
                const double ds = sn - sv.v[r];
                ps += ds * ds;
                so[r] = sn;
                to[r] = tn;
            }
            Vec<T, R>::store(S + off, so);
            Vec<T, R>::store(Th + off, to);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) Gn[(int64_t)g * d + i0 + r] = gacc[r];
    }
    double v[2] = {pf, ps};
    block_sum<2>(v, red);
    if (threadIdx.x == 0) {
        partials[(int64_t)blockIdx.x * PF_STRIDE + 0] += v[0];
        partials[(int64_t)blockIdx.x * PF_STRIDE + 2] += v[1];
    }
}

// Σ_j ‖S'_j‖ (report-only ℓ2,1 term): ‖S'_j‖ = max(0, 1 − t/‖B_j‖)·‖B_j‖
__global__ void k_l21_term(const double* __restrict__ bn, int64_t n, Ctl* __restrict__ ctl) {
    __shared__ double red[32];
    if (ctl->done) return;
    const double thr = ctl->thr;
    double s = 0.0, mn = INFINITY;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
        const double nr = bn[j];
        if (!(nr <= thr)) s += (1.0 - thr / nr) * nr;
        mn = fmin(mn, fabs(nr - thr));  // the column's support decision margin (solver.cpp:95)
    }
    double v[1] = {s};
    block_sum<1>(v, red);
    mn = block_min(mn, red);
    if (threadIdx.x == 0) {
        ctl->sparse_term = v[0];
        ctl->l21_smin = mn;
    }
}

// ---------------------------------------------------------------------------
// Ordered group sums: out[i,g] = Σ_{j∈g, ascending} f(j, i), with
//   mode 0 (D-form):  f = (x − s) + θ/ρ   (solver.cpp:163-164, summed at 61-65)
//   mode 1 (plain):   f = m[i,j]          (means_of / column_mean sums, kmeans.cpp:70-75)
// then optionally scaled by (1/n_g) (means_of, kmeans.cpp:76-80).
// ---------------------------------------------------------------------------
template <typename T, int R, int MODE>
__global__ void __launch_bounds__(256) k_group_sum(
    const T* __restrict__ X, const T* __restrict__ S, const T* __restrict__ Th,
    const int* __restrict__ goff, const int* __restrict__ members, const Ctl* __restrict__ ctl,
    double* __restrict__ out0, double* __restrict__ out1, int use_parity, int scale_by_count,
    int64_t d, int rowblocks, const int* __restrict__ gorder = nullptr) {
    // gorder: groups largest first (the longest member walks start first)
    const int gi = blockIdx.x / rowblocks;
    const int rb = blockIdx.x - gi * rowblocks;
    const int g = gorder ? __ldg(gorder + gi) : gi;
    const int64_t i0 = ((int64_t)rb * blockDim.x + threadIdx.x) * R;
    if (i0 >= d) return;
    double* __restrict__ out = (use_parity && ctl->parity) ? out1 : out0;
    const double rho = MODE == 0 ? ctl->rho : 1.0;
    const int beg = goff[g], end = goff[g + 1];
    double acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0;
    int t = beg;
    constexpr int U = MODE == 1 ? 8 : 4;
    for (; t + U <= end; t += U) {
        Vec<T, R> xv[U], sv[U], tv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t off = (int64_t)__ldg(members + t + u) * d + i0;
            xv[u].load(X + off);
            if (MODE == 0) {
                sv[u].load(S + off);
                tv[u].load(Th + off);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int r = 0; r < R; ++r)
                acc[r] += MODE == 0 ? (xv[u].v[r] - sv[u].v[r]) + tv[u].v[r] / rho : xv[u].v[r];
    }
    for (; t < end; ++t) {
        const int64_t off = (int64_t)__ldg(members + t) * d + i0;
        Vec<T, R> xv, sv, tv;
        xv.load(X + off);
        if (MODE == 0) {
            sv.load(S + off);
            tv.load(Th + off);
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
            acc[r] += MODE == 0 ? (xv.v[r] - sv.v[r]) + tv.v[r] / rho : xv.v[r];
    }
    const double inv = scale_by_count ? 1.0 / (double)(end - beg) : 1.0;
#pragma unroll
    for (int r = 0; r < R; ++r) out[(int64_t)g * d + i0 + r] = scale_by_count ? acc[r] * inv : acc[r];
}

// means_of (kmeans.cpp:66-82): out[i,g] = (Σ_{j∈g, ascending} m[i,j]) · (1/n_g).
// Each row's sum is a sequential chain over the group's members, so the only
// parallelism is over rows (and groups): a thread owns one row and keeps U
// member columns in flight (their indices staged in shared memory one batch
// ahead), so even the largest group — whose chains bound the kernel — streams
// at d·U·8 bytes in flight.  gorder: groups largest first.
constexpr int MS_U = 32, MS_T = 64;
template <typename T>
__global__ void __launch_bounds__(MS_T, 8) k_means_sum(const T* __restrict__ M, const int* __restrict__ goff,
                                                       const int* __restrict__ members,
                                                       const int* __restrict__ gorder, double* __restrict__ out,
                                                       int64_t d, int rowblocks, int scale = 1) {
    __shared__ int sidx[2][MS_U];
    const int gi = blockIdx.x / rowblocks;
    const int rb = blockIdx.x - gi * rowblocks;
    const int g = gorder ? __ldg(gorder + gi) : gi;
    const int64_t i = (int64_t)rb * MS_T + threadIdx.x;
    const bool row = i < d;
    const int beg = __ldg(goff + g), end = __ldg(goff + g + 1);
    double acc = 0.0;
    if (threadIdx.x < MS_U) sidx[0][threadIdx.x] = beg + (int)threadIdx.x < end ? __ldg(members + beg + threadIdx.x) : 0;
    __syncthreads();
    int b = 0;
    for (int t = beg; t < end; t += MS_U, b ^= 1) {
        double x[MS_U];
#pragma unroll
        for (int u = 0; u < MS_U; ++u)
            x[u] = (row && t + u < end) ? (double)__ldg(M + (int64_t)sidx[b][u] * d + i) : 0.0;
        if (threadIdx.x < MS_U) {  // the next batch's indices
            const int q = t + MS_U + (int)threadIdx.x;
            sidx[b ^ 1][threadIdx.x] = q < end ? __ldg(members + q) : 0;
        }
#pragma unroll
        for (int u = 0; u < MS_U; ++u)
            if (t + u < end) acc += x[u];  // ascending member order (kmeans.cpp:73)
        __syncthreads();
    }
    if (row) out[(int64_t)g * d + i] = scale ? acc * (1.0 / (double)(end - beg)) : acc;  // kmeans.cpp:78
}

// ---------------------------------------------------------------------------
// Finalize (one block): fixed-order combination of the Pass F partials, the
// report row, the stopping rule, and the scalars of iteration t+1.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_finalize(Ctl* __restrict__ ctl,
                                                   const double* __restrict__ partials,
                                                   int nparts, const int* __restrict__ goff,
                                                   double* __restrict__ mean_w, int c,
                                                   double* __restrict__ rep, int has_cond,
                                                   cudaGraphConditionalHandle cond,
                                                   double* __restrict__ marg) {
    __shared__ double red[32 * 5];
    pdl_enter();
    if (ctl->done) {
        if (threadIdx.x == 0 && has_cond) cudaGraphSetConditional(cond, 0u);
        return;
    }
    double v[5] = {0, 0, 0, 0, 0};
    double mn = INFINITY;
    for (int b = threadIdx.x; b < nparts; b += blockDim.x) {
#pragma unroll
        for (int q = 0; q < 5; ++q) v[q] += partials[(int64_t)b * PF_STRIDE + q];
        mn = fmin(mn, partials[(int64_t)b * PF_STRIDE + 5]);
    }
    block_sum<5>(v, red);
    mn = block_min(mn, red);
    __shared__ int s_done;
    if (threadIdx.x == 0) {
        Ctl& k = *ctl;
        const int t = k.iter;
        // fast-path verdict of Pass A (k_decide's counts): a label change or a
        // Hartigan move sends this iteration to the exact slow path
        if (k.changed || k.moves) k.slow = 1;
        const double feas = sqrt(v[0]) / k.xnorm;  // solver.cpp:20, 30
        const double dl = sqrt(v[1]) / k.xnorm;
        const double ds = sqrt(v[2]) / k.xnorm;
        const double sparse = k.l21 ? k.sparse_term : v[3];  // elementwise_l1 | l21_norm
        const double obj = k.lambda * v[4] + sparse;  // solver.cpp:191-195
        k.last_l1 = sparse;
        k.changed = 0;
        k.moves = 0;
        k.ambiguous = 0;
        rep[(int64_t)t * 4 + 0] = feas;
        rep[(int64_t)t * 4 + 1] = dl;
        rep[(int64_t)t * 4 + 2] = ds;
        rep[(int64_t)t * 4 + 3] = obj;
        // S-support margin of iteration t: min ||B| − 1/ρ|·ρ (solver.cpp:85 / 95)
        marg[t] = (k.l21 ? fmin(mn, k.l21_smin) : mn) / k.thr;
        if (!isfinite(feas) || !isfinite(dl) || !isfinite(ds)) k.nonfinite = 1;
        double mx = feas;  // std::max({feas, dl, ds})
        if (mx < dl) mx = dl;
        if (mx < ds) mx = ds;
        if (!k.fixed && !k.nonfinite) {  // solver.cpp:197
            if (!k.guard) {
                if (mx <= k.tol) k.converged = 1;
            } else if (k.force_exact) {
                k.stop_amb = 1;
            } else {
                // the reference's sums lie in [v·(1−ε), v·(1+ε)] (rounded outwards);
                // correctly rounded sqrt and / are monotone, so its residuals lie in
                // [sqrt(lo)/xn_hi, sqrt(hi)/xn_lo]
                const double om = __dadd_rd(1.0, -k.sum_eps), op = __dadd_ru(1.0, k.sum_eps);
                double lo = 0.0, hi = 0.0;
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const double a = sqrt(__dmul_rd(v[q], om)) / k.xn_hi;
                    const double b = sqrt(__dmul_ru(v[q], op)) / k.xn_lo;
                    lo = lo < a ? a : lo;
                    hi = hi < b ? b : hi;
                }
                if (hi <= k.tol) k.converged = 1;
                else if (!(lo > k.tol)) k.stop_amb = 1;  // decided on the chains (host)
            }
        }
        k.iter = t + 1;
        // advance ρ and the derived scalars to iteration t+1
        const double rho = k.rho_next;
        k.rho = rho;
        const double rn = rho * k.kappa;
        k.rho_next = (1e12 < rn) ? 1e12 : rn;  // std::min(ρκ, kRhoCap)
        const double two_lam = 2.0 * k.lambda;
        k.own_w = rho / (two_lam + rho);
        k.thr = 1.0 / rho;
        k.parity ^= 1;
        const int done = k.converged || k.slow || k.nonfinite || k.stop_amb || (t + 1 >= k.budget);
        k.done = done;
        s_done = done;
        if (has_cond) cudaGraphSetConditional(cond, done ? 0u : 1u);
    }
    __syncthreads();
    const double rho = ctl->rho, two_lam = 2.0 * ctl->lambda;
    for (int g = threadIdx.x; g < c; g += blockDim.x)  // solver.cpp:66-67
        mean_w[g] = two_lam / ((double)(goff[g + 1] - goff[g]) * (two_lam + rho));
    (void)s_done;
}

// ---------------------------------------------------------------------------
// The reference's residual sums as its own sequential chains, for a stop test
// the intervals of k_finalize could not decide (rare: the chain and the tree
// sum differ by ~1e-16 relative in practice, the rigorous bound is ~N·u):
//   chain 0: Σ_k ((x_k − l_k) − s_k)²   feas_residual   solver.cpp:23-31
//   chain 1: Σ_k (l_k − lp_k)²          rel_diff(L)      solver.cpp:14-21
//   chain 2: Σ_k (s_k − sp_k)²          rel_diff(S)
//   chain 3: Σ_k x_k²                   frob_norm(X)     matrix.cpp:99-103
// k in storage order (DenseMatrix::data()).  One CTA per chain: the terms are
// independent, so warps 1..7 stage the next tile's terms in shared memory while
// thread 0 adds the current tile's in order (the dependent adds are the cost:
// ≈N·4 cycles).  skip_x: chain 3 is not needed (‖X‖ already exact).
// ---------------------------------------------------------------------------
constexpr int CH_TILE = 2048;
template <typename T>
__global__ void __launch_bounds__(256) k_exact_chains(const T* __restrict__ X, const T* __restrict__ L,
                                                      const T* __restrict__ Lp, const T* __restrict__ S,
                                                      const T* __restrict__ Sp, int64_t N, int skip_x,
                                                      double* __restrict__ out) {
    __shared__ double buf[2][CH_TILE];
    const int q = blockIdx.x;
    if (q == 3 && skip_x) return;
    auto term = [&](int64_t k) -> double {
        if (q == 0) {
            const double r = (ld(X + k) - ld(L + k)) - ld(S + k);
            return r * r;
        }
        if (q == 1) {
            const double r = ld(L + k) - ld(Lp + k);
            return r * r;
        }
        if (q == 2) {
            const double r = ld(S + k) - ld(Sp + k);
            return r * r;
        }
        const double v = ld(X + k);
        return v * v;
    };
    auto fill = [&](int64_t tile, double* b) {
        const int64_t base = tile * CH_TILE;
        for (int e = (int)threadIdx.x - 32; e < CH_TILE; e += (int)blockDim.x - 32)
            b[e] = base + e < N ? term(base + e) : 0.0;
    };
    const int64_t ntiles = (N + CH_TILE - 1) / CH_TILE;
    if (threadIdx.x >= 32) fill(0, buf[0]);
    __syncthreads();
    double acc = 0.0;
    for (int64_t t = 0; t < ntiles; ++t) {
        if (threadIdx.x == 0) {
            const double* b = buf[t & 1];
            const int cnt = (int)((N - t * CH_TILE) < CH_TILE ? (N - t * CH_TILE) : CH_TILE);
#pragma unroll 16
            for (int e = 0; e < cnt; ++e) acc += b[e];
        } else if (threadIdx.x >= 32 && t + 1 < ntiles) {
            fill(t + 1, buf[(t + 1) & 1]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[q] = acc;
}

// fp32 storage: the exact fp64 copy of X the one-time kmeans(X) runs on
__global__ void k_widen(const float* __restrict__ src, double* __restrict__ dst, int64_t N) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < N; k += (int64_t)gridDim.x * blockDim.x)
        dst[k] = (double)src[k];
}

// mean_w for the current ρ (after the host rebuilt the member lists).
__global__ void k_mean_w(const Ctl* __restrict__ ctl, const int* __restrict__ goff,
                         double* __restrict__ mean_w, int c) {
    const double rho = ctl->rho, two_lam = 2.0 * ctl->lambda;
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < c; g += gridDim.x * blockDim.x)
        mean_w[g] = two_lam / ((double)(goff[g + 1] - goff[g]) * (two_lam + rho));
}

// ---------------------------------------------------------------------------
// Generic elementwise / reduction kernels (building blocks, L21 path, norms)
// ---------------------------------------------------------------------------

// sum of squares and |.| and non-finite flag, per-block partials (3 values)
template <typename T>
__global__ void __launch_bounds__(256) k_norms(const T* __restrict__ m, int64_t N,
                                               double* __restrict__ partials) {
    __shared__ double red[32 * 3];
    double sq = 0.0, ab = 0.0, bad = 0.0;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < N;
         k += (int64_t)gridDim.x * blockDim.x) {
        const double v = ld(m + k);
        sq += v * v;
        ab += fabs(v);
        if (!isfinite(v)) bad = 1.0;
    }
    double v[3] = {sq, ab, bad};
    block_sum<3>(v, red);
    if (threadIdx.x == 0)
        for (int q = 0; q < 3; ++q) partials[blockIdx.x * 3 + q] = v[q];
}

// generic residual sums for check_convergence: Σ((x−l)−s)², Σ(l−lp)², Σ(s−sp)²
__global__ void __launch_bounds__(256) k_triple(const double* __restrict__ x,
                                                const double* __restrict__ lp,
                                                const double* __restrict__ l,
                                                const double* __restrict__ sp,
                                                const double* __restrict__ s, int64_t N,
                                                double* __restrict__ partials) {
    __shared__ double red[32 * 3];
    double a = 0.0, b = 0.0, c = 0.0;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < N;
         k += (int64_t)gridDim.x * blockDim.x) {
        const double f = x[k] - l[k] - s[k];
        a += f * f;
        const double dl = l[k] - lp[k];
        b += dl * dl;
        const double ds = s[k] - sp[k];
        c += ds * ds;
    }
    double v[3] = {a, b, c};
    block_sum<3>(v, red);
    if (threadIdx.x == 0)
        for (int q = 0; q < 3; ++q) partials[blockIdx.x * 3 + q] = v[q];
}

__global__ void k_sum_partials(const double* __restrict__ partials, int nparts, int nv,
                               double* __restrict__ out) {
    __shared__ double red[32 * 5];
    double v[5] = {0, 0, 0, 0, 0};
    for (int b = threadIdx.x; b < nparts; b += blockDim.x)
        for (int q = 0; q < nv; ++q) v[q] += partials[(int64_t)b * nv + q];
    block_sum<5>(v, red);
    if (threadIdx.x == 0)
        for (int q = 0; q < nv; ++q) out[q] = v[q];
}

// L-update from a materialised D (building block l_update, solver.cpp:51-77)
template <int R>
__global__ void __launch_bounds__(256) k_l_blend(const double* __restrict__ D,
                                                 double* __restrict__ L,
                                                 const int* __restrict__ goff,
                                                 const int* __restrict__ members,
                                                 const double* __restrict__ G, double own_w,
                                                 double lambda, double rho, int64_t d,
                                                 int rowblocks) {
    const int g = blockIdx.x / rowblocks;
    const int rb = blockIdx.x - g * rowblocks;
    const int64_t i0 = ((int64_t)rb * blockDim.x + threadIdx.x) * R;
    if (i0 >= d) return;
    const int beg = goff[g], end = goff[g + 1];
    const double mw = 2.0 * lambda / ((double)(end - beg) * (2.0 * lambda + rho));
    double gs[R];
#pragma unroll
    for (int r = 0; r < R; ++r) gs[r] = G[(int64_t)g * d + i0 + r];
    for (int t = beg; t < end; ++t) {
        const int64_t off = (int64_t)members[t] * d + i0;
#pragma unroll
        for (int r = 0; r < R; ++r) L[off + r] = own_w * D[off + r] + mw * gs[r];
    }
}

// S = soft-threshold(B, t)   (solver.cpp:79-88)
__global__ void k_shrink_l1(const double* __restrict__ B, double* __restrict__ S, int64_t N,
                            double thr) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < N;
         k += (int64_t)gridDim.x * blockDim.x) {
        const double v = B[k];
        const double mag = fabs(v) - thr;
        S[k] = mag > 0.0 ? copysign(mag, v) : 0.0;
    }
}

// Θ += ρ((x − L) − S)    (solver.cpp:104-109)
__global__ void k_multiplier(double* __restrict__ Th, const double* __restrict__ X,
                             const double* __restrict__ L, const double* __restrict__ S,
                             int64_t N, double rho) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < N;
         k += (int64_t)gridDim.x * blockDim.x)
        Th[k] += rho * (X[k] - L[k] - S[k]);
}

// Exact per-column sequential sums of squares (column_l2_norms order,
// matrix.cpp:117-125), warp-transposed so each lane owns one column and
// walks its rows in ascending order while the warp reads coalesced 32×32
// tiles.  mode 0: v = m;  mode 1 (B-form for L21): v = (x − l) + θ/ρ.
template <typename T, int MODE>
__global__ void __launch_bounds__(128) k_col_sumsq(const T* __restrict__ M,
                                                   const T* __restrict__ Lm,
                                                   const T* __restrict__ Tm, double rho,
                                                   int64_t d, int64_t n,
                                                   double* __restrict__ out) {
    __shared__ double tile[4][32][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t j0 = ((int64_t)blockIdx.x * 4 + w) * 32;
    if (j0 >= n) return;
    double acc = 0.0;
    for (int64_t i0 = 0; i0 < d; i0 += 32) {
        const int64_t i = i0 + lane;
        for (int cc = 0; cc < 32; ++cc) {
            const int64_t j = j0 + cc;
            double v = 0.0;
            if (j < n && i < d) {
                const int64_t e = j * d + i;
                if (MODE == 0) v = ld(M + e);
                else v = (ld(M + e) - ld(Lm + e)) + ld(Tm + e) / rho;
            }
            tile[w][cc][lane] = v;
        }
        __syncwarp();
        const int lim = (int)((d - i0) < 32 ? (d - i0) : 32);
        for (int r = 0; r < lim; ++r) {
            const double v = tile[w][lane][r];
            acc += v * v;
        }
        __syncwarp();
    }
    if (j0 + lane < n) out[j0 + lane] = sqrt(acc);
}

// column shrink for L21: S_j = norm_j <= t ? 0 : (1 − t/norm_j)·B_j  (solver.cpp:94-100)
// mode 0: B given; mode 1: B = (x − l) + θ/ρ computed on the fly.
template <typename T, int MODE>
__global__ void k_shrink_l21(const T* __restrict__ B, const T* __restrict__ Lm,
                             const T* __restrict__ Tm, double rho, const double* __restrict__ norms,
                             T* __restrict__ S, int64_t d, int64_t n, double thr) {
    const int64_t N = d * n;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < N;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = k / d;
        const double nr = norms[j];
        double out = 0.0;
        if (!(nr <= thr)) {
            const double scale = 1.0 - thr / nr;
            const double b = MODE == 0 ? ld(B + k) : (ld(B + k) - ld(Lm + k)) + ld(Tm + k) / rho;
            out = scale * b;
        }
        S[k] = (T)out;
    }
}

}  // namespace respca_dev
