// K-means kernels (the p-update, kmeans.cpp) — exact decisions on screened
// distances.
//
// Every discrete decision of the reference's K-means — nearest centroid
// (kmeans.cpp:29, strict <, lowest index wins ties), the Hartigan move test
// (kmeans.cpp:107-119, threshold −1e-12), the farthest-point repair
// (kmeans.cpp:49-56) — is made on the reference's own distance value
// sq_dist(a, b) = Σ_i fl(fl(a_i − b_i)²) summed sequentially over ascending i
// (kmeans.cpp:12-19).  Reproducing that chain costs d dependent adds per
// (column, centroid) pair, so the kernels below first compute a SCREENED
// distance with the expanded form ‖x‖² + ‖c‖² − 2x·c on the FP64 FMA pipe,
// together with a rigorous bound on its distance to the reference value:
//
//   |ref − approx| ≤ e = (2d + 8)·u·1.05·(‖x‖ + ‖c‖)² + 2u·|approx|,  u = 2⁻⁵³
//
// (γ_d bounds for the three length-d FMA chains, the 3u term error of each
// rounded (a−b)², the sequential-sum bound γ_{d−1} of the reference chain, and
// slack).  A decision is taken from [approx − e, approx + e] only when it is
// the same for every value in the interval (IEEE rounding is monotone, so the
// weights na/(na−1)·dist etc. are bounded by evaluating them at the interval
// ends).  Undecidable columns — ties and near-ties — are resolved by the exact
// sequential chain, so labels are bit-identical to the reference's.
#pragma once

#include "common.cuh"

namespace respca_dev {

constexpr double kU = 1.1102230246251565e-16;  // 2^-53

RESPCA_DEV double screen_err(double kappa_d, double nx, double nc, double approx) {
    const double s = nx + nc;
    return kappa_d * (s * s) + 2.0 * kU * fabs(approx) + 1e-300;
}

RESPCA_DEV void cp_async8(void* smem, const void* gmem, bool pred) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int sz = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
RESPCA_DEV void cp_async4(void* smem, const void* gmem, bool pred) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int sz = pred ? 4 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
RESPCA_DEV void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
RESPCA_DEV void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---------------------------------------------------------------------------
// ‖c_k‖² for the screen (FMA chain; only ever used inside the bound)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_col_sq_fma(const double* __restrict__ C, int64_t d,
                                                    double* __restrict__ out,
                                                    const int* __restrict__ ver = nullptr,
                                                    int c = 0) {
    __shared__ double red[32];
    const int k = blockIdx.x;
    const double* ck = C + ((int64_t)(ver ? ver[k] : 0) * c + k) * d;
    // eight loads in flight per thread (one L2 round trip per eight rows instead of one
    // per row: C4, d = 76,800, c = 3: 47 µs → a few µs), four chains; any order is
    // inside the bound that uses the value
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    for (int64_t i0 = threadIdx.x; i0 < d; i0 += 8 * (int64_t)blockDim.x) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t i = i0 + u * (int64_t)blockDim.x;
            v[u] = i < d ? __ldg(ck + i) : 0.0;
        }
        s0 = __fma_rn(v[0], v[0], s0);
        s1 = __fma_rn(v[1], v[1], s1);
        s2 = __fma_rn(v[2], v[2], s2);
        s3 = __fma_rn(v[3], v[3], s3);
        s0 = __fma_rn(v[4], v[4], s0);
        s1 = __fma_rn(v[5], v[5], s1);
        s2 = __fma_rn(v[6], v[6], s2);
        s3 = __fma_rn(v[7], v[7], s3);
    }
    double v[1] = {(s0 + s1) + (s2 + s3)};
    block_sum<1>(v, red);
    if (threadIdx.x == 0) out[k] = v[0];
}

// ---------------------------------------------------------------------------
// Screened distance GEMM:  part[s][j][k] = Σ_{i∈split s} M[i,j]·C[i,k]
//                          xxp[s][j]     = Σ_{i∈split s} M[i,j]²
// CTA tile TJ×TK outputs, thread tile RJ×RK, K-chunks of 32 rows staged in
// shared memory by a 2-stage cp.async pipeline (global column-major →
// shared row-major, so both operands are read as 128-bit rows in the inner
// loop).  FP64-FMA bound: intensity RJ·RK FMAs per (RJ+RK) smem doubles.
// ---------------------------------------------------------------------------
template <typename T, int RJ, int RK, int NTJ, int NTK>
__global__ void __launch_bounds__(NTJ* NTK) k_dist_screen(const T* __restrict__ M,
                                                          const double* __restrict__ C, int64_t d,
                                                          int n, int c, int chunks_per_split,
                                                          double* __restrict__ part,
                                                          double* __restrict__ xxp) {
    constexpr int TJ = RJ * NTJ, TK = RK * NTK, KI = 32, NT = NTJ * NTK;
    constexpr int MSTR = TJ + (sizeof(T) == 8 ? 2 : 4);  // 16-byte aligned rows
    constexpr int CSTR = TK + 2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* Ms = reinterpret_cast<T*>(smem_raw);                                      // [2][KI][MSTR]
    double* Cs = reinterpret_cast<double*>(smem_raw + sizeof(T) * 2 * KI * MSTR);  // [2][KI][CSTR]
    __shared__ double xred[NT];

    const int tid = threadIdx.x;
    const int tk = tid % NTK, tj = tid / NTK;
    const int j0 = blockIdx.x * TJ, k0 = blockIdx.y * TK, split = blockIdx.z;
    const int64_t ibeg = (int64_t)split * chunks_per_split * KI;
    int64_t iend = ibeg + (int64_t)chunks_per_split * KI;
    if (iend > d) iend = d;
    const int nch = ibeg < iend ? (int)((iend - ibeg + KI - 1) / KI) : 0;

    auto load = [&](int64_t i0, int buf) {
        T* mdst = Ms + buf * KI * MSTR;
        double* cdst = Cs + buf * KI * CSTR;
        for (int e = tid; e < TJ * KI; e += NT) {
            const int col = e / KI, ii = e - col * KI;
            const int j = j0 + col;
            const int64_t i = i0 + ii;
            const bool p = (j < n) && (i < iend);
            const T* src = p ? M + (int64_t)j * d + i : M;
            if (sizeof(T) == 8) cp_async8(mdst + ii * MSTR + col, src, p);
            else cp_async4(mdst + ii * MSTR + col, src, p);
        }
        for (int e = tid; e < TK * KI; e += NT) {
            const int kk = e / KI, ii = e - kk * KI;
            const int k = k0 + kk;
            const int64_t i = i0 + ii;
            const bool p = (k < c) && (i < iend);
            cp_async8(cdst + ii * CSTR + kk, p ? C + (int64_t)k * d + i : C, p);
        }
        cp_commit();
    };

    double acc[RJ][RK];
#pragma unroll
    for (int a = 0; a < RJ; ++a)
#pragma unroll
        for (int b = 0; b < RK; ++b) acc[a][b] = 0.0;
    // ‖x‖² helpers: NT/TJ threads per column, each a contiguous row range of the chunk
    constexpr int XPER = NT / TJ;  // threads per column
    constexpr int XROWS = KI / XPER;
    const int xcol = tid % TJ, xpart = tid / TJ;
    double xx = 0.0;

    if (nch > 0) load(ibeg, 0);
    for (int ch = 0; ch < nch; ++ch) {
        if (ch + 1 < nch) {
            load(ibeg + (int64_t)(ch + 1) * KI, (ch + 1) & 1);
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        const T* ms = Ms + (ch & 1) * KI * MSTR;
        const double* cs = Cs + (ch & 1) * KI * CSTR;
#pragma unroll 4
        for (int ii = 0; ii < KI; ++ii) {
            double a[RJ], b[RK];
#pragma unroll
            for (int x = 0; x < RJ; ++x) a[x] = (double)ms[ii * MSTR + tj * RJ + x];
#pragma unroll
            for (int y = 0; y < RK; ++y) b[y] = cs[ii * CSTR + tk * RK + y];
#pragma unroll
            for (int x = 0; x < RJ; ++x)
#pragma unroll
                for (int y = 0; y < RK; ++y) acc[x][y] = __fma_rn(a[x], b[y], acc[x][y]);
        }
#pragma unroll
        for (int r = 0; r < XROWS; ++r) {
            const double v = (double)ms[(xpart * XROWS + r) * MSTR + xcol];
            xx = __fma_rn(v, v, xx);
        }
        __syncthreads();
    }
#pragma unroll
    for (int x = 0; x < RJ; ++x) {
        const int j = j0 + tj * RJ + x;
        if (j >= n) continue;
#pragma unroll
        for (int y = 0; y < RK; ++y) {
            const int k = k0 + tk * RK + y;
            if (k < c) part[((int64_t)split * n + j) * c + k] = acc[x][y];
        }
    }
    xred[tid] = xx;
    __syncthreads();
    if (blockIdx.y == 0 && tid < TJ && j0 + tid < n) {
        double s = 0.0;
        for (int p = 0; p < XPER; ++p) s += xred[p * TJ + tid];
        xxp[(int64_t)split * n + j0 + tid] = s;
    }
}

// ---------------------------------------------------------------------------
// Screened distance GEMM on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64):
//   part[s][j][k] = Σ_{i∈split s} M[i,j]·C[i,k],   xxp[s][j] = Σ_{i∈split s} M[i,j]²
// A = Mᵀ (rows j, K = i) and B = C (K = i, cols k) are both staged in shared
// memory in their global (i-contiguous) layout by 16-byte cp.async — no
// transposes — with a row stride of 36 elements, which makes every fragment
// load (lane → row lane/4, k lane%4) conflict-free.  CTA = 8 warps, tile
// 128 (j) × TK (k); warp tile (MJ·8) × (NK·8); K-chunks of 32 rows, 2 stages.
// ---------------------------------------------------------------------------
RESPCA_DEV void dmma884(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}
// m16n8k8 f64 (sm_90+): A 16×8 row-major (a0 (g,t) a1 (g+8,t) a2 (g,t+4)
// a3 (g+8,t+4)), B 8×8 col-major (b0 (t,g) b1 (t+4,g)), C/D 16×8
// (c0,c1 (g, 2t..2t+1), c2,c3 (g+8, 2t..2t+1)); g = lane/4, t = lane%4
RESPCA_DEV void dmma1688(double& c0, double& c1, double& c2, double& c3, double a0, double a1,
                         double a2, double a3, double b0, double b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3)
        : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
}
RESPCA_DEV void cp_async16(void* smem, const void* gmem, int bytes) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}

template <typename T, int WK, int MJ, int NK>
__global__ void __launch_bounds__(256, 2) k_dist_dmma(const T* __restrict__ M,
                                                     const double* __restrict__ C,
                                                     const int* __restrict__ ver, int64_t d,
                                                     int n, int c, int chunks_per_split,
                                                     double* __restrict__ part,
                                                     double* __restrict__ xxp,
                                                     const int* __restrict__ kmap = nullptr,
                                                     int csub = 0) {
    // kmap: screen only the centroids kmap[0..csub) (the rest of `part` is
    // kept); k below runs over that subset, kmap[k] is the centroid
    constexpr int NW = 8, WJ = NW / WK;
    constexpr int TJ = WJ * MJ * 8, TK = WK * NK * 8, KI = 32;
    constexpr int AS = 36;  // row stride (elements) of both smem tiles
    constexpr int EPV = 16 / sizeof(T);  // elements per 16-byte copy
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* As = reinterpret_cast<T*>(smem_raw);  // [2][TJ][AS]
    double* Bs = reinterpret_cast<double*>(smem_raw + sizeof(T) * 2 * TJ * AS);  // [2][TK][AS]

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wj = warp / WK, wk = warp % WK;
    const int g = lane >> 2, t4 = lane & 3;
    const int j0 = blockIdx.x * TJ, k0 = blockIdx.y * TK, split = blockIdx.z;
    const int64_t ibeg = (int64_t)split * chunks_per_split * KI;
    int64_t iend = ibeg + (int64_t)chunks_per_split * KI;
    if (iend > d) iend = d;
    const int nch = ibeg < iend ? (int)((iend - ibeg + KI - 1) / KI) : 0;
    const int nk = kmap ? csub : c;  // centroids screened by this launch
    auto cid = [&](int k) { return kmap ? __ldg(kmap + k) : k; };
    // 16-byte copies need 16-byte aligned global rows: true when d is a
    // multiple of 16/sizeof(T); otherwise fall back to element copies.
    const bool vec_ok = (d % EPV) == 0;

    auto load = [&](int64_t i0, int buf) {
        T* adst = As + buf * TJ * AS;
        double* bdst = Bs + buf * TK * AS;
        if (vec_ok) {
            constexpr int AV = KI / EPV;  // 16-byte vectors per row chunk
            for (int e = tid; e < TJ * AV; e += 256) {
                const int row = e / AV, v = e - row * AV;
                const int j = j0 + row;
                const int64_t i = i0 + v * EPV;
                int bytes = 0;
                if (j < n && i < iend) bytes = (int)(sizeof(T) * ((iend - i) < EPV ? (iend - i) : EPV));
                cp_async16(adst + row * AS + v * EPV, bytes ? M + (int64_t)j * d + i : M, bytes);
            }
            for (int e = tid; e < TK * (KI / 2); e += 256) {
                const int row = e / (KI / 2), v = e - row * (KI / 2);
                const int k = k0 + row;
                const int64_t i = i0 + v * 2;
                int bytes = 0;
                if (k < nk && i < iend) bytes = (int)(8 * ((iend - i) < 2 ? (iend - i) : 2));
                const int kc = k < nk ? cid(k) : 0;
                const double* ck = C + ((int64_t)(ver && k < nk ? ver[kc] : 0) * c + kc) * d;
                cp_async16(bdst + row * AS + v * 2, bytes ? ck + i : C, bytes);
            }
        } else {
            for (int e = tid; e < TJ * KI; e += 256) {
                const int row = e / KI, ii = e - row * KI;
                const int j = j0 + row;
                const int64_t i = i0 + ii;
                const bool p = j < n && i < iend;
                if (sizeof(T) == 8) cp_async8(adst + row * AS + ii, p ? M + (int64_t)j * d + i : M, p);
                else cp_async4(adst + row * AS + ii, p ? M + (int64_t)j * d + i : M, p);
            }
            for (int e = tid; e < TK * KI; e += 256) {
                const int row = e / KI, ii = e - row * KI;
                const int k = k0 + row;
                const int64_t i = i0 + ii;
                const bool p = k < nk && i < iend;
                const int kc = k < nk ? cid(k) : 0;
                const double* ck = C + ((int64_t)(ver && k < nk ? ver[kc] : 0) * c + kc) * d;
                cp_async8(bdst + row * AS + ii, p ? ck + i : C, p);
            }
        }
        cp_commit();
    };

    double acc[MJ][NK][2];
#pragma unroll
    for (int a = 0; a < MJ; ++a)
#pragma unroll
        for (int b = 0; b < NK; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    double xx[MJ];
#pragma unroll
    for (int a = 0; a < MJ; ++a) xx[a] = 0.0;

    if (nch > 0) load(ibeg, 0);
    for (int ch = 0; ch < nch; ++ch) {
        if (ch + 1 < nch) {
            load(ibeg + (int64_t)(ch + 1) * KI, (ch + 1) & 1);
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        const T* as = As + (ch & 1) * TJ * AS + (wj * MJ * 8 + g) * AS + t4;
        const double* bs = Bs + (ch & 1) * TK * AS + (wk * NK * 8 + g) * AS + t4;
#pragma unroll
        for (int kk = 0; kk < KI; kk += 8) {
            // m16n8k8: 8-row groups 2x2 and 2x2+1 form one 16-row A tile
            double a[MJ][2], b[NK][2];
#pragma unroll
            for (int x = 0; x < MJ; ++x) {
                a[x][0] = (double)as[x * 8 * AS + kk];
                a[x][1] = (double)as[x * 8 * AS + kk + 4];
            }
#pragma unroll
            for (int y = 0; y < NK; ++y) {
                b[y][0] = bs[y * 8 * AS + kk];
                b[y][1] = bs[y * 8 * AS + kk + 4];
            }
#pragma unroll
            for (int x2 = 0; x2 < MJ / 2; ++x2)
#pragma unroll
                for (int y = 0; y < NK; ++y)
                    dmma1688(acc[2 * x2][y][0], acc[2 * x2][y][1], acc[2 * x2 + 1][y][0],
                             acc[2 * x2 + 1][y][1], a[2 * x2][0], a[2 * x2 + 1][0], a[2 * x2][1],
                             a[2 * x2 + 1][1], b[y][0], b[y][1]);
            if (wk == 0)
#pragma unroll
                for (int x = 0; x < MJ; ++x)
                    xx[x] = __fma_rn(a[x][1], a[x][1], __fma_rn(a[x][0], a[x][0], xx[x]));
        }
        __syncthreads();
    }
    // epilogue: D[row g][col 2·t4 + {0,1}] of every 8×8 tile
#pragma unroll
    for (int x = 0; x < MJ; ++x) {
        const int j = j0 + (wj * MJ + x) * 8 + g;
        if (j >= n) continue;
        double* dst = part + ((int64_t)split * n + j) * c;
#pragma unroll
        for (int y = 0; y < NK; ++y) {
            const int k = k0 + (wk * NK + y) * 8 + 2 * t4;
            if (k < nk) dst[cid(k)] = acc[x][y][0];
            if (k + 1 < nk) dst[cid(k + 1)] = acc[x][y][1];
        }
    }
    if (wk == 0) {
#pragma unroll
        for (int x = 0; x < MJ; ++x) {
            double v = xx[x];
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            v += __shfl_xor_sync(0xffffffffu, v, 2);
            const int j = j0 + (wj * MJ + x) * 8 + g;
            if (t4 == 0 && j < n && blockIdx.y == 0) xxp[(int64_t)split * n + j] = v;
        }
    }
}

// Screened distance of (j, k) from the split partials (fixed split order).
struct Screen {
    const double* part;
    const double* xxp;
    const double* cc;
    int nsplit, n, c;
    double kappa_d;
    double abs_e = 0.0;  // absolute half-width term (TMA screen: FP32 underflow of ‖x‖² chunk sums)
    // BF16 screens: operands below the FP32/BF16 normal range are subnormal or
    // flushed (|error| ≤ 2⁻¹²⁶ per operand and product, not relative), so the
    // half-width gets lin_e·(‖x‖ + ‖c‖) on top of abs_e
    double lin_e = 0.0;
    // tcgen05 screens: their error flag (an mbarrier wait timed out, the
    // accumulators are not valid); set → every interval is unbounded, i.e. every
    // decision goes to the exact chains
    const int* err = nullptr;
    // split partials in split order; loads four at a time (the padding zeros
    // leave the sums unchanged: they never start from −0)
    RESPCA_DEV double xx(int j) const {
        double s = 0.0;
        for (int p0 = 0; p0 < nsplit; p0 += 4) {
            double a[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) a[u] = p0 + u < nsplit ? xxp[(int64_t)(p0 + u) * n + j] : 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u) s += a[u];
        }
        return s;
    }
    RESPCA_DEV void get(int j, int k, double xxj, double nx, double& lo, double& hi,
                        double& mid) const {
        double dot = 0.0;
        for (int p0 = 0; p0 < nsplit; p0 += 4) {
            double a[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) a[u] = p0 + u < nsplit ? part[((int64_t)(p0 + u) * n + j) * c + k] : 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u) dot += a[u];
        }
        interval(xxj, nx, dot, cc[k], lo, hi, mid);
    }
    RESPCA_DEV void interval(double xxj, double nx, double dot, double ck, double& lo, double& hi,
                             double& mid) const {
        mid = (xxj + ck) - 2.0 * dot;
        const double nc = sqrt(fabs(ck));
        const double e = screen_err(kappa_d, nx, nc, mid) + abs_e + lin_e * (nx + nc);
        if (!isfinite(mid) || !isfinite(e) || (err && __ldg(err) != 0)) {
            lo = -INFINITY;
            hi = INFINITY;
        } else {
            lo = mid - e;
            hi = mid + e;
        }
    }
};

// debug/test: materialise the screened intervals (approx, half-width)
__global__ void k_screen_dump(Screen sc, int n, int c, double* __restrict__ approx,
                              double* __restrict__ err) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)n * c) return;
    const int j = (int)(e / c), k = (int)(e % c);
    const double xxj = sc.xx(j);
    double lo, hi, mid;
    sc.get(j, k, xxj, sqrt(fabs(xxj)), lo, hi, mid);
    approx[e] = mid;
    err[e] = hi - mid;
}

// warp-wide lexicographic argmin on (value, index)
RESPCA_DEV void warp_argmin(double& v, int& k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int ok = __shfl_xor_sync(0xffffffffu, k, o);
        if (ov < v || (ov == v && ok < k)) {
            v = ov;
            k = ok;
        }
    }
}
// warp_min: common.cuh

// Decision status of one column
enum : int { ST_STABLE = 0, ST_CHANGED = 1, ST_MOVE = 2, ST_AMBIG = 3 };

// ---------------------------------------------------------------------------
// Per-column decision (one warp per column) on [lo, hi] intervals of the
// reference's distances:
//   1. label = argmin_k dist (kmeans.cpp:27-33)  — certain or ambiguous
//   2. if HART and the label is certain and unchanged: does the first
//      Hartigan pass move this column? (kmeans.cpp:103-121)
// DistFn(j, k, lo, hi, mid) supplies the interval (exact: lo = hi = mid).
// Returns the status and (for certain labels) the new label.
// ---------------------------------------------------------------------------
template <typename DistFn>
RESPCA_DEV int decide_column(int j, int c, int old_label, const int* __restrict__ counts,
                             bool hart, const DistFn& dist, int& new_label) {
    const int lane = threadIdx.x & 31;
    // candidate argmin on the midpoint
    double bv = INFINITY;
    int bk = 0x7fffffff;
    for (int k = lane; k < c; k += 32) {
        double lo, hi, mid;
        dist(j, k, lo, hi, mid);
        if (mid < bv) {  // ascending k per lane: strict < keeps the lowest index
            bv = mid;
            bk = k;
        }
    }
    warp_argmin(bv, bk);
    if (bk >= c) bk = 0;  // all-NaN guard: treated as ambiguous below
    double klo, khi, kmid;
    dist(j, bk, klo, khi, kmid);
    bool ok = true;
    for (int k = lane; k < c; k += 32) {
        if (k == bk) continue;
        double lo, hi, mid;
        dist(j, k, lo, hi, mid);
        if (k < bk) ok &= khi < lo;
        else ok &= khi <= lo;
    }
    ok = __all_sync(0xffffffffu, ok) && isfinite(khi);
    if (!ok) return ST_AMBIG;
    new_label = bk;
    if (bk != old_label) return ST_CHANGED;
    if (!hart) return ST_STABLE;
    const int from = bk;
    const int cf = counts[from];
    if (cf <= 1) return ST_STABLE;  // kmeans.cpp:105
    const double na = (double)cf;
    const double wa = na / (na - 1.0);
    const double gain_hi = wa * khi, gain_lo = wa * klo;
    bool surely_none = true, surely_move = false;
    for (int k = lane; k < c; k += 32) {
        if (k == from) continue;
        double lo, hi, mid;
        dist(j, k, lo, hi, mid);
        const double nb = (double)counts[k];
        const double wb = nb / (nb + 1.0);
        const double dlo = wb * lo - gain_hi;
        const double dhi = wb * hi - gain_lo;
        surely_none &= !(dlo < -1e-12);
        surely_move |= dhi < -1e-12;
    }
    surely_none = __all_sync(0xffffffffu, surely_none);
    surely_move = __any_sync(0xffffffffu, surely_move);
    if (surely_none) return ST_STABLE;
    if (surely_move) return ST_MOVE;
    return ST_AMBIG;
}

// Same decision with each lane's intervals (k = lane + 32q, q < KPL) computed
// once into registers; the candidate's interval is broadcast by shuffle.
template <int KPL>
RESPCA_DEV int decide_column_cached(int c, int old_label, const int (&cq)[KPL],
                                    bool hart, const double (&lo)[KPL], const double (&hi)[KPL],
                                    const double (&mid)[KPL], int& new_label) {
    const int lane = threadIdx.x & 31;
    double bv = INFINITY;
    int bk = 0x7fffffff;
#pragma unroll
    for (int q = 0; q < KPL; ++q) {
        const int k = lane + 32 * q;
        if (k < c && mid[q] < bv) {
            bv = mid[q];
            bk = k;
        }
    }
    warp_argmin(bv, bk);
    if (bk >= c) bk = 0;
    auto fetch = [&](int k, double& l, double& h, double& m) {
        const int q = k >> 5, src = k & 31;
        double tl = 0.0, th = 0.0, tm = 0.0;
#pragma unroll
        for (int qq = 0; qq < KPL; ++qq)
            if (qq == q) {
                tl = lo[qq];
                th = hi[qq];
                tm = mid[qq];
            }
        l = __shfl_sync(0xffffffffu, tl, src);
        h = __shfl_sync(0xffffffffu, th, src);
        m = __shfl_sync(0xffffffffu, tm, src);
    };
    double klo, khi, kmid;
    fetch(bk, klo, khi, kmid);
    bool ok = true;
#pragma unroll
    for (int q = 0; q < KPL; ++q) {
        const int k = lane + 32 * q;
        if (k >= c || k == bk) continue;
        if (k < bk) ok &= khi < lo[q];
        else ok &= khi <= lo[q];
    }
    ok = __all_sync(0xffffffffu, ok) && isfinite(khi);
    if (!ok) return ST_AMBIG;
    new_label = bk;
    if (bk != old_label) return ST_CHANGED;
    if (!hart) return ST_STABLE;
    const int from = bk;
    int cf = 0;  // counts[from], from the lane that holds it
    {
        const int q = from >> 5;
        int t = 0;
#pragma unroll
        for (int qq = 0; qq < KPL; ++qq)
            if (qq == q) t = cq[qq];
        cf = __shfl_sync(0xffffffffu, t, from & 31);
    }
    if (cf <= 1) return ST_STABLE;  // kmeans.cpp:105
    const double na = (double)cf;
    const double wa = na / (na - 1.0);
    const double gain_hi = wa * khi, gain_lo = wa * klo;
    bool surely_none = true, surely_move = false;
#pragma unroll
    for (int q = 0; q < KPL; ++q) {
        const int k = lane + 32 * q;
        if (k >= c || k == from) continue;
        const double nb = (double)cq[q];
        const double wb = nb / (nb + 1.0);
        surely_none &= !(wb * lo[q] - gain_hi < -1e-12);
        surely_move |= (wb * hi[q] - gain_lo) < -1e-12;
    }
    surely_none = __all_sync(0xffffffffu, surely_none);
    surely_move = __any_sync(0xffffffffu, surely_move);
    if (surely_none) return ST_STABLE;
    if (surely_move) return ST_MOVE;
    return ST_AMBIG;
}

// Decide all columns from the screen.  mode: 0 = Lloyd assignment only,
// 1 = ALM fast-path check (assignment + first Hartigan pass).
// Output labels are written to new_labels; ambiguous columns are appended to
// amb_list and keep their old label for now.
__global__ void __launch_bounds__(256, 4) k_decide(Screen sc, int n, int c,
                                                const int* __restrict__ old_labels,
                                                const int* __restrict__ counts, int mode,
                                                int* __restrict__ new_labels,
                                                int* __restrict__ amb_list, Ctl* __restrict__ ctl,
                                                int diag) {
    const int lane = threadIdx.x & 31;
    const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (j >= n) return;
    // every load of the column is issued before the first use (the done flag,
    // labels and group sizes included): one memory latency round per warp
    const int done = *(volatile const int*)&ctl->done;
    const int old = old_labels ? old_labels[j] : -1;
    int cq[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int k = lane + 32 * q;
        cq[q] = (counts && k < c) ? __ldg(counts + k) : 0;
    }
    const double xxj = sc.xx(j);
    const double nx = sqrt(fabs(xxj));
    auto fn = [&](int jj, int k, double& lo, double& hi, double& mid) {
        sc.get(jj, k, xxj, nx, lo, hi, mid);
    };
    int nl = old;
    int st;
    if (c <= 128) {  // intervals computed once per lane (KPL = 4)
        double lo[4], hi[4], mid[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int k = lane + 32 * q;
            if (k < c) fn(j, k, lo[q], hi[q], mid[q]);
            else lo[q] = hi[q] = mid[q] = INFINITY;
        }
        if (done) return;
        st = decide_column_cached<4>(c, old, cq, mode == 1, lo, hi, mid, nl);
    } else {
        if (done) return;
        st = decide_column(j, c, old, counts, mode == 1, fn, nl);
    }
    if (diag && mode == 1 && old >= 0 && counts[old] > 1) {
        // diagnostics: smallest Hartigan/argmin margin of this column relative
        // to (‖x‖ + ‖c‖)² — what a lower-precision screen would have to resolve
        double flo, fhi, fmid;
        fn(j, old, flo, fhi, fmid);
        const double na = (double)counts[old];
        const double ga = na / (na - 1.0) * fmid;
        double mrel = INFINITY;
        for (int k = lane; k < c; k += 32) {
            if (k == old) continue;
            double lo, hi, mid;
            fn(j, k, lo, hi, mid);
            const double nb = (double)counts[k];
            const double delta = nb / (nb + 1.0) * mid - ga;
            const double sc_ = nx + sqrt(fabs(sc.cc[k]));
            mrel = fmin(mrel, fabs(delta + 1e-12) / (sc_ * sc_));
        }
        mrel = warp_min(mrel);
        if (lane == 0)
            for (int q = 0; q < 6; ++q)
                if (mrel < 0.1 / (double)(q == 0 ? 1 : (q == 1 ? 10 : (q == 2 ? 100 : (q == 3 ? 1000 : (q == 4 ? 10000 : 100000))))))
                    atomicAdd(&ctl->margin_hist[q], 1u);
    }
    if (lane == 0) {
        new_labels[j] = st == ST_AMBIG ? old : nl;
        if (st == ST_CHANGED) atomicAdd(&ctl->changed, 1u);
        if (st == ST_MOVE) atomicAdd(&ctl->moves, 1u);
        if (st == ST_AMBIG) {
            const unsigned slot = atomicAdd(&ctl->ambiguous, 1u);
            amb_list[slot] = j;
        }
    }
}

// k_decide for c ≤ 32·KPL centroids and ≤ 4 screen splits: every load of the
// column (split partials, ‖x‖² partials, ‖c‖², labels, group sizes, the done
// flag) is issued in one basic block — one memory latency round per warp —
// and the intervals are Screen::get's arithmetic, term for term.
template <int KPL>
__global__ void __launch_bounds__(256, KPL == 2 ? 4 : 3) k_decide_fast(Screen sc, int n, int c,
                                                        const int* __restrict__ old_labels,
                                                        const int* __restrict__ counts, int mode,
                                                        int* __restrict__ new_labels,
                                                        int* __restrict__ amb_list, Ctl* __restrict__ ctl) {
    const int lane = threadIdx.x & 31;
    pdl_enter();
    const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (j >= n) return;
    const int ns = sc.nsplit;
    const int done = *(volatile const int*)&ctl->done;
    const int old = old_labels ? old_labels[j] : -1;
    double xp[4], pa[KPL][4], ccq[KPL];
    int cq[KPL];
#pragma unroll
    for (int p = 0; p < 4; ++p) xp[p] = p < ns ? __ldg(sc.xxp + (int64_t)p * n + j) : 0.0;
#pragma unroll
    for (int q = 0; q < KPL; ++q) {
        const int k = lane + 32 * q;
        const bool kk = k < c;
        cq[q] = (counts && kk) ? __ldg(counts + k) : 0;
        ccq[q] = kk ? __ldg(sc.cc + k) : 0.0;
#pragma unroll
        for (int p = 0; p < 4; ++p)
            pa[q][p] = (kk && p < ns) ? __ldg(sc.part + ((int64_t)p * n + j) * c + k) : 0.0;
    }
    double xxj = 0.0;  // Screen::xx: splits in order (trailing zeros leave the sum unchanged)
#pragma unroll
    for (int p = 0; p < 4; ++p) xxj += xp[p];
    const double nx = sqrt(fabs(xxj));
    double lo[KPL], hi[KPL], mid[KPL];
#pragma unroll
    for (int q = 0; q < KPL; ++q) {
        if (lane + 32 * q < c) {
            double dot = 0.0;
#pragma unroll
            for (int p = 0; p < 4; ++p) dot += pa[q][p];
            sc.interval(xxj, nx, dot, ccq[q], lo[q], hi[q], mid[q]);
        } else {
            lo[q] = hi[q] = mid[q] = INFINITY;
        }
    }
    if (done) return;
    int nl = old;
    const int st = decide_column_cached<KPL>(c, old, cq, mode == 1, lo, hi, mid, nl);
    if (lane == 0) {
        new_labels[j] = st == ST_AMBIG ? old : nl;
        if (st == ST_CHANGED) atomicAdd(&ctl->changed, 1u);
        if (st == ST_MOVE) atomicAdd(&ctl->moves, 1u);
        if (st == ST_AMBIG) {
            const unsigned slot = atomicAdd(&ctl->ambiguous, 1u);
            amb_list[slot] = j;
        }
    }
}

// Exact sequential distances (kmeans.cpp:12-19) of listed columns to all
// centroids: out[idx][k].  One block per listed column, one thread per
// centroid, ascending i — the reference's chain.
template <typename T>
__global__ void __launch_bounds__(128) k_exact_cols(const T* __restrict__ M,
                                                    const double* __restrict__ C, int64_t d,
                                                    int c, const int* __restrict__ list,
                                                    const unsigned* __restrict__ count,
                                                    double* __restrict__ out) {
    const unsigned cnt = count ? *count : gridDim.x;
    for (unsigned idx = blockIdx.x; idx < cnt; idx += gridDim.x) {
        const int j = list[idx];
        const T* x = M + (int64_t)j * d;
        for (int k = threadIdx.x; k < c; k += blockDim.x) {
            const double* cv = C + (int64_t)k * d;
            double s = 0.0;
            for (int64_t i = 0; i < d; ++i) {
                const double t = (double)__ldg(x + i) - __ldg(cv + i);
                s += t * t;
            }
            out[(int64_t)idx * c + k] = s;
        }
    }
}

// The same exact chains, warp-transposed for long lists (many undecidable
// columns, e.g. near-identical video frames): lane = listed column, each lane
// runs KC centroids' chains (ascending i, the reference's order) on 32×32
// column tiles and KC×32 centroid tiles streamed through a cp.async ring.
// Grid: (warp groups of 32 listed columns, centroid chunks of KC).
template <typename T, int KC>
__global__ void __launch_bounds__(64) k_exact_cols_tile(const T* __restrict__ M, const double* __restrict__ C,
                                                        int64_t d, int c, const int* __restrict__ list,
                                                        const unsigned* __restrict__ count,
                                                        double* __restrict__ out) {
    constexpr int PD = 4, W = 2;
    extern __shared__ __align__(16) unsigned char ex_sm[];
    auto tile = reinterpret_cast<T(*)[PD][32][33]>(ex_sm);                                // [W][PD][32][33]
    auto ctile = reinterpret_cast<double(*)[PD][KC][32]>(ex_sm + sizeof(T) * W * PD * 32 * 33);  // [W][PD][KC][32]
    const unsigned cnt = *count;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned e0 = (blockIdx.x * W + w) * 32u;
    if (e0 >= cnt) return;
    const int k0 = blockIdx.y * KC;
    const int64_t ntile = (d + 31) / 32;
    // lane's column (list entry e0 + lane; past the end: repeat entry e0, not stored)
    const bool mine = e0 + lane < cnt;
    int cols[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) cols[q] = __ldg(list + (e0 + q < cnt ? e0 + q : e0));
    auto issue = [&](int64_t t) {
        const int slot = (int)(t % PD);
        const int64_t i = t * 32 + lane;
        const bool okr = i < d;
#pragma unroll
        for (int q = 0; q < 32; ++q) {
            const T* src = okr ? M + (int64_t)cols[q] * d + i : M;
            if (sizeof(T) == 8) cp_async8(&tile[w][slot][q][lane], src, okr);
            else cp_async4(&tile[w][slot][q][lane], src, okr);
        }
#pragma unroll
        for (int k = 0; k < KC; ++k) {
            const bool ok = okr && k0 + k < c;
            cp_async8(&ctile[w][slot][k][lane], ok ? C + (int64_t)(k0 + k) * d + i : C, ok);
        }
        cp_commit();
    };
    for (int64_t t = 0; t < PD - 1; ++t) {
        if (t < ntile) issue(t);
        else cp_commit();
    }
    double s[KC];
#pragma unroll
    for (int k = 0; k < KC; ++k) s[k] = 0.0;
    for (int64_t t = 0; t < ntile; ++t) {
        if (t + PD - 1 < ntile) issue(t + PD - 1);
        else cp_commit();
        cp_wait<PD - 1>();
        __syncwarp();
        const int slot = (int)(t % PD);
        const int lim = (int)((d - t * 32) < 32 ? (d - t * 32) : 32);
        for (int r = 0; r < lim; ++r) {
            const double x = (double)tile[w][slot][lane][r];
#pragma unroll
            for (int k = 0; k < KC; ++k) {
                const double tt = x - ctile[w][slot][k][r];  // kmeans.cpp:15-16
                s[k] += tt * tt;
            }
        }
        __syncwarp();
    }
    if (mine)
#pragma unroll
        for (int k = 0; k < KC; ++k)
            if (k0 + k < c) out[(int64_t)(e0 + lane) * c + k0 + k] = s[k];
}

// Re-decide the listed (ambiguous) columns with exact distances.
__global__ void __launch_bounds__(256) k_redecide(const double* __restrict__ exact, int c,
                                                  const int* __restrict__ list,
                                                  const unsigned* __restrict__ count,
                                                  const int* __restrict__ old_labels,
                                                  const int* __restrict__ counts, int mode,
                                                  int* __restrict__ new_labels,
                                                  Ctl* __restrict__ ctl) {
    const int lane = threadIdx.x & 31;
    if (ctl->done) return;
    const unsigned cnt = *count;
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl->exact_fallbacks += cnt;
    const unsigned w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned nw = (gridDim.x * blockDim.x) >> 5;
    for (unsigned idx = w0; idx < cnt; idx += nw) {
        const int j = list[idx];
        auto fn = [&](int, int k, double& lo, double& hi, double& mid) {
            mid = exact[(int64_t)idx * c + k];
            lo = hi = mid;
        };
        const int old = old_labels ? old_labels[j] : -1;
        int nl = old;
        const int st = decide_column(j, c, old, counts, mode == 1, fn, nl);
        if (lane == 0) {
            new_labels[j] = nl;
            if (st == ST_CHANGED) atomicAdd(&ctl->changed, 1u);
            if (st == ST_MOVE) atomicAdd(&ctl->moves, 1u);
        }
    }
}

// k_exact_cols and k_redecide in one launch (short lists: one block per listed
// column computes its exact chains, then its first warp re-decides it).  With
// nothing ambiguous — the common iteration — this is one empty launch, not two.
template <typename T>
__global__ void __launch_bounds__(128) k_exact_redecide(const T* __restrict__ M, const double* __restrict__ C,
                                                        int64_t d, int c, const int* __restrict__ list,
                                                        const unsigned* __restrict__ count,
                                                        double* __restrict__ exact,
                                                        const int* __restrict__ old_labels,
                                                        const int* __restrict__ counts, int mode,
                                                        int* __restrict__ new_labels, Ctl* __restrict__ ctl) {
    pdl_enter();
    if (ctl->done) return;
    const unsigned cnt = *count;
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl->exact_fallbacks += cnt;
    const int lane = threadIdx.x & 31;
    for (unsigned idx = blockIdx.x; idx < cnt; idx += gridDim.x) {
        const int j = list[idx];
        const T* x = M + (int64_t)j * d;
        for (int k = threadIdx.x; k < c; k += blockDim.x) {  // k_exact_cols' chains
            const double* cv = C + (int64_t)k * d;
            double s = 0.0;
            for (int64_t i = 0; i < d; ++i) {
                const double t = (double)__ldg(x + i) - __ldg(cv + i);
                s += t * t;
            }
            exact[(int64_t)idx * c + k] = s;
        }
        __syncthreads();
        if (threadIdx.x < 32) {  // k_redecide's decision
            auto fn = [&](int, int k, double& lo, double& hi, double& mid) {
                mid = exact[(int64_t)idx * c + k];
                lo = hi = mid;
            };
            const int old = old_labels ? old_labels[j] : -1;
            int nl = old;
            const int st = decide_column(j, c, old, counts, mode == 1, fn, nl);
            if (lane == 0) {
                new_labels[j] = nl;
                if (st == ST_CHANGED) atomicAdd(&ctl->changed, 1u);
                if (st == ST_MOVE) atomicAdd(&ctl->moves, 1u);
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// k-means++ distance update (kmeans.cpp:188-191):
//   d2[j] = std::min(d2[j], sq_dist(col_j, col_last))
// Warp-transposed exact chains: lane = column, 32×32 tiles read coalesced.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(64) k_pp_d2(const T* __restrict__ M, int64_t d, int n, int last,
                                              double* __restrict__ d2) {
    // lane = column; rows stream through a PD-deep cp.async ring of 32×32
    // tiles per warp so the per-column sequential chain (the latency floor:
    // d dependent adds) is not also waiting on memory
    constexpr int PD = 4, W = 2;
    extern __shared__ __align__(16) unsigned char pp_sm[];
    auto tile = reinterpret_cast<T(*)[PD][32][33]>(pp_sm);                       // [W][PD][32][33]
    auto lastv = reinterpret_cast<T(*)[PD][32]>(pp_sm + sizeof(T) * W * PD * 32 * 33);  // [W][PD][32]
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int j0 = (blockIdx.x * W + w) * 32;
    if (j0 >= n) return;
    const int64_t ntile = (d + 31) / 32;
    auto issue = [&](int64_t t) {
        const int slot = (int)(t % PD);
        const int64_t i = t * 32 + lane;
        const bool okr = i < d;
        if (sizeof(T) == 8) cp_async8(&lastv[w][slot][lane], okr ? M + (int64_t)last * d + i : M, okr);
        else cp_async4(&lastv[w][slot][lane], okr ? M + (int64_t)last * d + i : M, okr);
        for (int cc = 0; cc < 32; ++cc) {
            const int j = j0 + cc;
            const bool ok = okr && j < n;
            const T* src = ok ? M + (int64_t)j * d + i : M;
            if (sizeof(T) == 8) cp_async8(&tile[w][slot][cc][lane], src, ok);
            else cp_async4(&tile[w][slot][cc][lane], src, ok);
        }
        cp_commit();
    };
    for (int64_t t = 0; t < PD - 1; ++t) {
        if (t < ntile) issue(t);
        else cp_commit();
    }
    double s = 0.0;
    for (int64_t t = 0; t < ntile; ++t) {
        if (t + PD - 1 < ntile) issue(t + PD - 1);
        else cp_commit();
        cp_wait<PD - 1>();
        __syncwarp();
        const int slot = (int)(t % PD);
        const int lim = (int)((d - t * 32) < 32 ? (d - t * 32) : 32);
        for (int r = 0; r < lim; ++r) {
            const double tt = (double)tile[w][slot][lane][r] - (double)lastv[w][slot][r];
            s += tt * tt;
        }
        __syncwarp();
    }
    const int j = j0 + lane;
    if (j < n) {
        const double old = d2[j];
        d2[j] = (s < old) ? s : old;
    }
}

// dst[:, list[y]] = src[:, list[y]] for the listed columns (d-long)
__global__ void k_copy_cols(const double* __restrict__ src, double* __restrict__ dst, int64_t d,
                            const int* __restrict__ list) {
    const int64_t k = __ldg(list + blockIdx.y);
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); i < d; i += (int64_t)gridDim.x * blockDim.x)
        dst[k * d + i] = src[k * d + i];
}

// k-means++ distance update of R restarts seeded side by side: one pass over
// the columns updates d2[r·n + j] = min(d2[r·n + j], sq_dist(col_j, col_last[r]))
// for every restart (each chain exact, ascending i, as k_pp_d2).
struct PPLast {
    int v[8];
};
template <typename T, int R>
__global__ void __launch_bounds__(64) k_pp_d2_multi(const T* __restrict__ M, int64_t d, int n, PPLast last,
                                                    double* __restrict__ d2) {
    constexpr int PD = 4, W = 2;
    extern __shared__ __align__(16) unsigned char pp_sm[];
    auto tile = reinterpret_cast<T(*)[PD][32][33]>(pp_sm);                           // [W][PD][32][33]
    auto lastv = reinterpret_cast<T(*)[PD][R][32]>(pp_sm + sizeof(T) * W * PD * 32 * 33);  // [W][PD][R][32]
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int j0 = (blockIdx.x * W + w) * 32;
    if (j0 >= n) return;
    const int64_t ntile = (d + 31) / 32;
    auto issue = [&](int64_t t) {
        const int slot = (int)(t % PD);
        const int64_t i = t * 32 + lane;
        const bool okr = i < d;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const T* src = okr ? M + (int64_t)last.v[r] * d + i : M;
            if (sizeof(T) == 8) cp_async8(&lastv[w][slot][r][lane], src, okr);
            else cp_async4(&lastv[w][slot][r][lane], src, okr);
        }
        for (int cc = 0; cc < 32; ++cc) {
            const int j = j0 + cc;
            const bool ok = okr && j < n;
            const T* src = ok ? M + (int64_t)j * d + i : M;
            if (sizeof(T) == 8) cp_async8(&tile[w][slot][cc][lane], src, ok);
            else cp_async4(&tile[w][slot][cc][lane], src, ok);
        }
        cp_commit();
    };
    for (int64_t t = 0; t < PD - 1; ++t) {
        if (t < ntile) issue(t);
        else cp_commit();
    }
    double s[R];
#pragma unroll
    for (int r = 0; r < R; ++r) s[r] = 0.0;
    for (int64_t t = 0; t < ntile; ++t) {
        if (t + PD - 1 < ntile) issue(t + PD - 1);
        else cp_commit();
        cp_wait<PD - 1>();
        __syncwarp();
        const int slot = (int)(t % PD);
        const int lim = (int)((d - t * 32) < 32 ? (d - t * 32) : 32);
        if (lim == 32) {
            // full tile: rows in batches of 8 (the shared-memory loads of a batch
            // issue together; each chain still adds in ascending row order)
#pragma unroll
            for (int q0 = 0; q0 < 32; q0 += 8) {
                double x[8], lv[R][8];
#pragma unroll
                for (int u = 0; u < 8; ++u) x[u] = (double)tile[w][slot][lane][q0 + u];
#pragma unroll
                for (int r = 0; r < R; ++r)
#pragma unroll
                    for (int u = 0; u < 8; ++u) lv[r][u] = (double)lastv[w][slot][r][q0 + u];
#pragma unroll
                for (int u = 0; u < 8; ++u)
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const double tt = x[u] - lv[r][u];
                        s[r] += tt * tt;
                    }
            }
        } else {
            for (int q = 0; q < lim; ++q) {
                const double x = (double)tile[w][slot][lane][q];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const double tt = x - (double)lastv[w][slot][r][q];
                    s[r] += tt * tt;
                }
            }
        }
        __syncwarp();
    }
    const int j = j0 + lane;
    if (j < n)
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const double old = d2[(int64_t)r * n + j];
            d2[(int64_t)r * n + j] = (s[r] < old) ? s[r] : old;
        }
}

// Exact own-centroid distance sq_dist(col_j, C[:, label_j]) for every column
// (inertia_of, kmeans.cpp:84-91; repair_empty, kmeans.cpp:51).  Lane = column:
// each lane runs its column's chain in ascending i (the reference's order) on
// 32×32 tiles of the 32 columns and of their 32 own centroids, both streamed
// through a cp.async ring (coalesced 32-element rows), so the chain never
// waits on a global load — it is the d dependent adds per column that bound
// the kernel (C3: 5 ms → 0.3 ms per restart at the end of kmeans(X)).
constexpr int OWN_PD = 4, OWN_W = 2;
template <typename T>
constexpr size_t own_exact_smem() {
    return (size_t)OWN_W * OWN_PD * 32 * 33 * (sizeof(T) + sizeof(double));
}
template <typename T>
__global__ void __launch_bounds__(OWN_W * 32) k_own_exact(const T* __restrict__ M,
                                                          const double* __restrict__ C, int64_t d, int n,
                                                          const int* __restrict__ labels,
                                                          double* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char own_sm[];
    auto tile = reinterpret_cast<T(*)[OWN_PD][32][33]>(own_sm);  // [W][PD][column][row]
    auto ctile = reinterpret_cast<double(*)[OWN_PD][32][33]>(own_sm + sizeof(T) * OWN_W * OWN_PD * 32 * 33);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int j0 = (blockIdx.x * OWN_W + w) * 32;
    if (j0 >= n) return;
    const int j = j0 + lane;
    const int64_t ntile = (d + 31) / 32;
    int64_t moff[32], coff[32];  // column q of the tile: its data and its own centroid
#pragma unroll
    for (int q = 0; q < 32; ++q) {
        const int jj = j0 + q < n ? j0 + q : j0;
        moff[q] = (int64_t)jj * d;
        coff[q] = (int64_t)__ldg(labels + jj) * d;
    }
    auto issue = [&](int64_t t) {
        const int slot = (int)(t % OWN_PD);
        const int64_t i = t * 32 + lane;
        const bool ok = i < d;
#pragma unroll
        for (int q = 0; q < 32; ++q) {
            const T* src = ok ? M + moff[q] + i : M;
            if (sizeof(T) == 8) cp_async8(&tile[w][slot][q][lane], src, ok);
            else cp_async4(&tile[w][slot][q][lane], src, ok);
            cp_async8(&ctile[w][slot][q][lane], ok ? C + coff[q] + i : C, ok);
        }
        cp_commit();
    };
    for (int64_t t = 0; t < OWN_PD - 1; ++t) {
        if (t < ntile) issue(t);
        else cp_commit();
    }
    double s = 0.0;
    for (int64_t t = 0; t < ntile; ++t) {
        if (t + OWN_PD - 1 < ntile) issue(t + OWN_PD - 1);
        else cp_commit();
        cp_wait<OWN_PD - 1>();
        __syncwarp();
        const int slot = (int)(t % OWN_PD);
        const int lim = (int)((d - t * 32) < 32 ? (d - t * 32) : 32);
        if (lim == 32) {
#pragma unroll
            for (int r = 0; r < 32; ++r) {
                const double tt = (double)tile[w][slot][lane][r] - ctile[w][slot][lane][r];  // kmeans.cpp:15-16
                s += tt * tt;
            }
        } else {
            for (int r = 0; r < lim; ++r) {
                const double tt = (double)tile[w][slot][lane][r] - ctile[w][slot][lane][r];
                s += tt * tt;
            }
        }
        __syncwarp();
    }
    if (j < n) out[j] = s;
}

template <typename T>
__global__ void k_gather_cols(const T* __restrict__ M, int64_t d, const int* __restrict__ idx,
                              int c, double* __restrict__ C) {
    const int k = blockIdx.y;
    const int64_t src = (int64_t)idx[k] * d;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d;
         i += (int64_t)gridDim.x * blockDim.x)
        C[(int64_t)k * d + i] = (double)M[src + i];
}

// Lloyd stop test partials (kmeans.cpp:148-153): Σ(next−C)², ΣC²
__global__ void __launch_bounds__(256) k_moved_scale(const double* __restrict__ next,
                                                     const double* __restrict__ C, int64_t N,
                                                     double* __restrict__ partials) {
    __shared__ double red[64];
    double a = 0.0, b = 0.0;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < N;
         k += (int64_t)gridDim.x * blockDim.x) {
        const double t = next[k] - C[k];
        a += t * t;
        b += C[k] * C[k];
    }
    double v[2] = {a, b};
    block_sum<2>(v, red);
    if (threadIdx.x == 0) {
        partials[blockIdx.x * 2] = v[0];
        partials[blockIdx.x * 2 + 1] = v[1];
    }
}

// The reference's exact sequential chains for the Lloyd stop (used only when
// the tree-summed test lands within 1e-9 of its threshold).
// The reference's sequential chains (kmeans.cpp:150-155) on one thread; the
// other threads stage the next chunk of both operands in shared memory, so the
// chain runs at add latency instead of load latency.
constexpr int MSE_CH = 1024;
__global__ void __launch_bounds__(256) k_moved_scale_exact(const double* __restrict__ next,
                                                           const double* __restrict__ C, int64_t N,
                                                           double* __restrict__ out) {
    __shared__ double sn[2][MSE_CH], sc[2][MSE_CH];
    const int tid = threadIdx.x;
    double moved = 0.0, scale = 0.0;
    const int64_t nch = (N + MSE_CH - 1) / MSE_CH;
    auto stage = [&](int64_t ch, int b) {
        const int64_t k0 = ch * MSE_CH;
        for (int i = tid; i < MSE_CH; i += blockDim.x) {
            const int64_t k = k0 + i;
            sn[b][i] = k < N ? next[k] : 0.0;
            sc[b][i] = k < N ? C[k] : 0.0;
        }
    };
    if (nch > 0) stage(0, 0);
    __syncthreads();
    for (int64_t ch = 0; ch < nch; ++ch) {
        const int b = (int)(ch & 1);
        if (tid == 0) {
            const int lim = (int)(N - ch * MSE_CH < MSE_CH ? N - ch * MSE_CH : MSE_CH);
            for (int i = 0; i < lim; ++i) {
                const double t = sn[b][i] - sc[b][i];
                moved += t * t;
                scale += sc[b][i] * sc[b][i];
            }
        } else if (ch + 1 < nch) {
            // threads 1.. stage the next chunk meanwhile
            const int64_t k0 = (ch + 1) * MSE_CH;
            for (int i = tid - 1; i < MSE_CH; i += blockDim.x - 1) {
                const int64_t k = k0 + i;
                sn[b ^ 1][i] = k < N ? next[k] : 0.0;
                sc[b ^ 1][i] = k < N ? C[k] : 0.0;
            }
        }
        __syncthreads();
    }
    if (tid == 0) {
        out[0] = moved;
        out[1] = scale;
    }
}

__global__ void k_count_labels(const int* __restrict__ labels, int n, int* __restrict__ counts) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
        atomicAdd(&counts[labels[j]], 1);
}

// ---------------------------------------------------------------------------
// repair_empty (kmeans.cpp:40-64), one block: for each empty cluster e in
// ascending order, steal the farthest point (strict > keeps the first index)
// among clusters with more than one member.  own[] holds the exact
// sq_dist(col_j, C[label_j]) values; the stolen point's entry is recomputed
// against its new centroid, exactly as the reference's next scan sees it.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(1024) k_repair(const T* __restrict__ M,
                                                 const double* __restrict__ C, int64_t d, int n,
                                                 int c, int* __restrict__ labels,
                                                 int* __restrict__ counts,
                                                 double* __restrict__ own, int* __restrict__ err) {
    __shared__ double sv[32];
    __shared__ int sj[32];
    __shared__ int s_steal;
    __shared__ double s_worst;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int e = 0; e < c; ++e) {
        if (counts[e] > 0) continue;
        double best = -1.0;
        int bj = 0x7fffffff;
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
            if (counts[labels[j]] <= 1) continue;
            const double v = own[j];
            if (v > best) {  // ascending j per thread: strict > keeps the first
                best = v;
                bj = j;
            }
        }
        // argmax, ties → lowest j
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, best, o);
            const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
            if (ov > best || (ov == best && oj < bj)) {
                best = ov;
                bj = oj;
            }
        }
        if (lane == 0) {
            sv[w] = best;
            sj[w] = bj;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double b = -1.0;
            int jj = 0x7fffffff;
            for (int q = 0; q < (int)(blockDim.x >> 5); ++q)
                if (sv[q] > b || (sv[q] == b && sj[q] < jj)) {
                    b = sv[q];
                    jj = sj[q];
                }
            s_worst = b;
            s_steal = jj;
            if (b < 0.0) {
                *err = 1;  // "kmeans: cannot repair empty cluster"
            } else {
                counts[labels[jj]] -= 1;
                labels[jj] = e;
                counts[e] += 1;
                double s = 0.0;  // exact chain against the new centroid
                for (int64_t i = 0; i < d; ++i) {
                    const double t = (double)M[(int64_t)jj * d + i] - C[(int64_t)e * d + i];
                    s += t * t;
                }
                own[jj] = s;
            }
        }
        __syncthreads();
        if (s_worst < 0.0) return;
    }
}

}  // namespace respca_dev
