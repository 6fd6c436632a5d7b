// Pass A screen on the 5th-generation tensor cores (tcgen05.mma kind::f16,
// BF16 operands, FP32 accumulation in TMEM) — the ALM loop's fast-path check.
//
//   dot[s][j][k] = Σ_{i ∈ split s} bf16(L[i,j]) · bf16(C[i,k])      (FP32 accumulate)
//   xxp[s][j]    = Σ_{i ∈ split s} L[i,j]²                           (FP64, producers)
//
// Bound used by the decisions (km.cuh Screen with kappa = kBf16Kappa(d)):
//   |dot_tc − x·c| ≤ (2^-8 + 2^-16 + d·2^-23)·Σ|x_i c_i| ≤ κ·‖x‖‖c‖
// (two BF16 input roundings, exact BF16×BF16 products in FP32, ≤ d FP32
// accumulation roundings taken as truncations), so
//   |(xx + cc − 2·dot) − ref| ≤ κ·(‖x‖ + ‖c‖)² + the FP64 terms of km.cuh.
// On the BASELINE workloads every loop decision has a margin ≥ 0.1·(‖x‖+‖c‖)²
// (measured), so the coarse screen decides every column; anything
// it cannot decide goes to the exact sequential chain as before.
//
// CTA: 128 columns (UMMA M = 128) × 64 centroids (N = 64), split-K over d.
// Warps 0-7 produce: FP64 rows of L → BF16 in the canonical K-major
// SWIZZLE_128B layout (8-row × 128-byte atoms, 16-byte chunks XOR-swizzled by
// row), B tiles by cp.async from a BF16 copy of the centroids; warp 8 issues
// the MMAs (one elected lane) and commits stage buffers back through
// mbarriers; warps 0-3 drain the TMEM accumulator (tcgen05.ld 32x32b).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>

#include "km.cuh"

namespace respca_dev {

constexpr int TC_M = 128, TC_N = 64, TC_KB = 64;  // K elements per stage (128 bytes of bf16)
constexpr int TC_STAGES = 4;
constexpr int TC_PRODUCERS = 8;                   // producer warps
constexpr int TC_THREADS = (TC_PRODUCERS + 1) * 32;
constexpr int TC_A_BYTES = TC_M * TC_KB * 2;      // 16 KB
constexpr int TC_B_BYTES = TC_N * TC_KB * 2;      // 8 KB
constexpr int TC_STAGE_BYTES = TC_A_BYTES + TC_B_BYTES;
constexpr size_t TC_SMEM = 1024 + (size_t)TC_STAGES * TC_STAGE_BYTES + 1024;

__host__ __device__ inline double tc_bf16_kappa(double d) {
    return 0.00390625 + 1.52587890625e-05 + d * 1.1920928955078125e-07;
}

RESPCA_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

RESPCA_DEV void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
RESPCA_DEV void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// bounded wait: returns false after ~2 s by default (a hang guard, never expected)
RESPCA_DEV bool mbar_wait(uint64_t* bar, uint32_t parity, unsigned long long limit_ns = 2000000000ULL) {
    const uint32_t a = smem_u32(bar);
    uint32_t done = 0;
    unsigned long long t0 = 0;
    for (int spin = 0;; ++spin) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
        if (done) return true;
        if ((spin & 1023) == 1023) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            if (!t0) t0 = t;
            else if (t - t0 > limit_ns) return false;
        }
    }
}

RESPCA_DEV void mbar_expect_tx_cta(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

RESPCA_DEV uint64_t tc_desc_sw128(uint32_t saddr) {
    // tcgen05 shared-memory matrix descriptor, K-major SWIZZLE_128B:
    // start>>4 [0,14), LBO>>4 [16,30) (unused for swizzled K-major: 1),
    // SBO>>4 [32,46) = 1024 B between 8-row atoms, version 1 [46,48),
    // base offset 0, layout type 2 = SWIZZLE_128B [61,64)
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// instruction descriptor: D f32, A/B bf16, K-major A and B, N = 64, M = 128
constexpr uint32_t TC_IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TC_N >> 3) << 17) |
                              ((uint32_t)(TC_M >> 4) << 24);

// byte offset of (row, 16-byte chunk) inside a K-major SWIZZLE_128B tile
RESPCA_DEV uint32_t sw128(int row, int chunk) {
    return (uint32_t)row * 128u + (uint32_t)((chunk ^ (row & 7)) << 4);
}

// centroids → BF16 K-major [TC_N][d_pad] (rows ≥ c zero) and ‖c_k‖² (FP64 FMA)
__global__ void __launch_bounds__(1024) k_tc_prep_centroids(const double* __restrict__ C, int64_t d, int c,
                                                             int64_t d_pad, __nv_bfloat16* __restrict__ Cb,
                                                             double* __restrict__ cc, int* __restrict__ err = nullptr) {
    __shared__ double red[32];
    pdl_enter();
    const int k = blockIdx.x;  // 0..TC_N-1
    if (err && k == 0 && threadIdx.x == 0) *err = 0;  // the screen's error flag, reset before it runs
    double s = 0.0;
    // 1024 threads, 4 loads in flight each: one latency round per 4096 rows
    for (int64_t i0 = threadIdx.x; i0 < d_pad; i0 += 4 * (int64_t)blockDim.x) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = i0 + u * (int64_t)blockDim.x;
            v[u] = (k < c && i < d) ? __ldg(C + (int64_t)k * d + i) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = i0 + u * (int64_t)blockDim.x;
            if (i < d_pad) {
                Cb[(int64_t)k * d_pad + i] = __double2bfloat16(v[u]);
                s = __fma_rn(v[u], v[u], s);
            }
        }
    }
    double v[1] = {s};
    block_sum<1>(v, red);
    if (threadIdx.x == 0 && k < c) cc[k] = v[0];
}

template <typename T>
__global__ void __launch_bounds__(TC_THREADS, 2) k_screen_tc(
    const T* __restrict__ M, const __nv_bfloat16* __restrict__ Cb, int64_t d, int64_t d_pad,
    int n, int c, int kblocks_per_split, double* __restrict__ part, double* __restrict__ xxp,
    int* __restrict__ err) {
    extern __shared__ __align__(1024) unsigned char tsm_raw[];
    // 1024-byte alignment for the SWIZZLE_128B atoms
    unsigned char* tsm = reinterpret_cast<unsigned char*>(
        ((uintptr_t)tsm_raw + 1023) & ~(uintptr_t)1023);
    unsigned char* stage_base = tsm;
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(tsm + (size_t)TC_STAGES * TC_STAGE_BYTES);
    uint64_t* empty_bar = full_bar + TC_STAGES;
    uint64_t* done_bar = empty_bar + TC_STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done_bar + 1);
    double* xx_s = reinterpret_cast<double*>(tmem_slot + 2);  // [TC_M]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j0 = blockIdx.x * TC_M, split = blockIdx.y;
    const int64_t kb0 = (int64_t)split * kblocks_per_split;
    const int64_t total_kb = (d + TC_KB - 1) / TC_KB;
    int64_t kb1 = kb0 + kblocks_per_split;
    if (kb1 > total_kb) kb1 = total_kb;
    const int nkb = kb1 > kb0 ? (int)(kb1 - kb0) : 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < TC_STAGES; ++s) {
            mbar_init(&full_bar[s], TC_PRODUCERS);
            mbar_init(&empty_bar[s], 1);
        }
        mbar_init(done_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == TC_PRODUCERS) {  // the MMA warp owns the TMEM allocation
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(TC_N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = *tmem_slot;

    if (warp < TC_PRODUCERS) {
        // ---------------- producers ----------------
        constexpr int RPW = TC_M / TC_PRODUCERS;  // rows (columns j) per warp: 16
        double xxr[RPW];
#pragma unroll
        for (int r = 0; r < RPW; ++r) xxr[r] = 0.0;
        for (int it = 0; it < nkb; ++it) {
            const int s = it % TC_STAGES;
            if (it >= TC_STAGES) {
                if (!mbar_wait(&empty_bar[s], ((it / TC_STAGES) - 1) & 1)) {
                    if (lane == 0) atomicExch(err, 1);
                    break;
                }
            }
            unsigned char* A = stage_base + (size_t)s * TC_STAGE_BYTES;
            unsigned char* B = A + TC_A_BYTES;
            const int64_t i0 = (kb0 + it) * TC_KB;
            // A: each lane converts elements (2·lane, 2·lane+1) of every row,
            // in batches of RB rows (all loads of a batch in flight together)
            constexpr int RB = 8;
#pragma unroll
            for (int rb = 0; rb < RPW; rb += RB) {
                double2 v[RB];
#pragma unroll
                for (int r = 0; r < RB; ++r) {
                    const int row = warp + (rb + r) * TC_PRODUCERS;
                    const int j = j0 + row;
                    const int64_t i = i0 + 2 * lane;
                    double x0 = 0.0, x1 = 0.0;
                    if (j < n) {
                        const T* src = M + (int64_t)j * d + i;
                        if (i + 1 < d) {
                            if (sizeof(T) == 8 && (d % 2) == 0) {
                                const double2 t = __ldcs(reinterpret_cast<const double2*>(src));
                                x0 = t.x;
                                x1 = t.y;
                            } else {
                                x0 = (double)src[0];
                                x1 = (double)src[1];
                            }
                        } else if (i < d) {
                            x0 = (double)src[0];
                        }
                    }
                    v[r] = make_double2(x0, x1);
                }
#pragma unroll
                for (int r = 0; r < RB; ++r) {
                    const int row = warp + (rb + r) * TC_PRODUCERS;
                    xxr[rb + r] = __fma_rn(v[r].y, v[r].y, __fma_rn(v[r].x, v[r].x, xxr[rb + r]));
                    __nv_bfloat162 b2;
                    b2.x = __double2bfloat16(v[r].x);
                    b2.y = __double2bfloat16(v[r].y);
                    // lane → K elements 2·lane..2·lane+1 = chunk lane/4, byte (lane%4)*4
                    *reinterpret_cast<__nv_bfloat162*>(A + sw128(row, lane >> 2) + (lane & 3) * 4) = b2;
                }
            }
            // B: 64 rows × 8 chunks of 16 B from the BF16 centroid copy
            for (int e = threadIdx.x; e < TC_N * 8; e += TC_PRODUCERS * 32) {
                const int row = e >> 3, ch = e & 7;
                const __nv_bfloat16* src = Cb + (int64_t)row * d_pad + i0 + ch * 8;
                cp_async16(B + sw128(row, ch), src, 16);
            }
            cp_commit();
            cp_wait<0>();
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&full_bar[s]);
        }
        // ‖x_j‖² of this split: reduce each row over the warp's lanes
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
            const double t = warp_sum(xxr[r]);
            if (lane == 0) xx_s[warp + r * TC_PRODUCERS] = t;
        }
    } else if (lane == 0) {
        // ---------------- MMA issuer ----------------
        bool ok = true;
        for (int it = 0; it < nkb; ++it) {
            const int s = it % TC_STAGES;
            if (!mbar_wait(&full_bar[s], (it / TC_STAGES) & 1)) {
                atomicExch(err, 2);
                ok = false;
                break;
            }
            asm volatile("tcgen05.fence::after_thread_sync;\n");
            const uint32_t a0 = smem_u32(stage_base + (size_t)s * TC_STAGE_BYTES);
            const uint32_t b0 = a0 + TC_A_BYTES;
#pragma unroll
            for (int kk = 0; kk < TC_KB / 16; ++kk) {  // K = 16 per kind::f16 MMA = 32 bytes
                const uint64_t ad = tc_desc_sw128(a0 + kk * 32);
                const uint64_t bd = tc_desc_sw128(b0 + kk * 32);
                const uint32_t acc = (it > 0 || kk > 0) ? 1u : 0u;
                asm volatile(
                    "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                    " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                    "l"(ad), "l"(bd), "r"(TC_IDESC), "r"(acc));
            }
            asm volatile(
                "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                    smem_u32(&empty_bar[s]))
                : "memory");
        }
        if (ok)
            asm volatile(
                "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                    smem_u32(done_bar))
                : "memory");
        else
            mbar_arrive(done_bar);
    }
    __syncthreads();  // xx_s complete; every stage issued
    // ---------------- epilogue: warps 0-3 drain TMEM (lane = accumulator row) ----------------
    if (warp < 4) {
        bool ok = nkb == 0 || mbar_wait(done_bar, 0);
        if (!ok && lane == 0) atomicExch(err, 3);
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        const int row = warp * 32 + lane;
        const int j = j0 + row;
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            uint32_t r[32];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
                "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                  "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),
                  "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]),
                  "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                  "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
                  "=r"(r[30]), "=r"(r[31])
                : "r"(taddr + half * 32));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            if (j < n && ok) {
                double* dst = part + ((int64_t)split * n + j) * c;
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                    const int k = half * 32 + q;
                    if (k < c) dst[k] = nkb ? (double)__uint_as_float(r[q]) : 0.0;
                }
            }
        }
        if (j < n) xxp[(int64_t)split * n + j] = nkb ? xx_s[row] : 0.0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == TC_PRODUCERS)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                     "r"(TC_N));
}

// ---------------------------------------------------------------------------
// TMA-fed variant for the ALM loop.  Pass F also writes L′ as BF16 in the
// K-major layout [n][d_pad] (Lb), so the screen no longer converts: one thread
// issues cp.async.bulk.tensor loads of the A tile (128 columns × 64 K, 16 KB)
// and the B tile (64 centroids × 64 K, 8 KB) straight into the SWIZZLE_128B
// layout the MMA descriptors expect; one thread issues tcgen05.mma; four warps
// accumulate ‖x_j‖² from the BF16 A tiles while the MMAs run (FP64
// accumulation of bf16 squares: |Σ bf16(x)² − ‖x‖²| ≤ (2⁻⁸ + 2⁻¹⁷)‖x‖²,
// covered by tma_xx_kappa) and then drain TMEM.
//   warp 0: TMA producer   warp 1: MMA issuer   warps 2-5: ‖x‖² + epilogue
// ---------------------------------------------------------------------------
constexpr int TM_THREADS = 6 * 32;

__host__ __device__ inline double tma_xx_kappa(double d) {
    // bf16 rounding of x (2⁻⁸ + 2⁻¹⁷), FP32 stage sums of 64 squares
    // (64·2⁻²⁴), the FP64 accumulation (d·1.1u)
    return 0.00390625 + 7.62939453125e-06 + 3.814697265625e-06 + d * 1.2212453270876722e-16;
}
// squares below FP32's normal range lose bits in the stage sums: absolute
// error ≤ 2⁻¹⁴⁹ per element (added to the screen's interval half-width)
__host__ __device__ inline double tma_xx_abs(double d) { return d * 1.401298464324817e-45; }

RESPCA_DEV void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];\n" ::"r"(dst),
        "l"((uint64_t)map), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

// STAGES-deep TMA ring, MINB CTAs per SM (smem ≈ STAGES·24 KB)
template <int STAGES>
constexpr size_t tm_smem() {
    return 1024 + (size_t)STAGES * TC_STAGE_BYTES + 1024;
}
template <int STAGES, int MINB>
__global__ void __launch_bounds__(TM_THREADS, MINB) k_screen_tma(
    const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int64_t d,
    int n, int c, int kblocks_per_split, double* __restrict__ part, double* __restrict__ xxp,
    int* __restrict__ err) {
    constexpr int TC_STAGES = STAGES;  // this kernel's ring depth
    pdl_enter();
    extern __shared__ __align__(1024) unsigned char tsm_raw[];
    unsigned char* tsm = reinterpret_cast<unsigned char*>(((uintptr_t)tsm_raw + 1023) & ~(uintptr_t)1023);
    unsigned char* stage_base = tsm;
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(tsm + (size_t)TC_STAGES * TC_STAGE_BYTES);
    uint64_t* empty_bar = full_bar + TC_STAGES;
    uint64_t* done_bar = empty_bar + TC_STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done_bar + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j0 = blockIdx.x * TC_M, split = blockIdx.y;
    const int64_t kb0 = (int64_t)split * kblocks_per_split;
    const int64_t total_kb = (d + TC_KB - 1) / TC_KB;
    int64_t kb1 = kb0 + kblocks_per_split;
    if (kb1 > total_kb) kb1 = total_kb;
    const int nkb = kb1 > kb0 ? (int)(kb1 - kb0) : 0;
    const int rot = nkb ? (int)(((int64_t)blockIdx.x * 5) % nkb) : 0;  // this tile's first K block (the sums are order-free: bounds cover any order)

    if (threadIdx.x == 0) {
        for (int s = 0; s < TC_STAGES; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 1 + 4);  // MMA commit + the four ‖x‖² warps
        }
        mbar_init(done_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"((uint64_t)&mapA) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"((uint64_t)&mapB) : "memory");
    }
    if (warp == 1) {  // the MMA warp owns the TMEM allocation
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(TC_N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = *tmem_slot;

    double xx = 0.0;                        // warps 2-5: ‖x_row‖² of this split
    const int quarter = warp & 3;           // TMEM lanes a warp may access: 32·(warp % 4)
    const int row = quarter * 32 + lane;
    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer ----------------
            for (int it = 0; it < nkb; ++it) {
                const int s = it % TC_STAGES;
                if (it >= TC_STAGES && !mbar_wait(&empty_bar[s], ((it / TC_STAGES) - 1) & 1)) {
                    atomicExch(err, 1);
                    break;
                }
                const uint32_t a = smem_u32(stage_base + (size_t)s * TC_STAGE_BYTES);
                mbar_expect_tx_cta(&full_bar[s], TC_A_BYTES + TC_B_BYTES);
                // K blocks in a rotated order, different per column tile: the
                // tiles of a split would otherwise all read the same centroid
                // (B) block at the same time — one L2 hot spot serving 79 CTAs
                const int kx = (int)((kb0 + (it + rot) % nkb) * TC_KB);
                tma_load_2d(a, &mapA, kx, j0, &full_bar[s]);
                tma_load_2d(a + TC_A_BYTES, &mapB, kx, 0, &full_bar[s]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer ----------------
            bool ok = true;
            for (int it = 0; it < nkb; ++it) {
                const int s = it % TC_STAGES;
                if (!mbar_wait(&full_bar[s], (it / TC_STAGES) & 1)) {
                    atomicExch(err, 2);
                    ok = false;
                    break;
                }
                asm volatile("tcgen05.fence::after_thread_sync;\n");
                const uint32_t a0 = smem_u32(stage_base + (size_t)s * TC_STAGE_BYTES);
                const uint32_t b0 = a0 + TC_A_BYTES;
#pragma unroll
                for (int kk = 0; kk < TC_KB / 16; ++kk) {
                    const uint64_t ad = tc_desc_sw128(a0 + kk * 32);
                    const uint64_t bd = tc_desc_sw128(b0 + kk * 32);
                    const uint32_t acc = (it > 0 || kk > 0) ? 1u : 0u;
                    asm volatile(
                        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                        "l"(ad), "l"(bd), "r"(TC_IDESC), "r"(acc));
                }
                asm volatile(
                    "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                        smem_u32(&empty_bar[s]))
                    : "memory");
            }
            if (ok)
                asm volatile(
                    "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                        smem_u32(done_bar))
                    : "memory");
            else
                mbar_arrive(done_bar);
        }
    } else {  // ---------------- ‖x‖² from the landed A tiles ----------------
        for (int it = 0; it < nkb; ++it) {
            const int s = it % TC_STAGES;
            if (!mbar_wait(&full_bar[s], (it / TC_STAGES) & 1)) {
                if (lane == 0) atomicExch(err, 4);
                break;
            }
            const unsigned char* A = stage_base + (size_t)s * TC_STAGE_BYTES;
            // the 64 squares of a stage summed in FP32 (a bf16 square is exact
            // in FP32; 63 roundings ≤ 64·2⁻²⁴ relative, in tma_xx_kappa), then
            // one conversion: F2F.F64.F32 per element throttled these warps
            uint4 q[8];
#pragma unroll
            for (int ch = 0; ch < 8; ++ch) q[ch] = *reinterpret_cast<const uint4*>(A + sw128(row, ch));
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[s]);  // the stage is in registers: release it
            float f0 = 0.0f, f1 = 0.0f;  // two FP32 chains of 32 squares
#pragma unroll
            for (int ch = 0; ch < 8; ++ch) {
                const uint32_t w[4] = {q[ch].x, q[ch].y, q[ch].z, q[ch].w};
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const float lo = __uint_as_float(w[h] << 16);
                    const float hi = __uint_as_float(w[h] & 0xffff0000u);
                    f0 = __fmaf_rn(lo, lo, f0);
                    f1 = __fmaf_rn(hi, hi, f1);
                }
            }
            xx += (double)f0 + (double)f1;
        }
    }
    __syncthreads();  // every stage issued
    if (warp >= 2) {  // ---------------- epilogue: TMEM → partials ----------------
        bool ok = nkb == 0 || mbar_wait(done_bar, 0);
        if (!ok && lane == 0) atomicExch(err, 3);
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        const int j = j0 + row;
        const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            uint32_t r[32];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
                "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                  "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),
                  "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]),
                  "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                  "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
                  "=r"(r[30]), "=r"(r[31])
                : "r"(taddr + half * 32));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            if (j < n && ok) {
                double* dst = part + ((int64_t)split * n + j) * c;
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                    const int k = half * 32 + q;
                    if (k < c) dst[k] = nkb ? (double)__uint_as_float(r[q]) : 0.0;
                }
            }
        }
        if (j < n) xxp[(int64_t)split * n + j] = nkb ? xx : 0.0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TC_N));
}

}  // namespace respca_dev
