// Device assembly of the "respca-synth-1" rpca workloads (csrc/synth.c;
// SURVEY §8(f) item 2).  The O((d+n)·r) normal factors U, V come from the host
// generator (glibc log/cos, as synth.c); the O(d·n) part — L0 = U·Vᵀ summed
// over k in ascending order, the Bernoulli(p) support and U[lo, hi] values of
// S0 from the same counter-based draws — runs here, so X is byte-identical to
// synth.c's while a 40,000² matrix takes milliseconds instead of seconds.
#pragma once

#include <stdint.h>

#include "common.cuh"

namespace respca_dev {

RESPCA_DEV uint64_t sy_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
RESPCA_DEV uint64_t sy_draw(uint64_t key, uint64_t idx) {
    return sy_mix64(key ^ (idx * 0xD1B54A32D192ED03ULL + 0x632BE59BD9B4E019ULL));
}
RESPCA_DEV double sy_unit01(uint64_t u) { return (double)(u >> 11) * (1.0 / 9007199254740992.0); }

// one CTA per (row block, column): acc = Σ_k U[i,k]·V[j,k] (k ascending,
// unfused multiply-add as synth.c under -ffp-contract=off), then S0
template <typename T>
__global__ void __launch_bounds__(256) k_synth_rpca(const double* __restrict__ U, const double* __restrict__ V,
                                                    int64_t d, int r, double p, double lo, double span,
                                                    uint64_t ks, uint64_t kval, int64_t j_base,
                                                    T* __restrict__ X) {
    extern __shared__ double vj[];
    const int64_t j = blockIdx.y;
    for (int k = threadIdx.x; k < r; k += blockDim.x) vj[k] = V[j * r + k];
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= d) return;
    double acc = 0.0;
    for (int k = 0; k < r; ++k) acc = __dadd_rn(acc, __dmul_rn(U[(int64_t)k * d + i], vj[k]));
    const uint64_t e = (uint64_t)(j_base + j) * (uint64_t)d + (uint64_t)i;  // global element: the draws' counter
    double s = 0.0;
    if (sy_unit01(sy_draw(ks, e)) < p) s = __dadd_rn(lo, __dmul_rn(span, sy_unit01(sy_draw(kval, e))));
    X[j * d + i] = (T)__dadd_rn(acc, s);
}

// ---------------------------------------------------------------------------
// io::synth_generate (io.cpp:232-294) with its O(d·n) assembly on the device.
// The libstdc++ draws stay on the host in the reference's order (c·d uniform
// prototype entries, then per corruption one position, one sign and one
// magnitude draw, then d·n normal draws when noise_sigma > 0); the device
// writes L0 (each column = its group's prototype), scatters the nnz
// corruptions into S0, forms X = L0 + S0 and adds the noise chunk by chunk.
// ---------------------------------------------------------------------------
// column j's group under the reference's near-equal contiguous blocks
RESPCA_DEV uint64_t sg_label(uint64_t j, uint64_t base, uint64_t rem) {
    const uint64_t big = (base + 1) * rem;  // columns covered by the `rem` groups of base+1
    return j < big ? j / (base + 1) : rem + (j - big) / base;
}

__global__ void __launch_bounds__(256) k_sg_fill(const double* __restrict__ proto, uint64_t d, uint64_t n,
                                                 uint64_t base, uint64_t rem, double* __restrict__ L0,
                                                 double* __restrict__ S0) {
    const uint64_t j = blockIdx.y;
    const uint64_t g = sg_label(j, base, rem);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d; i += (uint64_t)gridDim.x * blockDim.x) {
        L0[j * d + i] = __ldg(proto + g * d + i);
        S0[j * d + i] = 0.0;
    }
}

__global__ void __launch_bounds__(256) k_sg_scatter(const uint64_t* __restrict__ pos, const double* __restrict__ val,
                                                    uint64_t nnz, double* __restrict__ S0) {
    const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < nnz) S0[pos[k]] = val[k];  // positions are distinct (a partial permutation)
}

__global__ void __launch_bounds__(256) k_sg_sum(const double* __restrict__ L0, const double* __restrict__ S0,
                                                uint64_t N, double* __restrict__ X) {
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < N; e += (uint64_t)gridDim.x * blockDim.x)
        X[e] = __dadd_rn(L0[e], S0[e]);
}

__global__ void __launch_bounds__(256) k_sg_noise(const double* __restrict__ z, uint64_t cnt, double* __restrict__ X) {
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += (uint64_t)gridDim.x * blockDim.x)
        X[e] = __dadd_rn(X[e], z[e]);
}

}  // namespace respca_dev
