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

}  // namespace respca_dev
