// Shared device definitions for the RES-PCA engine.
//
// Numerical contract: this translation unit is compiled with --fmad=false, so
// every `a*b + c` below is a rounded multiply followed by a rounded add —
// the reference's x86-64 (SSE2, no FMA) arithmetic.  Division and sqrt are the
// IEEE correctly-rounded variants (nvcc defaults -prec-div/-prec-sqrt).  Where
// a kernel deliberately uses FMA (the screened distance kernel), it calls
// __fma_rn explicitly and its result is only ever used through a rigorous
// error bound.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <utility>

#define RESPCA_DEV __device__ __forceinline__

namespace respca_dev {

constexpr int kMaxBlocks = 4096;

// Device-resident control block of the ALM loop (one per context).  The
// finalize kernel advances it, so the captured graph needs no host scalars.
struct Ctl {
    // scalars of the current iteration t
    double rho;       // ρ_t
    double rho_next;  // ρ_{t+1} = min(ρ_t κ, 1e12)         (solver.cpp:110)
    double own_w;     // ρ_t / (2λ + ρ_t)                   (solver.cpp:58)
    double thr;       // 1 / ρ_t                            (solver.cpp:175)
    double lambda, kappa, tol, xnorm;
    int iter;         // t
    int budget;       // fixed_iters.value_or(max_iter)    (solver.cpp:152)
    int fixed;        // fixed_iters set → never stop early (solver.cpp:197)
    int parity;       // which G buffer holds G_t
    int converged;
    int slow;         // p-update of iteration t changed labels / moved a point
    int nonfinite;
    int done;         // loop finished (converged, budget, or slow → host)
    unsigned int changed, moves, ambiguous;  // counters of the decide pass
    int amb_list_len;
    double last_l1;   // ‖S‖₁ of the last finalized iteration (objective patch-up)
    unsigned int margin_hist[6];  // diagnostics: columns whose relative decision margin < 1e-1..1e-6
    int l21;          // sparse_norm = L21: the sparse term comes from `sparse_term`
    double sparse_term;
    unsigned long long exact_fallbacks;
    // ALM stop guard (solver.cpp:197 on the sequential chains of solver.cpp:14-31
    // and matrix.cpp:99-103): the three residual sums are tree sums here; the
    // reference's chain of the same N non-negative terms lies within
    // sum_eps·(tree sum) of it, so the reference's decision max(...) <= tol is
    // known exactly unless tol falls inside the interval — then stop_amb sends
    // the iteration to the host, which recomputes the chains in the
    // reference's order (Alm::resolve_stop).
    int guard;        // 1: decide on intervals (fp64 storage); 0: on the tree values
    int force_exact;  // RESPCA_ALM_STOP_FORCE_EXACT=1: every stop test goes to the chains
    int stop_amb;     // the stop test of the last finalized iteration was undecidable
    double sum_eps;   // relative bound |chain − tree| ≤ sum_eps·tree (rounded up)
    double xn_lo, xn_hi;  // bounds on the reference's ‖X‖ (= xnorm once it is the chain value)
    double l21_smin;      // ℓ2,1: min over columns of |‖B_j‖ − 1/ρ| (k_l21_term)
};

// Pass F partials per CTA: Σ feas², Σ dL², Σ dS², Σ|S|, Σ scatter, and the
// minimum over the CTA's elements of ||B| − 1/ρ| (the S-support margin)
constexpr int PF_STRIDE = 6;

RESPCA_DEV double warp_min(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
// block minimum (all threads get it); `red` holds ≥ 32 doubles
RESPCA_DEV double block_min(double v, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    v = warp_min(v);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    v = warp_min(lane < nw ? red[lane] : INFINITY);
    __syncthreads();
    return v;
}

RESPCA_DEV double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block reduction of NV doubles in fixed order (deterministic).  All threads
// get the totals.  `red` must hold 32*NV doubles.
template <int NV>
RESPCA_DEV void block_sum(double (&v)[NV], double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int q = 0; q < NV; ++q) v[q] = warp_sum(v[q]);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < NV; ++q) red[q * 32 + warp] = v[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        double t = lane < nw ? red[q * 32 + lane] : 0.0;
        v[q] = warp_sum(t);
    }
    __syncthreads();
}

template <typename T>
RESPCA_DEV double ld(const T* p) {
    return (double)__ldg(p);
}

// Programmatic dependent launch (PDL).  Kernels launched through pdl_launch
// start with pdl_enter(): griddepcontrol.wait blocks until the previous
// kernel on the stream has COMPLETED and its writes are visible (so every
// read below it sees exactly what a plain launch would), then the kernel
// allows its own dependent to be scheduled.  The gain is only the launch and
// CTA rasterisation latency at each kernel boundary, hidden under the
// predecessor's tail.  Without the launch attribute both instructions are
// no-ops.  RESPCA_PDL=0 launches plainly.
RESPCA_DEV void pdl_enter() {
    asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory");
}

}  // namespace respca_dev

namespace respca_host {
inline bool pdl_on() {  // read per launch: the captured graph's key includes it
    const char* e = std::getenv("RESPCA_PDL");
    return e ? std::atoi(e) != 0 : true;
}
template <class... P, class... A>
inline cudaError_t pdl_launch(void (*kf)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              A&&... args) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = grid;
    lc.blockDim = block;
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = pdl_on() ? 1 : 0;
    return cudaLaunchKernelEx(&lc, kf, std::forward<A>(args)...);
}
}  // namespace respca_host
