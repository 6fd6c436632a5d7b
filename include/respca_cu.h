/* respca_cu.h — C-ABI of the B200-native RES-PCA solver (librespca_cu.so).
 *
 * This is the drop-in boundary.  The reference exposes the solver only as a C++
 * API (/root/reference/proj/include/respca/solver.hpp:67-88,
 * kmeans.hpp:28-43, matrix.hpp:82-98); there is no plugin registry or FFI.
 * A host binding (the C++ facade in include/respca_b200/respca.hpp, the Python
 * mirror in paper_1904_07497_b200/respca.py, or a user's own FFI) calls these
 * entry points with plain pointers and sizes.  No torch or C++ types cross it,
 * no exceptions cross it: every function returns a status code and
 * respca_cu_last_error(ctx) holds the reference's message text.
 *
 * Matrices are column-major d×n (leading dimension d), exactly the reference's
 * DenseMatrix layout (matrix.hpp:26-31).  Labels are uint64 (the reference's
 * std::size_t, matrix.hpp:77).  All pointers below are HOST pointers; the
 * library owns device memory, streams and graphs inside the context.
 */
#ifndef RESPCA_CU_H
#define RESPCA_CU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (map 1:1 onto the reference's exception classes). */
enum {
    RESPCA_OK = 0,
    RESPCA_EINVAL = 1,    /* std::invalid_argument (solver.cpp:41-46, 129-132, ...) */
    RESPCA_ERUNTIME = 2,  /* std::runtime_error ("kmeans: cannot repair empty cluster", kmeans.cpp:58) */
    RESPCA_ENOMEM = 3,    /* device allocation failed */
    RESPCA_ECUDA = 4,     /* CUDA runtime / driver error, or no usable sm_100 device */
    RESPCA_ENONFINITE = 5,/* a non-finite value appeared inside the loop (device flag) */
    RESPCA_EIO = 6        /* respca::io::IoError family (io.hpp:13-33): open / magic / truncation */
};

enum { RESPCA_F64 = 0, RESPCA_F32 = 1 };    /* storage type of X, L, S, Θ */
enum { RESPCA_L1 = 0, RESPCA_L21 = 1 };     /* SparseNorm, solver.hpp:11 */

typedef struct respca_cu_ctx respca_cu_ctx;

/* SolverConfig + KMeansConfig, field for field (solver.hpp:13-28, kmeans.hpp:11-17). */
typedef struct {
    int has_lambda;          /* 0 → λ = sqrt(max(d, n))  (solver.cpp:35-38) */
    double lambda;
    double rho0;             /* 1e-4 */
    double kappa;            /* 1.5 */
    double tol;              /* 1e-3 */
    uint64_t max_iter;       /* 500 */
    uint64_t c;              /* 1 */
    int sparse_norm;         /* RESPCA_L1 */
    uint64_t km_max_iters;   /* 100 */
    uint64_t km_n_restarts;  /* 1 (the initial clustering forces >= 5, solver.cpp:147) */
    uint64_t km_seed;        /* 0 */
    double km_tol;           /* 1e-6 */
    int has_fixed_iters;     /* solver.hpp:26-27 */
    uint64_t fixed_iters;
} respca_cu_config;

/* ConvergenceReport (solver.hpp:39-46) + timings.  The four arrays are caller
 * allocated with room for fixed_iters (if set) else max_iter entries; the
 * solver writes exactly `iters` entries. */
typedef struct {
    double* feas;
    double* delta_l;
    double* delta_s;
    double* objective;
    uint64_t iters;
    int converged;
    double lambda;          /* resolved λ (DecompositionResult::lambda) */
    double wall_time;       /* seconds, the reference's window: after validation → results on host */
    double init_ms;         /* one-time kmeans(X) on the device */
    double loop_ms;         /* ALM loop on the device */
    double h2d_ms, d2h_ms;
    uint64_t slow_iters;    /* iterations whose p-update changed labels or moved a point */
    uint64_t hartigan_moves;/* total exact Hartigan moves (initial clustering + loop) */
    uint64_t exact_fallbacks;/* distance decisions resolved by exact sequential chains */
    uint64_t stop_resolves; /* ALM stop tests decided on the reference's own sequential
                               residual chains (the tree-sum interval straddled tol) */
} respca_cu_report;

/* Decision margins of the last respca_cu_solve on a context (SURVEY.md
 * Appendix A): how far each discrete decision of the reference sat from its
 * threshold, so a run whose decisions come near reduction-order noise
 * (~1e-14 relative) is visible.  Relative margins; +inf where a decision did
 * not occur. */
typedef struct {
    double alm_stop;        /* min over iterations of |max(feas, dL, dS)/tol − 1|  (solver.cpp:197) */
    double alm_stop_final;  /* the same at the last iteration */
    double s_support;       /* min over iterations and entries of ||B| − 1/ρ|·ρ (ℓ1, solver.cpp:85);
                               ℓ2,1: min over columns of |‖B_j‖ − 1/ρ|·ρ (solver.cpp:95) */
    double lloyd_stop;      /* initial kmeans(X): min over Lloyd steps of |√moved − tol·√scale|/(tol·√scale)
                               (kmeans.cpp:155) */
    double restart_gap;     /* initial kmeans(X): (second smallest − smallest inertia)/smallest over the
                               restarts (kmeans.cpp:246) */
    uint64_t stop_resolves; /* stop tests decided on the reference's own chains */
} respca_cu_margins;

void respca_cu_default_config(respca_cu_config* cfg);

/* Context: owns the device buffers, streams and CUDA graphs.  One context per
 * host thread; a context is not thread-safe, distinct contexts are. */
int respca_cu_create(int device, respca_cu_ctx** out);
void respca_cu_destroy(respca_cu_ctx* ctx);
const char* respca_cu_last_error(const respca_cu_ctx* ctx);
/* number of kernels this context launched (graph nodes count per execution) */
uint64_t respca_cu_kernel_launches(const respca_cu_ctx* ctx);

/* respca::solve (solver.cpp:127-210 / solver.hpp:88).  x, L_out, S_out are
 * d·n elements of `dtype`; labels_out has n entries.  Validation and error
 * messages follow the reference.  dtype = RESPCA_F32 is an API extension
 * (the reference is fp64-only). */
int respca_cu_solve(respca_cu_ctx* ctx, const void* x, uint64_t d, uint64_t n, int dtype,
                    const respca_cu_config* cfg, void* L_out, void* S_out,
                    uint64_t* labels_out, respca_cu_report* rep);

/* --- building blocks (solver.hpp:67-84, kmeans.hpp:28-43, matrix.hpp:82-98),
 *     fp64, same semantics and error text as the reference functions ------- */
int respca_cu_l_update(respca_cu_ctx* ctx, const double* D, uint64_t d, uint64_t n,
                       const uint64_t* labels, uint64_t c, double lambda, double rho,
                       double* L_out);
int respca_cu_s_update_l1(respca_cu_ctx* ctx, const double* B, uint64_t d, uint64_t n,
                          double threshold, double* S_out);
int respca_cu_s_update_l21(respca_cu_ctx* ctx, const double* B, uint64_t d, uint64_t n,
                           double threshold, double* S_out);
/* Θ += ρ(X − L − S); ρ = min(ρκ, 1e12).  theta and rho are in/out. */
int respca_cu_multiplier_update(respca_cu_ctx* ctx, double* theta, const double* x,
                                const double* L, const double* S, uint64_t d, uint64_t n,
                                double* rho, double kappa);
int respca_cu_check_convergence(respca_cu_ctx* ctx, const double* x, const double* l_prev,
                                const double* l, const double* s_prev, const double* s,
                                uint64_t d, uint64_t n, double tol, int* converged,
                                double* feas, double* delta_l, double* delta_s);
int respca_cu_kmeans(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n,
                     uint64_t c, uint64_t max_iters, uint64_t n_restarts, uint64_t seed,
                     double tol, uint64_t* labels_out, double* centroids_out,
                     double* inertia, uint64_t* iters_run);
int respca_cu_kmeans_warm(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n,
                          uint64_t c, uint64_t max_iters, double tol,
                          const uint64_t* init_labels, uint64_t* labels_out,
                          double* centroids_out, double* inertia, uint64_t* iters_run);
/* std::mt19937_64 seeded with `seed` (the reference takes the engine by
 * reference; a fresh engine with this seed reproduces its first call). */
int respca_cu_kmeans_pp_init(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n,
                             uint64_t c, uint64_t seed, double* centroids_out);
/* Same, drawing from the CALLER's engine through two callbacks (the
 * reference's kmeans_pp_init advances the std::mt19937_64& it is given):
 *   draw_first(user, n)   must return uniform_int_distribution<size_t>(0, n-1)(rng)
 *   draw_real(user, total) must return uniform_real_distribution<double>(0, total)(rng) */
int respca_cu_kmeans_pp_init_cb(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n,
                                uint64_t c, uint64_t (*draw_first)(void*, uint64_t),
                                double (*draw_real)(void*, double), void* user,
                                double* centroids_out);
int respca_cu_lloyd_step(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n,
                         const double* centroids, uint64_t c, uint64_t* labels_out,
                         double* next_out);
int respca_cu_group_scatter(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n,
                            const uint64_t* labels, uint64_t c, double* out);
int respca_cu_frob_norm(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n,
                        double* out);
int respca_cu_elementwise_l1(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n,
                             double* out);
int respca_cu_l21_norm(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n,
                       double* out);
int respca_cu_column_l2_norms(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n,
                              double* out);
int respca_cu_column_mean(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n,
                          const uint64_t* cols, uint64_t ncols, double* out);

/* Test hook: the screened K-means distance of every (column j, centroid k)
 * pair and the rigorous half-width of its interval around the reference's
 * sq_dist (kmeans.cpp:12-19); row-major n×c outputs. */
int respca_cu_debug_screen(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n,
                           const double* centroids, uint64_t c, double* approx_out,
                           double* err_out);

/* Same for the tcgen05 BF16 screen used by the ALM fast path (c <= 64). */
int respca_cu_debug_screen_tc(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n,
                              const double* centroids, uint64_t c, double* approx_out,
                              double* err_out);

/* Test hook for device memory checking (compute-sanitizer is unavailable on
 * the GPU pool): with RESPCA_GUARD=1 in the environment every device
 * allocation is poisoned with 0xFF bytes and followed by a 4 KiB guard;
 * returns the number of guards found overwritten (guard mode never frees
 * device memory, so every buffer ever allocated is checked), -1 when
 * RESPCA_GUARD is off; `msg` (may be NULL) describes the first ones. */
int respca_cu_debug_guards(char* msg, uint64_t cap);

/* Decision margins of the context's last solve (respca_cu_margins). */
int respca_cu_last_margins(const respca_cu_ctx* ctx, respca_cu_margins* out);

/* --- benchmark hooks (device-resident state, no host copies) ------------- */
/* Upload X and run validation + the one-time initial clustering; leaves the
 * context ready to step the ALM loop.  init_ms receives the device time. */
int respca_cu_bench_prepare(respca_cu_ctx* ctx, const void* x, uint64_t d, uint64_t n,
                            int dtype, const respca_cu_config* cfg, double* init_ms);
/* Run exactly `iters` ALM iterations (fixed-iteration semantics) on the
 * resident state; *ms receives the CUDA-event time of the whole region and
 * *pass_f_ms the summed time of the fused elementwise kernel.  Returns the
 * number of slow-path iterations through *slow. */
int respca_cu_bench_steps(respca_cu_ctx* ctx, uint64_t iters, double* ms, double* pass_f_ms,
                          double* pass_a_ms, uint64_t* slow);

/* ---- file I/O straight to / from HBM, outlier scores ------- */

/* RESPCA1 binary header (io.hpp:66-69: magic "RESPCA1\0", u64le rows, u64le
 * cols, then rows*cols f64le column-major).  Host only (no GPU needed);
 * RESPCA_EIO with the reference's message on a missing file, bad magic, short
 * header or a payload shorter than rows*cols doubles (io.cpp:138-153). */
int respca_cu_binary_info(const char* path, uint64_t* rows, uint64_t* cols, char* err,
                          size_t err_len);

/* solve() on a RESPCA1 file: the payload streams from disk into HBM through
 * two pinned chunks (the read of chunk k+1 overlaps the copy of chunk k; fp32
 * mode converts on the device), and L / S stream back out as RESPCA1 files
 * (device→host copy of chunk k+1 overlaps the write of chunk k).  l_path /
 * s_path may be NULL (not written).  d, n are taken from the file. */
int respca_cu_solve_file(respca_cu_ctx* ctx, const char* x_path, int dtype,
                         const respca_cu_config* cfg, const char* l_path, const char* s_path,
                         uint64_t* labels_out, uint64_t labels_cap, respca_cu_report* rep);

/* io::outlier_scores (io.cpp:296-306): scores[j] = ‖S_j‖₂ (column_l2_norms
 * order, matrix.cpp:117-125), flagged = ascending j with scores[j] >= threshold
 * (*n_flagged entries of `flagged`, capacity n).  threshold < 0 → EINVAL. */
int respca_cu_outlier_scores(respca_cu_ctx* ctx, const double* s, uint64_t d, uint64_t n,
                             double threshold, double* scores, uint64_t* flagged,
                             uint64_t* n_flagged);

/* The "respca-synth-1" rpca workload generator (paper_1904_07497_b200/csrc/
 * synth.c) with its O(d·n) assembly on the device: X = U·Vᵀ + S0, U (d×r),
 * V (n×r) i.i.d. N(0, sigma²), S0 Bernoulli(p) support with U[lo, hi] values.
 * Byte-identical to the host generator; X_out (host, d×n column-major, F64 or
 * F32 per dtype) receives the result. */
int respca_cu_synth_rpca(respca_cu_ctx* ctx, uint64_t d, uint64_t n, uint64_t r, double sigma, double p,
                         double lo, double hi, uint64_t seed, int dtype, void* X_out);

/* io::synth_generate (proj/src/io.cpp:232-294, declared at proj/include/respca/
 * io.hpp:88) with its O(d·n) assembly on the device: near-equal contiguous
 * groups of identical uniform(0,1) prototype columns (L0), round(sparsity·d·n)
 * corruptions at partial-Fisher–Yates positions with a random sign and a
 * magnitude in [magnitude/2, magnitude) (S0), X = L0 + S0 (+ N(0, noise_sigma²)
 * per element when noise_sigma > 0).  The libstdc++ draws run on the host in
 * the reference's order, so every output is byte-identical to the reference's.
 * X_out / L0_out / S0_out (host, d×n column-major fp64) and labels_out (n) may
 * each be NULL.  Invalid specs → EINVAL with the reference's message. */
int respca_cu_synth_generate(respca_cu_ctx* ctx, uint64_t d, uint64_t n, uint64_t c, double sparsity,
                             double magnitude, double noise_sigma, uint64_t seed, double* X_out,
                             double* L0_out, double* S0_out, uint64_t* labels_out);

#ifdef __cplusplus
}
#endif

#endif
