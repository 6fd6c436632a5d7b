/* TEST INFRASTRUCTURE — not product code.
 *
 * Plain-C ABI shared by the two CPU checkers under oracle/:
 *   - orc_*  : respca_oracle.c, a C restatement of the reference algorithm
 *              (each function cites the reference file:line it follows);
 *   - ref_*  : oracle/_ref/librespca_ref.so, the UNMODIFIED reference sources
 *              (/root/reference/proj/src/{matrix,kmeans,solver}.cpp) compiled
 *              by oracle/Makefile together with ref_shim.cpp.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load these libraries.
 *
 * Status codes mirror the reference's exception classes:
 *   0 = ok, 1 = std::invalid_argument, 2 = std::runtime_error, 3 = other.
 */
#ifndef RESPCA_ORACLE_ABI_H
#define RESPCA_ORACLE_ABI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Field-for-field image of SolverConfig + KMeansConfig
 * (reference proj/include/respca/solver.hpp:13-28, kmeans.hpp:11-17). */
typedef struct {
    int has_lambda;          /* 0 → λ = sqrt(max(d, n)) (solver.cpp:35-38) */
    double lambda;
    double rho0;             /* default 1e-4 */
    double kappa;            /* default 1.5 */
    double tol;              /* default 1e-3 */
    uint64_t max_iter;       /* default 500 */
    uint64_t c;              /* default 1 */
    int sparse_norm;         /* 0 = L1, 1 = L21 */
    uint64_t km_max_iters;   /* default 100 */
    uint64_t km_n_restarts;  /* default 1 (solve forces >= 5) */
    uint64_t km_seed;        /* default 0 */
    double km_tol;           /* default 1e-6 */
    int has_fixed_iters;
    uint64_t fixed_iters;
} orc_config;

#define ORC_DECLARE(P)                                                          \
    const char* P##_last_error(void);                                           \
    int P##_solve(const double* x, uint64_t d, uint64_t n,                      \
                  const orc_config* cfg, double* L, double* S,                  \
                  uint64_t* labels, double* feas, double* dl, double* ds,       \
                  double* obj, uint64_t* iters, int* converged,                 \
                  double* lambda_out, double* wall);                            \
    int P##_kmeans(const double* m, uint64_t d, uint64_t n, uint64_t c,         \
                   uint64_t max_iters, uint64_t n_restarts, uint64_t seed,      \
                   double tol, uint64_t* labels, double* centroids,             \
                   double* inertia, uint64_t* iters_run);                       \
    int P##_kmeans_warm(const double* m, uint64_t d, uint64_t n, uint64_t c,    \
                        uint64_t max_iters, double tol,                         \
                        const uint64_t* init_labels, uint64_t* labels,          \
                        double* centroids, double* inertia,                     \
                        uint64_t* iters_run);                                   \
    int P##_kmeans_pp_init(const double* m, uint64_t d, uint64_t n,             \
                           uint64_t c, uint64_t seed, double* centroids);       \
    int P##_lloyd_step(const double* m, uint64_t d, uint64_t n,                 \
                       const double* centroids, uint64_t c, uint64_t* labels,   \
                       double* next);                                           \
    int P##_l_update(const double* D, uint64_t d, uint64_t n,                   \
                     const uint64_t* labels, uint64_t c, double lambda,         \
                     double rho, double* L);                                    \
    int P##_s_update_l1(const double* B, uint64_t d, uint64_t n, double thr,    \
                        double* S);                                             \
    int P##_s_update_l21(const double* B, uint64_t d, uint64_t n, double thr,   \
                         double* S);                                            \
    int P##_multiplier_update(double* theta, const double* x, const double* L,  \
                              const double* S, uint64_t d, uint64_t n,          \
                              double* rho, double kappa);                       \
    int P##_check_convergence(const double* x, const double* l_prev,            \
                              const double* l, const double* s_prev,            \
                              const double* s, uint64_t d, uint64_t n,          \
                              double tol, int* conv, double* feas, double* dl,  \
                              double* ds);                                      \
    int P##_group_scatter(const double* m, uint64_t d, uint64_t n,              \
                          const uint64_t* labels, uint64_t c, double* out);     \
    int P##_frob_norm(const double* m, uint64_t d, uint64_t n, double* out);    \
    int P##_elementwise_l1(const double* m, uint64_t d, uint64_t n,             \
                           double* out);                                        \
    int P##_l21_norm(const double* m, uint64_t d, uint64_t n, double* out);     \
    int P##_column_l2_norms(const double* m, uint64_t d, uint64_t n,            \
                            double* out);                                       \
    int P##_column_mean(const double* m, uint64_t d, uint64_t n,                \
                        const uint64_t* cols, uint64_t ncols, double* out);     \
    int P##_uniform_int(uint64_t seed, uint64_t lo, uint64_t hi,                \
                        uint64_t count, uint64_t* out);                         \
    int P##_uniform_real(uint64_t seed, double a, double b, uint64_t count,     \
                         double* out);

ORC_DECLARE(orc)
ORC_DECLARE(ref)

/* Reference-only: replay of the ALM loop (solver.cpp:157-201) through the
 * reference's public building blocks, starting from a given assignment
 * instead of the one-time kmeans(X) (solver.cpp:148).  Used by the bench's
 * reference arm to time bounded samples of the loop.  iter_seconds[t] is the
 * wall time of iteration t. */
int ref_replay(const double* x, uint64_t d, uint64_t n, const orc_config* cfg,
               const uint64_t* init_labels, uint64_t n_iters, double* L,
               double* S, uint64_t* labels, double* feas, double* dl,
               double* ds, double* obj, double* iter_seconds);

#ifdef __cplusplus
}
#endif

#endif
