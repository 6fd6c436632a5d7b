// TEST INFRASTRUCTURE — not product code.
//
// extern "C" shim over the UNMODIFIED reference library.  oracle/Makefile
// compiles this file together with /root/reference/proj/src/{matrix,kmeans,
// solver}.cpp (reference flags: -std=gnu++20 -O3 -DNDEBUG, no -march) into
// oracle/_ref/librespca_ref.so.  Nothing here re-implements the algorithm: every
// entry point marshals plain buffers into the reference's own types and calls
// the reference's public API (proj/include/respca/{solver,kmeans,matrix}.hpp).

#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "respca/kmeans.hpp"
#include "respca/matrix.hpp"
#include "respca/solver.hpp"

#include "oracle_abi.h"

using namespace respca;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        g_err.clear();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

DenseMatrix wrap(const double* p, uint64_t d, uint64_t n) {
    return DenseMatrix(d, n, std::vector<double>(p, p + d * n));
}

void unwrap(const DenseMatrix& m, double* out) {
    std::memcpy(out, m.data().data(), m.size() * sizeof(double));
}

GroupAssignment wrap_labels(const uint64_t* l, uint64_t n, uint64_t c) {
    return GroupAssignment(std::vector<std::size_t>(l, l + n), c);
}

void unwrap_labels(const GroupAssignment& g, uint64_t* out) {
    for (std::size_t j = 0; j < g.size(); ++j) out[j] = g.label(j);
}

SolverConfig to_cfg(const orc_config* c) {
    SolverConfig s;
    if (c->has_lambda) s.lambda = c->lambda;
    s.rho0 = c->rho0;
    s.kappa = c->kappa;
    s.tol = c->tol;
    s.max_iter = c->max_iter;
    s.c = c->c;
    s.sparse_norm = c->sparse_norm ? SparseNorm::L21 : SparseNorm::L1;
    s.kmeans.max_iters = c->km_max_iters;
    s.kmeans.n_restarts = c->km_n_restarts;
    s.kmeans.seed = c->km_seed;
    s.kmeans.tol = c->km_tol;
    if (c->has_fixed_iters) s.fixed_iters = c->fixed_iters;
    return s;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_solve(const double* x, uint64_t d, uint64_t n, const orc_config* cfg,
              double* L, double* S, uint64_t* labels, double* feas, double* dl,
              double* ds, double* obj, uint64_t* iters, int* converged,
              double* lambda_out, double* wall) {
    return guarded([&] {
        // zero-filled ctor + copy: leaves the finite check to solve() itself
        // (solver.cpp:130), as a caller holding a mutated matrix would see it
        DenseMatrix xm(d, n);
        std::memcpy(xm.data().data(), x, d * n * sizeof(double));
        const DecompositionResult r = solve(xm, to_cfg(cfg));
        unwrap(r.L, L);
        unwrap(r.S, S);
        unwrap_labels(r.assignment, labels);
        for (std::size_t t = 0; t < r.report.iters; ++t) {
            feas[t] = r.report.feas[t];
            dl[t] = r.report.delta_l[t];
            ds[t] = r.report.delta_s[t];
            obj[t] = r.report.objective[t];
        }
        *iters = r.report.iters;
        *converged = r.report.converged ? 1 : 0;
        *lambda_out = r.lambda;
        *wall = r.wall_time;
    });
}

int ref_kmeans(const double* m, uint64_t d, uint64_t n, uint64_t c,
               uint64_t max_iters, uint64_t n_restarts, uint64_t seed,
               double tol, uint64_t* labels, double* centroids, double* inertia,
               uint64_t* iters_run) {
    return guarded([&] {
        KMeansConfig k;
        k.c = c;
        k.max_iters = max_iters;
        k.n_restarts = n_restarts;
        k.seed = seed;
        k.tol = tol;
        const KMeansResult r = kmeans(wrap(m, d, n), k);
        unwrap_labels(r.assignment, labels);
        unwrap(r.centroids, centroids);
        *inertia = r.inertia;
        *iters_run = r.iters_run;
    });
}

int ref_kmeans_warm(const double* m, uint64_t d, uint64_t n, uint64_t c,
                    uint64_t max_iters, double tol, const uint64_t* init_labels,
                    uint64_t* labels, double* centroids, double* inertia,
                    uint64_t* iters_run) {
    return guarded([&] {
        KMeansConfig k;
        k.c = c;
        k.max_iters = max_iters;
        k.tol = tol;
        const KMeansResult r =
            kmeans_warm(wrap(m, d, n), k, wrap_labels(init_labels, n, c));
        unwrap_labels(r.assignment, labels);
        unwrap(r.centroids, centroids);
        *inertia = r.inertia;
        *iters_run = r.iters_run;
    });
}

int ref_kmeans_pp_init(const double* m, uint64_t d, uint64_t n, uint64_t c,
                       uint64_t seed, double* centroids) {
    return guarded([&] {
        std::mt19937_64 rng(seed);
        unwrap(kmeans_pp_init(wrap(m, d, n), c, rng), centroids);
    });
}

int ref_lloyd_step(const double* m, uint64_t d, uint64_t n,
                   const double* centroids, uint64_t c, uint64_t* labels,
                   double* next) {
    return guarded([&] {
        auto [g, nx] = lloyd_step(wrap(m, d, n), wrap(centroids, d, c));
        unwrap_labels(g, labels);
        unwrap(nx, next);
    });
}

int ref_l_update(const double* D, uint64_t d, uint64_t n, const uint64_t* labels,
                 uint64_t c, double lambda, double rho, double* L) {
    return guarded([&] {
        unwrap(l_update(wrap(D, d, n), wrap_labels(labels, n, c), lambda, rho), L);
    });
}

int ref_s_update_l1(const double* B, uint64_t d, uint64_t n, double thr,
                    double* S) {
    return guarded([&] { unwrap(s_update_l1(wrap(B, d, n), thr), S); });
}

int ref_s_update_l21(const double* B, uint64_t d, uint64_t n, double thr,
                     double* S) {
    return guarded([&] { unwrap(s_update_l21(wrap(B, d, n), thr), S); });
}

int ref_multiplier_update(double* theta, const double* x, const double* L,
                          const double* S, uint64_t d, uint64_t n, double* rho,
                          double kappa) {
    return guarded([&] {
        SolverState st;
        st.L = wrap(L, d, n);
        st.S = wrap(S, d, n);
        st.Theta = wrap(theta, d, n);
        st.rho = *rho;
        multiplier_update(st, wrap(x, d, n), kappa);
        unwrap(st.Theta, theta);
        *rho = st.rho;
    });
}

int ref_check_convergence(const double* x, const double* l_prev, const double* l,
                          const double* s_prev, const double* s, uint64_t d,
                          uint64_t n, double tol, int* conv, double* feas,
                          double* dl, double* ds) {
    return guarded([&] {
        auto [ok, r] = check_convergence(wrap(x, d, n), wrap(l_prev, d, n),
                                         wrap(l, d, n), wrap(s_prev, d, n),
                                         wrap(s, d, n), tol);
        *conv = ok ? 1 : 0;
        *feas = r.feas;
        *dl = r.delta_l;
        *ds = r.delta_s;
    });
}

int ref_group_scatter(const double* m, uint64_t d, uint64_t n,
                      const uint64_t* labels, uint64_t c, double* out) {
    return guarded([&] {
        *out = group_scatter(wrap(m, d, n), wrap_labels(labels, n, c));
    });
}

int ref_frob_norm(const double* m, uint64_t d, uint64_t n, double* out) {
    return guarded([&] { *out = frob_norm(wrap(m, d, n)); });
}

int ref_elementwise_l1(const double* m, uint64_t d, uint64_t n, double* out) {
    return guarded([&] { *out = elementwise_l1(wrap(m, d, n)); });
}

int ref_l21_norm(const double* m, uint64_t d, uint64_t n, double* out) {
    return guarded([&] { *out = l21_norm(wrap(m, d, n)); });
}

int ref_column_l2_norms(const double* m, uint64_t d, uint64_t n, double* out) {
    return guarded([&] {
        const auto v = column_l2_norms(wrap(m, d, n));
        std::memcpy(out, v.data(), v.size() * sizeof(double));
    });
}

int ref_column_mean(const double* m, uint64_t d, uint64_t n, const uint64_t* cols,
                    uint64_t ncols, double* out) {
    return guarded([&] {
        std::vector<std::size_t> idx(cols, cols + ncols);
        const auto v = column_mean(wrap(m, d, n), idx);
        std::memcpy(out, v.data(), v.size() * sizeof(double));
    });
}

int ref_uniform_int(uint64_t seed, uint64_t lo, uint64_t hi, uint64_t count,
                    uint64_t* out) {
    return guarded([&] {
        std::mt19937_64 rng(seed);
        std::uniform_int_distribution<std::size_t> u(lo, hi);
        for (uint64_t k = 0; k < count; ++k) out[k] = u(rng);
    });
}

int ref_uniform_real(uint64_t seed, double a, double b, uint64_t count,
                     double* out) {
    return guarded([&] {
        std::mt19937_64 rng(seed);
        for (uint64_t k = 0; k < count; ++k) {
            std::uniform_real_distribution<double> u(a, b);
            out[k] = u(rng);
        }
    });
}

// Loop replay through the reference's public building blocks, statement for
// statement as solve() runs it (solver.cpp:152-201), minus the initial
// kmeans(X) at solver.cpp:148, which is replaced by `init_labels`.
int ref_replay(const double* x, uint64_t d, uint64_t n, const orc_config* cfg,
               const uint64_t* init_labels, uint64_t n_iters, double* L,
               double* S, uint64_t* labels, double* feas, double* dl,
               double* ds, double* obj, double* iter_seconds) {
    return guarded([&] {
        const SolverConfig sc = to_cfg(cfg);
        sc.validate();
        const DenseMatrix xm = wrap(x, d, n);
        const double x_norm = frob_norm(xm);
        const double lambda = sc.resolve_lambda(d, n);
        SolverState st;
        st.L = xm;
        st.S = DenseMatrix(d, n);
        st.Theta = DenseMatrix(d, n);
        st.rho = sc.rho0;
        st.assignment = wrap_labels(init_labels, n, sc.c);
        KMeansConfig km = sc.kmeans;
        km.c = sc.c;
        km.n_restarts = 1;
        DenseMatrix dm(d, n);
        for (uint64_t t = 0; t < n_iters; ++t) {
            const auto t0 = std::chrono::steady_clock::now();
            const DenseMatrix l_prev = st.L;
            const DenseMatrix s_prev = st.S;
            for (std::size_t k = 0; k < xm.size(); ++k)
                dm.data()[k] = xm.data()[k] - st.S.data()[k] + st.Theta.data()[k] / st.rho;
            st.L = l_update(dm, st.assignment, lambda, st.rho);
            st.assignment = kmeans_warm(st.L, km, st.assignment).assignment;
            for (std::size_t k = 0; k < xm.size(); ++k)
                dm.data()[k] = xm.data()[k] - st.L.data()[k] + st.Theta.data()[k] / st.rho;
            const double thr = 1.0 / st.rho;
            st.S = sc.sparse_norm == SparseNorm::L1 ? s_update_l1(dm, thr)
                                                     : s_update_l21(dm, thr);
            multiplier_update(st, xm, sc.kappa);
            // residual triple exactly as solve() inlines it (solver.cpp:183-186
            // via the file-local helpers at solver.cpp:14-31)
            double sq_f = 0.0, sq_l = 0.0, sq_s = 0.0;
            for (std::size_t k = 0; k < xm.size(); ++k) {
                const double a = xm.data()[k] - st.L.data()[k] - st.S.data()[k];
                sq_f += a * a;
            }
            for (std::size_t k = 0; k < xm.size(); ++k) {
                const double a = st.L.data()[k] - l_prev.data()[k];
                sq_l += a * a;
            }
            for (std::size_t k = 0; k < xm.size(); ++k) {
                const double a = st.S.data()[k] - s_prev.data()[k];
                sq_s += a * a;
            }
            feas[t] = std::sqrt(sq_f) / x_norm;
            dl[t] = std::sqrt(sq_l) / x_norm;
            ds[t] = std::sqrt(sq_s) / x_norm;
            const double sparse = sc.sparse_norm == SparseNorm::L1
                                      ? elementwise_l1(st.S)
                                      : l21_norm(st.S);
            obj[t] = lambda * group_scatter(st.L, st.assignment) + sparse;
            iter_seconds[t] = std::chrono::duration<double>(
                std::chrono::steady_clock::now() - t0).count();
        }
        unwrap(st.L, L);
        unwrap(st.S, S);
        unwrap_labels(st.assignment, labels);
    });
}

}  // extern "C"
