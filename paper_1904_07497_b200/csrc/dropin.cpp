// librespca_b200.so — the reference's C++ API (include/respca_b200/respca.hpp)
// implemented over the C-ABI of respca_cu.h.  Host-side type validation
// (DenseMatrix / GroupAssignment constructors, SolverConfig::validate) follows
// the reference (matrix.cpp:8-61, solver.cpp:35-49); every numerical
// operation runs on the GPU.  Status codes become the reference's exception
// classes: RESPCA_EINVAL → std::invalid_argument, RESPCA_ERUNTIME →
// std::runtime_error, anything else → std::runtime_error with the CUDA text.
#include "respca_b200/respca.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <memory>
#include <stdexcept>
#include <string>

#include "respca_cu.h"

namespace respca {

namespace {

struct CtxDeleter {
    void operator()(respca_cu_ctx* c) const { respca_cu_destroy(c); }
};

// one context per (host thread, device): contexts are not thread-safe
respca_cu_ctx* ctx_for(int device) {
    thread_local std::unique_ptr<respca_cu_ctx, CtxDeleter> slots[16];
    if (device < 0 || device >= 16) throw std::invalid_argument("respca: bad device id");
    auto& s = slots[device];
    if (!s) {
        respca_cu_ctx* c = nullptr;
        if (respca_cu_create(device, &c) != RESPCA_OK)
            throw std::runtime_error("respca: no usable sm_100 CUDA device (there is no CPU fallback)");
        s.reset(c);
    }
    return s.get();
}

void ck(respca_cu_ctx* c, int rc) {
    if (rc == RESPCA_OK) return;
    const std::string msg = respca_cu_last_error(c);
    if (rc == RESPCA_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

respca_cu_ctx* C0() { return ctx_for(0); }

std::vector<std::uint64_t> u64(const GroupAssignment& g) {
    return std::vector<std::uint64_t>(g.labels().begin(), g.labels().end());
}

GroupAssignment from_u64(const std::vector<std::uint64_t>& l, std::size_t c) {
    return GroupAssignment(std::vector<std::size_t>(l.begin(), l.end()), c);
}

respca_cu_config to_c(const SolverConfig& s) {
    respca_cu_config c;
    respca_cu_default_config(&c);
    c.has_lambda = s.lambda.has_value();
    c.lambda = s.lambda.value_or(0.0);
    c.rho0 = s.rho0;
    c.kappa = s.kappa;
    c.tol = s.tol;
    c.max_iter = s.max_iter;
    c.c = s.c;
    c.sparse_norm = s.sparse_norm == SparseNorm::L21 ? RESPCA_L21 : RESPCA_L1;
    c.km_max_iters = s.kmeans.max_iters;
    c.km_n_restarts = s.kmeans.n_restarts;
    c.km_seed = s.kmeans.seed;
    c.km_tol = s.kmeans.tol;
    c.has_fixed_iters = s.fixed_iters.has_value();
    c.fixed_iters = s.fixed_iters.value_or(0);
    return c;
}

}  // namespace

// ---- core -------------------------------------------------------------------
DenseMatrix::DenseMatrix(std::size_t rows, std::size_t cols)
    : rows_(rows), cols_(cols), data_(rows * cols, 0.0) {
    if (rows == 0 || cols == 0) throw std::invalid_argument("DenseMatrix: dimensions must be >= 1");
}

DenseMatrix::DenseMatrix(std::size_t rows, std::size_t cols, std::vector<double> data)
    : rows_(rows), cols_(cols), data_(std::move(data)) {
    if (rows == 0 || cols == 0) throw std::invalid_argument("DenseMatrix: dimensions must be >= 1");
    if (data_.size() != rows * cols)
        throw std::invalid_argument("DenseMatrix: data size does not match dimensions");
    if (!all_finite()) throw std::invalid_argument("DenseMatrix: non-finite value in input");
}

bool DenseMatrix::all_finite() const {
    return std::all_of(data_.begin(), data_.end(), [](double v) { return std::isfinite(v); });
}

GroupAssignment::GroupAssignment(std::vector<std::size_t> labels, std::size_t c)
    : labels_(std::move(labels)), c_(c) {
    if (c == 0) throw std::invalid_argument("GroupAssignment: c must be >= 1");
    std::vector<char> seen(c, 0);
    for (std::size_t l : labels_) {
        if (l >= c) throw std::invalid_argument("GroupAssignment: label out of range");
        seen[l] = 1;
    }
    if (std::find(seen.begin(), seen.end(), 0) != seen.end())
        throw std::invalid_argument("GroupAssignment: empty group");
}

std::vector<std::vector<std::size_t>> GroupAssignment::group_indices() const {
    std::vector<std::vector<std::size_t>> out(c_);
    for (std::size_t j = 0; j < labels_.size(); ++j) out[labels_[j]].push_back(j);
    return out;
}

std::vector<std::size_t> GroupAssignment::group_sizes() const {
    std::vector<std::size_t> out(c_, 0);
    for (std::size_t l : labels_) ++out[l];
    return out;
}

std::vector<double> column_mean(const DenseMatrix& m, std::span<const std::size_t> columns) {
    std::vector<std::uint64_t> cols(columns.begin(), columns.end());
    std::vector<double> out(m.rows());
    auto* c = C0();
    ck(c, respca_cu_column_mean(c, m.data().data(), m.rows(), m.cols(), cols.data(), cols.size(),
                                out.data()));
    return out;
}

double group_scatter(const DenseMatrix& m, const GroupAssignment& g) {
    if (g.size() != m.cols())
        throw std::invalid_argument("group_scatter: assignment length != column count");
    auto l = u64(g);
    double out = 0.0;
    auto* c = C0();
    ck(c, respca_cu_group_scatter(c, m.data().data(), m.rows(), m.cols(), l.data(), g.groups(),
                                  &out));
    return out;
}

#define RESPCA_SCALAR(fn, cfn)                                               \
    double fn(const DenseMatrix& m) {                                        \
        double out = 0.0;                                                    \
        auto* c = C0();                                                      \
        ck(c, cfn(c, m.data().data(), m.rows(), m.cols(), &out));            \
        return out;                                                          \
    }
RESPCA_SCALAR(frob_norm, respca_cu_frob_norm)
RESPCA_SCALAR(elementwise_l1, respca_cu_elementwise_l1)
RESPCA_SCALAR(l21_norm, respca_cu_l21_norm)
#undef RESPCA_SCALAR

std::vector<double> column_l2_norms(const DenseMatrix& m) {
    std::vector<double> out(m.cols());
    auto* c = C0();
    ck(c, respca_cu_column_l2_norms(c, m.data().data(), m.rows(), m.cols(), out.data()));
    return out;
}

// ---- clustering ---------------------------------------------------------------
namespace {
std::uint64_t draw_first(void* u, std::uint64_t n) {
    std::uniform_int_distribution<std::size_t> d(0, n - 1);
    return d(*static_cast<std::mt19937_64*>(u));
}
double draw_real(void* u, double total) {
    std::uniform_real_distribution<double> d(0.0, total);
    return d(*static_cast<std::mt19937_64*>(u));
}
}  // namespace

DenseMatrix kmeans_pp_init(const DenseMatrix& m, std::size_t c, std::mt19937_64& rng) {
    if (c == 0) throw std::invalid_argument("kmeans_pp_init: c must be >= 1");
    if (c > m.cols()) throw std::invalid_argument("kmeans_pp_init: c exceeds column count");
    DenseMatrix out(m.rows(), c);
    auto* cx = C0();
    ck(cx, respca_cu_kmeans_pp_init_cb(cx, m.data().data(), m.rows(), m.cols(), c, draw_first,
                                       draw_real, &rng, out.data().data()));
    return out;
}

std::pair<GroupAssignment, DenseMatrix> lloyd_step(const DenseMatrix& m,
                                                   const DenseMatrix& centroids) {
    if (centroids.cols() == 0 || centroids.rows() != m.rows())
        throw std::invalid_argument("lloyd_step: bad centroid matrix");
    std::vector<std::uint64_t> lab(m.cols());
    DenseMatrix next(m.rows(), centroids.cols());
    auto* c = C0();
    ck(c, respca_cu_lloyd_step(c, m.data().data(), m.rows(), m.cols(), centroids.data().data(),
                               centroids.cols(), lab.data(), next.data().data()));
    return {from_u64(lab, centroids.cols()), std::move(next)};
}

KMeansResult kmeans(const DenseMatrix& m, const KMeansConfig& cfg) {
    if (cfg.c == 0) throw std::invalid_argument("kmeans: c must be >= 1");
    if (cfg.c > m.cols()) throw std::invalid_argument("kmeans: c exceeds column count");
    std::vector<std::uint64_t> lab(m.cols());
    KMeansResult r;
    r.centroids = DenseMatrix(m.rows(), cfg.c);
    std::uint64_t it = 0;
    auto* c = C0();
    ck(c, respca_cu_kmeans(c, m.data().data(), m.rows(), m.cols(), cfg.c, cfg.max_iters,
                           cfg.n_restarts, cfg.seed, cfg.tol, lab.data(),
                           r.centroids.data().data(), &r.inertia, &it));
    r.assignment = from_u64(lab, cfg.c);
    r.iters_run = it;
    return r;
}

KMeansResult kmeans_warm(const DenseMatrix& m, const KMeansConfig& cfg,
                         const GroupAssignment& init) {
    if (init.size() != m.cols() || init.groups() != cfg.c)
        throw std::invalid_argument("kmeans_warm: assignment does not match");
    auto il = u64(init);
    std::vector<std::uint64_t> lab(m.cols());
    KMeansResult r;
    r.centroids = DenseMatrix(m.rows(), cfg.c);
    std::uint64_t it = 0;
    auto* c = C0();
    ck(c, respca_cu_kmeans_warm(c, m.data().data(), m.rows(), m.cols(), cfg.c, cfg.max_iters,
                                cfg.tol, il.data(), lab.data(), r.centroids.data().data(),
                                &r.inertia, &it));
    r.assignment = from_u64(lab, cfg.c);
    r.iters_run = it;
    return r;
}

// ---- solver ---------------------------------------------------------------------
double SolverConfig::resolve_lambda(std::size_t rows, std::size_t cols) const {
    if (lambda) return *lambda;
    return std::sqrt(static_cast<double>(std::max(rows, cols)));
}

void SolverConfig::validate() const {
    if (lambda && *lambda <= 0.0) throw std::invalid_argument("lambda must be > 0");
    if (rho0 <= 0.0) throw std::invalid_argument("rho0 must be > 0");
    if (kappa <= 1.0) throw std::invalid_argument("kappa must be > 1");
    if (tol <= 0.0) throw std::invalid_argument("tol must be > 0");
    if (c == 0) throw std::invalid_argument("c must be >= 1");
    if (max_iter == 0) throw std::invalid_argument("max_iter must be >= 1");
}

double Residuals::max() const { return std::max({feas, delta_l, delta_s}); }

DenseMatrix l_update(const DenseMatrix& d, const GroupAssignment& g, double lambda, double rho) {
    if (rho <= 0.0) throw std::invalid_argument("l_update: rho must be > 0");
    if (lambda < 0.0) throw std::invalid_argument("l_update: lambda must be >= 0");
    if (g.size() != d.cols()) throw std::invalid_argument("l_update: assignment length != column count");
    auto l = u64(g);
    DenseMatrix out(d.rows(), d.cols());
    auto* c = C0();
    ck(c, respca_cu_l_update(c, d.data().data(), d.rows(), d.cols(), l.data(), g.groups(), lambda,
                             rho, out.data().data()));
    return out;
}

DenseMatrix s_update_l1(const DenseMatrix& b, double threshold) {
    if (threshold < 0.0) throw std::invalid_argument("s_update_l1: negative threshold");
    DenseMatrix out(b.rows(), b.cols());
    auto* c = C0();
    ck(c, respca_cu_s_update_l1(c, b.data().data(), b.rows(), b.cols(), threshold,
                                out.data().data()));
    return out;
}

DenseMatrix s_update_l21(const DenseMatrix& b, double threshold) {
    if (threshold < 0.0) throw std::invalid_argument("s_update_l21: negative threshold");
    DenseMatrix out(b.rows(), b.cols());
    auto* c = C0();
    ck(c, respca_cu_s_update_l21(c, b.data().data(), b.rows(), b.cols(), threshold,
                                 out.data().data()));
    return out;
}

void multiplier_update(SolverState& st, const DenseMatrix& x, double kappa) {
    if (kappa <= 1.0) throw std::invalid_argument("multiplier_update: kappa must be > 1");
    auto* c = C0();
    ck(c, respca_cu_multiplier_update(c, st.Theta.data().data(), x.data().data(),
                                      st.L.data().data(), st.S.data().data(), x.rows(), x.cols(),
                                      &st.rho, kappa));
}

std::pair<bool, Residuals> check_convergence(const DenseMatrix& x, const DenseMatrix& l_prev,
                                             const DenseMatrix& l, const DenseMatrix& s_prev,
                                             const DenseMatrix& s, double tol) {
    Residuals r;
    int conv = 0;
    auto* c = C0();
    ck(c, respca_cu_check_convergence(c, x.data().data(), l_prev.data().data(), l.data().data(),
                                      s_prev.data().data(), s.data().data(), x.rows(), x.cols(),
                                      tol, &conv, &r.feas, &r.delta_l, &r.delta_s));
    return {conv != 0, r};
}

DecompositionResult b200::solve(const DenseMatrix& x, const SolverConfig& cfg,
                                const b200::Options& opt, b200::Timings* tm) {
    cfg.validate();  // solver.cpp:128-132 (finite / non-zero are checked on the device)
    if (cfg.c > x.cols()) throw std::invalid_argument("solve: c exceeds column count");
    const auto t0 = std::chrono::steady_clock::now();
    // allocation only (>= 1 entry); the solver writes rep.iters entries, 0 for fixed_iters = 0
    const std::size_t budget = std::max<std::size_t>(cfg.fixed_iters.value_or(cfg.max_iter), 1);
    DecompositionResult out;
    out.L = DenseMatrix(x.rows(), x.cols());
    out.S = DenseMatrix(x.rows(), x.cols());
    std::vector<std::uint64_t> lab(x.cols());
    std::vector<double> f(budget), dl(budget), ds(budget), ob(budget);
    respca_cu_report rep{};
    rep.feas = f.data();
    rep.delta_l = dl.data();
    rep.delta_s = ds.data();
    rep.objective = ob.data();
    const respca_cu_config cc = to_c(cfg);
    auto* c = ctx_for(opt.device);
    if (opt.precision == Precision::F32) {
        std::vector<float> xf(x.data().begin(), x.data().end()), Lf(x.size()), Sf(x.size());
        ck(c, respca_cu_solve(c, xf.data(), x.rows(), x.cols(), RESPCA_F32, &cc, Lf.data(),
                              Sf.data(), lab.data(), &rep));
        std::copy(Lf.begin(), Lf.end(), out.L.data().begin());
        std::copy(Sf.begin(), Sf.end(), out.S.data().begin());
    } else {
        ck(c, respca_cu_solve(c, x.data().data(), x.rows(), x.cols(), RESPCA_F64, &cc,
                              out.L.data().data(), out.S.data().data(), lab.data(), &rep));
    }
    out.assignment = from_u64(lab, cfg.c);
    f.resize(rep.iters);
    dl.resize(rep.iters);
    ds.resize(rep.iters);
    ob.resize(rep.iters);
    out.report.feas = std::move(f);
    out.report.delta_l = std::move(dl);
    out.report.delta_s = std::move(ds);
    out.report.objective = std::move(ob);
    out.report.converged = rep.converged != 0;
    out.report.iters = rep.iters;
    out.lambda = rep.lambda;
    out.wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (tm) {
        tm->init_ms = rep.init_ms;
        tm->loop_ms = rep.loop_ms;
        tm->h2d_ms = rep.h2d_ms;
        tm->d2h_ms = rep.d2h_ms;
        tm->hartigan_moves = rep.hartigan_moves;
        tm->slow_iters = rep.slow_iters;
        tm->exact_fallbacks = rep.exact_fallbacks;
    }
    return out;
}

DecompositionResult solve(const DenseMatrix& x, const SolverConfig& cfg) {
    return b200::solve(x, cfg, b200::Options{});
}

}  // namespace respca
