// respca_b200/respca.hpp — C++ drop-in facade of the B200-native RES-PCA
// solver.  It re-declares the reference's public C++ API
// (/root/reference/proj/include/respca/{matrix,kmeans,solver}.hpp) with the
// same names, types, class layouts and error behaviour, so code written
// against the reference recompiles (and, with identical layouts, relinks)
// against librespca_b200.so.  Every computation is forwarded through the C-ABI
// of respca_cu.h to the sm_100a engine — there is no CPU path.
//
// Extension: solve(x, cfg, b200::Options{...}) selects fp32 storage and the
// device.
#pragma once

#include <cstddef>
#include <cstdint>
#include <optional>
#include <random>
#include <span>
#include <utility>
#include <vector>

namespace respca {

// ---- core (matrix.hpp:11-98) ---------------------------------------------
class DenseMatrix {
public:
    DenseMatrix() = default;
    DenseMatrix(std::size_t rows, std::size_t cols);                            // zero-filled
    DenseMatrix(std::size_t rows, std::size_t cols, std::vector<double> data);  // finite check

    std::size_t rows() const { return rows_; }
    std::size_t cols() const { return cols_; }
    std::size_t size() const { return data_.size(); }
    double operator()(std::size_t i, std::size_t j) const { return data_[j * rows_ + i]; }
    double& operator()(std::size_t i, std::size_t j) { return data_[j * rows_ + i]; }
    std::span<const double> col(std::size_t j) const { return {data_.data() + j * rows_, rows_}; }
    std::span<double> col(std::size_t j) { return {data_.data() + j * rows_, rows_}; }
    const std::vector<double>& data() const { return data_; }
    std::vector<double>& data() { return data_; }
    bool same_shape(const DenseMatrix& o) const { return rows_ == o.rows_ && cols_ == o.cols_; }
    bool all_finite() const;

private:
    std::size_t rows_ = 0;
    std::size_t cols_ = 0;
    std::vector<double> data_;
};

class GroupAssignment {
public:
    GroupAssignment() = default;
    GroupAssignment(std::vector<std::size_t> labels, std::size_t c);  // validates
    std::size_t size() const { return labels_.size(); }
    std::size_t groups() const { return c_; }
    std::size_t label(std::size_t j) const { return labels_[j]; }
    const std::vector<std::size_t>& labels() const { return labels_; }
    std::vector<std::vector<std::size_t>> group_indices() const;
    std::vector<std::size_t> group_sizes() const;

private:
    std::vector<std::size_t> labels_;
    std::size_t c_ = 0;
};

std::vector<double> column_mean(const DenseMatrix& m, std::span<const std::size_t> columns);
double group_scatter(const DenseMatrix& m, const GroupAssignment& g);
double frob_norm(const DenseMatrix& m);
double elementwise_l1(const DenseMatrix& m);
double l21_norm(const DenseMatrix& m);
std::vector<double> column_l2_norms(const DenseMatrix& m);

// ---- clustering (kmeans.hpp:11-43) -----------------------------------------
struct KMeansConfig {
    std::size_t c = 1;
    std::size_t max_iters = 100;
    std::size_t n_restarts = 1;
    std::uint64_t seed = 0;
    double tol = 1e-6;
};

struct KMeansResult {
    GroupAssignment assignment;
    DenseMatrix centroids;
    double inertia = 0.0;
    std::size_t iters_run = 0;
};

// The engine is advanced exactly as the reference advances it (the k-means++
// draws run on the host through the same libstdc++ distributions).
DenseMatrix kmeans_pp_init(const DenseMatrix& m, std::size_t c, std::mt19937_64& rng);
std::pair<GroupAssignment, DenseMatrix> lloyd_step(const DenseMatrix& m,
                                                   const DenseMatrix& centroids);
KMeansResult kmeans(const DenseMatrix& m, const KMeansConfig& cfg);
KMeansResult kmeans_warm(const DenseMatrix& m, const KMeansConfig& cfg,
                         const GroupAssignment& init);

// ---- solver (solver.hpp:11-88) ---------------------------------------------
enum class SparseNorm { L1, L21 };

struct SolverConfig {
    std::optional<double> lambda;  // unset → sqrt(max(rows, cols))
    double rho0 = 1e-4;
    double kappa = 1.5;
    double tol = 1e-3;
    std::size_t max_iter = 500;
    std::size_t c = 1;
    SparseNorm sparse_norm = SparseNorm::L1;
    KMeansConfig kmeans;
    std::optional<std::size_t> fixed_iters;

    double resolve_lambda(std::size_t rows, std::size_t cols) const;
    void validate() const;
};

struct SolverState {
    DenseMatrix L;
    DenseMatrix S;
    DenseMatrix Theta;
    double rho = 0.0;
    GroupAssignment assignment;
    std::size_t iter = 0;
};

struct ConvergenceReport {
    std::vector<double> feas;
    std::vector<double> delta_l;
    std::vector<double> delta_s;
    std::vector<double> objective;
    bool converged = false;
    std::size_t iters = 0;
};

struct DecompositionResult {
    DenseMatrix L;
    DenseMatrix S;
    GroupAssignment assignment;
    ConvergenceReport report;
    double wall_time = 0.0;
    double lambda = 0.0;
};

struct Residuals {
    double feas = 0.0;
    double delta_l = 0.0;
    double delta_s = 0.0;
    double max() const;
};

DenseMatrix l_update(const DenseMatrix& d, const GroupAssignment& g, double lambda, double rho);
DenseMatrix s_update_l1(const DenseMatrix& b, double threshold);
DenseMatrix s_update_l21(const DenseMatrix& b, double threshold);
void multiplier_update(SolverState& state, const DenseMatrix& x, double kappa);
std::pair<bool, Residuals> check_convergence(const DenseMatrix& x, const DenseMatrix& l_prev,
                                             const DenseMatrix& l, const DenseMatrix& s_prev,
                                             const DenseMatrix& s, double tol);
DecompositionResult solve(const DenseMatrix& x, const SolverConfig& cfg);

// ---- B200 extension ---------------------------------------------------------
namespace b200 {
enum class Precision { F64, F32 };
struct Options {
    Precision precision = Precision::F64;
    int device = 0;
};
struct Timings {
    double init_ms = 0, loop_ms = 0, h2d_ms = 0, d2h_ms = 0;
    std::uint64_t hartigan_moves = 0, slow_iters = 0, exact_fallbacks = 0;
};
DecompositionResult solve(const DenseMatrix& x, const SolverConfig& cfg, const Options& opt,
                          Timings* timings = nullptr);
}  // namespace b200

}  // namespace respca
