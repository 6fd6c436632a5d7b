// TEST INFRASTRUCTURE — extern "C" shim over the UNMODIFIED reference I/O
// (proj/src/io.cpp: read_binary_matrix / write_binary_matrix 138-164,
// outlier_scores 296-306), built by oracle/Makefile into _ref/librespca_ref_io.so
// so that tests can pin the device tool's RESPCA1 streaming and outlier scores
// against the reference itself.  Status: 0 ok, 1 io::IoError, 2 other error;
// the exception text goes to err.
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>

#include "respca/io.hpp"

namespace {
void put_err(char* err, size_t len, const char* what) {
    if (err && len) {
        std::strncpy(err, what, len - 1);
        err[len - 1] = 0;
    }
}
}  // namespace

extern "C" {

int ref_write_binary(const char* path, const double* m, uint64_t rows, uint64_t cols, char* err,
                     size_t len) {
    try {
        respca::DenseMatrix a(rows, cols, std::vector<double>(m, m + rows * cols));
        respca::io::write_binary_matrix(path, a);
        return 0;
    } catch (const respca::io::IoError& e) {
        put_err(err, len, e.what());
        return 1;
    } catch (const std::exception& e) {
        put_err(err, len, e.what());
        return 2;
    }
}

int ref_read_binary(const char* path, double* out, uint64_t cap, uint64_t* rows, uint64_t* cols,
                    char* err, size_t len) {
    try {
        const respca::DenseMatrix a = respca::io::read_binary_matrix(path);
        *rows = a.rows();
        *cols = a.cols();
        if (out && a.size() <= cap) std::memcpy(out, a.data().data(), sizeof(double) * a.size());
        return 0;
    } catch (const respca::io::IoError& e) {
        put_err(err, len, e.what());
        return 1;
    } catch (const std::exception& e) {
        put_err(err, len, e.what());
        return 2;
    }
}

int ref_outlier_scores(const double* s, uint64_t d, uint64_t n, double threshold, double* scores,
                       uint64_t* flagged, uint64_t* n_flagged, char* err, size_t len) {
    try {
        respca::DenseMatrix a(d, n, std::vector<double>(s, s + d * n));
        const auto r = respca::io::outlier_scores(a, threshold);
        for (uint64_t j = 0; j < n; ++j) scores[j] = r.scores[j];
        for (size_t k = 0; k < r.flagged.size(); ++k) flagged[k] = r.flagged[k];
        *n_flagged = r.flagged.size();
        return 0;
    } catch (const respca::io::IoError& e) {
        put_err(err, len, e.what());
        return 1;
    } catch (const std::exception& e) {
        put_err(err, len, e.what());
        return 2;
    }
}

int ref_synth(uint64_t d, uint64_t n, uint64_t c, double sparsity, double magnitude, double sigma,
              uint64_t seed, double* x, double* l0, double* s0, uint64_t* labels, char* err, size_t len) {
    try {  // io::synth_generate (io.cpp:232-294)
        respca::io::SynthSpec spec;
        spec.d = d;
        spec.n = n;
        spec.c = c;
        spec.sparsity = sparsity;
        spec.magnitude = magnitude;
        spec.noise_sigma = sigma;
        spec.seed = seed;
        const auto data = respca::io::synth_generate(spec);
        std::memcpy(x, data.x.data().data(), sizeof(double) * d * n);
        std::memcpy(l0, data.l0.data().data(), sizeof(double) * d * n);
        std::memcpy(s0, data.s0.data().data(), sizeof(double) * d * n);
        for (uint64_t j = 0; j < n; ++j) labels[j] = data.assignment.label(j);
        return 0;
    } catch (const std::exception& e) {
        put_err(err, len, e.what());
        return 2;
    }
}

}  // extern "C"
