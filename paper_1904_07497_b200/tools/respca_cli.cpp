// respca_b200 — the reference command-line tool (proj/tools/respca_cli.cpp)
// on the B200 engine.  Subcommands and options mirror
// the reference: decompose, synth, bench, outliers (frames: PGM stacks are
// outside this build's scope).  Exit codes: 0 success, 2 usage/input error,
// 3 numerical failure (respca_cli.cpp:370-378).
//
// RESPCA1 inputs are solved through respca_cu_solve_file, which streams the
// file into HBM and the results back out in pinned chunks; CSV inputs are
// parsed on the host (io.cpp:60-121 semantics) and solved in memory.
#include <algorithm>
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <numeric>
#include <optional>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <sys/stat.h>
#include <vector>

#include "respca_cu.h"

namespace {

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct InputError : std::runtime_error {  // io::IoError family
    using std::runtime_error::runtime_error;
};
struct SolverError : std::runtime_error {
    int code;
    SolverError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// ---------------------------------------------------------------- arguments
struct Args {
    std::map<std::string, std::string> kv;
    bool has(const std::string& k) const { return kv.count(k) != 0; }
    std::string str(const std::string& k, const std::string& dflt = "") const {
        auto it = kv.find(k);
        return it == kv.end() ? dflt : it->second;
    }
    double num(const std::string& k, double dflt) const {
        if (!has(k)) return dflt;
        const std::string& v = kv.at(k);
        char* end = nullptr;
        const double x = std::strtod(v.c_str(), &end);
        if (end == v.c_str() || *end) throw UsageError("--" + k + ": not a number: " + v);
        return x;
    }
    uint64_t u(const std::string& k, uint64_t dflt) const {
        if (!has(k)) return dflt;
        const std::string& v = kv.at(k);
        uint64_t x = 0;
        auto [p, ec] = std::from_chars(v.data(), v.data() + v.size(), x);
        if (ec != std::errc() || p != v.data() + v.size()) throw UsageError("--" + k + ": not an integer: " + v);
        return x;
    }
};

Args parse(int argc, char** argv, int from, const std::vector<std::string>& allowed) {
    Args a;
    for (int i = from; i < argc; ++i) {
        std::string t = argv[i];
        if (t.rfind("--", 0) != 0) throw UsageError("unexpected argument: " + t);
        t = t.substr(2);
        std::string v;
        const auto eq = t.find('=');
        if (eq != std::string::npos) {
            v = t.substr(eq + 1);
            t = t.substr(0, eq);
        } else {
            if (i + 1 >= argc) throw UsageError("--" + t + " needs a value");
            v = argv[++i];
        }
        if (std::find(allowed.begin(), allowed.end(), t) == allowed.end())
            throw UsageError("unknown option --" + t);
        a.kv[t] = v;
    }
    return a;
}

// --------------------------------------------------------------- matrices
struct Matrix {  // column-major d×n, the reference's DenseMatrix layout
    uint64_t rows = 0, cols = 0;
    std::vector<double> v;
    double& at(uint64_t r, uint64_t c) { return v[c * rows + r]; }
};

bool exists(const std::string& p) {
    struct stat st;
    return ::stat(p.c_str(), &st) == 0;
}
bool is_dir(const std::string& p) {
    struct stat st;
    return ::stat(p.c_str(), &st) == 0 && S_ISDIR(st.st_mode);
}

enum class Format { Csv, Binary, PgmDir };

// respca_cli.cpp:33-46 — extension first, then the magic
Format detect_format(const std::string& in) {
    if (is_dir(in)) return Format::PgmDir;
    const auto dot = in.rfind('.');
    const std::string ext = dot == std::string::npos ? "" : in.substr(dot);
    if (ext == ".csv") return Format::Csv;
    if (ext == ".bin" || ext == ".respca") return Format::Binary;
    std::ifstream is(in, std::ios::binary);
    char magic[8] = {};
    is.read(magic, 8);
    if (is && std::memcmp(magic, "RESPCA1", 7) == 0) return Format::Binary;
    return Format::Csv;
}

// numeric CSV, no header; file row r / column c → entry (r, c)
Matrix read_csv(const std::string& path) {
    std::ifstream is(path);
    if (!is) throw InputError("cannot open " + path);
    std::vector<std::vector<double>> rows;
    std::string line;
    size_t lineno = 0;
    while (std::getline(is, line)) {
        ++lineno;
        if (!line.empty() && line.back() == '\r') line.pop_back();
        if (line.find_first_not_of(" \t") == std::string::npos) continue;
        std::vector<double> row;
        size_t pos = 0;
        while (true) {
            const size_t comma = line.find(',', pos);
            std::string cell = line.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
            const auto b = cell.find_first_not_of(" \t"), e = cell.find_last_not_of(" \t");
            cell = b == std::string::npos ? "" : cell.substr(b, e - b + 1);
            double x;
            auto [p, ec] = std::from_chars(cell.data(), cell.data() + cell.size(), x);
            if (ec != std::errc() || p != cell.data() + cell.size() || cell.empty())
                throw InputError("csv: non-numeric cell '" + cell + "' at line " + std::to_string(lineno));
            row.push_back(x);
            if (comma == std::string::npos) break;
            pos = comma + 1;
        }
        if (!rows.empty() && row.size() != rows.front().size())
            throw InputError("csv: ragged row at line " + std::to_string(lineno));
        rows.push_back(std::move(row));
    }
    if (rows.empty()) throw InputError("csv: empty file " + path);
    Matrix m;
    m.rows = rows.size();
    m.cols = rows.front().size();
    m.v.assign(m.rows * m.cols, 0.0);
    for (uint64_t r = 0; r < m.rows; ++r)
        for (uint64_t c = 0; c < m.cols; ++c) m.at(r, c) = rows[r][c];
    return m;
}

void write_csv(const std::string& path, const Matrix& m) {
    FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw InputError("cannot open " + path + " for writing");
    for (uint64_t r = 0; r < m.rows; ++r) {
        for (uint64_t c = 0; c < m.cols; ++c)
            std::fprintf(f, c + 1 < m.cols ? "%.17g," : "%.17g", m.v[c * m.rows + r]);
        std::fputc('\n', f);
    }
    std::fclose(f);
}

void write_binary(const std::string& path, const Matrix& m) {  // io.hpp:66-69
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw InputError("cannot open " + path + " for writing");
    unsigned char hdr[24];
    std::memcpy(hdr, "RESPCA1\0", 8);
    for (int i = 0; i < 8; ++i) hdr[8 + i] = (unsigned char)(m.rows >> (8 * i));
    for (int i = 0; i < 8; ++i) hdr[16 + i] = (unsigned char)(m.cols >> (8 * i));
    const bool ok = std::fwrite(hdr, 1, 24, f) == 24 &&
                    std::fwrite(m.v.data(), sizeof(double), m.v.size(), f) == m.v.size();
    std::fclose(f);
    if (!ok) throw InputError("cannot write " + path);
}

Matrix read_binary(const std::string& path) {
    uint64_t r = 0, c = 0;
    char err[512];
    if (respca_cu_binary_info(path.c_str(), &r, &c, err, sizeof err) != RESPCA_OK) throw InputError(err);
    Matrix m;
    m.rows = r;
    m.cols = c;
    m.v.resize(r * c);
    FILE* f = std::fopen(path.c_str(), "rb");
    const bool ok = f && std::fseek(f, 24, SEEK_SET) == 0 && std::fread(m.v.data(), 8, m.v.size(), f) == m.v.size();
    if (f) std::fclose(f);
    if (!ok) throw InputError("binary matrix: truncated payload in " + path);
    return m;
}

// ---------------------------------------------------------- synth_generate
// Restatement of io::synth_generate (io.cpp:232-294) with the same libstdc++
// engine and distributions, so the bytes match the reference tool's: near-
// equal contiguous groups of identical uniform(0,1) columns, exactly
// round(sparsity·d·n) corruptions at positions drawn by a partial
// Fisher–Yates shuffle with a random sign and a magnitude in
// [magnitude/2, magnitude), optional N(0, σ²) noise on X.
struct Synth {
    Matrix x, l0, s0;
    std::vector<uint64_t> labels;
};

Synth synth_generate(uint64_t d, uint64_t n, uint64_t c, double sparsity, double magnitude, double sigma,
                     uint64_t seed) {
    if (d == 0 || n == 0) throw UsageError("synth_generate: dimensions must be >= 1");
    if (c == 0 || c > n) throw UsageError("synth_generate: need 1 <= c <= n");
    if (sparsity < 0.0 || sparsity >= 1.0) throw UsageError("synth_generate: sparsity must be in [0,1)");
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> unit(0.0, 1.0);
    Synth s;
    s.labels.resize(n);
    {
        const uint64_t base = n / c, extra = n % c;
        uint64_t j = 0;
        for (uint64_t g = 0; g < c; ++g)
            for (uint64_t k = 0; k < base + (g < extra ? 1 : 0); ++k) s.labels[j++] = g;
    }
    std::vector<double> proto(c * d);  // group g's column, drawn group after group
    for (double& v : proto) v = unit(rng);
    for (Matrix* m : {&s.x, &s.l0, &s.s0}) {
        m->rows = d;
        m->cols = n;
        m->v.assign(d * n, 0.0);
    }
    for (uint64_t j = 0; j < n; ++j)
        std::copy(proto.begin() + s.labels[j] * d, proto.begin() + (s.labels[j] + 1) * d, s.l0.v.begin() + j * d);
    const uint64_t N = d * n;
    const uint64_t nnz = (uint64_t)std::llround(sparsity * (double)N);
    std::vector<uint64_t> perm(N);
    std::iota(perm.begin(), perm.end(), 0ULL);
    std::uniform_real_distribution<double> mag(magnitude / 2.0, magnitude);
    for (uint64_t k = 0; k < nnz; ++k) {
        std::uniform_int_distribution<std::size_t> pick((std::size_t)k, (std::size_t)(N - 1));
        std::swap(perm[k], perm[pick(rng)]);
        const double sign = unit(rng) < 0.5 ? -1.0 : 1.0;
        s.s0.v[perm[k]] = sign * mag(rng);
    }
    for (uint64_t k = 0; k < N; ++k) s.x.v[k] = s.l0.v[k] + s.s0.v[k];
    if (sigma > 0.0) {
        std::normal_distribution<double> noise(0.0, sigma);
        for (double& v : s.x.v) v += noise(rng);
    }
    return s;
}

// ------------------------------------------------------------------ solver
const std::vector<std::string> kSolveOpts = {"input", "groups", "lambda", "rho0", "kappa", "tol",
                                             "max-iter", "norm", "seed", "precision", "device"};

respca_cu_config to_config(const Args& a) {  // respca_cli.cpp:113-124
    respca_cu_config cfg;
    respca_cu_default_config(&cfg);
    const std::string lam = a.str("lambda", "auto");
    if (lam != "auto") {
        cfg.has_lambda = 1;
        cfg.lambda = a.num("lambda", 0.0);
    }
    cfg.rho0 = a.num("rho0", 1e-4);
    cfg.kappa = a.num("kappa", 1.5);
    cfg.tol = a.num("tol", 1e-3);
    cfg.max_iter = a.u("max-iter", 500);
    cfg.c = a.u("groups", 1);
    const std::string norm = a.str("norm", "l1");
    if (norm != "l1" && norm != "l21") throw UsageError("--norm must be l1 or l21");
    cfg.sparse_norm = norm == "l21" ? RESPCA_L21 : RESPCA_L1;
    cfg.km_seed = a.u("seed", 0);
    return cfg;
}

struct Ctx {
    respca_cu_ctx* h = nullptr;
    explicit Ctx(int device) {
        if (respca_cu_create(device, &h) != RESPCA_OK)
            throw SolverError(RESPCA_ECUDA, "no usable sm_100 CUDA device (this tool has no CPU fallback)");
    }
    ~Ctx() { respca_cu_destroy(h); }
    void check(int rc) const {
        if (rc == RESPCA_OK) return;
        const std::string msg = respca_cu_last_error(h);
        if (rc == RESPCA_EINVAL) throw UsageError(msg);
        if (rc == RESPCA_EIO) throw InputError(msg);
        throw SolverError(rc, msg);
    }
};

struct Result {
    std::vector<double> feas, dl, ds, obj;
    respca_cu_report rep{};
    std::vector<uint64_t> labels;
    Matrix L, S;
    void init(const respca_cu_config& cfg, uint64_t n) {
        const uint64_t budget = std::max<uint64_t>(cfg.has_fixed_iters ? cfg.fixed_iters : cfg.max_iter, 1);
        for (auto* v : {&feas, &dl, &ds, &obj}) v->assign(budget, 0.0);
        rep.feas = feas.data();
        rep.delta_l = dl.data();
        rep.delta_s = ds.data();
        rep.objective = obj.data();
        labels.assign(n, 0);
    }
};

Result solve_matrix(Ctx& ctx, const Matrix& x, const respca_cu_config& cfg, int dtype) {
    Result r;
    r.init(cfg, x.cols);
    r.L.rows = r.S.rows = x.rows;
    r.L.cols = r.S.cols = x.cols;
    if (dtype == RESPCA_F64) {
        r.L.v.resize(x.v.size());
        r.S.v.resize(x.v.size());
        ctx.check(respca_cu_solve(ctx.h, x.v.data(), x.rows, x.cols, RESPCA_F64, &cfg, r.L.v.data(), r.S.v.data(),
                                  r.labels.data(), &r.rep));
    } else {
        std::vector<float> xf(x.v.begin(), x.v.end()), lf(x.v.size()), sf(x.v.size());
        ctx.check(respca_cu_solve(ctx.h, xf.data(), x.rows, x.cols, RESPCA_F32, &cfg, lf.data(), sf.data(),
                                  r.labels.data(), &r.rep));
        r.L.v.assign(lf.begin(), lf.end());
        r.S.v.assign(sf.begin(), sf.end());
    }
    return r;
}

void write_report(const std::string& path, const Result& r, const respca_cu_config& cfg) {
    FILE* f = std::fopen(path.c_str(), "w");  // respca_cli.cpp:62-85, JSON lines
    if (!f) throw InputError("cannot open " + path + " for writing");
    for (uint64_t t = 0; t < r.rep.iters; ++t)
        std::fprintf(f, "{\"iter\":%llu,\"feas\":%.17g,\"dL\":%.17g,\"dS\":%.17g,\"objective\":%.17g}\n",
                     (unsigned long long)(t + 1), r.feas[t], r.dl[t], r.ds[t], r.obj[t]);
    std::fprintf(f,
                 "{\"converged\":%s,\"iters\":%llu,\"lambda\":%.17g,\"rho0\":%.17g,\"kappa\":%.17g,"
                 "\"tol\":%.17g,\"groups\":%llu,\"wall_time\":%.17g,\"final_feas\":%.17g}\n",
                 r.rep.converged ? "true" : "false", (unsigned long long)r.rep.iters, r.rep.lambda, cfg.rho0,
                 cfg.kappa, cfg.tol, (unsigned long long)cfg.c, r.rep.wall_time,
                 r.rep.iters ? r.feas[r.rep.iters - 1] : 0.0);
    std::fclose(f);
}

int dtype_of(const Args& a) {
    const std::string p = a.str("precision", "f64");
    if (p != "f64" && p != "f32") throw UsageError("--precision must be f64 or f32");
    return p == "f32" ? RESPCA_F32 : RESPCA_F64;
}

void need_input(const Args& a) {
    if (!a.has("input")) throw UsageError("--input is required");
    if (!a.has("groups")) throw UsageError("--groups is required");
    if (!exists(a.str("input"))) throw UsageError("input does not exist: " + a.str("input"));
}

uint64_t column_count(const std::string& in, Format fmt, Matrix* loaded) {
    if (fmt == Format::Binary) {
        uint64_t r = 0, c = 0;
        char err[512];
        if (respca_cu_binary_info(in.c_str(), &r, &c, err, sizeof err) != RESPCA_OK) throw InputError(err);
        return c;
    }
    *loaded = read_csv(in);
    return loaded->cols;
}

int run_decompose(const Args& a) {
    need_input(a);
    const std::string in = a.str("input");
    const Format fmt = detect_format(in);
    if (fmt == Format::PgmDir) throw UsageError("PGM frame directories are not supported by this build");
    Matrix x;
    const uint64_t n = column_count(in, fmt, &x);
    const respca_cu_config cfg = to_config(a);
    if (cfg.c == 0 || cfg.c > n) throw UsageError("--groups must be in [1, " + std::to_string(n) + "]");
    const int dtype = dtype_of(a);
    Ctx ctx((int)a.u("device", 0));
    Result r;
    const std::string ol = a.str("out-l"), os = a.str("out-s");
    if (fmt == Format::Binary) {  // disk → HBM → disk, streamed
        r.init(cfg, n);
        ctx.check(respca_cu_solve_file(ctx.h, in.c_str(), dtype, &cfg, ol.empty() ? nullptr : ol.c_str(),
                                       os.empty() ? nullptr : os.c_str(), r.labels.data(), n, &r.rep));
    } else {
        r = solve_matrix(ctx, x, cfg, dtype);
        if (!ol.empty()) write_csv(ol, r.L);
        if (!os.empty()) write_csv(os, r.S);
    }
    if (a.has("report")) write_report(a.str("report"), r, cfg);
    std::cout << "converged=" << (r.rep.converged ? "true" : "false") << " iters=" << r.rep.iters
              << " lambda=" << r.rep.lambda << " final_feas=" << (r.rep.iters ? r.feas[r.rep.iters - 1] : 0.0)
              << " wall_time=" << r.rep.wall_time << "\n";
    return 0;
}

int run_outliers(const Args& a) {  // respca_cli.cpp:229-264
    need_input(a);
    const std::string in = a.str("input");
    const Format fmt = detect_format(in);
    if (fmt == Format::PgmDir) throw UsageError("PGM frame directories are not supported by this build");
    Matrix x = fmt == Format::Binary ? read_binary(in) : read_csv(in);
    const respca_cu_config cfg = to_config(a);
    if (cfg.c == 0 || cfg.c > x.cols) throw UsageError("--groups must be in [1, " + std::to_string(x.cols) + "]");
    Ctx ctx((int)a.u("device", 0));
    const Result r = solve_matrix(ctx, x, cfg, dtype_of(a));
    const std::optional<double> thr = a.has("threshold") ? std::optional<double>(a.num("threshold", 0.0)) : std::nullopt;
    std::vector<double> sc(x.cols);
    std::vector<uint64_t> fl(x.cols);
    uint64_t nf = 0;
    ctx.check(respca_cu_outlier_scores(ctx.h, r.S.v.data(), x.rows, x.cols, thr.value_or(0.0), sc.data(), fl.data(),
                                       &nf));
    if (thr) {
        std::cout << "# threshold=" << *thr << "\n";
        for (uint64_t j = 0; j < x.cols; ++j)
            std::cout << j << ' ' << sc[j] << (sc[j] >= *thr ? " FLAGGED" : "") << '\n';
    } else {  // all scores, largest first
        std::vector<uint64_t> order(x.cols);
        std::iota(order.begin(), order.end(), 0ULL);
        std::sort(order.begin(), order.end(), [&](uint64_t p, uint64_t q) { return sc[p] > sc[q]; });
        for (uint64_t j : order) std::cout << j << ' ' << sc[j] << '\n';
    }
    return 0;
}

int run_synth(const Args& a) {  // respca_cli.cpp:166-185
    const uint64_t d = a.u("d", 100), n = a.u("n", 200), c = a.u("c", 3);
    Synth s;
    if (a.has("device")) {  // the d×n assembly on the GPU (respca_cu_synth_generate), same bytes
        if (d == 0 || n == 0) throw UsageError("synth_generate: dimensions must be >= 1");
        Ctx ctx((int)a.u("device", 0));
        for (Matrix* m : {&s.x, &s.l0, &s.s0}) {
            m->rows = d;
            m->cols = n;
            m->v.assign(d * n, 0.0);
        }
        s.labels.assign(n, 0);
        const int rc = respca_cu_synth_generate(ctx.h, d, n, c, a.num("sparsity", 0.05), a.num("magnitude", 1.0),
                                                a.num("noise-sigma", 0.0), a.u("seed", 0), s.x.v.data(),
                                                s.l0.v.data(), s.s0.v.data(), s.labels.data());
        ctx.check(rc);
    } else {
        s = synth_generate(d, n, c, a.num("sparsity", 0.05), a.num("magnitude", 1.0), a.num("noise-sigma", 0.0),
                           a.u("seed", 0));
    }
    if (a.has("out-x")) write_binary(a.str("out-x"), s.x);
    if (a.has("out-l0")) write_binary(a.str("out-l0"), s.l0);
    if (a.has("out-s0")) write_binary(a.str("out-s0"), s.s0);
    if (a.has("out-labels")) {
        std::ofstream os(a.str("out-labels"));
        for (uint64_t g : s.labels) os << g << '\n';
    }
    std::cout << "wrote synthetic problem d=" << d << " n=" << n << " c=" << c << "\n";
    return 0;
}

int run_bench(const Args& a) {  // respca_cli.cpp:187-227
    const std::string mode = a.str("mode", "n");
    if (mode != "n" && mode != "d") throw UsageError("--mode must be n or d");
    std::vector<uint64_t> sizes;
    {
        std::stringstream ss(a.str("sizes"));
        std::string tok;
        while (std::getline(ss, tok, ','))
            if (!tok.empty()) sizes.push_back(std::stoull(tok));
    }
    if (sizes.empty()) throw UsageError("empty size list");
    const uint64_t fixed = a.u("fixed", 500), repeats = a.u("repeats", 10), iters = a.u("iters", 30),
                   seed = a.u("seed", 0);
    std::ofstream file;
    std::ostream* os = &std::cout;
    if (a.has("out")) {
        file.open(a.str("out"));
        os = &file;
    }
    Ctx ctx((int)a.u("device", 0));
    *os << "mode,d,n,iters,repeats,mean_time,stddev_time\n";
    for (uint64_t size : sizes) {
        const uint64_t d = mode == "d" ? size : fixed, n = mode == "d" ? fixed : size;
        const Synth s = synth_generate(d, n, 3, 0.05, 1.0, 0.0, seed);
        respca_cu_config cfg;
        respca_cu_default_config(&cfg);
        cfg.c = 3;
        cfg.has_fixed_iters = 1;
        cfg.fixed_iters = iters;
        cfg.km_seed = seed;
        std::vector<double> times;
        for (uint64_t r = 0; r < repeats; ++r) times.push_back(solve_matrix(ctx, s.x, cfg, RESPCA_F64).rep.wall_time);
        const double mean = std::accumulate(times.begin(), times.end(), 0.0) / (double)times.size();
        double var = 0.0;
        for (double t : times) var += (t - mean) * (t - mean);
        const double sd = times.size() > 1 ? std::sqrt(var / (double)(times.size() - 1)) : 0.0;
        *os << mode << ',' << d << ',' << n << ',' << iters << ',' << repeats << ',' << mean << ',' << sd << '\n';
    }
    return 0;
}

void usage(std::ostream& os) {
    os << "respca_b200: SVD-free robust PCA (low-rank + sparse) on a B200\n"
          "subcommands:\n"
          "  decompose --input X --groups c [--lambda auto|v] [--rho0 v] [--kappa v] [--tol v]\n"
          "            [--max-iter n] [--norm l1|l21] [--seed s] [--precision f64|f32] [--device i]\n"
          "            [--out-l path] [--out-s path] [--report path.jsonl]\n"
          "  synth     [--d] [--n] [--c] [--sparsity] [--magnitude] [--noise-sigma] [--seed]\n"
          "            [--out-x] [--out-l0] [--out-s0] [--out-labels]\n"
          "  bench     [--mode n|d] --sizes a,b,... [--fixed] [--repeats] [--iters] [--seed] [--out]\n"
          "  outliers  (decompose options) [--threshold t]\n"
          "inputs: RESPCA1 binary (.bin/.respca, streamed to the GPU) or numeric CSV\n";
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage(std::cerr);
        return 2;
    }
    const std::string sub = argv[1];
    if (sub == "--help" || sub == "-h") {
        usage(std::cout);
        return 0;
    }
    try {
        if (sub == "decompose") {
            auto o = kSolveOpts;
            for (const char* k : {"out-l", "out-s", "report"}) o.push_back(k);
            return run_decompose(parse(argc, argv, 2, o));
        }
        if (sub == "outliers") {
            auto o = kSolveOpts;
            o.push_back("threshold");
            return run_outliers(parse(argc, argv, 2, o));
        }
        if (sub == "synth")
            return run_synth(parse(argc, argv, 2,
                                   {"d", "n", "c", "sparsity", "magnitude", "noise-sigma", "seed", "out-x",
                                    "out-l0", "out-s0", "out-labels", "device"}));
        if (sub == "bench")
            return run_bench(parse(argc, argv, 2, {"mode", "sizes", "fixed", "repeats", "iters", "seed", "out", "device"}));
        if (sub == "frames") throw UsageError("frames: PGM frame stacks are not supported by this build");
        throw UsageError("unknown subcommand: " + sub);
    } catch (const UsageError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    } catch (const InputError& e) {
        std::cerr << "input error: " << e.what() << "\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "solver error: " << e.what() << "\n";
        return 3;
    }
}
