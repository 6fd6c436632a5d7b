// librespca_cu.so — B200-native RES-PCA engine behind the C-ABI of
// include/respca_cu.h.
//
// Build (see paper_1904_07497_b200/build.py):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false
//        -Xcompiler -fPIC -shared engine.cu -o librespca_cu.so
// --fmad=false is load-bearing: it makes the device arithmetic the reference's
// (no FMA contraction, solver.cpp / kmeans.cpp compiled for baseline x86-64).
#include <cuda_profiler_api.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "alm.cuh"
#include "engine.cuh"
#include "binio.cuh"
#include "synth.h"
#include "synth_dev.cuh"
#include "kmeans_engine.cuh"
#include "km.cuh"

using namespace respca_host;
using namespace respca_dev;

struct AlmBase {
    virtual ~AlmBase() = default;
};

struct respca_cu_ctx {
    int device = 0;
    cudaStream_t st = nullptr;
    std::string err;
    uint64_t launches = 0;
    std::unique_ptr<AlmBase> resident;  // bench-resident solver state
    StreamBufs io;                       // pinned chunks for file streaming
    Arena arena;                         // N-sized solve state reused across solves
    std::unique_ptr<PoolBase> lanes[2];  // k-means restart lanes (fp64, fp32 storage)
    std::unique_ptr<PoolBase> engines[2];  // solve()'s k-means engine (fp64, fp32 storage)
    std::unique_ptr<AlmBase> solver[2];    // solve()'s ALM state + captured graphs, reused
    respca_cu_margins margins{};          // decision margins of the last solve
};

namespace {

using Clock = std::chrono::steady_clock;

void check_dims(uint64_t d, uint64_t n) {
    if (d == 0 || n == 0) throw InvalidArg("DenseMatrix: dimensions must be >= 1");
    if (n > 0x7fffffffULL) throw InvalidArg("respca_cu: more than 2^31-1 columns");
    if (d > (1ULL << 40) || d * n > (1ULL << 40)) throw InvalidArg("respca_cu: matrix too large");
}

void validate_cfg(const respca_cu_config& c) {  // solver.cpp:40-47
    if (c.has_lambda && c.lambda <= 0.0) throw InvalidArg("lambda must be > 0");
    if (c.rho0 <= 0.0) throw InvalidArg("rho0 must be > 0");
    if (c.kappa <= 1.0) throw InvalidArg("kappa must be > 1");
    if (c.tol <= 0.0) throw InvalidArg("tol must be > 0");
    if (c.c == 0) throw InvalidArg("c must be >= 1");
    if (c.max_iter == 0) throw InvalidArg("max_iter must be >= 1");
}

// labels uint64 (API) → int (device) with GroupAssignment validation (matrix.cpp:36-47)
std::vector<int> to_int_labels(const uint64_t* l, uint64_t n, uint64_t c) {
    if (c == 0) throw InvalidArg("GroupAssignment: c must be >= 1");
    std::vector<int> out(n);
    std::vector<char> seen(c, 0);
    for (uint64_t j = 0; j < n; ++j) {
        if (l[j] >= c) throw InvalidArg("GroupAssignment: label out of range");
        out[j] = (int)l[j];
        seen[l[j]] = 1;
    }
    for (uint64_t k = 0; k < c; ++k)
        if (!seen[k]) throw InvalidArg("GroupAssignment: empty group");
    return out;
}

// ---------------------------------------------------------------------------
// The ALM solver (solver.cpp:127-210), device resident.
// ---------------------------------------------------------------------------
template <typename T>
struct Alm : AlmBase {
    respca_cu_ctx* ctx;
    cudaStream_t st;
    Launch ln;
    Stats stats;
    int64_t d = 0;
    int n = 0, c = 0;
    respca_cu_config cfg{};
    double lambda = 0.0;
    uint64_t budget = 0;
    int R = 1, rowblocks = 0, nbF = 0;
    int nbP = 0;          // Pass F partials (CTAs) of the fast path
    bool pf_ring = false;  // Pass F as k_pass_f_ring (few groups)
    // Pass F as streams (k_pass_f_stream): RESPCA_PASSF_STREAM = 0 never, 1 always
    // (where d allows 16-byte copies), default: c = 1; RESPCA_STREAM_RB = rows per stream
    int passf_stream_env = [] {
        const char* e = std::getenv("RESPCA_PASSF_STREAM");
        return e ? std::atoi(e) : -1;
    }();
    bool pf_stream = false;
    // RESPCA_STREAM_NS=3 (fp64): 3-stage pipeline, 3 CTAs per SM (else 5 stages, 2 per SM)
    bool stream_ns3 = [] {
        const char* e = std::getenv("RESPCA_STREAM_NS");
        return e && e[0] == '3';
    }();
    int stream_rb = 32, stream_nrb = 0;
    // fp32 storage: the element chain in FP32 arithmetic (k_pass_f_ring F32A);
    // RESPCA_F32_ARITH=64 keeps the FP64 chain (A/B: C3-f32 0.69 -> 0.78 of HBM)
    bool f32_arith = [] {
        const char* e = std::getenv("RESPCA_F32_ARITH");
        return !(e && std::atoi(e) == 64);
    }();
    int ring_cfg() const {  // RESPCA_RING_CFG (tuning)
        if (const char* e = std::getenv("RESPCA_RING_CFG")) {
            const int r = std::atoi(e);
            if (r == 5 || ((r == 10 || r == 16) && d % 2 == 0) || (r == 33 && sizeof(T) == 4 && d % 4 == 0))
                return r;
        }
        // measured on B200 (fraction of the HBM copy bandwidth):
        //  5: a row per thread, 4-deep ring, 2-member batches — few groups (C5 0.755)
        //  10: two rows per thread, 128-thread CTAs, 4-deep — fp64 up to 256 MB
        //      (C2 0.685), fp32 storage with d % 4 != 0
        //  16: two rows per thread, 256-thread CTAs, 8-deep, 4-member batches —
        //      fp64 larger (C3 0.926)
        //  33: fp32 storage, four rows per thread (16-byte copies), 64-thread CTAs,
        //      8-deep (C3-f32 0.78, C4 0.82; 8-byte copies: 0.71 / 0.79)
        if (d % 2 != 0 || c * ceil_div(d, 512) < 2 * 148) return 5;
        if (sizeof(T) == 4) return d % 4 == 0 ? 33 : 10;
        if ((double)d * (double)n * sizeof(T) <= 256e6) return 10;
        return 16;
    }
    int ring_nt() const {  // rows per CTA of the ring variant
        const int r = ring_cfg();
        return r == 16 ? 512 : (r == 10 || r == 33) ? 256 : 64;
    }
    DBuf<T> X, L, S, Th;
    DBuf<double> G, Cw, Ck, mean_w, partials, rep, marg, nrm, bn;
    bool l21 = false;
    DBuf<int> labels, labels_new;
    DBuf<Ctl> ctl;
    KMeansEngine<T> own_km;  // bench-resident state keeps its own engine
    KMeansEngine<T>& km;     // solve(): the context's engine (buffers reused)
    WhileGraph wg;
    PlainGraph rest;
    double init_ms = 0.0, xnorm = 0.0, xsq_tree = 0.0;
    double m_lloyd = INFINITY, m_gap = INFINITY;  // initial kmeans(X) decision margins
    // (column end, event) per uploaded chunk of X, recorded by a chunked fill
    std::vector<std::pair<int64_t, cudaEvent_t>> chunk_events;
    // fp32 storage: the fp64 copy of X widened chunk by chunk during the upload
    cudaStream_t wide_st = nullptr;
    std::vector<cudaEvent_t> wide_evs;
    bool xd_ready = false;
    ~Alm() override {
        for (cudaEvent_t e : wide_evs) cudaEventDestroy(e);
        if (wide_st) cudaStreamDestroy(wide_st);
    }
    // exact ALM stop (resolve_stop): the start of the loop it replays from, and
    // ‖X‖ as the reference's chain once computed
    Ctl ctl0{};
    std::vector<int> labels0_h;
    bool xnorm_chain_ok = false;
    double xnorm_chain = 0.0;
    uint64_t stop_resolves = 0;  // iterations whose stop test went to the chains
    DBuf<T> Lp, Sp;
    DBuf<double> chains;
    int force_exact_env = [] {  // RESPCA_ALM_STOP_FORCE_EXACT=1: every stop test on the chains
        const char* e = std::getenv("RESPCA_ALM_STOP_FORCE_EXACT");
        return e && e[0] == '1' ? 1 : 0;
    }();
    bool use_tc = [] {
        const char* e = std::getenv("RESPCA_TC_SCREEN");
        return !(e && e[0] == '0');
    }();
    // Pass F → BF16 L′ → TMA-fed screen (RESPCA_TC_SCREEN=1 keeps the
    // converting producers, =0 the FP64 DMMA screen)
    bool use_tma = [] {
        const char* e = std::getenv("RESPCA_TC_SCREEN");
        return !(e && (e[0] == '0' || e[0] == '1'));
    }();
    bool lb_on = false;
    // the BF16 screens (κ ≈ 2⁻⁸·(‖x‖+‖c‖)²) decide nothing when the clusters
    // are tight relative to the data norm (e.g. near-identical video frames):
    // then the FP64 DMMA screen runs instead (set per solve from kmeans(X))
    bool tc_useless = false;
    int64_t dpad = 0;
    DBuf<__nv_bfloat16> Lb;

    bool use_arena = false;  // solve(): borrow the context's arena for X, L, S, Θ, Lb

    // per-solve counters of a reused solver
    void begin_solve() {
        stats = Stats{};
        slow_iters = 0;
        init_ms = 0.0;
        km.st = st;
        km.ln = ln;
        km.stats = &stats;
        km.gram_early = false;
        if constexpr (sizeof(T) == 4) Alm<double>::shared_engine(ctx).gram_early = false;
        for (cudaEvent_t e : wide_evs) cudaEventDestroy(e);
        wide_evs.clear();
        xd_ready = false;
    }
    static KMeansEngine<T>& shared_engine(respca_cu_ctx* cx) {
        auto& h = cx->engines[sizeof(T) == 8 ? 0 : 1];
        if (!h) h.reset(new EngineHolder<T>());
        return static_cast<EngineHolder<T>*>(h.get())->e;
    }
    explicit Alm(respca_cu_ctx* cx, bool shared = false)
        : ctx(cx), st(cx->st), ln{&cx->launches}, km(shared ? shared_engine(cx) : own_km) {
        km.st = st;
        km.ln = ln;
        km.stats = &stats;
        auto& pool = ctx->lanes[sizeof(T) == 8 ? 0 : 1];
        if (!pool) pool.reset(new LanePool<T>());
        km.lane_pool = static_cast<LanePool<T>*>(pool.get());
    }

    Ctl read_ctl() {
        Ctl h;
        CK(cudaMemcpyAsync(&h, ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        return h;
    }
    void write_ctl(const Ctl& h) {
        CK(cudaMemcpyAsync(ctl.p, &h, sizeof(Ctl), cudaMemcpyHostToDevice, st));
    }

    // upload + device-side validation (finite, ‖X‖ ≠ 0)  (solver.cpp:128-132)
    void upload(const T* x, uint64_t dd, uint64_t nn, const respca_cu_config& c_) {
        upload_with(dd, nn, c_, [&](T* dst) {
            CK(cudaMemcpyAsync(dst, x, sizeof(T) * (size_t)(dd * nn), cudaMemcpyHostToDevice, st));
        });
    }
    // fill(X) writes the d×n input into device memory on `st`
    template <class Fill>
    void upload_with(uint64_t dd, uint64_t nn, const respca_cu_config& c_, Fill&& fill) {
        cfg = c_;
        validate_cfg(cfg);
        if (cfg.c > nn) throw InvalidArg("solve: c exceeds column count");
        d = (int64_t)dd;
        n = (int)nn;
        c = (int)cfg.c;
        const int64_t N = d * n;
        if (use_arena) {
            X.borrow(ctx->arena.get("X", sizeof(T) * N), N);
            L.borrow(ctx->arena.get("L", sizeof(T) * N), N);
            S.borrow(ctx->arena.get("S", sizeof(T) * N), N);
            Th.borrow(ctx->arena.get("Th", sizeof(T) * N), N);
        } else {
            X.ensure(N);
            L.ensure(N);
            S.ensure(N);
            Th.ensure(N);
        }
        fill(X.p);
        const int blocks = std::min<int64_t>(2048, ceil_div(N, 256));
        // the initial clustering's Gram matrix starts on its own stream while X
        // is still arriving (the fill recorded chunk events), before the
        // validation below synchronises
        const char* ge = std::getenv("RESPCA_GRAM_EARLY");  // =0: G after the upload (round 1)
        if (!chunk_events.empty() && c > 1 && !(ge && ge[0] == '0')) {
            if constexpr (sizeof(T) == 8) {
                km.bind(X.p, d, n, c);
                if (km.gram_fits()) km.compute_gram_banded(chunk_events);
            } else {
                // fp32 storage: each chunk widened to the fp64 copy the initial
                // clustering runs on (its own stream), G banded behind the widening
                KMeansEngine<double>& kd = Alm<double>::shared_engine(ctx);
                kd.st = st;
                kd.ln = ln;
                kd.stats = &stats;
                double* Xd = static_cast<double*>(ctx->arena.get("Xd", sizeof(double) * N));
                kd.bind(Xd, d, n, c);
                if (kd.gram_fits()) {
                    if (!wide_st) CK(cudaStreamCreateWithFlags(&wide_st, cudaStreamNonBlocking));
                    std::vector<std::pair<int64_t, cudaEvent_t>> wev;
                    int64_t j0 = 0;
                    for (const auto& ch : chunk_events) {
                        CK(cudaStreamWaitEvent(wide_st, ch.second, 0));
                        const int64_t cnt = (ch.first - j0) * d;
                        k_widen<<<std::min<int64_t>(4 * 148 * 8, ceil_div(cnt, 256)), 256, 0, wide_st>>>(
                            X.p + j0 * d, Xd + j0 * d, cnt);
                        ln.add();
                        cudaEvent_t e;
                        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                        wide_evs.push_back(e);
                        CK(cudaEventRecord(e, wide_st));
                        wev.emplace_back(ch.first, e);
                        j0 = ch.first;
                    }
                    kd.compute_gram_banded(wev);
                    xd_ready = true;
                }
            }
        }
        chunk_events.clear();
        nrm.ensure(3 * 2048 + 8);
        k_norms<T><<<blocks, 256, 0, st>>>(X.p, N, nrm.p);
        k_sum_partials<<<1, 256, 0, st>>>(nrm.p, blocks, 3, nrm.p + 3 * 2048);
        ln.add(2);
        double h[3];
        CK(cudaMemcpyAsync(h, nrm.p + 3 * 2048, sizeof(h), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (h[2] != 0.0) throw InvalidArg("solve: non-finite X");
        xsq_tree = h[0];
        xnorm = std::sqrt(h[0]);
        if (xnorm == 0.0) throw InvalidArg("solve: all-zero X");
    }

    void setup_state() {
        const int64_t N = d * n;
        tc_useless = false;
        lambda = cfg.has_lambda ? cfg.lambda : std::sqrt((double)std::max<int64_t>(d, n));
        budget = cfg.has_fixed_iters ? cfg.fixed_iters : cfg.max_iter;
        CK(cudaMemcpyAsync(L.p, X.p, sizeof(T) * N, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemsetAsync(S.p, 0, sizeof(T) * N, st));
        CK(cudaMemsetAsync(Th.p, 0, sizeof(T) * N, st));
        G.ensure((size_t)2 * d * c);
        Cw.ensure((size_t)d * c);
        Ck.ensure((size_t)d * c);
        mean_w.ensure(c);
        labels.ensure(n);
        labels_new.ensure(n);
        rep.ensure(std::max<uint64_t>(budget, 1) * 4);
        marg.ensure(std::max<uint64_t>(budget, 1));
        ctl.ensure(1);
        R = (d % 2 == 0) ? 2 : 1;
        rowblocks = ceil_div(d, 256 * R);
        dpad = ((d + TC_KB - 1) / TC_KB) * TC_KB;
        lb_on = use_tc && use_tma && c > 1 && c <= TC_N && cfg.sparse_norm != RESPCA_L21;
        if (lb_on) {
            if (use_arena) Lb.borrow(ctx->arena.get("Lb", sizeof(__nv_bfloat16) * (size_t)n * dpad), (size_t)n * dpad);
            else Lb.ensure((size_t)n * dpad);
            CK(cudaMemsetAsync(Lb.p, 0, sizeof(__nv_bfloat16) * (size_t)n * dpad, st));  // K padding stays 0
        }
        nbF = rowblocks * c;
        // ℓ1: Pass F as k_pass_f_ring (a private cp.async ring per thread, ring_cfg());
        // round 1 measured it faster than a register-batched walk on every shape
        // (C3 1.026 -> 0.974 ms, C5 24.8 -> 18.4, C4 0.74 -> 0.45)
        pf_ring = !(cfg.sparse_norm == RESPCA_L21);
        nbP = pf_ring ? ceil_div(d, ring_nt()) * c : nbF;
        // c = 1 ("rank unknown"): one-thread-per-row walks cannot fill the GPU; Pass F
        // runs as row-block streams (measured fraction of HBM, ring → stream: C2-c1
        // 0.06 → 0.57, C3-c1 0.31 → 0.77, C5 0.73 → 0.85).  Every stream lasts the whole
        // kernel, so the rows per stream decide (sweeps in profiles/round2_ncu.md):
        //  * one wave only — the c·⌈d/rb⌉ streams fit the 2·148 resident CTAs, and
        //    at least ≈200 of them so that most SMs hold two;
        //  * segments on 64-byte boundaries (DRAM moves 64 bytes at a time: rb = 34
        //    at C3-c1 reads 12 % more than algorithmic), better on 128-byte ones;
        //  * a stage's 256 chunks well used: ⌊256/(rb/VEC)⌋·(rb/VEC) close to 256.
        pf_stream = false;
        if (!(cfg.sparse_norm == RESPCA_L21) && d % (16 / (int64_t)sizeof(T)) == 0 &&
            (passf_stream_env > 0 || (passf_stream_env < 0 && c == 1))) {
            const int vec = 16 / (int)sizeof(T), al = 64 / (int)sizeof(T), rbmax = 256;
            const int64_t slots = (stream_ns3 ? 3 : 2) * 148;
            double best = -1.0;
            for (int r = al; r <= rbmax; r += al) {
                const int lpc = r / vec;
                if (lpc > 256) break;
                const int64_t ns = (int64_t)c * ceil_div(d, (int64_t)r);
                if (ns > slots) continue;
                const double util = (double)((256 / lpc) * lpc) / 256.0;
                const double score = util + (r % (2 * al) == 0 ? 0.08 : 0.0) -
                                     (ns < 200 ? (double)(200 - ns) / 200.0 : 0.0);
                if (score > best) {
                    best = score;
                    stream_rb = r;
                }
            }
            pf_stream = best >= 0.0;  // d beyond 296·256 rows: the ring walks
            const int rbmax_env = rbmax;
            if (const char* e = std::getenv("RESPCA_STREAM_RB")) {
                const int r = std::atoi(e);
                if (r >= vec && r <= rbmax_env && r % vec == 0) {
                    stream_rb = r;
                    pf_stream = true;
                }
            }
            if (pf_stream) {
                stream_nrb = (int)ceil_div(d, (int64_t)stream_rb);
                nbP = c * stream_nrb;
            }
        }
        partials.ensure((size_t)std::max(nbF, nbP) * PF_STRIDE);
        Ctl h{};
        h.rho = cfg.rho0;
        const double rn = cfg.rho0 * cfg.kappa;
        h.rho_next = (1e12 < rn) ? 1e12 : rn;
        h.own_w = cfg.rho0 / (2.0 * lambda + cfg.rho0);
        h.thr = 1.0 / cfg.rho0;
        h.lambda = lambda;
        h.kappa = cfg.kappa;
        h.tol = cfg.tol;
        h.xnorm = xnorm;
        h.iter = 0;
        h.budget = (int)std::min<uint64_t>(budget, 0x7fffffff);
        h.fixed = cfg.has_fixed_iters ? 1 : 0;
        l21 = cfg.sparse_norm == RESPCA_L21;
        h.l21 = l21 ? 1 : 0;
        h.done = budget == 0 ? 1 : 0;  // fixed_iters = 0: no iteration (solver.cpp:152, 157)
        // stop guard: fp64 storage decides like the reference (fp32 storage has
        // no reference chain to match)
        h.guard = sizeof(T) == 8 ? 1 : 0;
        h.force_exact = force_exact_env;
        h.stop_amb = 0;
        {
            // recursive summation of N non-negative terms, any order: |sum − exact| ≤
            // γ_{N−1}·exact (γ_m = m·u/(1 − m·u)); chain vs tree: ≤ 2γ/(1−γ) of the tree
            const double u = std::ldexp(1.0, -53), m = (double)(N - 1);
            const double gam = m * u / (1.0 - m * u);
            h.sum_eps = 2.0 * gam / (1.0 - gam) * 1.0001;
            const double e2 = h.sum_eps + 4.0 * u;  // covers this host rounding
            h.xn_lo = std::sqrt(std::nextafter(xsq_tree * (1.0 - e2), 0.0));
            h.xn_hi = std::sqrt(std::nextafter(xsq_tree * (1.0 + e2), HUGE_VAL));
        }
        xnorm_chain_ok = false;
        stop_resolves = 0;
        ctl0 = h;
        write_ctl(h);
    }

    // initial grouping: kmeans(X) with >= 5 restarts (solver.cpp:143-150)
    void init_labels() {
        const auto ti0 = Clock::now();
        auto tr = [&](const char* what) {
            if (trace_on()) {
                CK(cudaStreamSynchronize(st));
                std::fprintf(stderr, "[respca] init: %s at %.3fs\n", what,
                             std::chrono::duration<double>(Clock::now() - ti0).count());
            }
        };
        km.bind(X.p, d, n, c);
        tr("bind");
        if (c == 1) {
            CK(cudaMemsetAsync(labels.p, 0, sizeof(int) * n, st));
            km.h_labels.assign(n, 0);
        } else {
            const uint64_t restarts = std::max<uint64_t>(cfg.km_n_restarts, 5);
            double inertia = 0.0;
            if constexpr (sizeof(T) == 4) {
                // fp32 storage: kmeans(X) on an exact fp64 copy of X — the same values,
                // so the same labels, but the FP64 tensor-core Gram and screens read
                // doubles instead of widening every float in their inner loops
                // (C3-f32 init 207 -> fp64's time)
                const int64_t N = d * n;
                double* Xd = static_cast<double*>(ctx->arena.get("Xd", sizeof(double) * N));
                if (xd_ready) {  // widened during the upload
                    CK(cudaStreamWaitEvent(st, wide_evs.back(), 0));
                } else {
                    k_widen<<<std::min<int64_t>(4 * 148 * 8, ceil_div(N, 256)), 256, 0, st>>>(X.p, Xd, N);
                    ln.add();
                }
                KMeansEngine<double>& kd = Alm<double>::shared_engine(ctx);
                kd.st = st;
                kd.ln = ln;
                kd.stats = &stats;
                auto& pool = ctx->lanes[0];
                if (!pool) pool.reset(new LanePool<double>());
                kd.lane_pool = static_cast<LanePool<double>*>(pool.get());
                kd.bind(Xd, d, n, c);
                kd.kmeans(cfg.km_max_iters, restarts, cfg.km_seed, cfg.km_tol, labels.p, Ck.p, &inertia, nullptr);
                kd.fetch_labels(labels.p);
                km.h_labels = kd.h_labels;
            } else {
                km.kmeans(cfg.km_max_iters, restarts, cfg.km_seed, cfg.km_tol, labels.p, Ck.p, &inertia,
                          nullptr);
            }
            // mean squared distance to the own centroid vs the scale (‖x‖+‖c‖)² ≈ 4‖x‖²
            // of the BF16 bound: below 1/32 its intervals straddle every decision
            {  // decision margins of the initial clustering
                const KMeansEngine<double>* kk = nullptr;
                if constexpr (sizeof(T) == 4) kk = &Alm<double>::shared_engine(ctx);
                const double lm = kk ? kk->lloyd_margin : km.lloyd_margin;
                const std::vector<double>& ri = kk ? kk->restart_inertia : km.restart_inertia;
                double b1 = INFINITY, b2 = INFINITY;
                for (double v : ri) {
                    if (!(v == v)) continue;
                    if (v < b1) {
                        b2 = b1;
                        b1 = v;
                    } else if (v < b2) {
                        b2 = v;
                    }
                }
                m_lloyd = lm;
                m_gap = (b2 < INFINITY && b1 > 0.0) ? (b2 - b1) / b1 : INFINITY;
            }
            tc_useless = !(inertia >= xnorm * xnorm * 4.0 / 32.0);
            if (tc_useless && lb_on) lb_on = false;
            tr("kmeans");
            if constexpr (sizeof(T) == 8) km.fetch_labels(labels.p);
        }
        labels0_h = km.h_labels;
        km.bind(L.p, d, n, c);  // from here on the p-update clusters L
        km.groups.build(km.h_labels.data(), n, c);
        km.upload_groups();
        tr("groups");
    }

    template <int K, int NS, int RBMAX>
    void launch_stream() {
        auto kf = k_pass_f_stream<T, K, NS, RBMAX>;
        constexpr int sm = StreamCfg<T, K, NS, RBMAX>::SMEM;
        CK(cudaFuncSetAttribute((const void*)kf, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        double* G1 = G.p + (size_t)d * c;
        kf<<<c * stream_nrb, PFS_THREADS, sm, st>>>(X.p, L.p, S.p, Th.p, km.goff.p, km.members.p,
                                             c > 1 ? km.gsize_ord.p : nullptr, G.p, G1, G.p, G1, Cw.p,
                                             mean_w.p, ctl.p, partials.p, d, stream_rb, stream_nrb,
                                             lb_on ? Lb.p : nullptr, dpad, c == 1 ? 1 : 0);
    }

    void launch_group_D() {  // G_t = Σ_{j∈g} ((x − s) + θ/ρ) into G[parity]
        if (R == 2)
            k_group_sum<T, 2, 0><<<nbF, 256, 0, st>>>(X.p, S.p, Th.p, km.goff.p, km.members.p,
                                                      ctl.p, G.p, G.p + (size_t)d * c, 1, 0, d,
                                                      rowblocks);
        else
            k_group_sum<T, 1, 0><<<nbF, 256, 0, st>>>(X.p, S.p, Th.p, km.goff.p, km.members.p,
                                                      ctl.p, G.p, G.p + (size_t)d * c, 1, 0, d,
                                                      rowblocks);
        k_mean_w<<<ceil_div(c, 256), 256, 0, st>>>(ctl.p, km.goff.p, mean_w.p, c);
        ln.add(2);
    }

    void prepare(const T* x, uint64_t dd, uint64_t nn, const respca_cu_config& c_) {
        upload(x, dd, nn, c_);
        Events ev;
        CK(cudaEventRecord(ev.a, st));
        setup_state();
        init_labels();
        launch_group_D();
        CK(cudaEventRecord(ev.b, st));
        CK(cudaEventSynchronize(ev.b));
        init_ms = ev.ms();
        capture();
    }

    // ---- one iteration of the fast path, captured ----------------------
    void launch_pass_f() {
        if (l21) {  // ℓ2,1: F1 only (the S/Θ half runs after the column norms)
            double* G1 = G.p + (size_t)d * c;
            if (R == 2)
                k_pass_f1<T, 2><<<nbF, 256, 0, st>>>(X.p, L.p, S.p, Th.p, km.goff.p, km.members.p,
                                                    G.p, G1, Cw.p, mean_w.p, ctl.p, partials.p, d,
                                                    rowblocks);
            else
                k_pass_f1<T, 1><<<nbF, 256, 0, st>>>(X.p, L.p, S.p, Th.p, km.goff.p, km.members.p,
                                                    G.p, G1, Cw.p, mean_w.p, ctl.p, partials.p, d,
                                                    rowblocks);
            ln.add();
            return;
        }
        if (pf_stream) {
            if constexpr (sizeof(T) == 8) {
                if (stream_ns3) launch_stream<1, 3, 128>();
                else if (stream_rb > 128) launch_stream<1, 5, 256>();
                else launch_stream<1, 5, 128>();
            } else {
                launch_stream<1, 4, 256>();
            }
            ln.add();
            return;
        }
        if (pf_ring) {
            double* G1 = G.p + (size_t)d * c;
            auto go = [&](auto kf, int nt, int u, int rw = 1) {
                const size_t sm = (size_t)u * 4 * nt * rw * sizeof(T);
                CK(cudaFuncSetAttribute((const void*)kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
                const int rbr = ceil_div(d, (int64_t)nt * rw);
                kf<<<rbr * c, nt, sm, st>>>(X.p, L.p, S.p, Th.p, km.goff.p, km.members.p, G.p, G1, G.p, G1, Cw.p,
                                            mean_w.p, ctl.p, partials.p, d, rbr, lb_on ? Lb.p : nullptr, dpad);
            };
            // the three configurations ring_cfg() chooses from (RESPCA_RING_CFG: the
            // tuning sweep's numbering, kept for reproducibility)
            const int rc = ring_cfg();
            if constexpr (sizeof(T) == 4) {
                if (f32_arith) {
                    switch (rc) {
                        case 33: go(k_pass_f_ring<T, 8, 64, 2, 4, true>, 64, 8, 4); break;
                        case 10: go(k_pass_f_ring<T, 4, 128, 2, 2, true>, 128, 4, 2); break;
                        case 16: go(k_pass_f_ring<T, 8, 256, 4, 2, true>, 256, 8, 2); break;
                        default: go(k_pass_f_ring<T, 4, 64, 2, 1, true>, 64, 4); break;
                    }
                    ln.add();
                    return;
                }
                if (rc == 33) {
                    go(k_pass_f_ring<T, 8, 64, 2, 4>, 64, 8, 4);
                    ln.add();
                    return;
                }
            }
            switch (rc) {
                case 10: go(k_pass_f_ring<T, 4, 128, 2, 2>, 128, 4, 2); break;
                case 16: go(k_pass_f_ring<T, 8, 256, 4, 2>, 256, 8, 2); break;
                default: go(k_pass_f_ring<T, 4, 64, 2>, 64, 4); break;
            }
            ln.add();
            return;
        }
    }
    void launch_pass_a() {
        if (c <= 1) return;
        if (lb_on) km.screen_tma(Lb.p, dpad, Cw.p);         // tcgen05, operands by TMA from Pass F's BF16 L′
        else if (use_tc && !tc_useless && km.tc_ok()) km.screen_tc(Cw.p);  // tcgen05, fp64 → bf16 producers
        else km.screen(Cw.p);                               // FP64 DMMA screen
        km.decide(Cw.p, labels.p, km.counts.p, 1, labels_new.p, ctl.p);  // verdict: k_finalize
    }
    // ℓ2,1 second half: ‖B_j‖, S'/Θ'/G_{t+1}, the ℓ2,1 report term
    void launch_post() {
        if (!l21) return;
        bn.ensure(n);
        double* G1 = G.p + (size_t)d * c;
        k_bnorms<T><<<ceil_div(n, 128), 128, 0, st>>>(X.p, L.p, Th.p, ctl.p, d, n, bn.p);
        if (R == 2)
            k_pass_f2<T, 2><<<nbF, 256, 0, st>>>(X.p, L.p, S.p, Th.p, km.goff.p, km.members.p,
                                                bn.p, G.p, G1, ctl.p, partials.p, d, rowblocks);
        else
            k_pass_f2<T, 1><<<nbF, 256, 0, st>>>(X.p, L.p, S.p, Th.p, km.goff.p, km.members.p,
                                                bn.p, G.p, G1, ctl.p, partials.p, d, rowblocks);
        k_l21_term<<<1, 1024, 0, st>>>(bn.p, n, ctl.p);
        ln.add(3);
    }
    void launch_finalize(bool cond) {
        CK(pdl_launch(k_finalize, dim3(1), dim3(1024), 0, st, ctl.p, partials.p, l21 ? nbF : nbP, km.goff.p,
                      mean_w.p, c, rep.p, cond ? 1 : 0, cond ? wg.handle : cudaGraphConditionalHandle{}, marg.p));
        ln.add();
    }
    int kernels_per_iter() const { return 1 + (c > 1 ? 2 + km.decide_kernels() : 0) + 1 + (l21 ? 3 : 0); }

    // the captured graphs bake in pointers and shapes: re-capture only when
    // one of them (or any device allocation) changed since the last capture
    uint64_t cap_key[13] = {};
    bool cap_valid = false;
    void capture_if_needed() {
        const uint64_t key[13] = {(uint64_t)d, (uint64_t)n, (uint64_t)c, (uint64_t)l21, (uint64_t)lb_on,
                                  (uint64_t)(use_tc && !tc_useless), (uint64_t)R, (uint64_t)rowblocks, (uint64_t)nbF,
                                  ((uint64_t)pf_stream << 44) ^ ((uint64_t)stream_rb << 45), (uint64_t)dpad, g_alloc_gen.load(),
                                  (uint64_t)pdl_on()};
        if (cap_valid && std::equal(key, key + 13, cap_key)) return;
        cap_valid = false;
        try {
            capture();
        } catch (...) {  // never leave the stream in capture mode
            cudaStreamCaptureStatus cs;
            if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
                cudaGraph_t g = nullptr;
                cudaStreamEndCapture(st, &g);
                if (g) cudaGraphDestroy(g);
            }
            cudaGetLastError();
            throw;
        }
        std::copy(key, key + 13, cap_key);
        cap_valid = true;
    }
    void capture() {
        const uint64_t saved = *ln.counter;  // captured launches are not executions
        // WHILE graph: the product loop
        wg.begin(st);
        launch_pass_f();
        launch_pass_a();
        launch_post();
        launch_finalize(true);
        wg.end(st);
        // plain graph of everything after Pass F (bench timing of Pass F by events)
        rest.begin(st);
        launch_pass_a();
        launch_post();
        launch_finalize(false);
        rest.end(st);
        *ln.counter = saved;
    }

    // slow path: the p-update changed labels (or a Hartigan move) in the last
    // finalized iteration t → finish kmeans_warm exactly, refresh groups, G.
    void slow_path(Ctl& h) {
        Nvtx r_("ALM slow path (kmeans_warm)");
        const int t = h.iter - 1;
        CK(cudaMemcpyAsync(Ck.p, Cw.p, sizeof(double) * d * c, cudaMemcpyDeviceToDevice, st));
        km.h_labels.resize(n);
        CK(cudaMemcpyAsync(km.h_labels.data(), labels.p, sizeof(int) * n, cudaMemcpyDeviceToHost,
                           st));
        CK(cudaStreamSynchronize(st));
        km.lloyd_run(Ck.p, labels.p, cfg.km_max_iters, cfg.km_tol);  // kmeans_warm, kmeans.cpp:257
        // lloyd_run left goff/members/counts = labels_{t+1} and Ck = means_of(L', labels_{t+1})
        const double scatter = km.inertia(Ck.p, labels.p);
        const double obj = lambda * scatter + h.last_l1;
        CK(cudaMemcpyAsync(rep.p + (size_t)t * 4 + 3, &obj, sizeof(double), cudaMemcpyHostToDevice,
                           st));
        launch_group_D();  // G_{t+1} under the new labels, ρ_{t+1}
        h.slow = 0;
        h.changed = h.moves = h.ambiguous = 0;
        h.done = h.converged || h.nonfinite || (h.iter >= h.budget);
        write_ctl(h);
        CK(cudaStreamSynchronize(st));
    }

    // run the loop to completion (solver.cpp:157-201)
    uint64_t slow_iters = 0;
    void run_loop() {
        if (budget == 0) return;  // solver.cpp:157: no iteration, L = X, S = 0
        for (;;) {
            const int it0 = read_ctl().iter;
            wg.launch(st);
            Ctl h = read_ctl();
            ln.add((uint64_t)kernels_per_iter() * (uint64_t)(h.iter - it0));
            if (h.nonfinite) throw NonFinite("solve: non-finite value inside the ALM loop");
            if (h.stop_amb) {
                resolve_stop(h);  // also runs the iteration's slow path, if any
            } else if (h.slow) {
                ++slow_iters;
                slow_path(h);
                capture_if_needed();  // the exact continuation may have grown a buffer
            }
            if (h.nonfinite) throw NonFinite("solve: non-finite value inside the ALM loop");
            if (h.done) break;
        }
    }

    // ---- the exact ALM stop ------------------------------------------------
    // The stop test of iteration t was undecidable on the tree sums.  The
    // reference decides it on its chains over L_{t+1} − L_t and S_{t+1} − S_t,
    // but L_t, S_t were overwritten in place.  The solve is deterministic, so it
    // is replayed from the state after kmeans(X) (fixed-iteration mode, every
    // iteration — slow paths included — exactly as before) up to iteration t,
    // L_t and S_t are copied aside, iteration t runs again, and k_exact_chains
    // computes the reference's three chains (and ‖X‖'s once).  Costs one more
    // loop up to t plus ≈4 cycles per element and chain; never happens on the
    // BASELINE workloads without RESPCA_ALM_STOP_FORCE_EXACT=1.
    void reset_to_start(int target) {
        const int64_t N = d * n;
        CK(cudaMemcpyAsync(L.p, X.p, sizeof(T) * N, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemsetAsync(S.p, 0, sizeof(T) * N, st));
        CK(cudaMemsetAsync(Th.p, 0, sizeof(T) * N, st));
        CK(cudaMemcpyAsync(labels.p, labels0_h.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st));
        km.h_labels = labels0_h;
        km.groups.build(km.h_labels.data(), n, c);
        km.upload_groups();
        Ctl h = ctl0;
        h.fixed = 1;
        h.budget = target;
        h.done = target == 0 ? 1 : 0;
        write_ctl(h);
        launch_group_D();
        CK(cudaStreamSynchronize(st));
    }
    // fixed-mode iterations until ctl.iter == target (slow paths included)
    void advance(int target) {
        for (;;) {
            Ctl h = read_ctl();
            if (h.iter >= target) return;
            if (!h.done) {
                wg.launch(st);
                ln.add((uint64_t)kernels_per_iter() * (uint64_t)(read_ctl().iter - h.iter));
                h = read_ctl();
            }
            if (h.nonfinite) throw NonFinite("solve: non-finite value inside the ALM loop");
            if (h.slow) {
                slow_path(h);
                capture_if_needed();
            } else if (h.done && h.iter < target) {
                throw RuntimeErr("respca: replay of the ALM loop stopped early");
            }
        }
    }
    void resolve_stop(Ctl& h) {
        Nvtx r_("exact ALM stop (replay + chains)");
        const int t = h.iter - 1;
        const int64_t N = d * n;
        const Stats s0 = stats;
        const uint64_t slow0 = slow_iters;
        // the report rows so far (some may hold chain values already)
        std::vector<double> rows((size_t)t * 4 + 4);
        if (t > 0) CK(cudaMemcpyAsync(rows.data(), rep.p, sizeof(double) * 4 * t, cudaMemcpyDeviceToHost, st));
        Lp.ensure(N);
        Sp.ensure(N);
        chains.ensure(4);
        capture_if_needed();
        reset_to_start(t);
        advance(t);
        CK(cudaMemcpyAsync(Lp.p, L.p, sizeof(T) * N, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(Sp.p, S.p, sizeof(T) * N, cudaMemcpyDeviceToDevice, st));
        Ctl g = read_ctl();
        g.budget = t + 1;
        g.done = 0;
        write_ctl(g);
        wg.launch(st);
        ln.add((uint64_t)kernels_per_iter());
        g = read_ctl();
        if (g.nonfinite) throw NonFinite("solve: non-finite value inside the ALM loop");
        if (g.iter != t + 1) throw RuntimeErr("respca: replay of the ALM loop diverged");
        const Stats s1 = stats;
        const bool was_slow = g.slow != 0;
        if (was_slow) {
            slow_path(g);
            capture_if_needed();
            g = read_ctl();
        }
        const Stats s2 = stats;
        k_exact_chains<T><<<4, 256, 0, st>>>(X.p, L.p, Lp.p, S.p, Sp.p, N, xnorm_chain_ok ? 1 : 0, chains.p);
        ln.add();
        double ch[4];
        CK(cudaMemcpyAsync(ch, chains.p, sizeof(ch), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (!xnorm_chain_ok) {
            xnorm_chain = std::sqrt(ch[3]);  // frob_norm, matrix.cpp:99-103
            xnorm_chain_ok = true;
        }
        const double feas = std::sqrt(ch[0]) / xnorm_chain;  // solver.cpp:20, 30
        const double dl = std::sqrt(ch[1]) / xnorm_chain;
        const double ds = std::sqrt(ch[2]) / xnorm_chain;
        // restore the earlier report rows, this row's residuals from the chains
        if (t > 0) CK(cudaMemcpyAsync(rep.p, rows.data(), sizeof(double) * 4 * t, cudaMemcpyHostToDevice, st));
        const double r3[3] = {feas, dl, ds};
        CK(cudaMemcpyAsync(rep.p + (size_t)t * 4, r3, sizeof(r3), cudaMemcpyHostToDevice, st));
        const bool conv = !ctl0.fixed && std::max({feas, dl, ds}) <= cfg.tol;  // solver.cpp:197
        g.fixed = ctl0.fixed;
        g.budget = ctl0.budget;
        g.converged = conv ? 1 : 0;
        g.stop_amb = 0;
        g.slow = 0;
        g.exact_fallbacks = h.exact_fallbacks;
        std::copy(h.margin_hist, h.margin_hist + 6, g.margin_hist);
        g.xnorm = xnorm_chain;  // from here on the report divides by the reference's ‖X‖
        g.xn_lo = g.xn_hi = xnorm_chain;
        g.done = conv || g.nonfinite || g.iter >= g.budget;
        write_ctl(g);
        CK(cudaStreamSynchronize(st));
        stats = s0;
        stats.hartigan_moves += s2.hartigan_moves - s1.hartigan_moves;
        stats.exact_fallbacks += s2.exact_fallbacks - s1.exact_fallbacks;
        stats.lloyd_steps += s2.lloyd_steps - s1.lloyd_steps;
        stats.hartigan_passes += s2.hartigan_passes - s1.hartigan_passes;
        slow_iters = slow0 + (was_slow ? 1 : 0);
        ++stop_resolves;
        if (trace_on())
            std::fprintf(stderr, "[respca] stop test of iteration %d on the chains: max %.17g vs tol %.17g -> %s\n",
                         t + 1, std::max({feas, dl, ds}), cfg.tol, conv ? "converged" : "continue");
        h = g;
    }

    void download(T* Lo, T* So, uint64_t* lab, respca_cu_report* rep_out) {
        const int64_t N = d * n;
        download_with(
            [&](const T* Ld) { CK(cudaMemcpyAsync(Lo, Ld, sizeof(T) * N, cudaMemcpyDeviceToHost, st)); },
            [&](const T* Sd) { CK(cudaMemcpyAsync(So, Sd, sizeof(T) * N, cudaMemcpyDeviceToHost, st)); },
            lab, rep_out);
    }
    // sinkL / sinkS read the device L / S (stream-ordered on `st`)
    template <class SinkL, class SinkS>
    void download_with(SinkL&& sinkL, SinkS&& sinkS, uint64_t* lab, respca_cu_report* rep_out) {
        const Ctl h = read_ctl();
        if (trace_on())
            std::fprintf(stderr,
                         "[respca] loop: %d iterations; columns x iterations with Hartigan margin "
                         "/ (|x|+|c|)^2 below 1e-1..1e-6: %u %u %u %u %u %u (of %lld)\n",
                         h.iter, h.margin_hist[0], h.margin_hist[1], h.margin_hist[2],
                         h.margin_hist[3], h.margin_hist[4], h.margin_hist[5],
                         (long long)h.iter * n);
        sinkL(L.p);
        sinkS(S.p);
        std::vector<int> hl(n);
        CK(cudaMemcpyAsync(hl.data(), labels.p, sizeof(int) * n, cudaMemcpyDeviceToHost, st));
        std::vector<double> hr((size_t)h.iter * 4 + 4), hm((size_t)h.iter + 1);
        if (h.iter > 0) {
            CK(cudaMemcpyAsync(hr.data(), rep.p, sizeof(double) * 4 * h.iter,
                               cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(hm.data(), marg.p, sizeof(double) * h.iter, cudaMemcpyDeviceToHost, st));
        }
        CK(cudaStreamSynchronize(st));
        {
            respca_cu_margins& mg = ctx->margins;
            mg = respca_cu_margins{};
            mg.alm_stop = mg.alm_stop_final = mg.s_support = INFINITY;
            for (int t = 0; t < h.iter; ++t) {
                const double mx = std::max({hr[(size_t)t * 4], hr[(size_t)t * 4 + 1], hr[(size_t)t * 4 + 2]});
                const double am = std::fabs(mx / cfg.tol - 1.0);
                if (!cfg.has_fixed_iters) {
                    mg.alm_stop = std::min(mg.alm_stop, am);
                    if (t + 1 == h.iter) mg.alm_stop_final = am;
                }
                mg.s_support = std::min(mg.s_support, hm[(size_t)t]);
            }
            mg.lloyd_stop = c > 1 ? m_lloyd : INFINITY;
            mg.restart_gap = c > 1 ? m_gap : INFINITY;
            mg.stop_resolves = stop_resolves;
            if (trace_on())
                std::fprintf(stderr,
                             "[respca] margins: ALM stop %.3g (final %.3g), S support %.3g, Lloyd stop %.3g, "
                             "restart gap %.3g, %llu stop test(s) on the chains\n",
                             mg.alm_stop, mg.alm_stop_final, mg.s_support, mg.lloyd_stop, mg.restart_gap,
                             (unsigned long long)mg.stop_resolves);
        }
        for (int j = 0; j < n; ++j) lab[j] = (uint64_t)hl[j];
        if (rep_out) {
            for (int t = 0; t < h.iter; ++t) {
                if (rep_out->feas) rep_out->feas[t] = hr[(size_t)t * 4 + 0];
                if (rep_out->delta_l) rep_out->delta_l[t] = hr[(size_t)t * 4 + 1];
                if (rep_out->delta_s) rep_out->delta_s[t] = hr[(size_t)t * 4 + 2];
                if (rep_out->objective) rep_out->objective[t] = hr[(size_t)t * 4 + 3];
            }
            rep_out->iters = (uint64_t)h.iter;
            rep_out->converged = h.converged;
            rep_out->lambda = lambda;
            rep_out->slow_iters = slow_iters;
            rep_out->hartigan_moves = stats.hartigan_moves;
            rep_out->exact_fallbacks = stats.exact_fallbacks + h.exact_fallbacks;
            rep_out->stop_resolves = stop_resolves;
        }
    }

    // ---- bench: exactly `iters` more iterations, events around Pass F ----
    void bench_steps(uint64_t iters, double* ms, double* pf_ms, double* pa_ms, uint64_t* slow) {
        Ctl h = read_ctl();
        if ((uint64_t)h.iter + iters > budget) {
            // grow the report buffer (fixed-iteration benchmark semantics)
            budget = (uint64_t)h.iter + iters;
            DBuf<double> nr;
            nr.ensure(budget * 4);
            if (h.iter > 0)
                CK(cudaMemcpyAsync(nr.p, rep.p, sizeof(double) * 4 * h.iter,
                                   cudaMemcpyDeviceToDevice, st));
            std::swap(rep.p, nr.p);
            std::swap(rep.cap, nr.cap);
            DBuf<double> nm;
            nm.ensure(budget);
            if (h.iter > 0)
                CK(cudaMemcpyAsync(nm.p, marg.p, sizeof(double) * h.iter, cudaMemcpyDeviceToDevice, st));
            std::swap(marg.p, nm.p);
            std::swap(marg.cap, nm.cap);
            CK(cudaStreamSynchronize(st));  // the old buffers are freed below
            capture();
        }
        h.budget = (int)(h.iter + iters);
        h.fixed = 1;
        h.done = 0;
        h.converged = 0;
        write_ctl(h);
        std::vector<Events> evf(iters), eva(iters);
        Events all;
        uint64_t remaining = iters, nslow = 0;
        // RESPCA_PROFILE_TIMED=1: scope an `ncu --profile-from-start off` capture
        // to exactly the timed iterations
        const char* prof = std::getenv("RESPCA_PROFILE_TIMED");
        const bool profiling = prof && prof[0] == '1' && iters > 1;
        // RESPCA_BENCH_EAGER=1: every kernel of the iteration launched on the
        // stream (no graph), so launch tracers that do not see graph nodes list them
        const char* eg = std::getenv("RESPCA_BENCH_EAGER");
        const bool eager = eg && eg[0] == '1';
        if (profiling) CK(cudaProfilerStart());
        double fsum = 0.0, asum = 0.0;
        CK(cudaEventRecord(all.a, st));
        while (remaining > 0) {
            const uint64_t base = iters - remaining;
            for (uint64_t t = 0; t < remaining; ++t) {
                CK(cudaEventRecord(evf[base + t].a, st));
                launch_pass_f();
                CK(cudaEventRecord(evf[base + t].b, st));
                CK(cudaEventRecord(eva[base + t].a, st));
                if (eager) {
                    const uint64_t l0 = *ln.counter;
                    launch_pass_a();
                    launch_post();
                    launch_finalize(false);
                    *ln.counter = l0;
                } else {
                    rest.launch(st);
                }
                ln.add(kernels_per_iter() - 1);
                CK(cudaEventRecord(eva[base + t].b, st));
            }
            Ctl g = read_ctl();
            const uint64_t done_iters = (uint64_t)g.iter - (uint64_t)(h.budget - iters);
            if (g.slow) {
                ++nslow;
                ++slow_iters;
                slow_path(g);
            }
            if (g.nonfinite) throw NonFinite("solve: non-finite value inside the ALM loop");
            remaining = iters - std::min<uint64_t>(iters, done_iters);
            if (remaining > 0) {
                g = read_ctl();
                g.done = 0;
                write_ctl(g);
            }
        }
        CK(cudaEventRecord(all.b, st));
        CK(cudaEventSynchronize(all.b));
        if (profiling) CK(cudaProfilerStop());
        for (uint64_t t = 0; t < iters; ++t) {
            fsum += evf[t].ms();
            asum += eva[t].ms();
        }
        *ms = all.ms();
        if (pf_ms) *pf_ms = fsum;
        if (pa_ms) *pa_ms = asum;
        if (slow) *slow = nslow;
    }
};

// solve() with the input coming from `fill(X)` and the outputs going to
// `sinkL(L)`, `sinkS(S)` (host buffers or streamed files)
template <typename T, class Fill, class SinkL, class SinkS>
void solve_core(respca_cu_ctx* ctx, uint64_t d, uint64_t n, const respca_cu_config& cfg, Fill&& fill,
                SinkL&& sinkL, SinkS&& sinkS, uint64_t* lab, respca_cu_report* rep) {
    check_dims(d, n);
    validate_cfg(cfg);
    if (cfg.c > n) throw InvalidArg("solve: c exceeds column count");
    const auto t0 = Clock::now();
    auto& slot = ctx->solver[sizeof(T) == 8 ? 0 : 1];
    if (!slot) {
        auto* fresh = new Alm<T>(ctx, /*shared=*/true);
        fresh->use_arena = true;
        slot.reset(fresh);
    }
    Alm<T>& a = *static_cast<Alm<T>*>(slot.get());
    a.begin_solve();
    Nvtx r_solve("respca::solve");
    Events ev;
    CK(cudaEventRecord(ev.a, ctx->st));
    {
        Nvtx r("upload + validate");
        a.upload_with(d, n, cfg, fill);
    }
    CK(cudaEventRecord(ev.b, ctx->st));
    CK(cudaEventSynchronize(ev.b));
    const double h2d = ev.ms();
    Events e2;
    CK(cudaEventRecord(e2.a, ctx->st));
    {
        Nvtx r("initial kmeans(X)");
        a.setup_state();
        a.init_labels();
        a.launch_group_D();
    }
    CK(cudaEventRecord(e2.b, ctx->st));
    CK(cudaEventSynchronize(e2.b));
    const double init_ms = e2.ms();
    a.capture_if_needed();
    Events e3;
    CK(cudaEventRecord(e3.a, ctx->st));
    {
        Nvtx r("ALM loop");
        a.run_loop();
    }
    CK(cudaEventRecord(e3.b, ctx->st));
    CK(cudaEventSynchronize(e3.b));
    const double loop_ms = e3.ms();
    Events e4;
    CK(cudaEventRecord(e4.a, ctx->st));
    {
        Nvtx r("download");
        a.download_with(sinkL, sinkS, lab, rep);
    }
    CK(cudaEventRecord(e4.b, ctx->st));
    CK(cudaEventSynchronize(e4.b));
    if (rep) {
        rep->init_ms = init_ms;
        rep->loop_ms = loop_ms;
        rep->h2d_ms = h2d;
        rep->d2h_ms = e4.ms();
        rep->wall_time = std::chrono::duration<double>(Clock::now() - t0).count();
    }
    if (trace_on())
        std::fprintf(stderr, "[respca] solve: h2d %.1f ms, init %.1f ms, loop %.1f ms, d2h %.1f ms, host wall %.1f ms\n",
                     h2d, init_ms, loop_ms, e4.ms(), 1e3 * std::chrono::duration<double>(Clock::now() - t0).count());
}

template <typename T>
void solve_impl(respca_cu_ctx* ctx, const T* x, uint64_t d, uint64_t n,
                const respca_cu_config& cfg, T* Lo, T* So, uint64_t* lab,
                respca_cu_report* rep) {
    const size_t N = (size_t)(d * n);
    cudaStream_t st = ctx->st;
    // X in column chunks (multiples of the Gram tile), an event after each: the
    // initial clustering's Gram matrix starts on the first chunks while the rest
    // are still crossing the host link
    std::vector<cudaEvent_t> evs;
    struct EvGuard {
        std::vector<cudaEvent_t>& v;
        ~EvGuard() {
            for (cudaEvent_t e : v) cudaEventDestroy(e);
        }
    } evg{evs};
    solve_core<T>(
        ctx, d, n, cfg,
        [&](T* X) {
            Alm<T>& a = *static_cast<Alm<T>*>(ctx->solver[sizeof(T) == 8 ? 0 : 1].get());
            const int64_t blk = 128, nchunk = (n >= 8 * blk && cfg.c > 1) ? 8 : 1;
            const int64_t per = ((int64_t)n / nchunk + blk - 1) / blk * blk;
            for (int64_t j0 = 0; j0 < (int64_t)n; j0 += per) {
                const int64_t j1 = std::min<int64_t>(n, j0 + per);
                CK(cudaMemcpyAsync(X + (size_t)j0 * d, x + (size_t)j0 * d, sizeof(T) * (size_t)(j1 - j0) * d,
                                   cudaMemcpyHostToDevice, st));
                if (nchunk > 1) {
                    cudaEvent_t e;
                    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                    evs.push_back(e);
                    CK(cudaEventRecord(e, st));
                    a.chunk_events.emplace_back(j1, e);
                }
            }
        },
        [&](const T* L) { CK(cudaMemcpyAsync(Lo, L, sizeof(T) * N, cudaMemcpyDeviceToHost, st)); },
        [&](const T* S) { CK(cudaMemcpyAsync(So, S, sizeof(T) * N, cudaMemcpyDeviceToHost, st)); }, lab, rep);
}

// solve() between RESPCA1 files
template <typename T>
void solve_file_impl(respca_cu_ctx* ctx, const char* xp, const respca_cu_config& cfg, const char* lp,
                     const char* sp, uint64_t* lab, uint64_t lab_cap, respca_cu_report* rep) {
    BinReader r(xp);
    const uint64_t d = r.rows, n = r.cols;
    check_dims(d, n);
    if (lab_cap < n) throw InvalidArg("respca_cu_solve_file: labels capacity smaller than the column count");
    cudaStream_t st = ctx->st;
    solve_core<T>(
        ctx, d, n, cfg, [&](T* X) { r.to_device<T>(X, (int64_t)(d * n), st, ctx->io, &ctx->launches); },
        [&](const T* L) {
            if (lp) write_binary_from_device<T>(lp, L, d, n, st, ctx->io, &ctx->launches);
        },
        [&](const T* S) {
            if (sp) write_binary_from_device<T>(sp, S, d, n, st, ctx->io, &ctx->launches);
        },
        lab, rep);
}

template <class F>
int guarded(respca_cu_ctx* ctx, F&& f) {
    if (!ctx) return RESPCA_EINVAL;
    try {
        CK(cudaSetDevice(ctx->device));
        f();
        ctx->err.clear();
        return RESPCA_OK;
    } catch (const InvalidArg& e) {
        ctx->err = e.what();
        return RESPCA_EINVAL;
    } catch (const RuntimeErr& e) {
        ctx->err = e.what();
        return RESPCA_ERUNTIME;
    } catch (const NoMem& e) {
        ctx->err = e.what();
        return RESPCA_ENOMEM;
    } catch (const NonFinite& e) {
        ctx->err = e.what();
        return RESPCA_ENONFINITE;
    } catch (const IoErr& e) {
        ctx->err = e.what();
        return RESPCA_EIO;
    } catch (const std::exception& e) {
        ctx->err = e.what();
        return RESPCA_ECUDA;
    }
}

// ---------------------------------------------------------------------------
// building-block helpers (fp64, host in / host out)
// ---------------------------------------------------------------------------
struct Dev64 {
    DBuf<double> b;
    double* up(cudaStream_t st, const double* h, size_t count) {
        b.ensure(count);
        CK(cudaMemcpyAsync(b.p, h, sizeof(double) * count, cudaMemcpyHostToDevice, st));
        return b.p;
    }
};

double sum_partials(cudaStream_t st, Launch& ln, double* part, int blocks, int nv, int q,
                    DBuf<double>& scratch) {
    scratch.ensure(8);
    k_sum_partials<<<1, 256, 0, st>>>(part, blocks, nv, scratch.p);
    ln.add();
    double h[5];
    CK(cudaMemcpyAsync(h, scratch.p, sizeof(double) * nv, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return h[q];
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

void respca_cu_default_config(respca_cu_config* c) {
    std::memset(c, 0, sizeof(*c));
    c->rho0 = 1e-4;
    c->kappa = 1.5;
    c->tol = 1e-3;
    c->max_iter = 500;
    c->c = 1;
    c->sparse_norm = RESPCA_L1;
    c->km_max_iters = 100;
    c->km_n_restarts = 1;
    c->km_seed = 0;
    c->km_tol = 1e-6;
}

int respca_cu_create(int device, respca_cu_ctx** out) {
    if (!out) return RESPCA_EINVAL;
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count <= device || device < 0) {
        cudaGetLastError();
        return RESPCA_ECUDA;
    }
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major < 10) return RESPCA_ECUDA;
    auto* ctx = new respca_cu_ctx();
    ctx->device = device;
    if (cudaSetDevice(device) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->st, cudaStreamNonBlocking) != cudaSuccess) {
        delete ctx;
        return RESPCA_ECUDA;
    }
    *out = ctx;
    return RESPCA_OK;
}

void respca_cu_destroy(respca_cu_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    ctx->resident.reset();
    if (ctx->st) cudaStreamDestroy(ctx->st);
    delete ctx;
}

const char* respca_cu_last_error(const respca_cu_ctx* ctx) {
    return ctx ? ctx->err.c_str() : "null context";
}

uint64_t respca_cu_kernel_launches(const respca_cu_ctx* ctx) { return ctx ? ctx->launches : 0; }

int respca_cu_solve(respca_cu_ctx* ctx, const void* x, uint64_t d, uint64_t n, int dtype,
                    const respca_cu_config* cfg, void* L_out, void* S_out, uint64_t* labels_out,
                    respca_cu_report* rep) {
    return guarded(ctx, [&] {
        if (!x || !cfg || !L_out || !S_out || !labels_out) throw InvalidArg("respca_cu_solve: null pointer");
        if (cfg->sparse_norm != RESPCA_L1 && cfg->sparse_norm != RESPCA_L21)
            throw InvalidArg("respca_cu_solve: unknown sparse_norm");
        const auto tw0 = Clock::now();
        if (dtype == RESPCA_F64)
            solve_impl<double>(ctx, (const double*)x, d, n, *cfg, (double*)L_out, (double*)S_out,
                               labels_out, rep);
        else if (dtype == RESPCA_F32)
            solve_impl<float>(ctx, (const float*)x, d, n, *cfg, (float*)L_out, (float*)S_out,
                              labels_out, rep);
        else
            throw InvalidArg("respca_cu_solve: unknown dtype");
        if (trace_on())
            std::fprintf(stderr, "[respca] respca_cu_solve total %.1f ms (incl. teardown)\n",
                         1e3 * std::chrono::duration<double>(Clock::now() - tw0).count());
    });
}

int respca_cu_bench_prepare(respca_cu_ctx* ctx, const void* x, uint64_t d, uint64_t n, int dtype,
                            const respca_cu_config* cfg, double* init_ms) {
    return guarded(ctx, [&] {
        check_dims(d, n);
        ctx->resident.reset();
        if (dtype == RESPCA_F64) {
            auto a = std::make_unique<Alm<double>>(ctx);
            a->prepare((const double*)x, d, n, *cfg);
            if (init_ms) *init_ms = a->init_ms;
            ctx->resident = std::move(a);
        } else {
            auto a = std::make_unique<Alm<float>>(ctx);
            a->prepare((const float*)x, d, n, *cfg);
            if (init_ms) *init_ms = a->init_ms;
            ctx->resident = std::move(a);
        }
    });
}

int respca_cu_bench_steps(respca_cu_ctx* ctx, uint64_t iters, double* ms, double* pf_ms,
                          double* pa_ms, uint64_t* slow) {
    return guarded(ctx, [&] {
        if (!ctx->resident) throw InvalidArg("respca_cu_bench_steps: call respca_cu_bench_prepare first");
        if (auto* a = dynamic_cast<Alm<double>*>(ctx->resident.get()))
            a->bench_steps(iters, ms, pf_ms, pa_ms, slow);
        else if (auto* b = dynamic_cast<Alm<float>*>(ctx->resident.get()))
            b->bench_steps(iters, ms, pf_ms, pa_ms, slow);
    });
}

// ---- building blocks ------------------------------------------------------

int respca_cu_l_update(respca_cu_ctx* ctx, const double* D, uint64_t d, uint64_t n,
                       const uint64_t* labels, uint64_t c, double lambda, double rho,
                       double* L_out) {
    return guarded(ctx, [&] {  // solver.cpp:51-77
        check_dims(d, n);
        const std::vector<int> lab = to_int_labels(labels, n, c);
        if (rho <= 0.0) throw InvalidArg("l_update: rho must be > 0");
        if (lambda < 0.0) throw InvalidArg("l_update: lambda must be >= 0");
        cudaStream_t st = ctx->st;
        Launch ln{&ctx->launches};
        KMeansEngine<double> km;
        km.st = st;
        km.ln = ln;
        Dev64 dD;
        const double* Dd = dD.up(st, D, d * n);
        km.bind(Dd, d, (int)n, (int)c);
        km.h_labels = lab;
        DBuf<double> G, Lb;
        G.ensure(d * c);
        Lb.ensure(d * n);
        // group sums of D in the reference order, then the blend
        km.groups.build(lab.data(), (int)n, (int)c);
        km.upload_groups();
        const bool r2 = d % 2 == 0;
        const int rb = ceil_div(d, 256 * (r2 ? 2 : 1));
        if (r2)
            k_group_sum<double, 2, 1><<<rb * (int)c, 256, 0, st>>>(
                Dd, nullptr, nullptr, km.goff.p, km.members.p, nullptr, G.p, nullptr, 0, 0, d, rb);
        else
            k_group_sum<double, 1, 1><<<rb * (int)c, 256, 0, st>>>(
                Dd, nullptr, nullptr, km.goff.p, km.members.p, nullptr, G.p, nullptr, 0, 0, d, rb);
        const double own_w = rho / (2.0 * lambda + rho);
        if (r2)
            k_l_blend<2><<<rb * (int)c, 256, 0, st>>>(Dd, Lb.p, km.goff.p, km.members.p, G.p, own_w,
                                                      lambda, rho, d, rb);
        else
            k_l_blend<1><<<rb * (int)c, 256, 0, st>>>(Dd, Lb.p, km.goff.p, km.members.p, G.p, own_w,
                                                      lambda, rho, d, rb);
        ln.add(2);
        CK(cudaMemcpyAsync(L_out, Lb.p, sizeof(double) * d * n, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    });
}

int respca_cu_s_update_l1(respca_cu_ctx* ctx, const double* B, uint64_t d, uint64_t n,
                          double thr, double* S_out) {
    return guarded(ctx, [&] {  // solver.cpp:79-88
        check_dims(d, n);
        if (thr < 0.0) throw InvalidArg("s_update_l1: negative threshold");
        cudaStream_t st = ctx->st;
        Dev64 db;
        double* p = db.up(st, B, d * n);
        k_shrink_l1<<<std::min<int64_t>(4096, ceil_div(d * n, 256)), 256, 0, st>>>(p, p, d * n, thr);
        ctx->launches++;
        CK(cudaMemcpyAsync(S_out, p, sizeof(double) * d * n, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    });
}

int respca_cu_s_update_l21(respca_cu_ctx* ctx, const double* B, uint64_t d, uint64_t n,
                           double thr, double* S_out) {
    return guarded(ctx, [&] {  // solver.cpp:90-102
        check_dims(d, n);
        if (thr < 0.0) throw InvalidArg("s_update_l21: negative threshold");
        cudaStream_t st = ctx->st;
        Dev64 db;
        double* p = db.up(st, B, d * n);
        DBuf<double> nr, so;
        nr.ensure(n);
        so.ensure(d * n);
        k_col_sumsq<double, 0><<<ceil_div(n, 128), 128, 0, st>>>(p, nullptr, nullptr, 1.0, d, n, nr.p);
        k_shrink_l21<double, 0><<<std::min<int64_t>(4096, ceil_div(d * n, 256)), 256, 0, st>>>(
            p, nullptr, nullptr, 1.0, nr.p, so.p, d, n, thr);
        ctx->launches += 2;
        CK(cudaMemcpyAsync(S_out, so.p, sizeof(double) * d * n, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    });
}

int respca_cu_multiplier_update(respca_cu_ctx* ctx, double* theta, const double* x,
                                const double* L, const double* S, uint64_t d, uint64_t n,
                                double* rho, double kappa) {
    return guarded(ctx, [&] {  // solver.cpp:104-111
        check_dims(d, n);
        if (kappa <= 1.0) throw InvalidArg("multiplier_update: kappa must be > 1");
        cudaStream_t st = ctx->st;
        Dev64 a, b, c2, e;
        double* th = a.up(st, theta, d * n);
        const double* xd = b.up(st, x, d * n);
        const double* ld_ = c2.up(st, L, d * n);
        const double* sd = e.up(st, S, d * n);
        k_multiplier<<<std::min<int64_t>(4096, ceil_div(d * n, 256)), 256, 0, st>>>(th, xd, ld_, sd,
                                                                                  d * n, *rho);
        ctx->launches++;
        CK(cudaMemcpyAsync(theta, th, sizeof(double) * d * n, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const double nr = *rho * kappa;
        *rho = (1e12 < nr) ? 1e12 : nr;
    });
}

int respca_cu_check_convergence(respca_cu_ctx* ctx, const double* x, const double* l_prev,
                                const double* l, const double* s_prev, const double* s,
                                uint64_t d, uint64_t n, double tol, int* conv, double* feas,
                                double* dl, double* ds) {
    return guarded(ctx, [&] {  // solver.cpp:113-125
        check_dims(d, n);
        cudaStream_t st = ctx->st;
        Launch ln{&ctx->launches};
        Dev64 a, b, c2, e, f;
        const double* xd = a.up(st, x, d * n);
        const double* lpd = b.up(st, l_prev, d * n);
        const double* ldd = c2.up(st, l, d * n);
        const double* spd = e.up(st, s_prev, d * n);
        const double* sd = f.up(st, s, d * n);
        const int blocks = std::min<int64_t>(2048, ceil_div(d * n, 256));
        DBuf<double> part, scr;
        part.ensure(3 * blocks);
        k_norms<double><<<blocks, 256, 0, st>>>(xd, d * n, part.p);
        ln.add();
        const double xn = std::sqrt(sum_partials(st, ln, part.p, blocks, 3, 0, scr));
        if (xn == 0.0) throw InvalidArg("check_convergence: all-zero X");
        k_triple<<<blocks, 256, 0, st>>>(xd, lpd, ldd, spd, sd, d * n, part.p);
        ln.add();
        double h[3];
        scr.ensure(8);
        k_sum_partials<<<1, 256, 0, st>>>(part.p, blocks, 3, scr.p);
        ln.add();
        CK(cudaMemcpyAsync(h, scr.p, sizeof(h), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        *feas = std::sqrt(h[0]) / xn;
        *dl = std::sqrt(h[1]) / xn;
        *ds = std::sqrt(h[2]) / xn;
        double mx = *feas;
        if (mx < *dl) mx = *dl;
        if (mx < *ds) mx = *ds;
        *conv = mx <= tol;
    });
}

static void km_common(respca_cu_ctx* ctx, KMeansEngine<double>& km, Dev64& dm, const double* m,
                      uint64_t d, uint64_t n, uint64_t c) {
    km.st = ctx->st;
    km.ln = Launch{&ctx->launches};
    const double* md = dm.up(ctx->st, m, d * n);
    km.bind(md, d, (int)n, (int)c);
}

int respca_cu_kmeans(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n, uint64_t c,
                     uint64_t max_iters, uint64_t n_restarts, uint64_t seed, double tol,
                     uint64_t* labels_out, double* centroids_out, double* inertia,
                     uint64_t* iters_run) {
    return guarded(ctx, [&] {  // kmeans.cpp:237-250
        check_dims(d, n);
        if (c == 0) throw InvalidArg("kmeans: c must be >= 1");
        if (c > n) throw InvalidArg("kmeans: c exceeds column count");
        KMeansEngine<double> km;
        Dev64 dm;
        km_common(ctx, km, dm, m, d, n, c);
        DBuf<int> lab;
        DBuf<double> cen;
        lab.ensure(n);
        cen.ensure(d * c);
        double in = 0.0;
        uint64_t it = 0;
        km.kmeans(max_iters, n_restarts, seed, tol, lab.p, cen.p, &in, &it);
        std::vector<int> hl(n);
        CK(cudaMemcpyAsync(hl.data(), lab.p, sizeof(int) * n, cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaMemcpyAsync(centroids_out, cen.p, sizeof(double) * d * c, cudaMemcpyDeviceToHost,
                           ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
        for (uint64_t j = 0; j < n; ++j) labels_out[j] = (uint64_t)hl[j];
        *inertia = in;
        *iters_run = it;
    });
}

int respca_cu_kmeans_warm(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n,
                          uint64_t c, uint64_t max_iters, double tol,
                          const uint64_t* init_labels, uint64_t* labels_out,
                          double* centroids_out, double* inertia, uint64_t* iters_run) {
    return guarded(ctx, [&] {  // kmeans.cpp:252-258
        check_dims(d, n);
        const std::vector<int> lab = to_int_labels(init_labels, n, c);
        KMeansEngine<double> km;
        Dev64 dm;
        km_common(ctx, km, dm, m, d, n, c);
        DBuf<int> dl;
        DBuf<double> cen;
        dl.ensure(n);
        cen.ensure(d * c);
        km.h_labels = lab;
        km.means(cen.p);  // means_of(m, init)
        const uint64_t it = km.lloyd_run(cen.p, dl.p, max_iters, tol);
        *inertia = km.inertia(cen.p, dl.p);
        std::vector<int> hl(n);
        CK(cudaMemcpyAsync(hl.data(), dl.p, sizeof(int) * n, cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaMemcpyAsync(centroids_out, cen.p, sizeof(double) * d * c, cudaMemcpyDeviceToHost,
                           ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
        for (uint64_t j = 0; j < n; ++j) labels_out[j] = (uint64_t)hl[j];
        *iters_run = it;
    });
}

int respca_cu_kmeans_pp_init(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n,
                             uint64_t c, uint64_t seed, double* centroids_out) {
    return guarded(ctx, [&] {  // kmeans.cpp:172-224
        check_dims(d, n);
        if (c == 0) throw InvalidArg("kmeans_pp_init: c must be >= 1");
        if (c > n) throw InvalidArg("kmeans_pp_init: c exceeds column count");
        KMeansEngine<double> km;
        Dev64 dm;
        km_common(ctx, km, dm, m, d, n, c);
        std::mt19937_64 rng(seed);
        const std::vector<int> ch = km.pp_init(rng);
        DBuf<double> cen;
        cen.ensure(d * c);
        km.gather(ch, cen.p);
        CK(cudaMemcpyAsync(centroids_out, cen.p, sizeof(double) * d * c, cudaMemcpyDeviceToHost,
                           ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
    });
}

int respca_cu_kmeans_pp_init_cb(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n,
                                uint64_t c, uint64_t (*draw_first)(void*, uint64_t),
                                double (*draw_real)(void*, double), void* user,
                                double* centroids_out) {
    return guarded(ctx, [&] {  // kmeans.cpp:172-224 with the caller's engine
        check_dims(d, n);
        if (!draw_first || !draw_real) throw InvalidArg("kmeans_pp_init: null draw callback");
        if (c == 0) throw InvalidArg("kmeans_pp_init: c must be >= 1");
        if (c > n) throw InvalidArg("kmeans_pp_init: c exceeds column count");
        KMeansEngine<double> km;
        Dev64 dm;
        km_common(ctx, km, dm, m, d, n, c);
        const std::vector<int> ch = km.pp_init_with(
            [&](uint64_t nn) { return draw_first(user, nn); },
            [&](double total) { return draw_real(user, total); });
        DBuf<double> cen;
        cen.ensure(d * c);
        km.gather(ch, cen.p);
        CK(cudaMemcpyAsync(centroids_out, cen.p, sizeof(double) * d * c, cudaMemcpyDeviceToHost,
                           ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
    });
}

int respca_cu_lloyd_step(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n,
                         const double* centroids, uint64_t c, uint64_t* labels_out,
                         double* next_out) {
    return guarded(ctx, [&] {  // kmeans.cpp:226-235
        check_dims(d, n);
        if (c == 0) throw InvalidArg("lloyd_step: bad centroid matrix");
        KMeansEngine<double> km;
        Dev64 dm, dc;
        km_common(ctx, km, dm, m, d, n, c);
        const double* C = dc.up(ctx->st, centroids, d * c);
        DBuf<int> lab;
        DBuf<double> nx;
        lab.ensure(n);
        nx.ensure(d * c);
        km.assign(C, lab.p);
        km.fetch_labels(lab.p);
        km.repair_if_needed(C, lab.p);
        km.means(nx.p);
        CK(cudaMemcpyAsync(next_out, nx.p, sizeof(double) * d * c, cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
        for (uint64_t j = 0; j < n; ++j) labels_out[j] = (uint64_t)km.h_labels[j];
    });
}

int respca_cu_group_scatter(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n,
                            const uint64_t* labels, uint64_t c, double* out) {
    return guarded(ctx, [&] {  // matrix.cpp:81-97
        check_dims(d, n);
        const std::vector<int> lab = to_int_labels(labels, n, c);
        KMeansEngine<double> km;
        Dev64 dm;
        km_common(ctx, km, dm, m, d, n, c);
        km.h_labels = lab;
        DBuf<double> cen;
        DBuf<int> dl;
        cen.ensure(d * c);
        dl.ensure(n);
        CK(cudaMemcpyAsync(dl.p, lab.data(), sizeof(int) * n, cudaMemcpyHostToDevice, ctx->st));
        km.means(cen.p);  // column_mean per group, matrix.cpp:63-79
        // per-group sequential sums in the reference's order: groups, then members
        smem_at_least((const void*)k_own_exact<double>, own_exact_smem<double>());
        k_own_exact<double><<<ceil_div(n, 32 * OWN_W), 32 * OWN_W, own_exact_smem<double>(), ctx->st>>>(
            km.M, cen.p, d, (int)n, dl.p, km.own.p);
        ctx->launches++;
        std::vector<double> own(n);
        CK(cudaMemcpyAsync(own.data(), km.own.p, sizeof(double) * n, cudaMemcpyDeviceToHost,
                           ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
        // report-grade total (tolerance, not bitwise: the reference's single chain
        // interleaves all groups' element terms)
        double total = 0.0;
        for (int k = 0; k < (int)c; ++k)
            for (int t = km.groups.goff[k]; t < km.groups.goff[k + 1]; ++t)
                total += own[km.groups.members[t]];
        *out = total;
    });
}

static double norm_kernel(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n, int q) {
    cudaStream_t st = ctx->st;
    Launch ln{&ctx->launches};
    Dev64 dm;
    const double* p = dm.up(st, m, d * n);
    const int blocks = std::min<int64_t>(2048, ceil_div(d * n, 256));
    DBuf<double> part, scr;
    part.ensure(3 * blocks);
    k_norms<double><<<blocks, 256, 0, st>>>(p, d * n, part.p);
    ln.add();
    return sum_partials(st, ln, part.p, blocks, 3, q, scr);
}

int respca_cu_frob_norm(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n,
                        double* out) {
    return guarded(ctx, [&] {  // matrix.cpp:99-103
        check_dims(d, n);
        *out = std::sqrt(norm_kernel(ctx, m, d, n, 0));
    });
}

int respca_cu_elementwise_l1(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n,
                             double* out) {
    return guarded(ctx, [&] {  // matrix.cpp:105-109
        check_dims(d, n);
        *out = norm_kernel(ctx, m, d, n, 1);
    });
}

int respca_cu_column_l2_norms(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n,
                              double* out) {
    return guarded(ctx, [&] {  // matrix.cpp:117-125 (exact sequential per column)
        check_dims(d, n);
        cudaStream_t st = ctx->st;
        Dev64 dm;
        const double* p = dm.up(st, m, d * n);
        DBuf<double> nr;
        nr.ensure(n);
        k_col_sumsq<double, 0><<<ceil_div(n, 128), 128, 0, st>>>(p, nullptr, nullptr, 1.0, d, n, nr.p);
        ctx->launches++;
        CK(cudaMemcpyAsync(out, nr.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    });
}

int respca_cu_l21_norm(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n, double* out) {
    return guarded(ctx, [&] {  // matrix.cpp:111-115
        check_dims(d, n);
        std::vector<double> nr(n);
        cudaStream_t st = ctx->st;
        Dev64 dm;
        const double* p = dm.up(st, m, d * n);
        DBuf<double> dn;
        dn.ensure(n);
        k_col_sumsq<double, 0><<<ceil_div(n, 128), 128, 0, st>>>(p, nullptr, nullptr, 1.0, d, n, dn.p);
        ctx->launches++;
        CK(cudaMemcpyAsync(nr.data(), dn.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        double s = 0.0;
        for (uint64_t j = 0; j < n; ++j) s += nr[j];
        *out = s;
    });
}

int respca_cu_debug_screen(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n,
                           const double* centroids, uint64_t c, double* approx_out,
                           double* err_out) {
    return guarded(ctx, [&] {  // test hook: the screened distance and its bound
        check_dims(d, n);
        KMeansEngine<double> km;
        Dev64 dm, dc;
        km_common(ctx, km, dm, m, d, n, c);
        const double* C = dc.up(ctx->st, centroids, d * c);
        km.screen(C);
        DBuf<double> a, e;
        a.ensure(n * c);
        e.ensure(n * c);
        k_screen_dump<<<ceil_div((int64_t)n * c, 256), 256, 0, ctx->st>>>(km.screen_view(), (int)n,
                                                                          (int)c, a.p, e.p);
        ctx->launches++;
        CK(cudaMemcpyAsync(approx_out, a.p, sizeof(double) * n * c, cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaMemcpyAsync(err_out, e.p, sizeof(double) * n * c, cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
    });
}

int respca_cu_last_margins(const respca_cu_ctx* ctx, respca_cu_margins* out) {
    if (!ctx || !out) return RESPCA_EINVAL;
    *out = ctx->margins;
    return RESPCA_OK;
}

int respca_cu_debug_guards(char* msg, uint64_t cap) {
    if (!guard_on()) return -1;
    std::string m;
    const int bad = guard_check(&m);
    if (msg && cap) {
        std::strncpy(msg, m.c_str(), (size_t)cap - 1);
        msg[cap - 1] = 0;
    }
    return bad;
}

int respca_cu_debug_screen_tc(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n,
                              const double* centroids, uint64_t c, double* approx_out,
                              double* err_out) {
    return guarded(ctx, [&] {  // test hook: the tcgen05 BF16 screen and its bound
        check_dims(d, n);
        if (c > (uint64_t)TC_N) throw InvalidArg("debug_screen_tc: c > 64");
        KMeansEngine<double> km;
        Dev64 dm, dc;
        km_common(ctx, km, dm, m, d, n, c);
        const double* C = dc.up(ctx->st, centroids, d * c);
        km.screen_tc(C);
        DBuf<double> a, e;
        a.ensure(n * c);
        e.ensure(n * c);
        k_screen_dump<<<ceil_div((int64_t)n * c, 256), 256, 0, ctx->st>>>(km.screen_view(), (int)n,
                                                                          (int)c, a.p, e.p);
        ctx->launches++;
        int errv = 0;
        CK(cudaMemcpyAsync(&errv, km.tcerr.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaMemcpyAsync(approx_out, a.p, sizeof(double) * n * c, cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaMemcpyAsync(err_out, e.p, sizeof(double) * n * c, cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
        if (errv) throw CudaErr("tcgen05 screen pipeline timed out (code " + std::to_string(errv) + ")");
    });
}

int respca_cu_column_mean(respca_cu_ctx* ctx, const double* m, uint64_t d, uint64_t n,
                          const uint64_t* cols, uint64_t ncols, double* out) {
    return guarded(ctx, [&] {  // matrix.cpp:63-79
        check_dims(d, n);
        if (ncols == 0) throw InvalidArg("column_mean: empty column set");
        for (uint64_t t = 0; t < ncols; ++t)
            if (cols[t] >= n) throw InvalidArg("column_mean: column index out of range");
        // one group whose member list is `cols` in the given order
        KMeansEngine<double> km;
        Dev64 dm;
        km_common(ctx, km, dm, m, d, n, 1);
        km.groups.goff = {0, (int)ncols};
        km.groups.members.assign(cols, cols + ncols);
        km.groups.counts = {(int)ncols};
        km.members.ensure(ncols);
        CK(cudaMemcpyAsync(km.goff.p, km.groups.goff.data(), sizeof(int) * 2, cudaMemcpyHostToDevice,
                           ctx->st));
        CK(cudaMemcpyAsync(km.members.p, km.groups.members.data(), sizeof(int) * ncols,
                           cudaMemcpyHostToDevice, ctx->st));
        DBuf<double> o;
        o.ensure(d);
        km.launch_group_mean(o.p);
        CK(cudaMemcpyAsync(out, o.p, sizeof(double) * d, cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
    });
}

int respca_cu_binary_info(const char* path, uint64_t* rows, uint64_t* cols, char* err, size_t err_len) {
    try {
        if (!path || !rows || !cols) throw InvalidArg("respca_cu_binary_info: null pointer");
        BinReader r(path);
        *rows = r.rows;
        *cols = r.cols;
        if (err && err_len) err[0] = 0;
        return RESPCA_OK;
    } catch (const std::exception& e) {
        if (err && err_len) {
            std::strncpy(err, e.what(), err_len - 1);
            err[err_len - 1] = 0;
        }
        return dynamic_cast<const IoErr*>(&e) ? RESPCA_EIO : RESPCA_EINVAL;
    }
}

int respca_cu_solve_file(respca_cu_ctx* ctx, const char* x_path, int dtype, const respca_cu_config* cfg,
                         const char* l_path, const char* s_path, uint64_t* labels_out, uint64_t labels_cap,
                         respca_cu_report* rep) {
    return guarded(ctx, [&] {
        if (!x_path || !cfg || !labels_out) throw InvalidArg("respca_cu_solve_file: null pointer");
        if (cfg->sparse_norm != RESPCA_L1 && cfg->sparse_norm != RESPCA_L21)
            throw InvalidArg("respca_cu_solve_file: unknown sparse_norm");
        if (dtype == RESPCA_F64)
            solve_file_impl<double>(ctx, x_path, *cfg, l_path, s_path, labels_out, labels_cap, rep);
        else if (dtype == RESPCA_F32)
            solve_file_impl<float>(ctx, x_path, *cfg, l_path, s_path, labels_out, labels_cap, rep);
        else
            throw InvalidArg("respca_cu_solve_file: unknown dtype");
    });
}

int respca_cu_outlier_scores(respca_cu_ctx* ctx, const double* s, uint64_t d, uint64_t n, double threshold,
                             double* scores, uint64_t* flagged, uint64_t* n_flagged) {
    return guarded(ctx, [&] {  // io.cpp:296-306
        if (!s || !scores) throw InvalidArg("respca_cu_outlier_scores: null pointer");
        if (threshold < 0.0) throw InvalidArg("outlier_scores: negative threshold");
        check_dims(d, n);
        cudaStream_t st = ctx->st;
        Dev64 dm;
        const double* p = dm.up(st, s, d * n);
        DBuf<double> nr;
        nr.ensure(n);
        k_col_sumsq<double, 0><<<ceil_div(n, 128), 128, 0, st>>>(p, nullptr, nullptr, 1.0, d, n, nr.p);
        ctx->launches++;
        CK(cudaMemcpyAsync(scores, nr.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        uint64_t m = 0;
        for (uint64_t j = 0; j < n; ++j)
            if (scores[j] >= threshold) {
                if (flagged) flagged[m] = j;
                ++m;
            }
        if (n_flagged) *n_flagged = m;
    });
}

int respca_cu_synth_rpca(respca_cu_ctx* ctx, uint64_t d, uint64_t n, uint64_t r, double sigma, double p,
                         double lo, double hi, uint64_t seed, int dtype, void* X_out) {
    return guarded(ctx, [&] {  // csrc/synth.c rpca, assembled on the device
        check_dims(d, n);
        if (!X_out) throw InvalidArg("respca_cu_synth_rpca: null pointer");
        if (r == 0) throw InvalidArg("respca_cu_synth_rpca: r must be >= 1");
        if (dtype != RESPCA_F64 && dtype != RESPCA_F32) throw InvalidArg("respca_cu_synth_rpca: unknown dtype");
        if (n > 65535 * 65535ULL) throw InvalidArg("respca_cu_synth_rpca: too many columns");
        synth_rpca_spec sp{d, n, r, sigma, p, lo, hi, seed};
        std::vector<double> U(d * r), V(n * r);
        if (synth_rpca_factors(&sp, U.data(), V.data()) != 0) throw InvalidArg("synth_rpca: bad spec");
        uint64_t ks = 0, kval = 0;
        synth_rpca_keys(&sp, &ks, &kval);
        cudaStream_t st = ctx->st;
        DBuf<double> du, dv;
        du.ensure(d * r);
        dv.ensure(n * r);
        CK(cudaMemcpyAsync(du.p, U.data(), sizeof(double) * d * r, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(dv.p, V.data(), sizeof(double) * n * r, cudaMemcpyHostToDevice, st));
        const size_t es = dtype == RESPCA_F64 ? 8 : 4;
        void* dx = ctx->arena.get("X", es * d * n);  // a later solve overwrites it anyway
        const dim3 grid(ceil_div(d, 256), 1, 1);
        for (uint64_t j0 = 0; j0 < n; j0 += 65535) {  // grid.y ≤ 65535 columns per launch
            const uint64_t nj = std::min<uint64_t>(65535, n - j0);
            const double* vp = dv.p + j0 * r;
            if (dtype == RESPCA_F64)
                k_synth_rpca<double><<<dim3(grid.x, (unsigned)nj), 256, sizeof(double) * r, st>>>(
                    du.p, vp, (int64_t)d, (int)r, p, lo, hi - lo, ks, kval, (int64_t)j0, (double*)dx + j0 * d);
            else
                k_synth_rpca<float><<<dim3(grid.x, (unsigned)nj), 256, sizeof(double) * r, st>>>(
                    du.p, vp, (int64_t)d, (int)r, p, lo, hi - lo, ks, kval, (int64_t)j0, (float*)dx + j0 * d);
            ctx->launches++;
        }
        CK(cudaMemcpyAsync(X_out, dx, es * d * n, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    });
}

int respca_cu_synth_generate(respca_cu_ctx* ctx, uint64_t d, uint64_t n, uint64_t c, double sparsity,
                             double magnitude, double noise_sigma, uint64_t seed, double* X_out, double* L0_out,
                             double* S0_out, uint64_t* labels_out) {
    return guarded(ctx, [&] {  // io::synth_generate (io.cpp:232-294)
        if (d == 0 || n == 0) throw InvalidArg("synth_generate: dimensions must be >= 1");
        if (c == 0 || c > n) throw InvalidArg("synth_generate: need 1 <= c <= n");
        if (!(sparsity >= 0.0) || sparsity >= 1.0) throw InvalidArg("synth_generate: sparsity must be in [0,1)");
        check_dims(d, n);
        if (n > 65535ULL) throw InvalidArg("synth_generate: too many columns for one launch");
        const uint64_t N = d * n;
        std::mt19937_64 rng(seed);
        std::uniform_real_distribution<double> unit(0.0, 1.0);
        const uint64_t base = n / c, rem = n % c;
        if (labels_out) {
            uint64_t col = 0;
            for (uint64_t g = 0; g < c; ++g)
                for (uint64_t k = 0; k < base + (g < rem ? 1 : 0); ++k) labels_out[col++] = g;
        }
        std::vector<double> proto(c * d);  // group after group, row after row (io.cpp:253-256)
        for (double& v : proto) v = unit(rng);
        // partial Fisher–Yates over positions 0..N-1 (io.cpp:267-273): only the
        // entries a swap has touched are stored
        const uint64_t nnz = (uint64_t)std::llround(sparsity * (double)N);
        std::vector<uint64_t> pos(nnz);
        std::vector<double> val(nnz);
        {
            std::unordered_map<uint64_t, uint64_t> moved;
            moved.reserve((size_t)(2 * nnz + 16));
            auto at = [&](uint64_t k) {
                auto it = moved.find(k);
                return it == moved.end() ? k : it->second;
            };
            std::uniform_real_distribution<double> mag(magnitude / 2.0, magnitude);
            for (uint64_t k = 0; k < nnz; ++k) {
                std::uniform_int_distribution<std::size_t> pick((std::size_t)k, (std::size_t)(N - 1));
                const uint64_t q = (uint64_t)pick(rng);
                const uint64_t vk = at(k), vq = at(q);
                moved[k] = vq;
                moved[q] = vk;
                const double sign = unit(rng) < 0.5 ? -1.0 : 1.0;
                pos[k] = vq;
                val[k] = sign * mag(rng);
            }
        }
        cudaStream_t st = ctx->st;
        DBuf<double> dproto, dval, dz;
        DBuf<uint64_t> dpos;
        dproto.ensure(c * d);
        CK(cudaMemcpyAsync(dproto.p, proto.data(), sizeof(double) * c * d, cudaMemcpyHostToDevice, st));
        double* dX = static_cast<double*>(ctx->arena.get("X", sizeof(double) * N));
        double* dL = static_cast<double*>(ctx->arena.get("L", sizeof(double) * N));
        double* dS = static_cast<double*>(ctx->arena.get("S", sizeof(double) * N));
        k_sg_fill<<<dim3((unsigned)std::min<uint64_t>(ceil_div(d, 256), 64), (unsigned)n), 256, 0, st>>>(
            dproto.p, d, n, base, rem, dL, dS);
        ctx->launches++;
        if (nnz) {
            dpos.ensure(nnz);
            dval.ensure(nnz);
            CK(cudaMemcpyAsync(dpos.p, pos.data(), sizeof(uint64_t) * nnz, cudaMemcpyHostToDevice, st));
            CK(cudaMemcpyAsync(dval.p, val.data(), sizeof(double) * nnz, cudaMemcpyHostToDevice, st));
            k_sg_scatter<<<(unsigned)ceil_div(nnz, 256), 256, 0, st>>>(dpos.p, dval.p, nnz, dS);
            ctx->launches++;
        }
        const unsigned gb = (unsigned)std::min<uint64_t>(ceil_div(N, 256), 148 * 16);
        k_sg_sum<<<gb, 256, 0, st>>>(dL, dS, N, dX);
        ctx->launches++;
        if (noise_sigma > 0.0) {  // io.cpp:279-282: one normal draw per element, in storage order
            std::normal_distribution<double> noise(0.0, noise_sigma);
            const uint64_t CH = 1ULL << 22;
            std::vector<double> z(std::min(CH, N));
            dz.ensure(z.size());
            for (uint64_t e0 = 0; e0 < N; e0 += CH) {
                const uint64_t cnt = std::min(CH, N - e0);
                for (uint64_t e = 0; e < cnt; ++e) z[e] = noise(rng);
                CK(cudaMemcpyAsync(dz.p, z.data(), sizeof(double) * cnt, cudaMemcpyHostToDevice, st));
                k_sg_noise<<<(unsigned)std::min<uint64_t>(ceil_div(cnt, 256), 148 * 16), 256, 0, st>>>(dz.p, cnt,
                                                                                                      dX + e0);
                ctx->launches++;
                CK(cudaStreamSynchronize(st));  // z is reused by the next chunk
            }
        }
        if (X_out) CK(cudaMemcpyAsync(X_out, dX, sizeof(double) * N, cudaMemcpyDeviceToHost, st));
        if (L0_out) CK(cudaMemcpyAsync(L0_out, dL, sizeof(double) * N, cudaMemcpyDeviceToHost, st));
        if (S0_out) CK(cudaMemcpyAsync(S0_out, dS, sizeof(double) * N, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    });
}

}  // extern "C"
