// Device K-means engine: kmeans / kmeans_warm / lloyd_run / hartigan_refine /
// kmeans_pp_init (reference kmeans.cpp) with bit-identical labels.
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <memory>
#include <mutex>
#include <random>
#include <thread>
#include <vector>

#include "alm.cuh"
#include "engine.cuh"
#include "km.cuh"
#include "hartigan.cuh"
#include "hart_gram.cuh"
#include "tc_screen.cuh"

namespace respca_host {

using namespace respca_dev;

struct Launch {
    uint64_t* counter;
    void add(uint64_t k = 1) { *counter += k; }
};

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// host counting sort → CSR member lists in ascending column order
// (GroupAssignment::group_indices, matrix.cpp:49-55)
struct Groups {
    std::vector<int> goff, members, counts;
    void build(const int* labels, int n, int c) {
        goff.assign(c + 1, 0);
        counts.assign(c, 0);
        for (int j = 0; j < n; ++j) counts[labels[j]]++;
        for (int k = 0; k < c; ++k) goff[k + 1] = goff[k] + counts[k];
        members.resize(n);
        std::vector<int> fill(goff.begin(), goff.end() - 1);
        for (int j = 0; j < n; ++j) members[fill[labels[j]]++] = j;
    }
};

struct Stats {
    uint64_t hartigan_moves = 0, exact_fallbacks = 0, lloyd_steps = 0, hartigan_passes = 0;
    uint64_t hartigan_rounds = 0, hartigan_refreshes = 0, pp_respeculated = 0;
    double t_pp = 0, t_lloyd = 0, t_hart = 0, t_inertia = 0;  // seconds (host clock, synced)
    double t_hart_kernel = 0;  // device span of the Hartigan round kernels
};

inline bool trace_on() {
    static const bool on = [] {
        const char* e = std::getenv("RESPCA_TRACE");
        return e && e[0] == '1';
    }();
    return on;
}
using HClock = std::chrono::steady_clock;
inline double since(HClock::time_point t) {
    return std::chrono::duration<double>(HClock::now() - t).count();
}

template <typename T>
struct KmLane;
// restart lanes kept by a context across solves (streams + buffers)
template <typename T>
struct LanePool : PoolBase {
    std::vector<std::unique_ptr<KmLane<T>>> lanes;
};

// cudaFuncSetAttribute only when a kernel needs more dynamic shared memory
// than already granted: the call is not free while other streams run kernels
// (restart lanes launch side by side), so each function is raised once.
inline void smem_at_least(const void* f, size_t bytes) {
    static std::mutex mu;
    static std::vector<std::pair<const void*, size_t>> granted;
    std::lock_guard<std::mutex> g(mu);
    for (auto& e : granted)
        if (e.first == f) {
            if (e.second >= bytes) return;
            CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
            e.second = bytes;
            return;
        }
    CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    granted.emplace_back(f, bytes);
}

template <typename T>
struct KMeansEngine {
    cudaStream_t st = nullptr;
    LanePool<T>* lane_pool = nullptr;  // context-owned lanes (nullptr: per call)
    // the tcgen05 B operand copy lives with the engine; a tensor map keyed on
    // (pointer, n, dpad) is rebuilt when any of them changes
    Launch ln{nullptr};
    Stats* stats = nullptr;
    const T* M = nullptr;
    int64_t d = 0;
    int n = 0, c = 0;
    int nsplit = 1;
    // buffers
    DBuf<double> part, xxp, cc, nextC, exact, own, msp, approx, err, d2, xx, scratch;
    DBuf<int> newlab, amb, counts, goff, members, modver, stamp, gidx, errflag;
    DBuf<Ctl> kctl;
    HBuf hst;
    Groups groups;
    std::vector<int> h_labels;

    void bind(const T* m, int64_t dd, int nn, int cc_) {
        M = m;
        d = dd;
        n = nn;
        c = cc_;
        // split-K for the screen: aim for >= 2 CTAs per SM
        const int tiles = ceil_div(n, tile_j()) * ceil_div(c, tile_k());
        const int chunks = ceil_div(d, 32);
        nsplit = std::max(1, std::min(chunks / 4, ceil_div(2 * 148, tiles)));
        nsplit = std::min(nsplit, 32);
        part.ensure((size_t)nsplit * n * c);
        xxp.ensure((size_t)nsplit * n);
        cc.ensure(c);
        nextC.ensure((size_t)d * c);
        exact.ensure((size_t)n * c);
        own.ensure(n);
        msp.ensure(2 * 512 + 2);
        newlab.ensure(n);
        amb.ensure(n);
        counts.ensure(c);
        goff.ensure(c + 1);
        members.ensure(n);
        kctl.ensure(1);
        errflag.ensure(1);
        scratch.ensure(std::max<int64_t>(c, 64));
    }
    // CTA tile of the DMMA screen: 128 columns × TK centroids
    int tk_tile() const { return c > 32 ? 64 : (c > 16 ? 32 : (c > 8 ? 16 : 8)); }
    int tile_j() const { return 128; }
    int tile_k() const { return tk_tile(); }

    template <int WK, int MJ, int NK>
    void launch_dmma(const T* Mp, int nn, const double* C, const int* ver, dim3 grid, int cps,
                     const int* kmap = nullptr, int csub = 0) {
        constexpr int NW = 8, WJ = NW / WK;
        constexpr int TJ = WJ * MJ * 8, TK = WK * NK * 8;
        static_assert(TJ == 128, "tile");
        const size_t sm = sizeof(T) * 2 * TJ * 36 + sizeof(double) * 2 * TK * 36;
        auto kf = k_dist_dmma<T, WK, MJ, NK>;
        smem_at_least((const void*)kf, (size_t)(sm));
        kf<<<grid, 256, sm, st>>>(Mp, C, ver, d, nn, c, cps, part.p, xxp.p, kmap, csub);
    }
    static int tk_for(int cc_) { return cc_ > 32 ? 64 : (cc_ > 16 ? 32 : (cc_ > 8 ? 16 : 8)); }
    // the Lloyd screen of only the centroids in `sub` (their values changed since
    // the last screen of these columns; the other partials in `part` stay valid:
    // unchanged member sets give bit-identical means and deterministic partials)
    DBuf<int> kmap;
    void screen_subset(const double* C, const std::vector<int>& sub) {
        if ((int)sub.size() == c || scr_n != n || tc_mode) {
            screen(C);
            return;
        }
        if (sub.empty()) return;
        const int cs = (int)sub.size();
        kmap.ensure(c);
        CK(cudaMemcpyAsync(kmap.p, sub.data(), sizeof(int) * cs, cudaMemcpyHostToDevice, st));
        k_col_sq_fma<<<c, 1024, 0, st>>>(C, d, cc.p, nullptr, c);
        // the split count of the full screen (the partial layout must not change)
        const int tiles = ceil_div(n, tile_j()) * ceil_div(c, tile_k());
        const int chunks = ceil_div(d, 32);
        int ns = std::max(1, std::min(chunks / 4, ceil_div(2 * 148, tiles)));
        ns = std::min(ns, 64);
        if (ns != scr_split) {
            screen(C);
            return;
        }
        const int cps = ceil_div(chunks, ns);
        const int tk = tk_for(cs);
        dim3 grid(ceil_div(n, tile_j()), ceil_div(cs, tk), ns);
        switch (tk) {
            case 64: launch_dmma<2, 4, 4>(M, n, C, nullptr, grid, cps, kmap.p, cs); break;
            case 32: launch_dmma<1, 2, 4>(M, n, C, nullptr, grid, cps, kmap.p, cs); break;
            case 16: launch_dmma<1, 2, 2>(M, n, C, nullptr, grid, cps, kmap.p, cs); break;
            default: launch_dmma<1, 2, 1>(M, n, C, nullptr, grid, cps, kmap.p, cs); break;
        }
        ln.add(2);
    }

    // ---- screened distances --------------------------------------------
    // columns [0, nn) of Mp against C; split-K sized for >= 2 CTAs per SM
    int scr_n = 0, scr_split = 1;
    // ver != nullptr: centroid k lives in slot ver[k] of a [2][c][d] store
    void screen_cols(const T* Mp, int nn, const double* C, const int* ver = nullptr) {
        k_col_sq_fma<<<c, 1024, 0, st>>>(C, d, cc.p, ver, c);
        const int tiles = ceil_div(nn, tile_j()) * ceil_div(c, tile_k());
        const int chunks = ceil_div(d, 32);
        int ns = std::max(1, std::min(chunks / 4, ceil_div(2 * 148, tiles)));
        ns = std::min(ns, 64);
        part.ensure((size_t)ns * nn * c);
        xxp.ensure((size_t)ns * nn);
        const int cps = ceil_div(chunks, ns);
        dim3 grid(ceil_div(nn, tile_j()), ceil_div(c, tile_k()), ns);
        switch (tk_tile()) {
            case 64: launch_dmma<2, 4, 4>(Mp, nn, C, ver, grid, cps); break;  // warps 4×2, warp 32×32
            case 32: launch_dmma<1, 2, 4>(Mp, nn, C, ver, grid, cps); break;  // warps 8×1, warp 16×32
            case 16: launch_dmma<1, 2, 2>(Mp, nn, C, ver, grid, cps); break;
            default: launch_dmma<1, 2, 1>(Mp, nn, C, ver, grid, cps); break;
        }
        ln.add(2);
        scr_n = nn;
        scr_split = ns;
        tc_mode = false;
        tma_mode = false;
    }
    void screen(const double* C) { screen_cols(M, n, C); }
    // bound factor of the screen (see km.cuh): γ-bounds of the length-d
    // chains of both the screen (FMA / DMMA accumulation, counted as 2 roundings
    // per step for safety) and the reference's sequential chain, plus slack
    double kappa_screen() const { return (3.0 * (double)d + 16.0) * kU * 1.1; }
    // ---- tensor-core (tcgen05, BF16) screen: the ALM fast path --------------
    // valid for c <= 64; intervals use the BF16 bound (tc_screen.cuh)
    DBuf<__nv_bfloat16> tcCb;
    DBuf<int> tcerr;
    bool tc_mode = false;
    bool tc_ok() const { return c <= TC_N; }
    void screen_tc(const double* C) {
        const int64_t d_pad = ((d + TC_KB - 1) / TC_KB) * TC_KB;
        tcCb.ensure((size_t)TC_N * d_pad);
        tcerr.ensure(1);
        CK(cudaMemsetAsync(tcerr.p, 0, sizeof(int), st));
        k_tc_prep_centroids<<<TC_N, 1024, 0, st>>>(C, d, c, d_pad, tcCb.p, cc.p);
        const int tiles = ceil_div(n, TC_M);
        const int64_t total_kb = d_pad / TC_KB;
        // two CTAs fit per SM (smem ~100 KB): one wave of <= 2·148 CTAs
        int ns = (int)std::max<int64_t>(1, std::min<int64_t>(total_kb / 4, (2 * 148) / tiles));
        ns = std::max(1, std::min(ns, 16));
        const int kbps = (int)((total_kb + ns - 1) / ns);
        part.ensure((size_t)ns * n * c);
        xxp.ensure((size_t)ns * n);
        auto kf = k_screen_tc<T>;
        smem_at_least((const void*)kf, (size_t)(TC_SMEM));
        kf<<<dim3(tiles, ns), TC_THREADS, TC_SMEM, st>>>(M, tcCb.p, d, d_pad, n, c, kbps, part.p,
                                                         xxp.p, tcerr.p);
        ln.add(2);
        scr_n = n;
        scr_split = ns;
        tc_mode = true;
        tma_mode = false;
    }
    // ---- the loop's screen with TMA-fed operands (tc_screen.cuh) -------------
    bool tma_mode = false;
    const void* tma_key_a = nullptr;
    int64_t tma_key_n = -1, tma_key_dpad = -1;
    CUtensorMap mapA{}, mapB{};
    static CUtensorMap make_map(const void* base, uint64_t inner, uint64_t outer, uint32_t box_outer) {
        using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
        static Encode enc = [] {
            void* fn = nullptr;
            cudaDriverEntryPointQueryResult q;
            CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
            if (!fn || q != cudaDriverEntryPointSuccess) throw CudaErr("cuTensorMapEncodeTiled unavailable");
            return reinterpret_cast<Encode>(fn);
        }();
        CUtensorMap m;
        const cuuint64_t dims[2] = {inner, outer};
        const cuuint64_t strides[1] = {inner * 2};
        const cuuint32_t box[2] = {(cuuint32_t)TC_KB, box_outer};
        const cuuint32_t es[2] = {1, 1};
        const CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                               es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) throw CudaErr("cuTensorMapEncodeTiled failed");
        return m;
    }
    // Lb: BF16 columns [n][dpad] written by Pass F; C: FP64 centroids
    void screen_tma(const __nv_bfloat16* Lbp, int64_t dpad, const double* C) {
        tcCb.ensure((size_t)TC_N * dpad);
        tcerr.ensure(1);
        CK(pdl_launch(k_tc_prep_centroids, dim3(TC_N), dim3(1024), 0, st, C, d, c, dpad, tcCb.p, cc.p, tcerr.p));
        // RESPCA_TC_FORCE_ERR=1 (tests): raise the screen's error flag as a timed-out
        // mbarrier wait would — every decision must then come from the exact chains
        if (env_int("RESPCA_TC_FORCE_ERR", 0)) CK(cudaMemsetAsync(tcerr.p, 0x7f, sizeof(int), st));
        if (tma_key_a != (const void*)Lbp || tma_key_n != n || tma_key_dpad != dpad) {
            mapA = make_map(Lbp, (uint64_t)dpad, (uint64_t)n, TC_M);
            mapB = make_map(tcCb.p, (uint64_t)dpad, (uint64_t)TC_N, TC_N);
            tma_key_a = Lbp;
            tma_key_n = n;
            tma_key_dpad = dpad;
        }
        const int tiles = ceil_div(n, TC_M);
        const int64_t total_kb = dpad / TC_KB;
        // RESPCA_TMA_CFG: 0 = 4 stages, 2 CTAs/SM; 1 = 3 stages, 3 CTAs/SM
        const int cfg3 = env_int("RESPCA_TMA_CFG", 0);
        const int per_sm = cfg3 ? 3 : 2;
        int ns = (int)std::max<int64_t>(1, std::min<int64_t>(total_kb / 4, (per_sm * 148) / tiles));
        ns = std::max(1, std::min(ns, 16));
        if (const char* e = std::getenv("RESPCA_TMA_NS")) ns = std::max(1, std::min(16, std::atoi(e)));
        const int kbps = (int)((total_kb + ns - 1) / ns);
        part.ensure((size_t)ns * n * c);
        xxp.ensure((size_t)ns * n);
        auto kf = cfg3 ? k_screen_tma<3, 3> : k_screen_tma<4, 2>;
        const size_t sm = cfg3 ? tm_smem<3>() : tm_smem<4>();
        smem_at_least((const void*)kf, sm);
        CK(pdl_launch(kf, dim3(tiles, ns), dim3(TM_THREADS), sm, st, mapA, mapB, d, n, c, kbps,
                      part.p, xxp.p, tcerr.p));
        ln.add(2);
        scr_n = n;
        scr_split = ns;
        tc_mode = true;
        tma_mode = true;
    }
    Screen screen_view() const {
        Screen s;
        s.part = part.p;
        s.xxp = xxp.p;
        s.cc = cc.p;
        s.nsplit = scr_split;
        s.n = scr_n;
        s.c = c;
        s.kappa_d = tc_mode ? tc_bf16_kappa((double)d) + kappa_screen() : kappa_screen();
        if (tma_mode) s.kappa_d = (s.kappa_d + tma_xx_kappa((double)d)) * 1.01;  // ‖x‖² from BF16 values
        if (tma_mode) s.abs_e = tma_xx_abs((double)d) * 1.01;
        if (tc_mode) {
            // per operand |η| ≤ 2⁻¹²⁶ (BF16 subnormal or flushed): Σ|η|(|x_i| + |c_i|) + η² per dot,
            // twice in the distance; products flushed below 2⁻¹²⁶: d·2⁻¹²⁶ per dot
            const double t = std::ldexp(1.0, -126);
            s.abs_e += 4.0 * (double)d * t * 1.01;
            s.lin_e = 2.0 * std::sqrt((double)d) * t * 1.01;
            s.err = tcerr.p;
        }
        return s;
    }

    // long chains over few centroids: the warp-transposed exact kernel
    bool exact_tiled() const {
        const int e = env_int("RESPCA_EXACT_TILED", -1);
        if (e >= 0) return e != 0;
        return c <= 16 && d >= 4096;
    }
    // decide (+ exact fallback for ambiguous columns); returns #ambiguous
    int decide_kernels() const { return exact_tiled() ? 3 : 2; }  // launches of decide()
    static bool decide_fast_env() {  // RESPCA_DECIDE_FAST=0: the general k_decide everywhere
        static const bool v = env_int("RESPCA_DECIDE_FAST", 1) != 0;
        return v;
    }
    void decide(const double* C, const int* old_labels, const int* cnts, int mode, int* out_labels,
                Ctl* ctl) {
        const Screen sv = screen_view();
        const unsigned nb = (unsigned)ceil_div((int64_t)n * 32, 256);
        if (!trace_on() && sv.nsplit <= 4 && c <= 64 && decide_fast_env())
            CK(pdl_launch(k_decide_fast<2>, dim3(nb), dim3(256), 0, st, sv, n, c, old_labels, cnts, mode,
                          out_labels, amb.p, ctl));
        else if (!trace_on() && sv.nsplit <= 4 && c <= 128 && decide_fast_env())
            CK(pdl_launch(k_decide_fast<4>, dim3(nb), dim3(256), 0, st, sv, n, c, old_labels, cnts, mode,
                          out_labels, amb.p, ctl));
        else
            k_decide<<<nb, 256, 0, st>>>(sv, n, c, old_labels, cnts, mode, out_labels, amb.p, ctl,
                                         trace_on() ? 1 : 0);
        if (exact_tiled()) {
            // the list length is known only on the device: a grid for all n
            // columns, warps past the count return at once
            constexpr int KC = 4;
            const size_t sm = sizeof(T) * 2 * 4 * 32 * 33 + sizeof(double) * 2 * 4 * KC * 32;
            smem_at_least((const void*)k_exact_cols_tile<T, KC>, sm);
            k_exact_cols_tile<T, KC><<<dim3(ceil_div(n, 64), ceil_div(c, KC)), 64, sm, st>>>(
                M, C, d, c, amb.p, &ctl->ambiguous, exact.p);
            k_redecide<<<std::min(ceil_div((int64_t)n * 32, 256), 4 * 148), 256, 0, st>>>(
                exact.p, c, amb.p, &ctl->ambiguous, old_labels, cnts, mode, out_labels, ctl);
            ln.add(3);
        } else {
            CK(pdl_launch(k_exact_redecide<T>, dim3(std::min(n, 4 * 148)), dim3(128), 0, st, M, C, d, c, amb.p,
                          &ctl->ambiguous, exact.p, old_labels, cnts, mode, out_labels, ctl));
            ln.add(2);
        }
    }

    // assign_nearest (kmeans.cpp:21-37) → labels (device)
    void assign(const double* C, int* labels, const std::vector<int>* changed = nullptr) {
        CK(cudaMemsetAsync(kctl.p, 0, sizeof(Ctl), st));
        if (changed) screen_subset(C, *changed);
        else screen(C);
        decide(C, nullptr, nullptr, 0, labels, kctl.p);
        Ctl h;
        CK(cudaMemcpyAsync(&h, kctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (stats) stats->exact_fallbacks += h.ambiguous;
    }

    void fetch_labels(const int* labels) {
        h_labels.resize(n);
        CK(cudaMemcpyAsync(h_labels.data(), labels, sizeof(int) * n, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    // groups by size, largest first (group-walk kernels schedule the longest
    // member walks first, so no single large group forms the tail)
    DBuf<int> gsize_ord;
    std::vector<int> h_gsize_ord;
    void upload_groups() {
        h_gsize_ord.resize(c);
        for (int k = 0; k < c; ++k) h_gsize_ord[k] = k;
        if ((int)groups.counts.size() == c)
            std::stable_sort(h_gsize_ord.begin(), h_gsize_ord.end(),
                             [&](int x, int y) { return groups.counts[x] > groups.counts[y]; });
        gsize_ord.ensure(c);
        CK(cudaMemcpyAsync(gsize_ord.p, h_gsize_ord.data(), sizeof(int) * c, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(goff.p, groups.goff.data(), sizeof(int) * (c + 1),
                           cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(members.p, groups.members.data(), sizeof(int) * n,
                           cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(counts.p, groups.counts.data(), sizeof(int) * c,
                           cudaMemcpyHostToDevice, st));
    }

    // repair_empty (kmeans.cpp:40-64); labels device, h_labels must be current
    void repair_if_needed(const double* C, int* labels) {
        groups.build(h_labels.data(), n, c);
        bool empty = false;
        for (int k = 0; k < c; ++k) empty |= groups.counts[k] == 0;
        if (!empty) return;
        CK(cudaMemcpyAsync(counts.p, groups.counts.data(), sizeof(int) * c,
                           cudaMemcpyHostToDevice, st));
        launch_own_exact(C, labels);
        CK(cudaMemsetAsync(errflag.p, 0, sizeof(int), st));
        k_repair<T><<<1, 1024, 0, st>>>(M, C, d, n, c, labels, counts.p, own.p, errflag.p);
        ln.add(2);
        int e = 0;
        CK(cudaMemcpyAsync(&e, errflag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        fetch_labels(labels);
        if (e) throw RuntimeErr("kmeans: cannot repair empty cluster");
    }

    // means_of (kmeans.cpp:66-82) for the labels in h_labels → Cout
    void means(double* Cout) {
        groups.build(h_labels.data(), n, c);
        upload_groups();
        launch_group_mean(Cout);
    }
    // means_of of only the groups in `changed` (their member sets changed); the
    // other columns of Cout are copied from Cprev (same member set → same bits)
    DBuf<int> kcopy;
    void means_subset(double* Cout, const double* Cprev, const std::vector<int>& changed) {
        groups.build(h_labels.data(), n, c);
        upload_groups();
        std::vector<char> is(c, 0);
        for (int k : changed) is[k] = 1;
        std::vector<int> keep;
        for (int k = 0; k < c; ++k)
            if (!is[k]) keep.push_back(k);
        if (!keep.empty()) {
            kcopy.ensure(c);
            CK(cudaMemcpyAsync(kcopy.p, keep.data(), sizeof(int) * keep.size(), cudaMemcpyHostToDevice, st));
            k_copy_cols<<<dim3(ceil_div(d, 256 * 4), (unsigned)keep.size()), 256, 0, st>>>(Cprev, Cout, d,
                                                                                        kcopy.p);
            ln.add();
        }
        if (!changed.empty()) launch_group_mean(Cout, &changed);
    }
    DBuf<int> gord;
    void launch_group_mean(double* Cout, const std::vector<int>* only = nullptr) {
        // groups largest first: the largest group's member walks bound the kernel
        std::vector<int> ord;
        if (only) ord = *only;
        else
            for (int k = 0; k < c; ++k) ord.push_back(k);
        if ((int)groups.counts.size() == c)
            std::stable_sort(ord.begin(), ord.end(),
                             [&](int x, int y) { return groups.counts[x] > groups.counts[y]; });
        gord.ensure(c);
        // pageable source: staged by the runtime before the call returns
        CK(cudaMemcpyAsync(gord.p, ord.data(), sizeof(int) * ord.size(), cudaMemcpyHostToDevice, st));
        const int rb = ceil_div(d, MS_T);
        k_means_sum<T><<<rb * (int)ord.size(), MS_T, 0, st>>>(M, goff.p, members.p, gord.p, Cout, d, rb);
        ln.add();
    }

    // Lloyd stop (kmeans.cpp:148-158): sqrt(moved) <= tol * max(sqrt(scale), 1e-300)
    bool stop_test(const double* nxt, const double* C, double tol) {
        const int64_t N = d * (int64_t)c;
        const int blocks = std::min(512, ceil_div(N, 256));
        k_moved_scale<<<blocks, 256, 0, st>>>(nxt, C, N, msp.p);
        k_sum_partials<<<1, 256, 0, st>>>(msp.p, blocks, 2, msp.p + 2 * 512);
        ln.add(2);
        double h[2];
        CK(cudaMemcpyAsync(h, msp.p + 2 * 512, sizeof(h), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        auto verdict = [&](double moved, double scale, double& margin) {
            const double s = std::sqrt(scale);
            const double thr = tol * std::max(s, 1e-300);
            const double m = std::sqrt(moved);
            margin = std::fabs(m - thr) / std::max(thr, 1e-300);
            return m <= thr;
        };
        double margin;
        bool v = verdict(h[0], h[1], margin);
        lloyd_margin = std::min(lloyd_margin, margin);
        if (margin < 1e-9 && h[0] != 0.0) {  // too close for a tree sum: reference chain
            if (trace_on())
                std::fprintf(stderr, "[respca] lloyd stop: exact chain (moved %.17g scale %.17g margin %.3g)\n", h[0],
                             h[1], margin);
            k_moved_scale_exact<<<1, 256, 0, st>>>(nxt, C, N, msp.p + 2 * 512);
            ln.add();
            CK(cudaMemcpyAsync(h, msp.p + 2 * 512, sizeof(h), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            v = verdict(h[0], h[1], margin);
        }
        return v;
    }

    // decision margins of the last kmeans(): the Lloyd stop
    // test's relative distance to its threshold, and every restart's inertia
    double lloyd_margin = INFINITY;
    std::vector<double> restart_inertia;

    // lloyd_run (kmeans.cpp:141-168).  C: in = start centroids, out = final
    // means; labels: device out.  Returns iters_run.
    uint64_t lloyd_run(double* C, int* labels, uint64_t max_iters, double tol) {
        if (max_iters == 0) throw InvalidArg("kmeans: max_iters must be >= 1");
        uint64_t it = 0;
        double* cur = C;
        double* nxt = nextC.p;
        const auto t_lloyd0 = HClock::now();
        double lph[5] = {0, 0, 0, 0, 0};
        // incremental steps: a centroid whose group kept its member set keeps
        // its bits (means_of sums the same columns in the same order), so the
        // next means and the next screen only touch the groups that changed
        std::vector<int> prevL, chg;
        bool have_chg = false;  // chg = groups changed between the last two assignments
        const bool incr = env_int("RESPCA_LLOYD_INCR", 1) != 0;
        for (; it < max_iters; ++it) {
            const auto ts0 = HClock::now();
            assign(cur, labels, (incr && have_chg && it >= 2) ? &chg : nullptr);
            const double ta = since(ts0);
            fetch_labels(labels);
            const double tf = since(ts0);
            repair_if_needed(cur, labels);
            const double tr = since(ts0);
            if (incr && it >= 1 && (int)prevL.size() == n) {
                std::vector<char> f(c, 0);
                for (int j = 0; j < n; ++j)
                    if (prevL[j] != h_labels[j]) f[prevL[j]] = f[h_labels[j]] = 1;
                chg.clear();
                for (int k = 0; k < c; ++k)
                    if (f[k]) chg.push_back(k);
                have_chg = true;
                means_subset(nxt, cur, chg);
            } else {
                have_chg = false;
                means(nxt);
            }
            prevL = h_labels;
            const double tm = since(ts0);
            if (stats) stats->lloyd_steps++;
            const bool stop = stop_test(nxt, cur, tol);
            if (trace_on()) {
                lph[0] += ta;
                lph[1] += tf - ta;
                lph[2] += tr - tf;
                lph[3] += tm - tr;
                lph[4] += since(ts0) - tm;
            }
            std::swap(cur, nxt);
            if (stop) {
                ++it;
                break;
            }
        }
        if (trace_on())
            std::fprintf(stderr, "[respca] lloyd %llu steps: assign %.4f fetch %.4f repair %.4f means %.4f stop %.4f\n",
                         (unsigned long long)it, lph[0], lph[1], lph[2], lph[3], lph[4]);
        if (cur != C) CK(cudaMemcpyAsync(C, cur, sizeof(double) * d * c, cudaMemcpyDeviceToDevice, st));
        if (stats) {
            CK(cudaStreamSynchronize(st));
            stats->t_lloyd += since(t_lloyd0);
        }
        // lanes enter the refinement together: a persistent grid holds its SMs,
        // and a lane's short Lloyd kernels queued behind another lane's long
        // refinement kernel on a shared hardware queue would wait for it
        if (before_hartigan) before_hartigan();
        const auto t_h0 = HClock::now();
        hartigan(C, labels);
        if (stats) stats->t_hart += since(t_h0);
        fetch_labels(labels);
        groups.build(h_labels.data(), n, c);
        for (int k = 0; k < c; ++k)
            if (groups.counts[k] == 0) throw InvalidArg("GroupAssignment: empty group");
        means(C);  // drop incremental rounding (kmeans.cpp:161)
        return it;
    }

    // hartigan_refine (kmeans.cpp:96-139), exact sequential semantics
    // (hartigan.cuh): ONE persistent cooperative launch for every pass; the
    // start intervals come from one full screen, later ones from the kernel's
    // lazy per-entry refresh.
    DBuf<double> hA, hE, hxx, hC2, hpart, hcand, hccp;
    DBuf<int> hver, hebuf;
    DBuf<HartGlobal> hglob;
    int hart_ctas = 0;  // CTAs of the Hartigan kernel (0: one per SM)
    std::function<void()> before_hartigan;  // restart lanes: wait for the others' seeding/Lloyd

    static int env_int(const char* name, int dflt) {
        const char* e = std::getenv(name);
        return e ? std::atoi(e) : dflt;
    }
    struct HartGeom {
        int G = 1, cpb = 1, B = 1, R = 8, stages = 2;
        bool cache = true;
        size_t smem = 0;
    };
    // shared memory of the Hartigan kernel (hartigan.cuh carve-up)
    size_t hart_smem(int cpb, bool cache, int B, int R, int stages) const {
        const size_t stage = R > 0 ? (size_t)stages * sizeof(double) * (size_t)(R + 4) *
                                         (size_t)(((B + 15) & ~15) + ((c + 15) & ~15))
                                   : 0;
        return (cache ? (size_t)cpb * d * sizeof(T) + 16 : 0) + sizeof(double) * 2 * (size_t)cpb * c +
               sizeof(double) * (4 * (size_t)c + HART_RED) + stage + sizeof(int) * 5 * (size_t)c + 2048;
    }
    HartGeom hart_geometry() const {
        int dev = 0, nsm = 148, optin = 0;
        CK(cudaGetDevice(&dev));
        CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        optin -= 4096;  // the kernel's static shared memory + headroom
        const int avail = std::min(HART_MAXG, hart_ctas > 0 ? std::min(hart_ctas, nsm) : nsm);
        if (const char* e = std::getenv("RESPCA_HART_GEOM")) {  // "cache,cpb,R,stages" (experiments)
            int ca = 1, cp = 2, rr = 16, stg = 3;
            if (std::sscanf(e, "%d,%d,%d,%d", &ca, &cp, &rr, &stg) == 4) {
                HartGeom g;
                g.cache = ca != 0;
                g.cpb = cp;
                g.G = std::max(1, std::min(avail, ceil_div(n, cp)));
                g.B = g.G * cp;
                g.R = rr;
                g.stages = stg;
                g.smem = hart_smem(cp, g.cache, g.B, rr, stg);
                if (g.smem <= (size_t)optin) return g;
            }
        }
        for (int pass = 0; pass < 2; ++pass) {
            const bool cache = pass == 0;  // owned columns cached in shared memory, else streamed
            for (int cpb = cache ? 8 : 4; cpb >= 1; --cpb) {
                HartGeom g;
                g.cache = cache;
                g.cpb = cpb;
                g.G = std::max(1, std::min(avail, ceil_div(n, cpb)));
                g.B = g.G * cpb;
                // refresh chunks: the most rows (32/16/8), then the most stages (3/2)
                for (int R : {32, 16, 8})
                    for (int stages : {3, 2}) {
                        if (R > 8 && (int64_t)R / 2 >= (d + g.G - 1) / g.G) continue;  // slice shorter
                        const size_t sm = hart_smem(cpb, cache, g.B, R, stages);
                        if (sm > (size_t)optin) continue;
                        g.R = R;
                        g.stages = stages;
                        g.smem = sm;
                        return g;
                    }
            }
        }
        throw InvalidArg("hartigan: c too large for the device's shared memory");
    }
    // ---- Gram-matrix refinement (hart_gram.cuh).  kmeans(X) computes
    //      G = XᵀX once; every restart's refinement borrows it for the call.
    const double* gram = nullptr;  // borrowed G, diag, norm bounds (nullptr: per-pass path)
    const double *gram_xx = nullptr, *gram_xn = nullptr, *gram_xl = nullptr;
    cudaEvent_t gram_ev = nullptr;  // G complete
    cudaStream_t gram_st = nullptr;  // G's own stream (restart lanes)
    DBuf<double> gG, gxx, gxn, gxl, gS;
    DBuf<GramScal> gsc;
    DBuf<int> glog;
    DBuf<unsigned long long> gstats;
    static constexpr int kGramMaxC = 256;

    static int gram_env() {  // RESPCA_HART_GRAM: 0 off, 1 on where it fits (default)
        static const int v = [] {
            const char* e = std::getenv("RESPCA_HART_GRAM");
            return e ? std::atoi(e) : 1;
        }();
        return v;
    }
    bool gram_fits() const {
        if (gram_env() == 0 || c < 2 || c > kGramMaxC || n > 32768) return false;
        size_t fr = 0, tot = 0;
        CK(cudaMemGetInfo(&fr, &tot));
        return (double)n * (double)n * 8.0 <= 0.4 * (double)fr;
    }
    bool gram_path() const { return gram != nullptr && c >= 2 && c <= kGramMaxC; }
    double gram_gamma() const { return (2.2 * (double)d + 4.0) * kU; }
    // G = MᵀM on the FP64 tensor cores + its diagonal bounds; the event marks completion
    // G's storage and pointers (lent to the restart lanes before G is computed;
    // its consumers wait on gram_ev)
    void alloc_gram() {
        gG.ensure((size_t)n * n);
        gxx.ensure(n);
        gxn.ensure(n);
        gxl.ensure(n);
        if (!gram_ev) CK(cudaEventCreateWithFlags(&gram_ev, cudaEventDisableTiming));
        gram = gG.p;
        gram_xx = gxx.p;
        gram_xn = gxn.p;
        gram_xl = gxl.p;
    }
    void compute_gram(cudaStream_t gs = nullptr) {
        if (!gs) gs = st;
        alloc_gram();
        const long long nb = ceil_div(n, GR_T);
        const long long tiles = nb * (nb + 1) / 2;
        const size_t sm = gram_smem<T>();
        smem_at_least((const void*)k_gram<T>, (size_t)(sm));
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (trace_on() && gs == st) {
            CK(cudaEventCreate(&e0));
            CK(cudaEventCreate(&e1));
            CK(cudaEventRecord(e0, gs));
        }
        const int gctas = env_int("RESPCA_GRAM_CTAS", 0);  // 0: one CTA per tile
        k_gram<T><<<(unsigned)(gctas > 0 ? std::min<long long>(gctas, tiles) : tiles), 256, sm, gs>>>(M, d, n, gG.p,
                                                                                                     tiles);
        if (trace_on() && gs == st) {
            CK(cudaEventRecord(e1, gs));
            CK(cudaEventSynchronize(e1));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            std::fprintf(stderr, "[respca] gram: n=%d d=%lld %lld tiles %.3f ms (%.1f TFLOP/s)\n", n, (long long)d,
                         tiles, ms, 2.0 * (double)tiles * GR_T * GR_T * (double)d / (ms * 1e-3) / 1e12);
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
        }
        k_gram_diag<<<ceil_div(n, 256), 256, 0, gs>>>(gG.p, n, gram_gamma(), gxx.p, gxn.p, gxl.p);
        ln.add(2);
        if (!gram_ev) CK(cudaEventCreateWithFlags(&gram_ev, cudaEventDisableTiming));
        CK(cudaEventRecord(gram_ev, gs));
        gram = gG.p;
        gram_xx = gxx.p;
        gram_xn = gxn.p;
        gram_xl = gxl.p;
    }
    // G computed while X still arrives: the upload records an event per column
    // chunk; the tiles of block rows up to a chunk's end (a contiguous range of
    // the row-major lower triangle) wait only for that chunk.  kmeans() then
    // finds G launched (gram_early) and only waits on gram_ev.
    bool gram_early = false;
    void compute_gram_banded(const std::vector<std::pair<int64_t, cudaEvent_t>>& chunks) {
        if (!gram_st) {
            int lo = 0, hi = 0;
            CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            CK(cudaStreamCreateWithPriority(&gram_st, cudaStreamNonBlocking, lo));
        }
        alloc_gram();
        const size_t sm = gram_smem<T>();
        smem_at_least((const void*)k_gram<T>, sm);
        long long t_prev = 0;
        for (const auto& ch : chunks) {
            const long long nbe = ceil_div((int64_t)std::min<int64_t>(ch.first, n), (int64_t)GR_T);
            const long long t_end = nbe * (nbe + 1) / 2;
            CK(cudaStreamWaitEvent(gram_st, ch.second, 0));
            if (t_end > t_prev) {
                k_gram<T><<<(unsigned)(t_end - t_prev), 256, sm, gram_st>>>(M, d, n, gG.p, t_end, t_prev);
                ln.add();
            }
            t_prev = t_end;
        }
        k_gram_diag<<<ceil_div(n, 256), 256, 0, gram_st>>>(gG.p, n, gram_gamma(), gxx.p, gxn.p, gxl.p);
        ln.add();
        CK(cudaEventRecord(gram_ev, gram_st));
        gram_early = true;
    }
    void lend_gram(KMeansEngine& o) const {
        o.gram = gram;
        o.gram_xx = gram_xx;
        o.gram_xn = gram_xn;
        o.gram_xl = gram_xl;
        o.gram_ev = gram_ev;
    }
    void drop_gram() {
        gram = gram_xx = gram_xn = gram_xl = nullptr;
    }
    void gram_reserve() {
        gS.ensure((size_t)n * c);
        gsc.ensure(c);
        glog.ensure((size_t)5 * 50 * n);
        gstats.ensure(16);
        hst.ensure<unsigned long long>(16);
    }
    // hartigan_refine on the Gram matrix: labels (device) in/out; C (device,
    // the start centroids = means_of(labels)) is scratch for exact fallbacks
    void hartigan_gram(double* C, int* labels) {
        upload_groups();
        gram_reserve();
        if (trace_on() && gram_ev) {
            const auto tw = HClock::now();
            CK(cudaEventSynchronize(gram_ev));
            std::fprintf(stderr, "[respca] hartigan(gram): waited %.4fs for G\n", since(tw));
        }
        if (gram_ev) CK(cudaStreamWaitEvent(st, gram_ev, 0));
        const double gamG = gram_gamma();
        {  // S⁰_k[j] = Σ_{m∈k} Ĝ[m][j]: the member-walk kernel of means_of over G's columns
            std::vector<int> ord(c);
            for (int k = 0; k < c; ++k) ord[k] = k;
            std::stable_sort(ord.begin(), ord.end(),
                             [&](int x, int y) { return groups.counts[x] > groups.counts[y]; });
            gord.ensure(c);
            CK(cudaMemcpyAsync(gord.p, ord.data(), sizeof(int) * c, cudaMemcpyHostToDevice, st));
            const int rb = ceil_div(n, MS_T);
            k_means_sum<double><<<rb * c, MS_T, 0, st>>>(gram, goff.p, members.p, gord.p, gS.p, n, rb, 0);
        }
        k_gram_scal<<<c, 256, 0, st>>>(gS.p, gram_xn, goff.p, members.p, n, c, gamG, gsc.p);
        GramArgs a{};
        a.G = gram;
        a.xx = gram_xx;
        a.xn = gram_xn;
        a.xl = gram_xl;
        a.S = gS.p;
        a.scal0 = gsc.p;
        a.labels = labels;
        a.counts = counts.p;
        a.Cs = C;
        a.log = glog.p;
        a.stats = gstats.p;
        a.M = M;
        a.d = d;
        a.n = n;
        a.c = c;
        a.max_pass = 50;  // kmeans.cpp:101
        a.force_exact = env_int("RESPCA_GRAM_FORCE_EXACT", 0);
        a.timing = trace_on() ? 1 : 0;
        a.gamG = gamG;
        a.gamc = ((double)d + 3.0) * kU * 1.02;
        // one cluster of CL CTAs (one SM each) per restart: 16 (the non-portable size,
        // halved below when the GPU cannot place it) — with the st.async exchange a
        // wider window costs nothing per window and saves windows at every size
        // (C2, n = 2000: refinement-dominated init 49 ms at CL = 1, 20 ms at 16; C1 27 → 18.5)
        int CL = 16;
        while (CL > 1 && (CL / 2) * GRAM_WARPS >= n) CL /= 2;  // tiny n: no CTA without a column
        if (const char* e = std::getenv("RESPCA_GRAM_CL")) CL = std::max(1, std::min(GRAM_MAXCL, std::atoi(e)));
        // the column → CTA map uses shifts: the cluster size is a power of two
        while (CL & (CL - 1)) CL &= CL - 1;
        auto smem_for = [&](int cl) -> size_t {
            const size_t cs = (size_t)((c + 1) & ~1), gl = (size_t)4 * GRAM_WARPS * cl;
            return (size_t)c * (sizeof(GramCoef) + sizeof(GramScal) + sizeof(double)) + sizeof(int) * cs +
                   sizeof(double) * (3 * GRAM_WARPS * cs + 3 * GRAM_WARPS * gl) + 80;
        };
        auto launch = [&](auto kf) {
            smem_at_least((const void*)kf, smem_for(CL));
            if (CL > 8) CK(cudaFuncSetAttribute((const void*)kf, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            for (;; CL = std::max(1, CL / 2)) {
                cudaLaunchConfig_t lc = {};
                lc.gridDim = dim3(CL);
                lc.blockDim = dim3(GRAM_THREADS);
                lc.dynamicSmemBytes = smem_for(CL);
                lc.stream = st;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = CL;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                lc.attrs = at;
                lc.numAttrs = 1;
                const cudaError_t e = cudaLaunchKernelEx(&lc, kf, a);
                if (e == cudaSuccess) break;
                if (CL == 1) CK(e);
                (void)cudaGetLastError();  // cluster not schedulable: halve it
            }
        };
        if (c <= 32) launch(k_hart_gram<T, 1>);
        else if (c <= 64) launch(k_hart_gram<T, 2>);
        else if (c <= 128) launch(k_hart_gram<T, 4>);
        else launch(k_hart_gram<T, 8>);
        ln.add(3);
        if (stats || trace_on()) {
            unsigned long long* hh = hst.ensure<unsigned long long>(16);
            CK(cudaMemcpyAsync(hh, gstats.p, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            if (stats) {
                stats->hartigan_moves += hh[0];
                stats->hartigan_passes += hh[1];
                stats->hartigan_rounds += hh[2];
                stats->exact_fallbacks += hh[3];
            }
            if (trace_on())
                std::fprintf(stderr, "[respca] hartigan(gram, CL=%d): %llu passes %llu windows %llu moves %llu fallbacks (replayed %llu moves); "
                             "s at 1.965GHz: elect %.3f far stores %.3f patch %.3f block change %.3f decide %.3f push %.3f exchange wait %.3f pending %.3f\n",
                             CL, hh[1], hh[2], hh[0], hh[3], hh[4], hh[5] / 1.965e9, hh[6] / 1.965e9, hh[7] / 1.965e9, hh[8] / 1.965e9, hh[9] / 1.965e9, hh[10] / 1.965e9,
                             hh[11] / 1.965e9, hh[12] / 1.965e9);
        }
    }

    void hart_reserve() {
        if (gram_path()) gram_reserve();
        const HartGeom g = hart_geometry();
        const size_t nc = (size_t)n * c;
        hA.ensure(nc);
        hE.ensure(nc);
        hxx.ensure(n);
        hC2.ensure((size_t)2 * d * c);
        hver.ensure(c);
        hebuf.ensure(ceil_div(n, g.B));
        hpart.ensure((size_t)2 * g.G * g.B * c);
        hcand.ensure((size_t)4 * n);
        hccp.ensure((size_t)2 * g.G * c);
        hglob.ensure(1);
        scratch.ensure(std::max(c, 64));
        hst.ensure<HartGlobal>(1);
    }

    void hartigan(double* C, int* labels) {
        if (c <= 1) return;  // no candidate target: never moves
        if (c >= 32768) throw InvalidArg("hartigan: c >= 32768 is not supported");
        groups.build(h_labels.data(), n, c);
        CK(cudaMemcpyAsync(counts.p, groups.counts.data(), sizeof(int) * c,
                           cudaMemcpyHostToDevice, st));
        if (gram_path()) {
            hartigan_gram(C, labels);
            return;
        }
        hart_reserve();
        const HartGeom hgm = hart_geometry();
        CK(cudaMemcpyAsync(hC2.p, C, sizeof(double) * d * c, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemsetAsync(hver.p, 0, sizeof(int) * c, st));
        CK(cudaMemsetAsync(hebuf.p, 0, sizeof(int) * ceil_div(n, hgm.B), st));
        CK(cudaMemsetAsync(hglob.p, 0, sizeof(HartGlobal), st));
        k_hart_first_reset<<<1, 1, 0, st>>>(hglob.p);
        // start intervals: one screen of every column against the start centroids
        screen_cols(M, n, hC2.p, nullptr);
        const double gam = ((double)d + 3.0) * kU * 1.02;
        k_hart_fill<<<ceil_div((int64_t)n * c, 256), 256, 0, st>>>(screen_view(), hA.p, hE.p, hxx.p, n, c, gam);
        ln.add(2);
        const int G = hgm.G, cpb = hgm.cpb;
        const bool cache = hgm.cache;
        const size_t smem = hgm.smem;
        auto kf = cpb <= 2 ? k_hart_all<T, 2> : (cpb <= 4 ? k_hart_all<T, 4> : k_hart_all<T, 8>);
        smem_at_least((const void*)kf, (size_t)(smem));
        HartArgs a{};
        a.g = hglob.p;
        a.labels = labels;
        a.counts = counts.p;
        a.Cs = hC2.p;
        a.ver = hver.p;
        a.A = hA.p;
        a.E = hE.p;
        a.ebuf = hebuf.p;
        a.part = hpart.p;
        a.stage_rows = hgm.R;
        a.stages = hgm.stages;
        a.diag = env_int("RESPCA_HART_DIAG", 0);
        a.xx = hxx.p;
        a.cc0 = cc.p;
        a.scratch = scratch.p;
        a.cand = hcand.p;
        a.ccp = hccp.p;
        a.gam = gam;
        a.d = d;
        a.n = n;
        a.c = c;
        a.cpb = cpb;
        a.cache_cols = cache ? 1 : 0;
        a.max_pass = 50;  // kmeans.cpp:101
        // + the reciprocal-multiply update used for ‖c′‖² and the dots (≤ 7.5u(‖x‖+‖c‖)²)
        a.kappa_d = kappa_screen() + 16.0 * kU;
        const T* Mp = M;
        void* args[] = {&Mp, &a};
        CK(cudaLaunchCooperativeKernel((const void*)kf, dim3(G), dim3(512), args, smem, st));
        ln.add(1);
        const dim3 cg(ceil_div(d, 256 * 8), std::min(c, 64));
        k_hart_consolidate<<<cg, 256, 0, st>>>(hC2.p, hver.p, d, c);
        CK(cudaMemcpyAsync(C, hC2.p, sizeof(double) * d * c, cudaMemcpyDeviceToDevice, st));
        ln.add(1);
        if (stats) {
            HartGlobal* hh = hst.ensure<HartGlobal>(1);
            CK(cudaMemcpyAsync(hh, hglob.p, sizeof(HartGlobal), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            stats->hartigan_moves += hh->moves;
            stats->exact_fallbacks += hh->exact_fallbacks;
            stats->hartigan_passes += hh->passes;
            stats->hartigan_rounds += hh->rounds;
            stats->hartigan_refreshes += hh->refreshed;
            stats->t_hart_kernel += 1e-9 * (double)hh->t_kernel;
            if (trace_on())
                std::fprintf(stderr,
                             "[respca] hartigan: G=%d cpb=%d R=%d %llu passes %llu blocks %llu rounds %llu moves "
                             "%llu refreshed, kernel %.3fs (block entries %.3fs; CTA0 stale/entry %.2f, heavy %llu, redo rounds %llu)\n",
                             G, cpb, hgm.R, (unsigned long long)hh->passes, (unsigned long long)hh->blocks,
                             (unsigned long long)hh->rounds, (unsigned long long)hh->moves,
                             (unsigned long long)hh->refreshed, 1e-9 * hh->t_kernel, 1e-9 * hh->t_load,
                             (double)hh->stale_sum / (double)std::max<uint64_t>(1, hh->blocks),
                             (unsigned long long)hh->heavy_blocks, (unsigned long long)hh->redos);
            if (trace_on())
                std::fprintf(stderr,
                             "[respca] hartigan CTA0 phases (s at 1.965 GHz): update %.3f entry-tiles %.3f entry-barrier %.3f "
                             "entry-reduce+wait %.3f decide %.3f barrier %.3f settle %.3f | tiles: issue %.3f wait %.3f compute %.3f\n",
                             hh->tm[0] / 1.965e9, hh->tm[1] / 1.965e9, hh->tm[2] / 1.965e9, hh->tm[3] / 1.965e9,
                             hh->tm[4] / 1.965e9, hh->tm[5] / 1.965e9, hh->tm[7] / 1.965e9, hh->tm[6] / 1.965e9,
                             hh->tsub1 / 1.965e9, hh->tsub2 / 1.965e9);
            if (trace_on())
                std::fprintf(stderr, "[respca] hartigan CTA0 active rounds %llu: phase-1 %.2f us (x_m pass + sum %.2f us)\n",
                             (unsigned long long)hh->act_rounds,
                             hh->act_cycles / 1965.0 / std::max<double>(1.0, (double)hh->act_rounds),
                             hh->dq_cycles / 1965.0 / std::max<double>(1.0, (double)hh->act_rounds));
            if (trace_on() && env_int("RESPCA_HART_DIAG", 0))
                std::fprintf(stderr,
                             "[respca] hartigan no-move margins / (|x|+|c|)^2 below 1e-1..1e-8: %llu %llu %llu %llu %llu %llu %llu %llu of %llu\n",
                             hh->hist[0], hh->hist[1], hh->hist[2], hh->hist[3], hh->hist[4], hh->hist[5], hh->hist[6],
                             hh->hist[7], hh->hist[8]);
        }
    }

    void k_col_sq_fma_T(const T* m, int cols, double* out);

    void launch_own_exact(const double* C, const int* labels) {
        smem_at_least((const void*)k_own_exact<T>, own_exact_smem<T>());
        k_own_exact<T><<<ceil_div(n, 32 * OWN_W), 32 * OWN_W, own_exact_smem<T>(), st>>>(M, C, d, n, labels, own.p);
    }
    // inertia_of (kmeans.cpp:84-91): exact per-column chains, sequential host sum
    double inertia(const double* C, const int* labels) {
        launch_own_exact(C, labels);
        ln.add();
        std::vector<double> h(n);
        CK(cudaMemcpyAsync(h.data(), own.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        double s = 0.0;
        for (int j = 0; j < n; ++j) s += h[j];
        return s;
    }

    // kmeans_pp_init (kmeans.cpp:172-224); RNG stays on the host (libstdc++)
    std::vector<int> pp_init(std::mt19937_64& rng) {
        return pp_init_with(
            [&](uint64_t nn) {
                std::uniform_int_distribution<std::size_t> first(0, (std::size_t)nn - 1);
                return (uint64_t)first(rng);
            },
            [&](double total) {
                std::uniform_real_distribution<double> u(0.0, total);
                return u(rng);
            });
    }
    // draw_first(n) = uniform_int_distribution<size_t>(0, n-1)(rng);
    // draw_real(total) = uniform_real_distribution<double>(0, total)(rng)
    template <class FirstFn, class RealFn>
    std::vector<int> pp_init_with(FirstFn&& draw_first, RealFn&& draw_real) {
        if (c == 0) throw InvalidArg("kmeans_pp_init: c must be >= 1");
        if ((int64_t)c > n) throw InvalidArg("kmeans_pp_init: c exceeds column count");
        std::vector<int> chosen;
        std::vector<char> is_chosen(n, 0);
        const uint64_t f0 = draw_first((uint64_t)n);
        if (f0 >= (uint64_t)n) throw InvalidArg("kmeans_pp_init: draw out of range");
        chosen.push_back((int)f0);
        is_chosen[chosen[0]] = 1;
        d2.ensure(n);
        std::vector<double> hd2(n, std::numeric_limits<double>::infinity());
        CK(cudaMemcpyAsync(d2.p, hd2.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
        while ((int)chosen.size() < c) {
            const int last = chosen.back();
            const size_t ppsm = sizeof(T) * 2 * 4 * (32 * 33 + 32);
            smem_at_least((const void*)k_pp_d2<T>, (size_t)(ppsm));
            k_pp_d2<T><<<ceil_div(n, 64), 64, ppsm, st>>>(M, d, n, last, d2.p);
            ln.add();
            CK(cudaMemcpyAsync(hd2.data(), d2.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            double total = 0.0;
            for (int j = 0; j < n; ++j) total += hd2[j];
            int pick = n;
            if (total > 0.0) {
                double r = draw_real(total);
                for (int j = 0; j < n; ++j) {
                    r -= hd2[j];
                    if (r <= 0.0 && !is_chosen[j]) {
                        pick = j;
                        break;
                    }
                }
            }
            if (pick == n) {
                for (int j = 0; j < n; ++j)
                    if (!is_chosen[j]) {
                        pick = j;
                        break;
                    }
            }
            chosen.push_back(pick);
            is_chosen[pick] = 1;
        }
        return chosen;
    }

    // k-means++ seedings (kmeans.cpp:172-224) of R ≤ 8 restarts side by side:
    // one pass over the columns per pick serves every restart's d² update
    // (k_pp_d2_multi); each restart draws from its own engine.  engs[r]: in =
    // the restart's start state, out = its state after the seeding's draws.
    template <int R>
    void launch_pp_multi(const PPLast& lasts) {
        const size_t sm = sizeof(T) * 2 * 4 * (32 * 33 + R * 32);
        smem_at_least((const void*)k_pp_d2_multi<T, R>, sm);
        k_pp_d2_multi<T, R><<<ceil_div(n, 64), 64, sm, st>>>(M, d, n, lasts, d2.p);
        ln.add();
    }
    HBuf hpp;
    template <int R>
    void launch_pp_gram(const PPLast& lasts) {
        k_pp_gram<R><<<ceil_div(n, 256), 256, 0, st>>>(gram, gram_xx, n, lasts, d2.p);
        ln.add();
    }
    // on_gram: the d² values come from the Gram matrix (k_pp_gram: one row of G
    // per restart and pick, no pass over the columns) with the rigorous bound
    // E = κ·(2·max‖x‖)² per value.  The reference's pick is the first column
    // where its running remainder r − Σ d² turns ≤ 0; the remainder computed
    // from the d̃ values differs from the reference's by at most B (derived
    // below), so the pick is the reference's whenever no remainder up to the
    // pick lies within ±B.  Otherwise the restart is seeded again on the exact
    // chains (pp_init) from its start state — the draws a restart consumes do
    // not depend on the d² values, only on `total > 0`.
    uint64_t pp_gram_fallbacks = 0;
    std::vector<std::vector<int>> pp_joint(std::vector<std::mt19937_64>& engs, bool on_gram = false) {
        const int R = (int)engs.size();
        if (R < 1 || R > 8) throw InvalidArg("pp_joint: 1..8 restarts");
        if (c == 0) throw InvalidArg("kmeans_pp_init: c must be >= 1");
        if ((int64_t)c > n) throw InvalidArg("kmeans_pp_init: c exceeds column count");
        const bool og = on_gram && gram != nullptr && gram_ev != nullptr && env_int("RESPCA_PP_GRAM", 1) != 0;
        double E = 0.0;
        if (og) {
            CK(cudaStreamWaitEvent(st, gram_ev, 0));
            std::vector<double> hx(n);
            CK(cudaMemcpyAsync(hx.data(), gram_xn, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            double xm = 0.0;
            for (int j = 0; j < n; ++j) xm = std::max(xm, hx[j]);
            const double kap = (gram_gamma() + ((double)d + 3.0) * kU * 1.02 + 8.0 * kU) * 1.01;
            E = kap * (2.0 * xm) * (2.0 * xm) * 1.0001;
            if (!(E == E) || std::isinf(E)) throw InvalidArg("kmeans_pp_init: non-finite Gram norms");
        }
        const std::vector<std::mt19937_64> start = engs;
        std::vector<char> amb(R, 0);
        const int force_amb = og ? env_int("RESPCA_PP_GRAM_FORCE_AMB", 0) : 0;  // tests: restart v−1 falls back
        std::vector<std::vector<int>> chosen(R);
        std::vector<std::vector<char>> is_chosen(R, std::vector<char>(n, 0));
        for (int r = 0; r < R; ++r) {
            std::uniform_int_distribution<std::size_t> first(0, (std::size_t)n - 1);
            const int f0 = (int)first(engs[r]);
            chosen[r].push_back(f0);
            is_chosen[r][f0] = 1;
        }
        d2.ensure((size_t)R * n);
        double* hd2 = hpp.ensure<double>((size_t)R * n);
        for (size_t e = 0; e < (size_t)R * n; ++e) hd2[e] = std::numeric_limits<double>::infinity();
        CK(cudaMemcpyAsync(d2.p, hd2, sizeof(double) * R * n, cudaMemcpyHostToDevice, st));
        for (int p = 1; p < c; ++p) {
            PPLast lasts{};
            for (int r = 0; r < 8; ++r) lasts.v[r] = chosen[r < R ? r : 0].back();
            if (og) {
                switch (R) {
                    case 1: launch_pp_gram<1>(lasts); break;
                    case 2: launch_pp_gram<2>(lasts); break;
                    case 3: launch_pp_gram<3>(lasts); break;
                    case 4: launch_pp_gram<4>(lasts); break;
                    case 5: launch_pp_gram<5>(lasts); break;
                    case 6: launch_pp_gram<6>(lasts); break;
                    case 7: launch_pp_gram<7>(lasts); break;
                    default: launch_pp_gram<8>(lasts); break;
                }
            } else {
                switch (R) {
                    case 1: launch_pp_multi<1>(lasts); break;
                    case 2: launch_pp_multi<2>(lasts); break;
                    case 3: launch_pp_multi<3>(lasts); break;
                    case 4: launch_pp_multi<4>(lasts); break;
                    case 5: launch_pp_multi<5>(lasts); break;
                    case 6: launch_pp_multi<6>(lasts); break;
                    case 7: launch_pp_multi<7>(lasts); break;
                    default: launch_pp_multi<8>(lasts); break;
                }
            }
            CK(cudaMemcpyAsync(hd2, d2.p, sizeof(double) * R * n, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            if (og) {
                for (int r = 0; r < R; ++r) {
                    if (amb[r]) continue;
                    if (force_amb > 0 && (force_amb - 1) % R == r && p == std::min(3, c - 1)) {
                        amb[r] = 1;
                        continue;
                    }
                    const double* h = hd2 + (size_t)r * n;
                    double total = 0.0;
                    for (int j = 0; j < n; ++j) total += h[j];
                    // |total − reference total|: n values within E, two recursive sums of n terms
                    const double gn = (double)n * kU * 1.01;
                    const double ET = (double)n * E * (1.0 + gn) + 2.02 * gn * total;
                    if (!(total > 2.0 * ET) || std::isinf(total)) {  // `total > 0` not certain
                        amb[r] = 1;
                        continue;
                    }
                    std::uniform_real_distribution<double> u(0.0, total);
                    double rr = u(engs[r]);
                    // start value within ET + 3u·total; each step adds ≤ E + u·(2·total + ET)
                    const double B = (ET + 3.0 * kU * total) + (double)n * E + 2.2 * (double)n * kU * (total + ET);
                    int pick = n, hit = n;
                    for (int j = 0; j < n; ++j) {
                        rr -= h[j];
                        if (rr <= B) {
                            hit = j;
                            break;
                        }
                    }
                    if (hit < n && rr >= -B) {  // the sign of the reference's remainder is not certain here
                        amb[r] = 1;
                        continue;
                    }
                    // certainly ≤ 0 from column `hit` on (it only decreases): the first unchosen one
                    for (int j = hit; j < n; ++j)
                        if (!is_chosen[r][j]) {
                            pick = j;
                            break;
                        }
                    if (pick == n)
                        for (int j = 0; j < n; ++j)
                            if (!is_chosen[r][j]) {
                                pick = j;
                                break;
                            }
                    chosen[r].push_back(pick);
                    is_chosen[r][pick] = 1;
                }
                continue;
            }
            for (int r = 0; r < R; ++r) {  // kmeans.cpp:192-221, restart by restart
                const double* h = hd2 + (size_t)r * n;
                double total = 0.0;
                for (int j = 0; j < n; ++j) total += h[j];
                int pick = n;
                if (total > 0.0) {
                    std::uniform_real_distribution<double> u(0.0, total);
                    double rr = u(engs[r]);
                    for (int j = 0; j < n; ++j) {
                        rr -= h[j];
                        if (rr <= 0.0 && !is_chosen[r][j]) {
                            pick = j;
                            break;
                        }
                    }
                }
                if (pick == n)
                    for (int j = 0; j < n; ++j)
                        if (!is_chosen[r][j]) {
                            pick = j;
                            break;
                        }
                chosen[r].push_back(pick);
                is_chosen[r][pick] = 1;
            }
        }
        if (og && trace_on()) {
            int na = 0;
            for (int r = 0; r < R; ++r) na += amb[r];
            std::fprintf(stderr, "[respca] k-means++ on G: %d restarts, %d picks each, bound per value %.3g, %d to the exact chains\n",
                         R, c - 1, E, na);
        }
        for (int r = 0; r < R; ++r)
            if (amb[r]) {  // exact chains from the restart's start state
                engs[r] = start[r];
                chosen[r] = pp_init(engs[r]);
                ++pp_gram_fallbacks;
                if (trace_on()) std::fprintf(stderr, "[respca] k-means++ on G: restart %d seeded again on the exact chains\n", r);
            }
        return chosen;
    }

    void gather(const std::vector<int>& idx, double* C) {
        gidx.ensure(c);
        CK(cudaMemcpyAsync(gidx.p, idx.data(), sizeof(int) * c, cudaMemcpyHostToDevice, st));
        k_gather_cols<T><<<dim3(ceil_div(d, 256 * 4), c), 256, 0, st>>>(M, d, gidx.p, c, C);
        ln.add();
    }

    // full-screen split of screen_cols(M, n, …) (same formula)
    void reserve_full_screen() {
        const int tiles = ceil_div(n, tile_j()) * ceil_div(c, tile_k());
        const int chunks = ceil_div(d, 32);
        int ns = std::max(1, std::min(chunks / 4, ceil_div(2 * 148, tiles)));
        ns = std::min(ns, 64);
        part.ensure((size_t)ns * n * c);
        xxp.ensure((size_t)ns * n);
    }

    // number of restarts run side by side (one lane = engine + stream + host
    // thread each); RESPCA_KM_LANES overrides (tests)
    int lanes_for(uint64_t n_restarts) const {
        if (const char* e = std::getenv("RESPCA_KM_LANES")) {
            const int v = std::atoi(e);
            if (v >= 1) return (int)std::min<uint64_t>((uint64_t)v, std::max<uint64_t>(n_restarts, 1));
        }
        // small problems too: the restarts' latency-bound refinements run side by side
        // (C1, 500²: init 18.7 ms in order, 5.2 ms on five lanes)
        if (n_restarts < 2) return 1;
        return (int)std::min<uint64_t>(n_restarts, 8);
    }

    // kmeans (kmeans.cpp:237-250).  labels/C device outputs.
    void kmeans(uint64_t max_iters, uint64_t n_restarts, uint64_t seed, double tol, int* labels,
                double* C, double* inertia_out, uint64_t* iters_out) {
        if (c == 0) throw InvalidArg("kmeans: c must be >= 1");
        if ((int64_t)c > n) throw InvalidArg("kmeans: c exceeds column count");
        const int L = lanes_for(n_restarts);
        lloyd_margin = INFINITY;
        restart_inertia.assign(n_restarts, std::numeric_limits<double>::quiet_NaN());
        struct GramScope {
            KMeansEngine* e;
            ~GramScope() {
                e->drop_gram();
                e->gram_early = false;
            }
        } gram_scope{this};
        const bool want_gram = gram_early || gram_fits();
        const bool overlap = L > 1 && env_int("RESPCA_GRAM_OVERLAP", 1) != 0;
        if (want_gram && !overlap && !gram_early) compute_gram();
        if (L > 1) {
            kmeans_lanes(L, max_iters, n_restarts, seed, tol, labels, C, inertia_out, iters_out, want_gram && overlap);
        } else {
            std::mt19937_64 rng(seed);
            double best = std::numeric_limits<double>::infinity();
            DBuf<int> lab;
            DBuf<double> cen;
            lab.ensure(n);
            cen.ensure((size_t)d * c);
            bool have = false;
            for (uint64_t r = 0; r < n_restarts; ++r) {
                const auto tp = HClock::now();
                const std::vector<int> chosen = pp_init(rng);
                gather(chosen, cen.p);
                if (stats) stats->t_pp += since(tp);
                const uint64_t it = lloyd_run(cen.p, lab.p, max_iters, tol);
                const auto ti = HClock::now();
                const double in = inertia(cen.p, lab.p);
                restart_inertia[r] = in;
                if (stats) stats->t_inertia += since(ti);
                if (in < best) {  // kmeans.cpp:246
                    best = in;
                    have = true;
                    CK(cudaMemcpyAsync(labels, lab.p, sizeof(int) * n, cudaMemcpyDeviceToDevice, st));
                    CK(cudaMemcpyAsync(C, cen.p, sizeof(double) * d * c, cudaMemcpyDeviceToDevice, st));
                    if (inertia_out) *inertia_out = in;
                    if (iters_out) *iters_out = it;
                }
            }
            CK(cudaStreamSynchronize(st));
            if (!have && n_restarts > 0) {
                // every restart had a NaN inertia: the reference returns the
                // default-constructed result; mirror that as an error
                throw RuntimeErr("kmeans: no restart produced a finite inertia");
            }
        }
        if (stats && trace_on())
            std::fprintf(stderr,
                         "[respca] kmeans(X): %d lane(s); pp %.3fs lloyd %.3fs (%llu steps) hartigan %.3fs "
                         "(%llu rounds, %llu moves, %llu passes, %llu refreshes, round kernels %.3fs) inertia %.3fs "
                         "fallbacks %llu\n",
                         L, stats->t_pp, stats->t_lloyd, (unsigned long long)stats->lloyd_steps,
                         stats->t_hart, (unsigned long long)stats->hartigan_rounds,
                         (unsigned long long)stats->hartigan_moves,
                         (unsigned long long)stats->hartigan_passes,
                         (unsigned long long)stats->hartigan_refreshes, stats->t_hart_kernel,
                         stats->t_inertia,
                         (unsigned long long)stats->exact_fallbacks);
    }

    // The restarts of kmeans() side by side.  Restart r's k-means++ draws
    // must follow restart r−1's (one libstdc++ engine, kmeans.cpp:240), so the
    // seeding steps take turns; Lloyd, Hartigan and inertia of different
    // restarts then overlap on their own streams, each Hartigan kernel on
    // 1/L of the SMs (so every lane's cooperative grid can be resident at
    // once).  The winner is the reference's: the first restart with the
    // smallest inertia (strict <, kmeans.cpp:246); the first restart that
    // throws decides the exception.
    void kmeans_lanes(int L, uint64_t max_iters, uint64_t n_restarts, uint64_t seed, double tol,
                      int* labels, double* C, double* inertia_out, uint64_t* iters_out, bool want_gram = false) {
        int dev = 0, nsm = 148;
        CK(cudaGetDevice(&dev));
        CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        using Lane = KmLane<T>;
        const auto t_k0 = HClock::now();
        LanePool<T> local;
        std::vector<std::unique_ptr<Lane>>& lanes = (lane_pool ? *lane_pool : local).lanes;
        cudaEvent_t ready;
        CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
        CK(cudaEventRecord(ready, st));  // M is complete on the caller's stream
        // G = MᵀM on its own stream, overlapping the seeding and the Lloyd
        // steps; the refinements wait for it (gram_ev)
        // G = MᵀM on its own stream, overlapping the seedings and the Lloyd steps
        // (RESPCA_GRAM_AFTER_PP=1: after the seedings; measured equal or slower)
        const int gram_when = env_int("RESPCA_GRAM_AFTER_PP", 0);
        auto launch_gram = [&](cudaEvent_t after) {
            if (!gram_st) {
                int lo = 0, hi = 0;
                CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
                CK(cudaStreamCreateWithPriority(&gram_st, cudaStreamNonBlocking, lo));
            }
            CK(cudaStreamWaitEvent(gram_st, after, 0));
            compute_gram(gram_st);
        };
        if (want_gram) alloc_gram();  // pointers lent to the lanes below
        if (want_gram && !gram_when && !gram_early) launch_gram(ready);
        while ((int)lanes.size() < L) {
            lanes.emplace_back(new Lane());
            {
                int lo = 0, hi = 0;
                CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
                CK(cudaStreamCreateWithPriority(&lanes.back()->e.st, cudaStreamNonBlocking, hi));
            }
        }
        for (int l = 0; l < L; ++l) {
            Lane& ln_ = *lanes[l];
            ln_.reset();
            CK(cudaStreamWaitEvent(ln_.e.st, ready, 0));
            ln_.e.ln = Launch{&ln_.launches};
            ln_.e.stats = stats ? &ln_.st : nullptr;
            ln_.e.hart_ctas = std::max(1, nsm / L);
            ln_.e.bind(M, d, n, c);
            ln_.e.lloyd_margin = INFINITY;
            lend_gram(ln_.e);
            // every buffer a lane touches is allocated before the lanes run
            // (cudaFree would synchronise the device under them)
            ln_.e.reserve_full_screen();
            ln_.e.hart_reserve();
            ln_.e.d2.ensure(n);
            ln_.e.gidx.ensure(c);
            ln_.wl.ensure(n);
            ln_.bl.ensure(n);
            ln_.wc.ensure((size_t)d * c);
            ln_.bc.ensure((size_t)d * c);
        }
        CK(cudaEventDestroy(ready));
        if (trace_on()) std::fprintf(stderr, "[respca] lanes: %d set up in %.3fs\n", L, since(t_k0));
        // Restart r's seeding draws continue restart r−1's (one libstdc++
        // engine, kmeans.cpp:240): 1 uniform_int, then 1 uniform_real per pick
        // whose d² total is positive (kmeans.cpp:196-211) — c−1 of them unless
        // the data degenerate.  Seedings therefore start from SPECULATED engine
        // states (that count assumed) and are checked against the true state
        // once restart r−1's seeding is known; a mismatch redoes the seeding.
        std::vector<std::mt19937_64> spec(n_restarts), truth(n_restarts + 1);
        std::vector<char> truth_known(n_restarts + 1, 0);
        {
            std::mt19937_64 sim(seed);
            for (uint64_t r = 0; r < n_restarts; ++r) {
                spec[r] = sim;
                std::uniform_int_distribution<std::size_t> first(0, (std::size_t)n - 1);
                (void)first(sim);
                for (int p = 1; p < c; ++p) {
                    std::uniform_real_distribution<double> u(0.0, 1.0);
                    (void)u(sim);
                }
            }
            truth[0] = std::mt19937_64(seed);
            truth_known[0] = 1;
        }
        // the first ≤ 8 restarts seed side by side from their speculated states
        // (one pass over the columns per pick for all of them)
        std::vector<std::vector<int>> joint_chosen;
        std::vector<std::mt19937_64> joint_eng;
        if (n_restarts > 1 && env_int("RESPCA_PP_JOINT", 1) != 0) {
            const auto tj = HClock::now();
            joint_eng.assign(spec.begin(), spec.begin() + (size_t)std::min<uint64_t>(n_restarts, 8));
            Nvtx r_pp("k-means++ seeding (joint)");
            joint_chosen = pp_joint(joint_eng, want_gram && !gram_when);
            if (stats) stats->t_pp += since(tj);
        }
        if (want_gram && gram_when && !gram_early) {
            cudaEvent_t seeded;
            CK(cudaEventCreateWithFlags(&seeded, cudaEventDisableTiming));
            CK(cudaEventRecord(seeded, st));
            launch_gram(seeded);
            CK(cudaEventDestroy(seeded));
        }
        std::mutex mu;
        std::condition_variable cv;
        uint64_t abort_at = UINT64_MAX;    // restarts after a failed one are skipped
        std::vector<std::exception_ptr> errs(n_restarts);
        // a persistent Hartigan grid holds its SMs until it ends: no lane
        // starts one before every lane is past its seeding and Lloyd steps
        // (they need the whole GPU); lanes that stop early count as arrived
        std::vector<char> arrived(L, 0);
        int n_arrived = 0;
        auto arrive = [&](int l) {  // caller holds mu
            if (!arrived[l]) {
                arrived[l] = 1;
                ++n_arrived;
                cv.notify_all();
            }
        };
        for (int l = 0; l < L; ++l)
            lanes[l]->e.before_hartigan = [&, l] {
                std::unique_lock<std::mutex> lk(mu);
                arrive(l);
                cv.wait(lk, [&] { return n_arrived == L; });
            };
        auto body = [&](int l) {
            Lane& ln_ = *lanes[l];
            KMeansEngine<T>& e = ln_.e;
            struct Done {  // every exit path counts as arrived
                std::mutex& m;
                std::function<void()> f;
                ~Done() {
                    std::lock_guard<std::mutex> g(m);
                    f();
                }
            } done{mu, [&, l] { arrive(l); }};
            try {
                CK(cudaSetDevice(dev));
            } catch (...) {
                std::lock_guard<std::mutex> g(mu);
                errs[l] = std::current_exception();
                abort_at = std::min<uint64_t>(abort_at, (uint64_t)l);
                cv.notify_all();
                return;
            }
            for (uint64_t r = (uint64_t)l; r < n_restarts; r += (uint64_t)L) {
                try {
                    // seeding from the speculated engine state, then confirmed
                    // against the true one (redone from it on a mismatch)
                    const auto tp = HClock::now();
                    std::mt19937_64 eng = spec[r];
                    std::vector<int> chosen;
                    if (r < joint_chosen.size()) {
                        eng = joint_eng[r];
                        chosen = joint_chosen[r];
                    } else {
                        chosen = e.pp_init(eng);
                    }
                    std::mt19937_64 start;
                    {
                        std::unique_lock<std::mutex> lk(mu);
                        cv.wait(lk, [&] { return truth_known[r] || r > abort_at; });
                        if (r > abort_at) return;
                        start = truth[r];
                    }
                    if (!(start == spec[r])) {
                        eng = start;
                        chosen = e.pp_init(eng);
                        if (e.stats) e.stats->pp_respeculated += 1;
                    }
                    {
                        std::lock_guard<std::mutex> g(mu);
                        truth[r + 1] = eng;
                        truth_known[r + 1] = 1;
                    }
                    cv.notify_all();
                    e.gather(chosen, ln_.wc.p);
                    if (e.stats) e.stats->t_pp += since(tp);
                    const double t_pp_end = since(t_k0);
                    Nvtx r_lane("restart: lloyd + hartigan");
                    const uint64_t it = e.lloyd_run(ln_.wc.p, ln_.wl.p, max_iters, tol);
                    const auto ti = HClock::now();
                    const double in = e.inertia(ln_.wc.p, ln_.wl.p);
                    {
                        std::lock_guard<std::mutex> g(mu);
                        restart_inertia[r] = in;
                    }
                    if (e.stats) e.stats->t_inertia += since(ti);
                    if (trace_on())
                        std::fprintf(stderr, "[respca] lane %d restart %llu: seeded at %.3fs, done at %.3fs (lloyd %.3fs, hartigan %.3fs)\n", l,
                                     (unsigned long long)r, t_pp_end, since(t_k0), ln_.st.t_lloyd, ln_.st.t_hart);
                    if (in < ln_.best_in) {
                        ln_.best_in = in;
                        ln_.best_r = (int)r;
                        ln_.best_it = it;
                        CK(cudaMemcpyAsync(ln_.bl.p, ln_.wl.p, sizeof(int) * n, cudaMemcpyDeviceToDevice, e.st));
                        CK(cudaMemcpyAsync(ln_.bc.p, ln_.wc.p, sizeof(double) * d * c,
                                           cudaMemcpyDeviceToDevice, e.st));
                    }
                    CK(cudaStreamSynchronize(e.st));
                } catch (...) {
                    std::lock_guard<std::mutex> g(mu);
                    errs[r] = std::current_exception();
                    abort_at = std::min(abort_at, r);
                    cv.notify_all();
                    return;
                }
            }
        };
        std::vector<std::thread> threads;
        for (int l = 0; l < L; ++l) threads.emplace_back(body, l);
        for (auto& t : threads) t.join();
        for (int l = 0; l < L; ++l) lanes[l]->e.drop_gram();
        if (trace_on()) std::fprintf(stderr, "[respca] lanes joined at %.3fs\n", since(t_k0));
        for (int l = 0; l < L; ++l) {
            auto& lp = lanes[l];
            *ln.counter += lp->launches;
            lloyd_margin = std::min(lloyd_margin, lp->e.lloyd_margin);
            if (stats) {
                const Stats& s2 = lp->st;
                stats->hartigan_moves += s2.hartigan_moves;
                stats->exact_fallbacks += s2.exact_fallbacks;
                stats->lloyd_steps += s2.lloyd_steps;
                stats->hartigan_passes += s2.hartigan_passes;
                stats->hartigan_rounds += s2.hartigan_rounds;
                stats->hartigan_refreshes += s2.hartigan_refreshes;
                stats->pp_respeculated += s2.pp_respeculated;
                stats->t_pp += s2.t_pp;
                stats->t_lloyd += s2.t_lloyd;
                stats->t_hart += s2.t_hart;
                stats->t_inertia += s2.t_inertia;
                stats->t_hart_kernel += s2.t_hart_kernel;
            }
        }
        for (uint64_t r = 0; r < n_restarts; ++r)
            if (errs[r]) std::rethrow_exception(errs[r]);
        int bl = -1;
        for (int l = 0; l < L; ++l) {
            const Lane& x = *lanes[l];
            if (x.best_r < 0) continue;
            if (bl < 0 || x.best_in < lanes[bl]->best_in ||
                (x.best_in == lanes[bl]->best_in && x.best_r < lanes[bl]->best_r))
                bl = l;
        }
        if (bl < 0) throw RuntimeErr("kmeans: no restart produced a finite inertia");
        const Lane& w = *lanes[bl];
        CK(cudaMemcpyAsync(labels, w.bl.p, sizeof(int) * n, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(C, w.bc.p, sizeof(double) * d * c, cudaMemcpyDeviceToDevice, st));
        CK(cudaStreamSynchronize(st));
        if (inertia_out) *inertia_out = w.best_in;
        if (iters_out) *iters_out = w.best_it;
    }
};

// a context's k-means engine for solve() (buffers reused across solves)
template <typename T>
struct EngineHolder : PoolBase {
    KMeansEngine<T> e;
};

template <typename T>
struct KmLane {
    KMeansEngine<T> e;
    uint64_t launches = 0;
    Stats st;
    DBuf<int> wl, bl;
    DBuf<double> wc, bc;
    int best_r = -1;
    double best_in = std::numeric_limits<double>::infinity();
    uint64_t best_it = 0;
    void reset() {
        launches = 0;
        st = Stats{};
        best_r = -1;
        best_in = std::numeric_limits<double>::infinity();
        best_it = 0;
    }
    ~KmLane() {
        if (e.st) cudaStreamDestroy(e.st);
    }
};

template <typename T>
__global__ void k_colsq_T(const T* __restrict__ M, int64_t d, double* __restrict__ out) {
    __shared__ double red[32];
    const int j = blockIdx.x;
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < d; i += blockDim.x) {
        const double v = (double)M[(int64_t)j * d + i];
        s = __fma_rn(v, v, s);
    }
    double v[1] = {s};
    block_sum<1>(v, red);
    if (threadIdx.x == 0) out[j] = v[0];
}

template <typename T>
void KMeansEngine<T>::k_col_sq_fma_T(const T* m, int cols, double* out) {
    k_colsq_T<T><<<cols, 256, 0, st>>>(m, d, out);
    ln.add();
}

}  // namespace respca_host
