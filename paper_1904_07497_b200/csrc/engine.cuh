// Host-side engine infrastructure: errors, device buffers, launch accounting,
// conditional CUDA graphs.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "respca_cu.h"
#include <nvtx3/nvToolsExt.h>

namespace respca_host {

struct InvalidArg : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct RuntimeErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NoMem : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NonFinite : std::runtime_error {
    using std::runtime_error::runtime_error;
};
// io::IoError and its subclasses (io.hpp:13-33): file open/format/size errors
struct IoErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void ck(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        throw NoMem(std::string("device allocation failed: ") + what);
    }
    throw CudaErr(std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) ::respca_host::ck((x), #x)

// ---------------------------------------------------------------------------
// Guarded allocations (RESPCA_GUARD=1; tests only).  compute-sanitizer is not
// available on the GPU pool, so device memory checking is done here: every
// allocation is poisoned (0xFF bytes: NaN doubles/floats, −1 ints — a read
// of memory no kernel wrote shows up as a result that differs from the
// oracle) and followed by a 4 KiB guard of 0xA5 bytes, which
// respca_cu_debug_guards() verifies (any write past the end of a buffer).
// ---------------------------------------------------------------------------
constexpr size_t kGuardBytes = 4096;
inline bool guard_on() {
    static const bool on = [] {
        const char* e = std::getenv("RESPCA_GUARD");
        return e && e[0] == '1';
    }();
    return on;
}
struct GuardRec {
    void* p;
    size_t bytes;
};
inline std::mutex& guard_mu() {
    static std::mutex m;
    return m;
}
inline std::vector<GuardRec>& guard_list() {
    static std::vector<GuardRec> v;
    return v;
}
inline cudaError_t dev_alloc(void** p, size_t bytes) {
    if (!guard_on()) return cudaMalloc(p, bytes);
    cudaError_t e = cudaMalloc(p, bytes + kGuardBytes);
    if (e != cudaSuccess) return e;
    // on a stream of its own: allocations also happen while another stream is
    // being captured into a graph, where device-wide synchronisation is illegal
    static cudaStream_t gs = [] {
        cudaStream_t s = nullptr;
        cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
        return s;
    }();
    cudaMemsetAsync(*p, 0xFF, bytes, gs);
    cudaMemsetAsync(static_cast<char*>(*p) + bytes, 0xA5, kGuardBytes, gs);
    cudaStreamSynchronize(gs);
    std::lock_guard<std::mutex> g(guard_mu());
    guard_list().push_back({*p, bytes});
    return cudaSuccess;
}
// number of guards found overwritten (the first few described in `msg`)
inline int guard_check(std::string* msg = nullptr) {
    if (!guard_on()) return 0;
    std::lock_guard<std::mutex> g(guard_mu());
    cudaDeviceSynchronize();
    int bad = 0;
    std::vector<unsigned char> h(kGuardBytes);
    for (const GuardRec& r : guard_list()) {
        cudaMemcpy(h.data(), static_cast<char*>(r.p) + r.bytes, kGuardBytes, cudaMemcpyDeviceToHost);
        size_t off = kGuardBytes;
        for (size_t k = 0; k < kGuardBytes; ++k)
            if (h[k] != 0xA5) {
                off = k;
                break;
            }
        if (off != kGuardBytes) {
            if (msg && bad < 8)
                *msg += "guard overwritten: buffer of " + std::to_string(r.bytes) + " bytes, first bad byte +" +
                        std::to_string(off) + "; ";
            ++bad;
        }
    }
    return bad;
}
// guard mode never returns memory: a freed buffer keeps its guard checked by
// guard_check() (tests are small), and no synchronising call can land inside
// a stream capture
inline void dev_free(void* p) {
    if (!p || guard_on()) return;
    cudaFree(p);
}

// bumped whenever device memory behind a DBuf / Arena slot changes address:
// captured CUDA graphs bake pointers in, so a graph is re-captured when this
// moved since its capture
inline std::atomic<uint64_t> g_alloc_gen{0};

template <class U>
struct DBuf {
    U* p = nullptr;
    size_t cap = 0;
    bool owned = true;  // false: memory lent by a context Arena
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() {
        if (p && owned) dev_free(p);
    }
    U* ensure(size_t count) {
        if (count == 0) count = 1;
        if (count > cap) {
            if (p && owned) dev_free(p);
            p = nullptr;
            cap = 0;
            owned = true;
            CK(dev_alloc(reinterpret_cast<void**>(&p), count * sizeof(U)));
            cap = count;
            g_alloc_gen.fetch_add(1);
        }
        return p;
    }
    void borrow(void* q, size_t count) {  // arena memory, never freed here
        if (p && owned) dev_free(p);
        if (p != q) g_alloc_gen.fetch_add(1);
        p = static_cast<U*>(q);
        cap = count;
        owned = false;
    }
    void release() {
        if (p && owned) dev_free(p);
        p = nullptr;
        cap = 0;
    }
};

// Device memory a context keeps across solves (named slots that only grow):
// repeated solves skip cudaMalloc/cudaFree of the N-sized state, whose cost
// (and cudaFree's implicit device synchronisation) is erratic at GB sizes.
struct Arena {
    struct Slot {
        void* p = nullptr;
        size_t bytes = 0;
    };
    std::vector<std::pair<std::string, Slot>> slots;
    void* get(const std::string& name, size_t bytes) {
        for (auto& kv : slots)
            if (kv.first == name) {
                if (kv.second.bytes < bytes) {
                    dev_free(kv.second.p);
                    kv.second.p = nullptr;
                    kv.second.bytes = 0;
                    CK(dev_alloc(&kv.second.p, bytes));
                    kv.second.bytes = bytes;
                    g_alloc_gen.fetch_add(1);
                }
                return kv.second.p;
            }
        Slot sl;
        CK(dev_alloc(&sl.p, bytes));
        sl.bytes = bytes;
        g_alloc_gen.fetch_add(1);
        slots.emplace_back(name, sl);
        return sl.p;
    }
    ~Arena() {
        for (auto& kv : slots)
            if (kv.second.p) dev_free(kv.second.p);
    }
};

// type-erased holder for per-context pools (k-means restart lanes)
struct PoolBase {
    virtual ~PoolBase() = default;
};

// pinned host staging buffer
struct HBuf {
    void* p = nullptr;
    size_t cap = 0;
    ~HBuf() {
        if (p) cudaFreeHost(p);
    }
    template <class U>
    U* ensure(size_t count) {
        size_t bytes = count * sizeof(U);
        if (bytes == 0) bytes = 8;
        if (bytes > cap) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            CK(cudaMallocHost(&p, bytes));
            cap = bytes;
        }
        return static_cast<U*>(p);
    }
};

struct Events {
    cudaEvent_t a = nullptr, b = nullptr;
    Events() {
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
    }
    ~Events() {
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
    }
    float ms() {
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, a, b));
        return t;
    }
};

// NVTX range for profilers (nsys / ncu --nvtx): solve phases, k-means phases
struct Nvtx {
    explicit Nvtx(const char* name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
    Nvtx(const Nvtx&) = delete;
    Nvtx& operator=(const Nvtx&) = delete;
};

// A graph whose body runs while the device keeps a conditional handle set.
struct WhileGraph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraph_t body = nullptr;
    cudaGraphConditionalHandle handle{};
    int kernels_per_iter = 0;
    ~WhileGraph() { reset(); }
    void reset() {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        exec = nullptr;
        graph = nullptr;
        body = nullptr;
    }
    bool ready() const { return exec != nullptr; }
    // begin: creates the outer graph + WHILE node and starts capturing `st`
    // into its body.  The captured kernels must set the handle to 0 to stop.
    void begin(cudaStream_t st) {
        reset();
        CK(cudaGraphCreate(&graph, 0));
        CK(cudaGraphConditionalHandleCreate(&handle, graph, 1u, cudaGraphCondAssignDefault));
        cudaGraphNodeParams prm = {};
        prm.type = cudaGraphNodeTypeConditional;
        prm.conditional.handle = handle;
        prm.conditional.type = cudaGraphCondTypeWhile;
        prm.conditional.size = 1;
        cudaGraphNode_t node;
        CK(cudaGraphAddNode(&node, graph, nullptr, 0, &prm));
        body = prm.conditional.phGraph_out[0];
        CK(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0,
                                         cudaStreamCaptureModeRelaxed));
    }
    void end(cudaStream_t st) {
        cudaGraph_t out = nullptr;
        CK(cudaStreamEndCapture(st, &out));
        CK(cudaGraphInstantiate(&exec, graph, 0));
    }
    void launch(cudaStream_t st) { CK(cudaGraphLaunch(exec, st)); }
};

// plain captured graph
struct PlainGraph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    ~PlainGraph() { reset(); }
    void reset() {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        exec = nullptr;
        graph = nullptr;
    }
    void begin(cudaStream_t st) {
        reset();
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
    }
    void end(cudaStream_t st) {
        CK(cudaStreamEndCapture(st, &graph));
        CK(cudaGraphInstantiate(&exec, graph, 0));
    }
    void launch(cudaStream_t st) { CK(cudaGraphLaunch(exec, st)); }
};

}  // namespace respca_host
