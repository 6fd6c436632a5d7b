// Host-side engine infrastructure: errors, device buffers, launch accounting,
// conditional CUDA graphs.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <stdexcept>
#include <string>
#include <vector>

#include "respca_cu.h"

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
        if (p && owned) cudaFree(p);
    }
    U* ensure(size_t count) {
        if (count == 0) count = 1;
        if (count > cap) {
            if (p && owned) cudaFree(p);
            p = nullptr;
            cap = 0;
            owned = true;
            CK(cudaMalloc(&p, count * sizeof(U)));
            cap = count;
            g_alloc_gen.fetch_add(1);
        }
        return p;
    }
    void borrow(void* q, size_t count) {  // arena memory, never freed here
        if (p && owned) cudaFree(p);
        if (p != q) g_alloc_gen.fetch_add(1);
        p = static_cast<U*>(q);
        cap = count;
        owned = false;
    }
    void release() {
        if (p && owned) cudaFree(p);
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
                    cudaFree(kv.second.p);
                    kv.second.p = nullptr;
                    kv.second.bytes = 0;
                    CK(cudaMalloc(&kv.second.p, bytes));
                    kv.second.bytes = bytes;
                    g_alloc_gen.fetch_add(1);
                }
                return kv.second.p;
            }
        Slot sl;
        CK(cudaMalloc(&sl.p, bytes));
        sl.bytes = bytes;
        g_alloc_gen.fetch_add(1);
        slots.emplace_back(name, sl);
        return sl.p;
    }
    ~Arena() {
        for (auto& kv : slots)
            if (kv.second.p) cudaFree(kv.second.p);
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
