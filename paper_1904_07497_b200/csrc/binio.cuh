// RESPCA1 binary matrices (io.hpp:66-69, io.cpp:138-164) streamed straight
// between disk and HBM.  Two pinned chunks per
// direction: the file read of chunk k+1 overlaps the host→device copy of
// chunk k, and the device→host copy of chunk k+1 overlaps the file write of
// chunk k.  The file payload is always f64; fp32 storage converts on the
// device.  Errors carry the reference's io::IoError messages.
#pragma once

#include <cstdio>
#include <cstring>
#include <string>

#include "engine.cuh"

namespace respca_dev {

template <typename T>
__global__ void k_f64_to(const double* __restrict__ a, T* __restrict__ b, int64_t n) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        b[k] = (T)a[k];
}
template <typename T>
__global__ void k_to_f64(const T* __restrict__ a, double* __restrict__ b, int64_t n) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        b[k] = (double)a[k];
}

}  // namespace respca_dev

namespace respca_host {

constexpr char kBinMagic[8] = {'R', 'E', 'S', 'P', 'C', 'A', '1', '\0'};
constexpr size_t kBinChunk = (size_t)8 << 20;  // doubles per streamed chunk (64 MB)

// pinned double-buffer + events, kept by the context across calls
struct StreamBufs {
    HBuf pin[2];
    cudaEvent_t ev[2] = {nullptr, nullptr};
    DBuf<double> stage;  // fp32 conversion staging
    void init() {
        for (int b = 0; b < 2; ++b)
            if (!ev[b]) CK(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming));
    }
    ~StreamBufs() {
        for (int b = 0; b < 2; ++b)
            if (ev[b]) cudaEventDestroy(ev[b]);
    }
};

// io.cpp:138-153: magic, rows, cols; the payload must hold rows*cols doubles
struct BinReader {
    FILE* f = nullptr;
    std::string path;
    uint64_t rows = 0, cols = 0;
    explicit BinReader(const std::string& p) : path(p) {
        f = std::fopen(p.c_str(), "rb");
        if (!f) throw IoErr("cannot open " + p);
        char magic[8];
        if (std::fread(magic, 1, 8, f) != 8) throw IoErr("binary matrix: file too short");
        if (std::memcmp(magic, kBinMagic, 8) != 0) throw IoErr("binary matrix: bad magic in " + p);
        rows = u64();
        cols = u64();
        const off_t here = ftello(f);
        if (fseeko(f, 0, SEEK_END) != 0) throw IoErr("cannot seek " + p);
        const unsigned long long avail = (unsigned long long)(ftello(f) - here);
        if (fseeko(f, here, SEEK_SET) != 0) throw IoErr("cannot seek " + p);
        const unsigned __int128 need = (unsigned __int128)rows * cols * 8u;
        if (need > (unsigned __int128)avail) throw IoErr("binary matrix: truncated payload in " + p);
    }
    uint64_t u64() {
        unsigned char b[8];
        if (std::fread(b, 1, 8, f) != 8) throw IoErr("binary matrix: truncated header");
        uint64_t v = 0;
        for (int i = 0; i < 8; ++i) v |= (uint64_t)b[i] << (8 * i);
        return v;
    }
    ~BinReader() {
        if (f) std::fclose(f);
    }
    // payload → device (T storage), N = rows*cols elements
    template <typename T>
    void to_device(T* dst, int64_t N, cudaStream_t st, StreamBufs& sb, uint64_t* launches) {
        sb.init();
        for (int64_t off = 0, k = 0; off < N; off += (int64_t)kBinChunk, ++k) {
            const size_t cnt = (size_t)std::min<int64_t>((int64_t)kBinChunk, N - off);
            double* hb = sb.pin[k & 1].ensure<double>(kBinChunk);
            if (k >= 2) CK(cudaEventSynchronize(sb.ev[k & 1]));  // its last copy is done
            if (std::fread(hb, sizeof(double), cnt, f) != cnt)
                throw IoErr("binary matrix: truncated payload in " + path);
            if (sizeof(T) == sizeof(double)) {
                CK(cudaMemcpyAsync((void*)(dst + off), hb, cnt * sizeof(double), cudaMemcpyHostToDevice, st));
            } else {
                double* dv = sb.stage.ensure(kBinChunk);
                CK(cudaMemcpyAsync(dv, hb, cnt * sizeof(double), cudaMemcpyHostToDevice, st));
                respca_dev::k_f64_to<T><<<592, 256, 0, st>>>(dv, dst + off, (int64_t)cnt);
                if (launches) ++*launches;
            }
            CK(cudaEventRecord(sb.ev[k & 1], st));
        }
    }
};

// io.cpp:156-164
template <typename T>
void write_binary_from_device(const std::string& path, const T* src, uint64_t rows, uint64_t cols,
                              cudaStream_t st, StreamBufs& sb, uint64_t* launches) {
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw IoErr("cannot open " + path + " for writing");
    struct Closer {
        FILE* f;
        ~Closer() {
            if (f) std::fclose(f);
        }
    } closer{f};
    unsigned char hdr[24];
    std::memcpy(hdr, kBinMagic, 8);
    for (int i = 0; i < 8; ++i) hdr[8 + i] = (unsigned char)(rows >> (8 * i));
    for (int i = 0; i < 8; ++i) hdr[16 + i] = (unsigned char)(cols >> (8 * i));
    if (std::fwrite(hdr, 1, 24, f) != 24) throw IoErr("cannot write " + path);
    sb.init();
    const int64_t N = (int64_t)(rows * cols);
    size_t prev_cnt = 0;
    int64_t k = 0;
    auto flush = [&](int64_t kk, size_t cnt) {
        CK(cudaEventSynchronize(sb.ev[kk & 1]));
        if (std::fwrite(sb.pin[kk & 1].p, sizeof(double), cnt, f) != cnt) throw IoErr("cannot write " + path);
    };
    for (int64_t off = 0; off < N; off += (int64_t)kBinChunk, ++k) {
        const size_t cnt = (size_t)std::min<int64_t>((int64_t)kBinChunk, N - off);
        double* hb = sb.pin[k & 1].ensure<double>(kBinChunk);
        if (sizeof(T) == sizeof(double)) {
            CK(cudaMemcpyAsync(hb, (const void*)(src + off), cnt * sizeof(double), cudaMemcpyDeviceToHost, st));
        } else {
            double* dv = sb.stage.ensure(kBinChunk);
            respca_dev::k_to_f64<T><<<592, 256, 0, st>>>(src + off, dv, (int64_t)cnt);
            if (launches) ++*launches;
            CK(cudaMemcpyAsync(hb, dv, cnt * sizeof(double), cudaMemcpyDeviceToHost, st));
        }
        CK(cudaEventRecord(sb.ev[k & 1], st));
        if (k >= 1) flush(k - 1, prev_cnt);  // overlaps this chunk's copy
        prev_cnt = cnt;
    }
    if (k >= 1) flush(k - 1, prev_cnt);
    if (std::fflush(f) != 0) throw IoErr("cannot write " + path);
}

}  // namespace respca_host
