// What a plain, perfectly coalesced kernel with Pass F's traffic mix (4 arrays in, 3 out, in place)
// reaches on this GPU, next to a 1:1 copy — the practical ceiling for the fused ALM pass.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_copy(const double2* __restrict__ a, double2* __restrict__ b, size_t n2) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void k_mix(const double2* __restrict__ x, double2* __restrict__ l, double2* __restrict__ s, double2* __restrict__ t,
                      size_t n2, double w) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
        const double2 X = __ldg(x + i), L = l[i], S = s[i], T = t[i];
        double2 ln, sn, tn;
        ln.x = w * ((X.x - S.x) + T.x) + L.x * 1e-30; ln.y = w * ((X.y - S.y) + T.y) + L.y * 1e-30;
        sn.x = (X.x - ln.x) + T.x; sn.y = (X.y - ln.y) + T.y;
        tn.x = T.x + w * ((X.x - ln.x) - sn.x); tn.y = T.y + w * ((X.y - ln.y) - sn.y);
        __stcs(l + i, ln); __stcs(s + i, sn); __stcs(t + i, tn);
    }
}
int main() {
    const size_t N = 100000000ull, n2 = N / 2;
    double2 *x, *l, *s, *t;
    cudaMalloc(&x, N * 8); cudaMalloc(&l, N * 8); cudaMalloc(&s, N * 8); cudaMalloc(&t, N * 8);
    cudaMemset(x, 0, N * 8); cudaMemset(l, 0, N * 8); cudaMemset(s, 0, N * 8); cudaMemset(t, 0, N * 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int grid : {148 * 4, 148 * 8, 148 * 16, 148 * 32}) for (int bs : {256, 512}) {
        float ms;
        for (int w = 0; w < 3; ++w) k_copy<<<grid, bs>>>(x, l, n2);
        cudaEventRecord(a); for (int r = 0; r < 20; ++r) k_copy<<<grid, bs>>>(x, l, n2); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b); const double copy = 2.0 * N * 8 / (ms / 20 * 1e-3) / 1e9;
        for (int w = 0; w < 3; ++w) k_mix<<<grid, bs>>>(x, l, s, t, n2, 0.5);
        cudaEventRecord(a); for (int r = 0; r < 20; ++r) k_mix<<<grid, bs>>>(x, l, s, t, n2, 0.5); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b); const double mix = 7.0 * N * 8 / (ms / 20 * 1e-3) / 1e9;
        printf("grid %5d block %3d: copy %.0f GB/s, 4-in/3-out %.0f GB/s (%.3f ms per pass, %.3f of this copy)\n", grid, bs, copy, mix, ms / 20, mix / copy);
    }
    return 0;
}
