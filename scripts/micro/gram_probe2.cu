#include <cstdio>
#include <cuda_runtime.h>
constexpr int kThreads = 512, kWarps = 16, kLd = 33;
template <int MODE>
__device__ void gram_ab(const double* A, const double* B, double* C, int n, int b) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int e = warp; e < b * b; e += kWarps) {
        const int j = e / b, i = e - j * b;
        if (i > j) continue;
        const double* a = A + (size_t)i * n;
        const double* c = B + (size_t)j * n;
        double s = 0.0;
        if (MODE != 2)
            for (int r = lane; r < n; r += 32) s = fma(a[r], c[r], s);
        if (MODE != 1) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        }
        if (lane == 0) { C[i + j * kLd] = s; C[j + i * kLd] = s; }
    }
    __syncthreads();
}
template <int MODE>
__global__ void k(double* out, long long* cyc, int n, int b, int reps) {
    extern __shared__ double sm[];
    double* X = sm; double* S = X + n * b;
    for (int e = threadIdx.x; e < n * b; e += kThreads) X[e] = 1.0 / (1 + e);
    __syncthreads();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) gram_ab<MODE>(X, X, S, n, b);
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = S[5]; }
}
__global__ void kf(float* out, long long* cyc, int reps) {  // float shuffle reduce chain only
    float s = threadIdx.x;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = s; }
}
__global__ void kd(double* out, long long* cyc, int reps) {
    double s = threadIdx.x;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = s; }
}
int main() {
    double* d; long long* c; long long h; float* f;
    cudaMalloc(&d, 64); cudaMalloc(&c, 64); cudaMalloc(&f, 64);
    const int sm = (100 * 16 + 33 * 32) * 8;
    k<0><<<1, 512, sm>>>(d, c, 100, 16, 100); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("full: %.0f cycles/call\n", h / 100.0);
    k<1><<<1, 512, sm>>>(d, c, 100, 16, 100); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("dot only: %.0f cycles/call\n", h / 100.0);
    k<2><<<1, 512, sm>>>(d, c, 100, 16, 100); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("shuffle only: %.0f cycles/call\n", h / 100.0);
    kf<<<1, 32>>>(f, c, 1000); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("1 warp float 5-level shfl reduce: %.0f cycles\n", h / 1000.0);
    kd<<<1, 32>>>(d, c, 1000); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("1 warp double 5-level shfl reduce: %.0f cycles\n", h / 1000.0);
    kd<<<1, 512>>>(d, c, 1000); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("16 warps double 5-level shfl reduce: %.0f cycles\n", h / 1000.0);
}
