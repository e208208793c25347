#include <cstdio>
#include <cuda_runtime.h>
constexpr int kThreads = 512, kWarps = 16, kLd = 33;
__device__ void gram_ab(const double* A, const double* B, double* C, int n, int b) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int e = warp; e < b * b; e += kWarps) {
        const int j = e / b, i = e - j * b;
        if (i > j) continue;
        const double* a = A + (size_t)i * n;
        const double* c = B + (size_t)j * n;
        double s = 0.0;
        for (int r = lane; r < n; r += 32) s = fma(a[r], c[r], s);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) { C[i + j * kLd] = s; C[j + i * kLd] = s; }
    }
    __syncthreads();
}
__global__ void k(double* out, long long* cyc, int n, int b, int reps) {
    extern __shared__ double sm[];
    double* X = sm; double* S = X + n * b;
    for (int e = threadIdx.x; e < n * b; e += kThreads) X[e] = 1.0 / (1 + e);
    __syncthreads();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) gram_ab(X, X, S, n, b);
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = S[5]; }
}
__global__ void k2(double* out, long long* cyc, int n, int b, int reps) {   // no sync variant timing per call split
    extern __shared__ double sm[];
    double* X = sm; double* S = X + n * b;
    for (int e = threadIdx.x; e < n * b; e += kThreads) X[e] = 1.0 / (1 + e);
    __syncthreads();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) { __syncthreads(); }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = S[5]; }
}
int main() {
    double* d; long long* c; long long h;
    cudaMalloc(&d, 64); cudaMalloc(&c, 64);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    k<<<1, 512, (100 * 16 + 33 * 32) * 8>>>(d, c, 100, 16, 100);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("gram_ab n=100 b=16: %.0f cycles per call (%.2f us)\n", h / 100.0, h / 100.0 / 1965.0);
    k2<<<1, 512, (100 * 16 + 33 * 32) * 8>>>(d, c, 100, 16, 1000);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("syncthreads: %.0f cycles\n", h / 1000.0);
    cudaError_t e = cudaGetLastError(); printf("%s\n", cudaGetErrorString(e));
}
