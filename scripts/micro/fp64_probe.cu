// Microbenchmark: DFMA / FFMA throughput + dependent latency, smem load latency.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_tput(double* out, int iters) {
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double b = 1.0000001, c = 1e-9;
    for (int i = 0; i < iters; ++i) {
        a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
        a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void ffma_tput(float* out, int iters) {
    float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const float b = 1.0000001f, c = 1e-9f;
    for (int i = 0; i < iters; ++i) {
        a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
        a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void dfma_lat(double* out, long long* cyc, int iters) {
    double a = threadIdx.x;
    const double b = 1.0000001, c = 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) a = fma(a, b, c);
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void smem_lat(double* out, long long* cyc, int iters) {
    __shared__ int idx[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i * 33 + 7) & 1023;
    __syncthreads();
    int p = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) p = idx[p];
    long long t1 = clock64();
    out[threadIdx.x] = p;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void sync_cost(double* out, long long* cyc, int iters) {
    __shared__ double s[512];
    double a = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        s[threadIdx.x] = a;
        __syncthreads();
        a += s[(threadIdx.x + 1) & 511];
        __syncthreads();
    }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    double* d; float* f; long long* cyc;
    cudaMalloc(&d, 148 * 1024 * 8 * 8); cudaMalloc(&f, 148 * 1024 * 8 * 4); cudaMalloc(&cyc, 64);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int iters = 20000; float ms;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a); dfma_tput<<<148 * 4, 512>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("DFMA throughput: %.2f TFLOP/s\n", 148.0 * 4 * 512 * 8 * iters * 2 / (ms * 1e-3) / 1e12);
        cudaEventRecord(a); ffma_tput<<<148 * 4, 512>>>(f, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("FFMA throughput: %.2f TFLOP/s\n", 148.0 * 4 * 512 * 8 * iters * 2 / (ms * 1e-3) / 1e12);
    }
    long long h;
    dfma_lat<<<1, 32>>>(d, cyc, 10000); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.1f cycles\n", h / 10000.0);
    smem_lat<<<1, 32>>>(d, cyc, 10000); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("LDS dependent latency: %.1f cycles\n", h / 10000.0);
    sync_cost<<<1, 512>>>(d, cyc, 10000); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("syncthreads x2 + STS/LDS round (512 thr): %.1f cycles\n", h / 10000.0);
    return 0;
}
