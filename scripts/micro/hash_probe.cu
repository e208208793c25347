// Ceiling probe for the sampler: stream a float tensor, SplitMix64 keep rule
// per element, count only (no compaction).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 hash_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256) probe(const float4* __restrict__ x, long long n4, unsigned long long seed,
                                             unsigned thr_hi, int mode, unsigned long long* out) {
    unsigned cnt = 0;
    float acc = 0.f;
    for (long long i = blockIdx.x * 256ll + threadIdx.x; i < n4; i += (long long)gridDim.x * 256) {
        const float4 v = __ldcs(x + i);
        if (mode == 0) { acc += v.x + v.y + v.z + v.w; continue; }
        const float xv[4] = {v.x, v.y, v.z, v.w};
        const unsigned long long z0 = seed + (unsigned long long)(4 * i + 1) * 0x9E3779B97F4A7C15ULL;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const unsigned long long z = z0 + (unsigned long long)j * 0x9E3779B97F4A7C15ULL;
            const unsigned zl = (unsigned)z, zh = (unsigned)(z >> 32);
            const unsigned al = zl ^ __funnelshift_r(zl, zh, 30), ah = zh ^ (zh >> 30);
            const unsigned long long pm = (unsigned long long)al * 0x1CE4E5B9u;
            const unsigned yl = (unsigned)pm;
            const unsigned yh = (unsigned)(pm >> 32) + al * 0xBF58476Du + ah * 0x1CE4E5B9u;
            const unsigned bl = yl ^ __funnelshift_r(yl, yh, 27), bh = yh ^ (yh >> 27);
            const unsigned zhi = __umulhi(bl, 0x133111EBu) + bl * 0x94D049BBu + bh * 0x133111EBu;
            const unsigned hhi = zhi ^ (zhi >> 31);
            cnt += (xv[j] != 0.f) & (hhi < thr_hi);
        }
    }
    if (acc == 12345.f) cnt += 1;
    atomicAdd(out, (unsigned long long)cnt);
}
int main() {
    const long long n = 134217728ll * 8;  // C5-size floats
    float* x; unsigned long long* out;
    cudaMalloc(&x, n * 4); cudaMalloc(&out, 8);
    cudaMemset(x, 0x3f, n * 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode = 0; mode < 2; ++mode)
        for (int per = 2; per <= 16; per *= 2) {
            float best = 1e9;
            for (int r = 0; r < 5; ++r) {
                cudaMemset(out, 0, 8);
                cudaEventRecord(a);
                probe<<<sms * per, 256>>>((const float4*)x, n / 4, 7, 0x0CCCCCCCu, mode, out);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
            }
            printf("mode %d ctas/sm %2d: %.3f ms  %.0f GB/s  %.2f Gel/s\n", mode, per, best, n * 4 / best / 1e6, n / best / 1e6);
        }
    return 0;
}
