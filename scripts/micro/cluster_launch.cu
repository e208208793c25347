// Launch overhead of a 16-CTA cluster kernel with large dynamic shared memory
// versus a plain one-CTA kernel (event-timed, back-to-back launches).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cluster(int* out) {
    extern __shared__ double sm[];
    cg::cluster_group c = cg::this_cluster();
    if (threadIdx.x == 0) sm[0] = 1.0;
    c.sync();
    if (threadIdx.x == 0 && c.block_rank() == 0) out[0] += static_cast<int>(sm[0]);
}
__global__ void k_plain(int* out) {
    extern __shared__ double sm[];
    if (threadIdx.x == 0) sm[0] = 1.0;
    __syncthreads();
    if (threadIdx.x == 0) out[0] += static_cast<int>(sm[0]);
}

int main() {
    int* d;
    cudaMalloc(&d, 4);
    cudaMemset(d, 0, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int smemkb : {16, 100, 200, 225}) {
        for (int cl : {1, 8, 16}) {
            const size_t smem = smemkb * 1024;
            cudaFuncSetAttribute(k_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            cudaFuncSetAttribute(k_plain, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(cl);
            cfg.blockDim = dim3(256);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cl;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            for (int w = 0; w < 10; ++w) cudaLaunchKernelEx(&cfg, k_cluster, d);
            cudaEventRecord(a);
            for (int i = 0; i < 100; ++i) cudaLaunchKernelEx(&cfg, k_cluster, d);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("cluster %2d smem %3d KB: %.2f us/launch (%s)\n", cl, smemkb, ms * 10, cudaGetErrorString(cudaGetLastError()));
        }
        for (int w = 0; w < 10; ++w) k_plain<<<1, 256, smemkb * 1024>>>(d);
        cudaEventRecord(a);
        for (int i = 0; i < 100; ++i) k_plain<<<1, 256, smemkb * 1024>>>(d);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("plain 1 CTA smem %3d KB: %.2f us/launch\n", smemkb, ms * 10);
    }
    return 0;
}
