// Dense route (reference: hosvd/hooi(DenseTensor), tucker.cpp:135-150,
// :171-180, and the dense pieces of the sparse route: mode_product
// tensor.cpp:224-239, matricize :180-200, densify :261-266, the entrywise fit
// tucker.cpp:40-64 and reconstruct :204-209).  Taken when a sampled tensor
// keeps >= 25% of its entries (kDensifyThreshold, tucker.cpp:66-69).
// Intermediates are fp64; each output is summed by one thread in a fixed
// order, so results are reproducible bit for bit.
#include <algorithm>

#include "sparse_ttm.cuh"

namespace machb {

namespace {

struct Split3 {
    long long inner, outer;
    int len;
};

Split3 split3(const std::vector<int>& dims, int mode) {
    Split3 s{1, 1, dims[static_cast<std::size_t>(mode)]};
    for (int m = 0; m < mode; ++m) s.inner *= dims[static_cast<std::size_t>(m)];
    for (int m = mode + 1; m < static_cast<int>(dims.size()); ++m) s.outer *= dims[static_cast<std::size_t>(m)];
    return s;
}

template <typename Tin>
__global__ void mode_product_kernel(const Tin* __restrict__ in, long long inner, int len, long long outer,
                                    const double* __restrict__ U, int J, int transpose, double* __restrict__ out) {
    const long long total = inner * J * outer;
    for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long a = idx % inner;
        const long long rest = idx / inner;
        const int q = static_cast<int>(rest % J);
        const long long c = rest / J;
        const Tin* src = in + a + inner * len * c;
        double s = 0.0;
        if (transpose) {
            const double* u = U + static_cast<long long>(q) * len;  // U is len x J
            for (int r = 0; r < len; ++r) s += static_cast<double>(src[inner * r]) * u[r];
        } else {
            for (int r = 0; r < len; ++r) s += static_cast<double>(src[inner * r]) * U[q + static_cast<long long>(J) * r];
        }
        out[idx] = s;
    }
}

// One thread per (a, c): the len input values of its fibre are read once and
// all J outputs accumulated in registers (the generic kernel above re-reads
// them J times).  U (len x J products) staged in shared memory when it fits.
template <typename Tin, int JB>
__global__ void __launch_bounds__(256) mode_product_fibre_kernel(const Tin* __restrict__ in, long long inner, int len,
                                                                 long long outer, const double* __restrict__ U, int J,
                                                                 int transpose, int stage, double* __restrict__ out) {
    extern __shared__ double us[];  // us[r * J + q] = M(q, r)
    const double* M = U;
    if (stage) {
        for (int e = threadIdx.x; e < len * J; e += blockDim.x) {
            const int r = e / J, q = e - (e / J) * J;
            us[e] = transpose ? U[r + static_cast<long long>(len) * q] : U[q + static_cast<long long>(J) * r];
        }
        __syncthreads();
    }
    const long long total = inner * outer;
    for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long a = idx % inner, c = idx / inner;
        const Tin* src = in + a + inner * len * c;
        double acc[JB];
#pragma unroll
        for (int q = 0; q < JB; ++q) acc[q] = 0.0;
        for (int r = 0; r < len; ++r) {
            const double x = static_cast<double>(src[inner * r]);
            if (stage) {
                const double* ur = us + r * J;
#pragma unroll
                for (int q = 0; q < JB; ++q)
                    if (q < J) acc[q] = fma(x, ur[q], acc[q]);
            } else {
#pragma unroll
                for (int q = 0; q < JB; ++q)
                    if (q < J) acc[q] = fma(x, transpose ? M[r + static_cast<long long>(len) * q] : M[q + static_cast<long long>(J) * r], acc[q]);
            }
        }
        double* o = out + a + inner * static_cast<long long>(J) * c;
#pragma unroll
        for (int q = 0; q < JB; ++q)
            if (q < J) o[inner * q] = acc[q];
    }
}

// Few fibres, long contraction (e.g. the dense route's Z0 = X x_0 U_0^T, 16 x
// 1024 x 1024, contracted over its last mode: only 16K fibres of length
// 1024): the contraction is split into chunks over blockIdx.y, each thread
// accumulating its fibre's chunk for all J outputs; partials are summed in
// chunk order by sum_chunks_kernel (deterministic).
template <typename Tin, int JB>
__global__ void __launch_bounds__(256) mode_product_fibre_split_kernel(const Tin* __restrict__ in, long long inner,
                                                                       int len, long long outer,
                                                                       const double* __restrict__ U, int J,
                                                                       int transpose, int chunk,
                                                                       double* __restrict__ part) {
    extern __shared__ double us[];  // us[(r - r0) * J + q] = M(q, r) for the chunk
    const int r0 = blockIdx.y * chunk, r1 = min(len, r0 + chunk);
    for (int e = threadIdx.x; e < (r1 - r0) * J; e += blockDim.x) {
        const int r = r0 + e / J, q = e - (e / J) * J;
        us[e] = transpose ? U[r + static_cast<long long>(len) * q] : U[q + static_cast<long long>(J) * r];
    }
    __syncthreads();
    const long long total = inner * outer;
    double* pp = part + static_cast<long long>(blockIdx.y) * total * J;
    for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long a = idx % inner, c = idx / inner;
        const Tin* src = in + a + inner * len * c;
        double acc[JB];
#pragma unroll
        for (int q = 0; q < JB; ++q) acc[q] = 0.0;
#pragma unroll 4
        for (int r = r0; r < r1; ++r) {
            const double x = static_cast<double>(src[inner * r]);
            const double* ur = us + (r - r0) * J;
#pragma unroll
            for (int q = 0; q < JB; ++q)
                if (q < J) acc[q] = fma(x, ur[q], acc[q]);
        }
        double* o = pp + a + inner * static_cast<long long>(J) * c;
#pragma unroll
        for (int q = 0; q < JB; ++q)
            if (q < J) o[inner * q] = acc[q];
    }
}

__global__ void sum_chunks_kernel(const double* __restrict__ part, int nchunk, long long n, double* __restrict__ out) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        double s = 0.0;
        for (int k = 0; k < nchunk; ++k) s += part[static_cast<long long>(k) * n + i];
        out[i] = s;
    }
}

// inner == 1 (contracting the fastest mode): a fibre is contiguous, so one
// warp takes it (lanes over r, coalesced), then reduces the J sums.
template <typename Tin, int JB>
__global__ void __launch_bounds__(256) mode_product_row_kernel(const Tin* __restrict__ in, int len, long long outer,
                                                               const double* __restrict__ U, int J, int transpose,
                                                               int stage, double* __restrict__ out) {
    extern __shared__ double us[];  // us[q * len + r] = M(q, r): lanes (consecutive r) hit consecutive banks
    if (stage) {
        for (int e = threadIdx.x; e < len * J; e += blockDim.x) {
            const int q = e / len, r = e - (e / len) * len;
            us[e] = transpose ? U[r + static_cast<long long>(len) * q] : U[q + static_cast<long long>(J) * r];
        }
        __syncthreads();
    }
    const int lane = threadIdx.x & 31;
    const long long nw = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
    for (long long c = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5; c < outer; c += nw) {
        const Tin* src = in + static_cast<long long>(len) * c;
        double acc[JB];
#pragma unroll
        for (int q = 0; q < JB; ++q) acc[q] = 0.0;
        for (int r = lane; r < len; r += 32) {
            const double x = static_cast<double>(src[r]);
#pragma unroll
            for (int q = 0; q < JB; ++q)
                if (q < J)
                    acc[q] = fma(x, stage ? us[q * len + r] : (transpose ? U[r + static_cast<long long>(len) * q] : U[q + static_cast<long long>(J) * r]), acc[q]);
        }
#pragma unroll
        for (int q = 0; q < JB; ++q) {
            if (q >= J) break;
            double v = acc[q];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) out[q + static_cast<long long>(J) * c] = v;
        }
    }
}

template <typename Tin, typename Tout>
__global__ void matricize_kernel(const Tin* __restrict__ in, long long inner, int len, long long outer,
                                 Tout* __restrict__ out) {
    const long long total = inner * len * outer;
    for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        // idx walks the source (coalesced reads); out(r, a + inner*c) = in[a + inner*(r + len*c)]
        const long long a = idx % inner;
        const long long rest = idx / inner;
        const int r = static_cast<int>(rest % len);
        const long long c = rest / len;
        out[r + static_cast<long long>(len) * (a + inner * c)] = static_cast<Tout>(in[idx]);
    }
}

template <typename T, typename IdxT>
__global__ void densify_kernel(const IdxT* __restrict__ idx, const T* __restrict__ val, long long nnz, T* __restrict__ out) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i < nnz) out[idx[i]] = val[i];
}

// values rounded to TF32 (round to nearest, ties away): the tensor core then reads them exactly
template <typename IdxT>
__global__ void densify_tf32_kernel(const IdxT* __restrict__ idx, const float* __restrict__ val, long long nnz,
                                    float* __restrict__ out) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= nnz) return;
    std::uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(val[i]));
    out[idx[i]] = __uint_as_float(r);
}

template <typename T, typename IdxT>
__global__ void scatter_sub_kernel(const IdxT* __restrict__ idx, const T* __restrict__ val, long long nnz,
                                   double* __restrict__ out) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i < nnz) out[idx[i]] -= static_cast<double>(val[i]);
}

constexpr int kRedBlocks = 1024;

template <typename T>
__global__ void __launch_bounds__(256) sumsq_diff_kernel(const T* __restrict__ x, const double* __restrict__ y, long long n,
                                                         double* __restrict__ part) {
    __shared__ double red[8];
    double s = 0.0;
    for (long long i = blockIdx.x * 256ll + threadIdx.x; i < n; i += 256ll * kRedBlocks) {
        const double dlt = static_cast<double>(x[i]) - y[i];
        s += dlt * dlt;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < 8; ++i) t += red[i];
        part[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(256) sum_final2_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
    __shared__ double red[8];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += 256) s += part[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < 8; ++i) t += red[i];
        *out = t;
    }
}

int grid_for(long long n) {
    long long b = (n + 255) / 256;
    if (b > 148 * 64) b = 148 * 64;
    if (b < 1) b = 1;
    return static_cast<int>(b);
}

}  // namespace

template <typename Tin>
void dense_mode_product(Ctx* ctx, const Tin* in, const std::vector<int>& dims, int mode, const double* U, int J,
                        bool transpose, double* out) {
    const Split3 s = split3(dims, mode);
    const long long total = s.inner * J * s.outer;
    if (total == 0) return;
    static const bool generic = std::getenv("MACH_DENSE_GENERIC") != nullptr;
    if (!generic && J <= 32) {
        const std::size_t ub = static_cast<std::size_t>(s.len) * J * sizeof(double);
        const int stage = ub <= 48 * 1024 ? 1 : 0;
        const long long fib = s.inner * s.outer;
        auto go = [&](auto mode_product_fibre_kernel_jb) {  // (the name is the profiler's kernel label)
            MB_LAUNCH(ctx, mode_product_fibre_kernel_jb, static_cast<unsigned>(std::min<long long>(grid_for(fib), 148 * 8)), 256, stage ? ub : 0, in, s.inner, s.len, s.outer, U,
                      J, transpose ? 1 : 0, stage, out);
        };
        if (s.inner == 1) {
            auto gr = [&](auto mode_product_row_kernel_jb) {  // (the name is the profiler's kernel label)
                MB_LAUNCH(ctx, mode_product_row_kernel_jb, static_cast<unsigned>(std::min<long long>(grid_for(s.outer * 32), 148 * 8)), 256, stage ? ub : 0, in, s.len, s.outer,
                          U, J, transpose ? 1 : 0, stage, out);
            };
            if (J <= 8) gr(mode_product_row_kernel<Tin, 8>);
            else if (J <= 16) gr(mode_product_row_kernel<Tin, 16>);
            else gr(mode_product_row_kernel<Tin, 32>);
            return;
        }
        if (fib < 148ll * 1024 && s.len >= 128) {
            // too few fibres to fill the GPU: split the contraction
            int nchunk = static_cast<int>(std::min<long long>(s.len / 32, (148ll * 2048 + fib - 1) / fib));
            nchunk = std::max(nchunk, static_cast<int>((static_cast<long long>(s.len) * J * 8 + 48 * 1024 - 1) / (48 * 1024)));
            const int chunk = (s.len + nchunk - 1) / nchunk;
            const int nc = (s.len + chunk - 1) / chunk;
            DBuf<double> part(ctx, static_cast<std::size_t>(nc) * total);
            const std::size_t cb = static_cast<std::size_t>(chunk) * J * sizeof(double);
            dim3 grid(static_cast<unsigned>(std::max<long long>(1, std::min<long long>((fib + 255) / 256, 148 * 8))),
                      static_cast<unsigned>(nc));
            auto gs = [&](auto mode_product_split_kernel_jb) {  // (the name is the profiler's kernel label)
                MB_LAUNCH(ctx, mode_product_split_kernel_jb, grid, 256, cb, in, s.inner, s.len, s.outer, U, J,
                          transpose ? 1 : 0, chunk, part.get());
            };
            if (J <= 8) gs(mode_product_fibre_split_kernel<Tin, 8>);
            else if (J <= 16) gs(mode_product_fibre_split_kernel<Tin, 16>);
            else gs(mode_product_fibre_split_kernel<Tin, 32>);
            MB_LAUNCH(ctx, sum_chunks_kernel, grid_for(total), 256, 0, part.get(), nc, total, out);
            return;
        }
        if (J <= 8) go(mode_product_fibre_kernel<Tin, 8>);
        else if (J <= 16) go(mode_product_fibre_kernel<Tin, 16>);
        else go(mode_product_fibre_kernel<Tin, 32>);
        return;
    }
    MB_LAUNCH(ctx, mode_product_kernel<Tin>, grid_for(total), 256, 0, in, s.inner, s.len, s.outer, U, J,
              transpose ? 1 : 0, out);
}
template void dense_mode_product<float>(Ctx*, const float*, const std::vector<int>&, int, const double*, int, bool, double*);
template void dense_mode_product<double>(Ctx*, const double*, const std::vector<int>&, int, const double*, int, bool, double*);

template <typename Tin, typename Tout>
void dense_matricize(Ctx* ctx, const Tin* in, const std::vector<int>& dims, int mode, Tout* out) {
    const Split3 s = split3(dims, mode);
    const long long total = s.inner * s.len * s.outer;
    if (total == 0) return;
    MB_LAUNCH(ctx, (matricize_kernel<Tin, Tout>), grid_for(total), 256, 0, in, s.inner, s.len, s.outer, out);
}
template void dense_matricize<float, float>(Ctx*, const float*, const std::vector<int>&, int, float*);
template void dense_matricize<double, double>(Ctx*, const double*, const std::vector<int>&, int, double*);
template void dense_matricize<float, double>(Ctx*, const float*, const std::vector<int>&, int, double*);

template <typename T>
void densify(Ctx* ctx, const mach_sparse* X, T* out) {
    MB_CUDA(cudaMemsetAsync(out, 0, static_cast<std::size_t>(X->numel) * sizeof(T), ctx->stream));
    if (X->nnz == 0) return;
    if (X->idx64)
        MB_LAUNCH(ctx, (densify_kernel<T, unsigned long long>), ceil_div(X->nnz, 256), 256, 0,
                  static_cast<const unsigned long long*>(X->idx), static_cast<const T*>(X->val), X->nnz, out);
    else
        MB_LAUNCH(ctx, (densify_kernel<T, unsigned int>), ceil_div(X->nnz, 256), 256, 0,
                  static_cast<const unsigned int*>(X->idx), static_cast<const T*>(X->val), X->nnz, out);
}
template void densify<float>(Ctx*, const mach_sparse*, float*);

void densify_tf32(Ctx* ctx, const mach_sparse* X, float* out) {
    MB_CUDA(cudaMemsetAsync(out, 0, static_cast<std::size_t>(X->numel) * sizeof(float), ctx->stream));
    if (X->nnz == 0) return;
    if (X->idx64)
        MB_LAUNCH(ctx, densify_tf32_kernel<unsigned long long>, ceil_div(X->nnz, 256), 256, 0,
                  static_cast<const unsigned long long*>(X->idx), static_cast<const float*>(X->val), X->nnz, out);
    else
        MB_LAUNCH(ctx, densify_tf32_kernel<unsigned int>, ceil_div(X->nnz, 256), 256, 0,
                  static_cast<const unsigned int*>(X->idx), static_cast<const float*>(X->val), X->nnz, out);
}
template void densify<double>(Ctx*, const mach_sparse*, double*);

template <typename T>
void scatter_sub(Ctx* ctx, const mach_sparse* X, double* dense) {
    if (X->nnz == 0) return;
    if (X->idx64)
        MB_LAUNCH(ctx, (scatter_sub_kernel<T, unsigned long long>), ceil_div(X->nnz, 256), 256, 0,
                  static_cast<const unsigned long long*>(X->idx), static_cast<const T*>(X->val), X->nnz, dense);
    else
        MB_LAUNCH(ctx, (scatter_sub_kernel<T, unsigned int>), ceil_div(X->nnz, 256), 256, 0,
                  static_cast<const unsigned int*>(X->idx), static_cast<const T*>(X->val), X->nnz, dense);
}
template void scatter_sub<float>(Ctx*, const mach_sparse*, double*);
template void scatter_sub<double>(Ctx*, const mach_sparse*, double*);

template <typename T>
void sumsq_diff(Ctx* ctx, const T* x, const double* y, long long n, double* scratch, double* out) {
    MB_LAUNCH(ctx, sumsq_diff_kernel<T>, kRedBlocks, 256, 0, x, y, n, scratch);
    MB_LAUNCH(ctx, sum_final2_kernel, 1, 256, 0, scratch, kRedBlocks, out);
}
template void sumsq_diff<float>(Ctx*, const float*, const double*, long long, double*, double*);
template void sumsq_diff<double>(Ctx*, const double*, const double*, long long, double*, double*);

}  // namespace machb
