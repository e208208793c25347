// accuracy(t, model) = 1 - |t - reconstruct(model)| / |t| (reference:
// proj/src/tucker.cpp:211-217, used by compare, proj/src/metrics.cpp:155-156)
// as one fused pass over the reference tensor: the reconstruction is never
// materialised (at C5 it would be 8.6 GB of fp64).
//
// W = core x_1 U_1 ... x_{d-1} U_{d-1} (every mode but the first; r_0 x
// numel / I_0 fp64, 134 MB at C5) is formed by the fp64 mode-product chain;
// then each thread owns one row i0 of X_(0), keeps U_0[i0, :] in registers
// and walks columns: x_hat = U_0[i0, :] . W[:, c] in fp64, (x - x_hat)^2
// accumulated in fp64.  Reads t once (coalesced along i0) and W once per
// 256-row block; block partials are summed in a fixed order (deterministic).
#include "common.cuh"
#include "sparse_ttm.cuh"

namespace machb {

namespace {

template <typename T, int R0>
__global__ void __launch_bounds__(256) residual_fused_kernel(const T* __restrict__ x, int I0, long long ncol,
                                                             const double* __restrict__ U0, int r0,
                                                             const double* __restrict__ W, long long cols_per_block,
                                                             double* __restrict__ part) {
    const int i0 = blockIdx.x * blockDim.x + threadIdx.x;
    double u[R0];
#pragma unroll
    for (int a = 0; a < R0; ++a) u[a] = (i0 < I0 && a < r0) ? U0[i0 + static_cast<long long>(I0) * a] : 0.0;
    const long long c0 = blockIdx.y * cols_per_block, c1 = min(ncol, c0 + cols_per_block);
    double acc = 0.0;
    if (i0 < I0) {
        for (long long c = c0; c < c1; ++c) {
            const double* w = W + static_cast<long long>(r0) * c;
            double xh = 0.0;
#pragma unroll
            for (int a = 0; a < R0; ++a)
                if (a < r0) xh = fma(u[a], __ldg(w + a), xh);
            const double dlt = static_cast<double>(x[i0 + static_cast<long long>(I0) * c]) - xh;
            acc = fma(dlt, dlt, acc);
        }
    }
    __shared__ double red[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += red[w];
        part[blockIdx.y * gridDim.x + blockIdx.x] = s;
    }
}

__global__ void sum_parts_ordered_kernel(const double* __restrict__ part, long long n, double* __restrict__ out) {
    // one warp: strided partial sums in lane order, then a fixed shuffle tree
    double s = 0.0;
    for (long long i = threadIdx.x; i < n; i += 32) s += part[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) *out = s;
}

}  // namespace

// |x - core x_0 U_0 ... x_{d-1} U_{d-1}|^2 over the whole dense grid
// (core, U on the device: U_m is I_m x r_m column-major)
template <typename T>
double residual2_fused(Ctx* ctx, const T* x, const std::vector<int>& dims, const std::vector<int>& ranks,
                       const double* core, const std::vector<const double*>& U) {
    const int d = static_cast<int>(dims.size());
    const int I0 = dims[0], r0 = ranks[0];
    // W: expand the core over modes 1..d-1 (first-mode-fastest: r0 x I1 x ...)
    std::vector<int> cur = ranks;
    DBuf<double> w;
    const double* src = core;
    for (int m = 1; m < d; ++m) {
        std::vector<int> nd = cur;
        nd[static_cast<std::size_t>(m)] = dims[static_cast<std::size_t>(m)];
        DBuf<double> z(ctx, static_cast<std::size_t>(checked_size(nd)));
        // expansion by U_m (I_m x r_m): out(q, r) with q < I_m, M(q, r) = U[q + I_m r]
        dense_mode_product<double>(ctx, src, cur, m, U[static_cast<std::size_t>(m)], dims[static_cast<std::size_t>(m)],
                                   false, z.get());
        w = std::move(z);
        src = w.get();
        cur = nd;
    }
    const long long ncol = checked_size(dims) / I0;
    const int bx = ceil_div(I0, 256);
    const long long want = 148ll * 8 / bx + 1;
    const long long cpb = std::max<long long>(1, (ncol + want - 1) / want);
    const long long by = (ncol + cpb - 1) / cpb;
    if (by > 65535) throw Error(MACH_ERR_INTERNAL, "residual: grid too large");
    DBuf<double> part(ctx, static_cast<std::size_t>(bx * by)), out(ctx, 1);
    dim3 grid(static_cast<unsigned>(bx), static_cast<unsigned>(by));
    if (r0 <= 8) MB_LAUNCH(ctx, (residual_fused_kernel<T, 8>), grid, 256, 0, x, I0, ncol, U[0], r0, src, cpb, part.get());
    else if (r0 <= 16) MB_LAUNCH(ctx, (residual_fused_kernel<T, 16>), grid, 256, 0, x, I0, ncol, U[0], r0, src, cpb, part.get());
    else if (r0 <= 32) MB_LAUNCH(ctx, (residual_fused_kernel<T, 32>), grid, 256, 0, x, I0, ncol, U[0], r0, src, cpb, part.get());
    else throw Error(MACH_ERR_INTERNAL, "residual: first-mode rank above 32");
    MB_LAUNCH(ctx, sum_parts_ordered_kernel, 1, 32, 0, part.get(), static_cast<long long>(bx) * by, out.get());
    double h = 0.0;
    to_host(ctx, &h, out.get(), 1);
    sync(ctx);
    return h;
}
template double residual2_fused<float>(Ctx*, const float*, const std::vector<int>&, const std::vector<int>&, const double*,
                                       const std::vector<const double*>&);
template double residual2_fused<double>(Ctx*, const double*, const std::vector<int>&, const std::vector<int>&,
                                        const double*, const std::vector<const double*>&);

namespace {
// subspace_sin (metrics.cpp:59-66): M = A - B (B^T A) over the leading r
// columns, H = M^T M (r x r) for the exact eigensolver; one CTA
__global__ void __launch_bounds__(256) ortho_residual_gram_kernel(const double* __restrict__ A, const double* __restrict__ Bm,
                                                                  int n, int r, double* __restrict__ M,
                                                                  double* __restrict__ H) {
    __shared__ double Cs[32 * 32];
    for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
        const int l = e % r, j = e / r;
        double s = 0.0;
        for (int i = 0; i < n; ++i) s = fma(Bm[i + static_cast<long long>(n) * l], A[i + static_cast<long long>(n) * j], s);
        Cs[l + 32 * j] = s;
    }
    __syncthreads();
    for (long long e = threadIdx.x; e < static_cast<long long>(n) * r; e += blockDim.x) {
        const int i = static_cast<int>(e % n), j = static_cast<int>(e / n);
        double v = A[e];
        for (int l = 0; l < r; ++l) v = fma(-Bm[i + static_cast<long long>(n) * l], Cs[l + 32 * j], v);
        M[e] = v;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
        const int a = e % r, b = e / r;
        double s = 0.0;
        for (int i = 0; i < n; ++i) s = fma(M[i + static_cast<long long>(n) * a], M[i + static_cast<long long>(n) * b], s);
        H[a + r * b] = s;
    }
}
}  // namespace

// largest principal-angle sine between the spans of the leading r columns of
// A and B (n x >= r, column-major, device)
double subspace_sin_dev(Ctx* ctx, const double* A, const double* Bm, int n, int r) {
    if (r < 1 || r > 32) throw_arg("subspace_sin: 1 <= r <= 32");
    DBuf<double> M(ctx, static_cast<std::size_t>(n) * r), H(ctx, static_cast<std::size_t>(r) * r), V(ctx, static_cast<std::size_t>(r)),
        sig(ctx, 1), work(ctx, eig_work_doubles(r, 1));
    DBuf<int> st(ctx, 3);
    MB_LAUNCH(ctx, ortho_residual_gram_kernel, 1, 256, 0, A, Bm, n, r, M.get(), H.get());
    eig_topk(ctx, H.get(), r, 1, work.get(), V.get(), sig.get(), st.get());
    double s = 0.0;
    to_host(ctx, &s, sig.get(), 1);
    sync(ctx);
    return s;  // sqrt(max(0, lambda_max)) as metrics.cpp:65
}

}  // namespace machb
