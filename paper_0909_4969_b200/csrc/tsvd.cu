// truncated_svd / leading_left_singular_vectors / low_rank_approx on the
// device (reference: proj/include/mach/linalg.hpp:11-30,
// proj/src/linalg.cpp:196-317).
//
// Same dispatch and assembly as the reference's assemble_svd
// (linalg.cpp:210-236): Gram of the short side (rows side when rows <= cols),
// its top-k eigenpairs (the warm-startable subspace solver with the exact
// selected-eigenpair fallback, eig_select), singular values sqrt(max(0,
// lambda)); then
//   rows side:    left = canonical_sign(V), right = orthonormal_columns(A^T
//                 left, canonicalize = false);
//   columns side: left = orthonormal_columns(A V, canonicalize = true) and the
//                 right vectors carry the left flips.
// A zero matrix gives the identity columns and zero singular values
// (zero_matrix_svd, linalg.cpp:196-207).  The reference switches the short
// side above 512 to subspace iteration on the implicit Gram; the device
// eigensolver returns the same subspace (to its residual certificate), so one
// path serves every size.
#include "basis_cta.cuh"
#include "common.cuh"
#include "sparse_ttm.cuh"

namespace machb {

namespace {

// orthonormal_columns (linalg.cpp:66-100) in one CTA: twice Gram-Schmidt with
// the rank (kRankFloor * sigma1) and collapse (1e-3) tests, deterministic
// completions, optional canonical signs; flips[i] = the sign applied.
__global__ void __launch_bounds__(kB) ortho_cols_kernel(const double* __restrict__ W, int n, int wc, int k,
                                                        const double* __restrict__ sig, int canon,
                                                        double* __restrict__ U, double* __restrict__ flips,
                                                        int* __restrict__ st, double* __restrict__ gv) {
    extern __shared__ double sm[];
    double* v = gv ? gv : sm;
    double* tcoef = gv ? sm : v + n;
    double* red = tcoef + k;
    int* redi = reinterpret_cast<int*>(red + 32);
    const double floor = sig[0] * kRankFloor;
    int fail = 0;
    for (int i = 0; i < k; ++i) {
        bool backed = false;
        if (i < wc) {
            for (int r = threadIdx.x; r < n; r += kB) v[r] = W[r + static_cast<std::size_t>(i) * n];
            double s = 0.0;
            for (int r = threadIdx.x; r < n; r += kB) s += v[r] * v[r];
            const double nv = sqrt(cta_sum(s, red));
            if (nv > floor) {
                if (i > 0) {
                    cta_project_out(U, n, i, v, tcoef, red);
                    cta_project_out(U, n, i, v, tcoef, red);
                }
                double s2 = 0.0;
                for (int r = threadIdx.x; r < n; r += kB) s2 += v[r] * v[r];
                const double res = sqrt(cta_sum(s2, red));
                if (res > kCollapseFloor * nv) {
                    for (int r = threadIdx.x; r < n; r += kB) U[r + static_cast<std::size_t>(i) * n] = v[r] / res;
                    __syncthreads();
                    backed = true;
                }
            }
        }
        if (!backed && !cta_completion(U, n, i, v, tcoef, red) && !fail) fail = i + 1;
        double f = 1.0;
        if (canon) {
            double* u = U + static_cast<std::size_t>(i) * n;
            const int p = cta_argmax_abs(u, n, red, redi);
            f = u[p] < 0.0 ? -1.0 : 1.0;
            __syncthreads();
            if (f < 0.0)
                for (int r = threadIdx.x; r < n; r += kB) u[r] = -u[r];
            __syncthreads();
        }
        if (threadIdx.x == 0) flips[i] = f;
    }
    if (threadIdx.x == 0) st[0] = fail;
}

// canonical_sign of each column (one CTA per column)
__global__ void __launch_bounds__(kB) canon_cols_kernel(double* __restrict__ V, int n) {
    __shared__ double red[32];
    __shared__ int redi[32];
    double* u = V + static_cast<std::size_t>(blockIdx.x) * n;
    const int p = cta_argmax_abs(u, n, red, redi);
    const bool flip = u[p] < 0.0;
    __syncthreads();
    if (flip)
        for (int r = threadIdx.x; r < n; r += kB) u[r] = -u[r];
}

__global__ void scale_cols_kernel(double* __restrict__ V, int n, int k, const double* __restrict__ f) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e < static_cast<long long>(n) * k) V[e] *= f[e / n];
}

__global__ void transpose_kernel(const double* __restrict__ a, int rows, int cols, double* __restrict__ t) {
    __shared__ double tile[32][33];
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int r = r0 + threadIdx.x, c = c0 + j;
        if (r < rows && c < cols) tile[j][threadIdx.x] = a[r + static_cast<std::size_t>(c) * rows];
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int c = c0 + threadIdx.x, r = r0 + j;
        if (r < rows && c < cols) t[c + static_cast<std::size_t>(r) * cols] = tile[threadIdx.x][j];
    }
}

// out (rows x cols) = left diag(sv) right^T
__global__ void low_rank_kernel(const double* __restrict__ L, const double* __restrict__ sv, const double* __restrict__ R,
                                int rows, int cols, int k, double* __restrict__ out) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= static_cast<long long>(rows) * cols) return;
    const int r = static_cast<int>(e % rows), c = static_cast<int>(e / rows);
    double s = 0.0;
    for (int i = 0; i < k; ++i) s = fma(L[r + static_cast<std::size_t>(i) * rows] * sv[i], R[c + static_cast<std::size_t>(i) * cols], s);
    out[e] = s;
}

void ortho_cols(Ctx* ctx, const double* W, int n, int wc, int k, const double* sig, bool canon, double* U, double* flips,
                int* st) {
    std::size_t smem = basis_smem(n, k);
    DBuf<double> g;
    if (smem > 160 * 1024) {
        g.alloc(ctx, static_cast<std::size_t>(n));
        smem = basis_smem(0, k);
    }
    MB_LAUNCH(ctx, ortho_cols_kernel, 1, kB, smem, W, n, wc, k, sig, canon ? 1 : 0, U, flips, st, g.get());
}

}  // namespace

// A: rows x cols column-major fp64 on the device; outputs on the device
// (left rows x k, sv k, right cols x k).  Throws like the reference.
void truncated_svd_dev(Ctx* ctx, const double* A, int rows, int cols, int k, double* left, double* sv, double* right) {
    if (rows < 1 || cols < 1) throw_arg("matrix must be nonempty");
    if (k < 1 || k > std::min(rows, cols)) throw_arg("k must satisfy 1 <= k <= min(rows, cols)");
    DBuf<double> scal(ctx, 2), red(ctx, sumsq_scratch());
    sumsq<double>(ctx, A, static_cast<long long>(rows) * cols, red.get(), scal.get());
    double n2 = 0.0;
    to_host(ctx, &n2, scal.get(), 1);
    sync(ctx);
    if (n2 == 0.0) {  // zero_matrix_svd
        std::vector<double> l(static_cast<std::size_t>(rows) * k, 0.0), r(static_cast<std::size_t>(cols) * k, 0.0),
            s(static_cast<std::size_t>(k), 0.0);
        for (int i = 0; i < k; ++i) {
            l[static_cast<std::size_t>(i) + static_cast<std::size_t>(i) * rows] = 1.0;
            r[static_cast<std::size_t>(i) + static_cast<std::size_t>(i) * cols] = 1.0;
        }
        to_device(ctx, left, l.data(), l.size());
        to_device(ctx, right, r.data(), r.size());
        to_device(ctx, sv, s.data(), s.size());
        sync(ctx);
        return;
    }
    const bool rows_side = rows <= cols;
    const int side = rows_side ? rows : cols;
    DBuf<double> G(ctx, static_cast<std::size_t>(side) * side), V(ctx, static_cast<std::size_t>(side) * k);
    DBuf<int> est(ctx, 3), st(ctx, 1);
    if (rows_side) gram<double>(ctx, A, rows, 1, cols, rows, G.get());
    else gram<double>(ctx, A, 1, rows, rows, cols, G.get());
    eig_select(ctx, G.get(), side, k, nullptr, 0, nullptr, eig_block(side, k), V.get(), sv, est.get());
    DBuf<double> flips(ctx, k);
    if (rows_side) {
        MB_LAUNCH(ctx, canon_cols_kernel, k, kB, 0, V.get(), rows);
        MB_CUDA(cudaMemcpyAsync(left, V.get(), V.n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
        DBuf<double> At(ctx, static_cast<std::size_t>(rows) * cols), W(ctx, static_cast<std::size_t>(cols) * k);
        MB_LAUNCH(ctx, transpose_kernel, dim3(ceil_div(cols, 32), ceil_div(rows, 32)), dim3(32, 8), 0, A, rows, cols, At.get());
        matmul_yv<double>(ctx, At.get(), cols, rows, left, k, W.get());  // A^T left
        ortho_cols(ctx, W.get(), cols, k, k, sv, false, right, flips.get(), st.get());
    } else {
        DBuf<double> W(ctx, static_cast<std::size_t>(rows) * k);
        matmul_yv<double>(ctx, A, rows, cols, V.get(), k, W.get());  // A V
        ortho_cols(ctx, W.get(), rows, k, k, sv, true, left, flips.get(), st.get());
        MB_CUDA(cudaMemcpyAsync(right, V.get(), V.n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
        MB_LAUNCH(ctx, scale_cols_kernel, ceil_div(static_cast<long long>(cols) * k, 256), 256, 0, right, cols, k, flips.get());
    }
    int fail = 0;
    to_host(ctx, &fail, st.get(), 1);
    sync(ctx);
    if (fail)
        throw Error(MACH_ERR_CONVERGENCE, "orthonormal completion found no free direction (singular index " +
                                              std::to_string(fail) + ")", fail);
}

void low_rank_dev(Ctx* ctx, const double* L, const double* sv, const double* R, int rows, int cols, int k, double* out) {
    MB_LAUNCH(ctx, low_rank_kernel, ceil_div(static_cast<long long>(rows) * cols, 256), 256, 0, L, sv, R, rows, cols, k, out);
}

}  // namespace machb
