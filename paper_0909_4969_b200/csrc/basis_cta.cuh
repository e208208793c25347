// CTA-level building blocks of the basis step (linalg.cu) shared with the
// merged fallback kernel (eig.cu): reductions, Gram-Schmidt projection,
// completion, canonical sign, basis_from_products, and the fused mode
// basis's fallback chain body.
#pragma once

#include "common.cuh"

namespace machb {

namespace {
constexpr double kRankFloor = 1e-6;      // linalg_internal.hpp:23
constexpr double kCollapseFloor = 1e-3;  // linalg.cpp:37
constexpr int kB = 256;                  // one-CTA kernels
constexpr int kW = kB / 32;

__device__ double cta_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < kW; ++i) s += red[i];
    return s;
}

// index of the largest |u_i|, lowest index on ties (canonical_sign, linalg.cpp:18-32)
__device__ int cta_argmax_abs(const double* u, int n, double* redv, int* redi) {
    double best = -1.0;
    int bi = 0x7fffffff;
    for (int i = threadIdx.x; i < n; i += kB) {
        const double a = fabs(u[i]);
        if (a > best) { best = a; bi = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) { redv[threadIdx.x >> 5] = best; redi[threadIdx.x >> 5] = bi; }
    __syncthreads();
    best = redv[0];
    bi = redi[0];
    for (int i = 1; i < kW; ++i)
        if (redv[i] > best || (redv[i] == best && redi[i] < bi)) { best = redv[i]; bi = redi[i]; }
    return bi;
}

// v -= B[:, :count] (B[:, :count]^T v), B column-major n x *, v in smem
__device__ void cta_project_out(const double* B, int n, int count, double* v, double* tcoef, double* red) {
    if (count <= 0) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    for (int c = warp; c < count; c += kW) {
        const double* b = B + static_cast<std::size_t>(c) * n;
        double s = 0.0;
        for (int r = lane; r < n; r += 32) s += b[r] * v[r];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) tcoef[c] = s;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < n; r += kB) {
        double s = v[r];
        for (int c = 0; c < count; ++c) s -= B[r + static_cast<std::size_t>(c) * n] * tcoef[c];
        v[r] = s;
    }
    __syncthreads();
}

// completion_column (linalg.cpp:41-51): lowest-index unit vector surviving
// two projections against the first `count` columns; written to column count.
__device__ bool cta_completion(double* B, int n, int count, double* v, double* tcoef, double* red) {
    for (int e = 0; e < n; ++e) {
        for (int r = threadIdx.x; r < n; r += kB) v[r] = (r == e) ? 1.0 : 0.0;
        cta_project_out(B, n, count, v, tcoef, red);
        cta_project_out(B, n, count, v, tcoef, red);
        double s = 0.0;
        for (int r = threadIdx.x; r < n; r += kB) s += v[r] * v[r];
        const double nv = sqrt(cta_sum(s, red));
        if (nv > 0.5) {
            for (int r = threadIdx.x; r < n; r += kB) B[r + static_cast<std::size_t>(count) * n] = v[r] / nv;
            __syncthreads();
            return true;
        }
    }
    return false;
}

__device__ void cta_canonical_sign(double* u, int n, double* redv, int* redi) {
    const int p = cta_argmax_abs(u, n, redv, redi);
    const bool flip = u[p] < 0.0;
    __syncthreads();
    if (flip)
        for (int r = threadIdx.x; r < n; r += kB) u[r] = -u[r];
    __syncthreads();
}

}  // namespace

std::size_t basis_smem(int n, int k);

namespace {
// CTA body (kB threads, shared memory basis_smem(n, k) at sm)
// gv: optional global scratch for the n-vector (tall matricizations whose
// n doubles do not fit in shared memory); then sm holds only the small parts
__device__ void basis_from_products_cta(const double* __restrict__ W, int n, int wc, int k, const double* __restrict__ sig,
                                        double* __restrict__ U, double* __restrict__ sv, int* __restrict__ st, double* sm,
                                        double* gv = nullptr) {
    double* v = gv ? gv : sm;
    double* tcoef = gv ? sm : v + n;
    double* red = tcoef + k;
    int* redi = reinterpret_cast<int*>(red + 32);
    const double sigma1 = sig[0];
    const double floor = sigma1 * kRankFloor;
    int nr = 0, completed = 0, fail = 0;
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
        if (!backed) {
            if (!cta_completion(U, n, i, v, tcoef, red) && !fail) fail = i + 1;
            completed = 1;
        } else {
            ++nr;
        }
        cta_canonical_sign(U + static_cast<std::size_t>(i) * n, n, red, redi);
        if (threadIdx.x == 0) sv[i] = (backed && i < wc) ? sig[i] : 0.0;
    }
    if (threadIdx.x == 0) { st[0] = nr; st[1] = completed; st[2] = fail; }
}


// the fused mode basis's fallback chain after the exact eigensolver, one CTA
// (kB threads, shared memory basis_smem(rows, k)):
//   flags[1]: W = Y V;  flags[2]: U from W (basis_from_products);
//   flags[3]: the row-major kernel copy of U.
template <typename T>
__device__ void mb_fallback_cta(const T* __restrict__ Y, int rows, int C, const double* __restrict__ V, int k,
                                double* __restrict__ W, const double* __restrict__ sig, double* __restrict__ U,
                                double* __restrict__ sv, int* __restrict__ st, T* __restrict__ Ur, int rs,
                                const int* __restrict__ flags, double* sm) {
    const int need_w = flags[1], need_basis = flags[2], need_rm = flags[3];
    if (!need_w && !need_basis && !need_rm) return;
    if (need_w) {
        for (long long idx = threadIdx.x; idx < static_cast<long long>(rows) * k; idx += kB) {
            const int i = static_cast<int>(idx % rows), j = static_cast<int>(idx / rows);
            double acc = 0.0;
            for (int c = 0; c < C; ++c)
                acc = fma(static_cast<double>(Y[i + static_cast<std::size_t>(c) * rows]), V[c + static_cast<std::size_t>(j) * C], acc);
            W[idx] = acc;
        }
        __syncthreads();
    }
    if (need_basis) basis_from_products_cta(W, rows, k, k, sig, U, sv, st, sm);
    __syncthreads();
    if (need_rm && Ur)
        for (long long idx = threadIdx.x; idx < static_cast<long long>(rows) * rs; idx += kB) {
            const int i = static_cast<int>(idx / rs), c = static_cast<int>(idx % rs);
            Ur[idx] = (c < k) ? static_cast<T>(U[i + static_cast<std::size_t>(c) * rows]) : T(0);
        }
}

}  // namespace
}  // namespace machb
