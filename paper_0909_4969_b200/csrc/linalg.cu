// Device building blocks of the eigen step and the Tucker bookkeeping:
//  - Gram of a matricized projection Y (row side Y Y^T or column side Y^T Y),
//    fp64 accumulation (linalg.cpp:340, :348);
//  - basis_from_side: numerical rank against kRankFloor, sign canonicalisation,
//    deterministic completion (linalg.cpp:261-276, :18-32, :41-51);
//  - orthonormal_columns / basis_from_products: twice Gram-Schmidt, rank and
//    collapse floors, completion, sign (linalg.cpp:66-100, :283-296);
//  - W = Y V, core = U_d^T Y_(d), deterministic sums of squares.
// All reductions run in a fixed order, so results are bitwise reproducible.
#include <algorithm>

#include "common.cuh"

#include "basis_cta.cuh"

namespace machb {


// ---------------------------------------------------------------------------
// G = A^T A with A(kk, j) = a[kk*sk + j*sn], A is K x N; G is N x N fp64.
// 32x32 output tile per block, fixed-order accumulation over K.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) gram_kernel(const T* __restrict__ a, long long sk, long long sn, int K, int N,
                                                   double* __restrict__ G) {
    __shared__ double As[32][33];
    __shared__ double Bs[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
    double acc[4] = {0, 0, 0, 0};
    for (int k0 = 0; k0 < K; k0 += 32) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            int kk, jj;
            if (sn == 1) { kk = ty + 8 * q; jj = tx; } else { kk = tx; jj = ty + 8 * q; }
            const int gk = k0 + kk;
            const int gi = i0 + jj, gj = j0 + jj;
            As[kk][jj] = (gk < K && gi < N) ? static_cast<double>(a[gk * sk + gi * sn]) : 0.0;
            Bs[kk][jj] = (gk < K && gj < N) ? static_cast<double>(a[gk * sk + gj * sn]) : 0.0;
        }
        __syncthreads();
#pragma unroll 8
        for (int kk = 0; kk < 32; ++kk) {
            const double x = As[kk][tx];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] += x * Bs[kk][ty + 8 * q];
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int i = i0 + tx, j = j0 + ty + 8 * q;
        if (i < N && j < N) G[i + static_cast<std::size_t>(j) * N] = acc[q];
    }
}

// Small-N Gram on the fp64 tensor cores: one warp per 8x8 tile (ti >= tj) and
// K-chunk, mma.m8n8k4 with operands straight from global memory (the matrix
// is L2-resident), eight k-steps of loads in flight.  Off-diagonal tiles are
// written to both triangles and diagonal tiles from their lower half, so G is
// exactly symmetric.  With nsplit > 1 the chunks go to `part` and are summed
// in chunk order.
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

template <typename T>
__global__ void __launch_bounds__(256) gram_mma_kernel(const T* __restrict__ a, long long sk, long long sn, int K, int N,
                                                       int nts, int kchunk, int nsplit, double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const long long w = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
    const int NT = nts * (nts + 1) / 2;
    if (w >= static_cast<long long>(NT) * nsplit) return;
    const int tile = static_cast<int>(w % NT), split = static_cast<int>(w / NT);
    int ti = static_cast<int>((sqrt(8.0 * tile + 1.0) - 1.0) * 0.5);
    while ((ti + 1) * (ti + 2) / 2 <= tile) ++ti;
    while (ti * (ti + 1) / 2 > tile) --ti;
    const int tj = tile - ti * (ti + 1) / 2;
    const int gr = lane >> 2, tq = lane & 3;
    const int i = ti * 8 + gr, j = tj * 8 + gr;
    const int k0 = split * kchunk, k1 = min(K, k0 + kchunk);
    const bool iv = i < N, jv = j < N;
    const T* pa = a + static_cast<long long>(iv ? i : 0) * sn;
    const T* pb = a + static_cast<long long>(jv ? j : 0) * sn;
    double c0 = 0.0, c1 = 0.0;
    for (int kb = k0; kb < k1; kb += 32) {
        double av[8], bv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int kk = kb + 4 * u + tq;
            const bool kv = kk < k1;
            av[u] = (kv && iv) ? static_cast<double>(pa[kk * sk]) : 0.0;
            bv[u] = (kv && jv) ? static_cast<double>(pb[kk * sk]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) dmma884(c0, c1, av[u], bv[u]);
    }
    double* G = out + static_cast<std::size_t>(split) * N * N;
    const int r = ti * 8 + gr;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int c = tj * 8 + 2 * tq + e;
        const double v = e ? c1 : c0;
        if (r < N && c < N && (ti != tj || r >= c)) {
            G[r + static_cast<std::size_t>(c) * N] = v;
            G[c + static_cast<std::size_t>(r) * N] = v;
        }
    }
}

__global__ void sum_parts_kernel(const double* __restrict__ part, int nsplit, long long n, double* __restrict__ G) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= n) return;
    double s = 0.0;
    for (int q = 0; q < nsplit; ++q) s += part[q * n + e];
    G[e] = s;
}

template <typename T>
void gram(Ctx* ctx, const T* a, long long sk, long long sn, int K, int N, double* G) {
    if (N <= 256 && K <= (1 << 20)) {
        const int nts = (N + 7) / 8;
        const int NT = nts * (nts + 1) / 2;
        const int kchunk_min = 1024;
        int nsplit = std::max(1, std::min(K / kchunk_min, 2368 / NT));
        nsplit = std::min(nsplit, 64);
        const int kchunk = ((ceil_div(K, nsplit) + 31) / 32) * 32;
        nsplit = ceil_div(K, kchunk);
        const long long warps = static_cast<long long>(NT) * nsplit;
        if (nsplit == 1) {
            MB_LAUNCH(ctx, gram_mma_kernel<T>, ceil_div(warps * 32, 256), 256, 0, a, sk, sn, K, N, nts, kchunk, 1, G);
        } else {
            DBuf<double> part(ctx, static_cast<std::size_t>(nsplit) * N * N);
            MB_LAUNCH(ctx, gram_mma_kernel<T>, ceil_div(warps * 32, 256), 256, 0, a, sk, sn, K, N, nts, kchunk, nsplit,
                      part.get());
            const long long n2 = static_cast<long long>(N) * N;
            MB_LAUNCH(ctx, sum_parts_kernel, ceil_div(n2, 256), 256, 0, part.get(), nsplit, n2, G);
        }
        return;
    }
    dim3 grid(ceil_div(N, 32), ceil_div(N, 32));
    MB_LAUNCH(ctx, gram_kernel<T>, grid, 256, 0, a, sk, sn, K, N, G);
}
template void gram<float>(Ctx*, const float*, long long, long long, int, int, double*);
template void gram<double>(Ctx*, const double*, long long, long long, int, int, double*);

// ---------------------------------------------------------------------------
// W (rows x kc, fp64) = Y (rows x C, col-major, T) * V (C x kc, fp64)
// ---------------------------------------------------------------------------
template <typename T, int KC>
__global__ void __launch_bounds__(128) matmul_yv_kernel(const T* __restrict__ Y, int rows, int C, const double* __restrict__ V,
                                                        int kc, double* __restrict__ W, const int* __restrict__ need) {
    pdl_enter();  // programmatic dependent launch: predecessor complete and visible
    if (need && need[0] == 0) return;
    // thread per row of W; V staged in shared memory (broadcast reads); the
    // column loop streams Y column by column (coalesced across the rows)
    extern __shared__ double vs[];
    for (int e = threadIdx.x; e < C * kc; e += blockDim.x) vs[e] = V[e];
    __syncthreads();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    double acc[KC];
#pragma unroll
    for (int j = 0; j < KC; ++j) acc[j] = 0.0;
#pragma unroll 4
    for (int c = 0; c < C; ++c) {
        const double y = static_cast<double>(Y[i + static_cast<std::size_t>(c) * rows]);
#pragma unroll
        for (int j = 0; j < KC; ++j)
            if (j < kc) acc[j] = fma(y, vs[c + j * C], acc[j]);
    }
#pragma unroll
    for (int j = 0; j < KC; ++j)
        if (j < kc) W[i + static_cast<std::size_t>(j) * rows] = acc[j];
}

template <typename T>
__global__ void matmul_yv_generic_kernel(const T* __restrict__ Y, int rows, int C, const double* __restrict__ V, int kc,
                                         double* __restrict__ W, const int* __restrict__ need) {
    pdl_enter();  // programmatic dependent launch: predecessor complete and visible
    if (need && need[0] == 0) return;
    const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (idx >= static_cast<long long>(rows) * kc) return;
    const int i = static_cast<int>(idx % rows), c2 = static_cast<int>(idx / rows);
    double s = 0.0;
    for (int c = 0; c < C; ++c) s += static_cast<double>(Y[i + static_cast<std::size_t>(c) * rows]) * V[c + static_cast<std::size_t>(c2) * C];
    W[idx] = s;
}

template <typename T>
void matmul_yv_gated(Ctx* ctx, const T* Y, int rows, int C, const double* V, int kc, double* W, const int* need) {
    const long long n = static_cast<long long>(rows) * kc;
    if (n == 0) return;
    const std::size_t vsm = static_cast<std::size_t>(C) * kc * sizeof(double);
    if (kc <= 32 && vsm <= 48 * 1024) {
        if (kc <= 16)
            MB_LAUNCH_PDL(ctx, (matmul_yv_kernel<T, 16>), ceil_div(rows, 128), 128, vsm, Y, rows, C, V, kc, W, need);
        else
            MB_LAUNCH_PDL(ctx, (matmul_yv_kernel<T, 32>), ceil_div(rows, 128), 128, vsm, Y, rows, C, V, kc, W, need);
        return;
    }
    MB_LAUNCH_PDL(ctx, matmul_yv_generic_kernel<T>, ceil_div(n, 256), 256, 0, Y, rows, C, V, kc, W, need);
}

template <typename T>
void matmul_yv(Ctx* ctx, const T* Y, int rows, int C, const double* V, int kc, double* W) {
    matmul_yv_gated<T>(ctx, Y, rows, C, V, kc, W, nullptr);
}
template void matmul_yv_gated<float>(Ctx*, const float*, int, int, const double*, int, double*, const int*);
template void matmul_yv_gated<double>(Ctx*, const double*, int, int, const double*, int, double*, const int*);
template void matmul_yv<float>(Ctx*, const float*, int, int, const double*, int, double*);
template void matmul_yv<double>(Ctx*, const double*, int, int, const double*, int, double*);

// ---------------------------------------------------------------------------
// basis_from_side (linalg.cpp:261-276) on device.  V: n x k eigenvectors
// (descending), sig: k.  Writes U (n x k), sv (k), st[0]=numerical rank,
// st[1]=completed.  eig_status[1]==1 marks an exactly zero matricization
// (linalg.cpp:326-333: identity basis, rank 0, completed).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kB) basis_from_side_kernel(const double* __restrict__ V, const double* __restrict__ sig,
                                                             int n, int k, const int* __restrict__ eig_status,
                                                             double* __restrict__ U, double* __restrict__ sv,
                                                             int* __restrict__ st, double* __restrict__ gv) {
    extern __shared__ double sm[];
    double* v = gv ? gv : sm;             // n (global scratch for tall n)
    double* tcoef = gv ? sm : v + n;      // k
    double* red = tcoef + k;   // 32
    int* redi = reinterpret_cast<int*>(red + 32);
    for (int idx = threadIdx.x; idx < n * k; idx += kB) U[idx] = V[idx];
    __syncthreads();
    if (eig_status[1] == 1) {
        for (int i = threadIdx.x; i < k; i += kB) sv[i] = 0.0;
        if (threadIdx.x == 0) { st[0] = 0; st[1] = 1; st[2] = 0; }
        return;
    }
    const double sigma1 = sig[0];
    int nr = 0;
    while (nr < k && sig[nr] > sigma1 * kRankFloor) ++nr;
    for (int i = 0; i < nr; ++i) cta_canonical_sign(U + static_cast<std::size_t>(i) * n, n, red, redi);
    for (int i = threadIdx.x; i < k; i += kB) sv[i] = (i < nr) ? sig[i] : 0.0;
    int fail = 0;
    for (int i = nr; i < k; ++i)
        if (!cta_completion(U, n, i, v, tcoef, red)) { fail = i + 1; break; }
    if (threadIdx.x == 0) { st[0] = nr; st[1] = nr < k ? 1 : 0; st[2] = fail; }
}

// ---------------------------------------------------------------------------
// basis_from_products (linalg.cpp:283-296) = orthonormal_columns(w, k, sigma1,
// canonicalize=true) + sv of the backed columns.  W: n x wc.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kB) basis_from_products_kernel(const double* __restrict__ W, int n, int wc, int k,
                                                                 const double* __restrict__ sig,
                                                                 const int* __restrict__ eig_status,
                                                                 double* __restrict__ U, double* __restrict__ sv,
                                                                 int* __restrict__ st, const int* __restrict__ skip,
                                                                 double* __restrict__ gv) {
    pdl_enter();  // programmatic dependent launch: predecessor complete and visible
    if (skip && skip[0] == 0) return;  // the CholQR2 fast path already produced U
    extern __shared__ double sm[];
    basis_from_products_cta(W, n, wc, k, sig, U, sv, st, sm, gv);
    (void)eig_status;
}

// The fused mode basis's fallback chain after the exact eigensolver, in one
// CTA (see mb_fallback_cta); on the fast path one no-op launch.
template <typename T>
__global__ void __launch_bounds__(kB) mb_fallback_kernel(const T* __restrict__ Y, int rows, int C, const double* __restrict__ V,
                                                         int k, double* __restrict__ W, const double* __restrict__ sig,
                                                         double* __restrict__ U, double* __restrict__ sv,
                                                         int* __restrict__ st, T* __restrict__ Ur, int rs,
                                                         const int* __restrict__ flags) {
    pdl_enter();  // programmatic dependent launch: predecessor complete and visible
    extern __shared__ double sm[];
    mb_fallback_cta<T>(Y, rows, C, V, k, W, sig, U, sv, st, Ur, rs, flags, sm);
}

template <typename T>
void mb_fallback(Ctx* ctx, const T* Y, int rows, int C, const double* V, int k, double* W, const double* sig, double* U,
                 double* sv, int* st, T* Ur, int rs, const int* flags) {
    MB_LAUNCH_PDL(ctx, mb_fallback_kernel<T>, 1, kB, basis_smem(rows, k), Y, rows, C, V, k, W, sig, U, sv, st, Ur, rs, flags);
}
template void mb_fallback<float>(Ctx*, const float*, int, int, const double*, int, double*, const double*, double*,
                                 double*, int*, float*, int, const int*);
template void mb_fallback<double>(Ctx*, const double*, int, int, const double*, int, double*, const double*, double*,
                                  double*, int*, double*, int, const int*);

std::size_t basis_smem(int n, int k) { return (static_cast<std::size_t>(n) + k + 32 + 32) * sizeof(double); }

// n-vector scratch of the one-CTA basis kernels: shared memory, or global
// memory for tall matricizations (C4's 65536-row time mode)
namespace {
constexpr std::size_t kBasisSmemMax = 160 * 1024;
struct BasisScratch {
    DBuf<double> g;
    std::size_t smem = 0;
    BasisScratch(Ctx* ctx, int n, int k) {
        smem = basis_smem(n, k);
        if (smem > kBasisSmemMax) {
            g.alloc(ctx, static_cast<std::size_t>(n));
            smem = basis_smem(0, k);
        }
    }
};
}  // namespace

void basis_from_side(Ctx* ctx, const double* V, const double* sig, int n, int k, const int* eig_status, double* U,
                     double* sv, int* st) {
    BasisScratch bs(ctx, n, k);
    MB_LAUNCH(ctx, basis_from_side_kernel, 1, kB, bs.smem, V, sig, n, k, eig_status, U, sv, st, bs.g.get());
}

// ---------------------------------------------------------------------------
// basis_from_products fast path.  W = Y V has (numerically) orthogonal columns
// of lengths sigma_i, so the reference's twice Gram-Schmidt (linalg.cpp:66-100)
// equals CholQR2 here: C = W^T W = R^T R gives every column's length
// (sqrt C_ii) and its residual after projecting out the earlier columns
// (R_ii), i.e. the same rank and collapse tests, and U = W R^{-1} (twice).
// When a column fails a test (rank deficiency / completion needed) the flag
// stays 1 and the full Gram-Schmidt kernel runs next in the stream.
// ---------------------------------------------------------------------------
constexpr int kFastK = 32;

__device__ void small_gram(const double* X, int n, int k, double* C, double* red) {
    // C (k x k, ld kFastK) = X^T X over n rows; one warp per (i <= j) pair
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int p = warp; p < k * (k + 1) / 2; p += kW) {
        int i = 0;
        while ((i + 1) * (i + 2) / 2 <= p) ++i;
        const int j = p - i * (i + 1) / 2;
        const double* a = X + static_cast<std::size_t>(i) * n;
        const double* b = X + static_cast<std::size_t>(j) * n;
        double s = 0.0;
        for (int r = lane; r < n; r += 32) s = fma(a[r], b[r], s);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
            C[i + j * kFastK] = s;
            C[j + i * kFastK] = s;
        }
    }
    __syncthreads();
    (void)red;
}

// upper Cholesky factor of C in place (thread 0), then Ri = R^{-1} (thread c
// solves column c).  Returns false on a non-positive pivot.
__device__ bool small_chol_inv(double* C, double* Ri, int k, double* diag, int* ok) {
    if (threadIdx.x == 0) {
        int good = 1;
        for (int j = 0; j < k && good; ++j) {
            double d = C[j + j * kFastK];
            for (int p = 0; p < j; ++p) d -= C[p + j * kFastK] * C[p + j * kFastK];
            if (!(d > 0.0)) { good = 0; break; }
            const double rjj = sqrt(d);
            C[j + j * kFastK] = rjj;
            diag[j] = rjj;
            for (int l = j + 1; l < k; ++l) {
                double v = C[j + l * kFastK];
                for (int p = 0; p < j; ++p) v -= C[p + j * kFastK] * C[p + l * kFastK];
                C[j + l * kFastK] = v / rjj;
            }
        }
        *ok = good;
    }
    __syncthreads();
    if (!*ok) return false;
    if (threadIdx.x < k) {
        const int c = threadIdx.x;
        for (int r = k - 1; r >= 0; --r) {
            double v = (r == c) ? 1.0 : 0.0;
            for (int p = r + 1; p < k; ++p) v -= C[r + p * kFastK] * Ri[p + c * kFastK];
            Ri[r + c * kFastK] = (r <= c) ? v / C[r + r * kFastK] : 0.0;
        }
    }
    __syncthreads();
    return true;
}

// Y (n x k) = X Ri, column-major, X and Y distinct
__device__ void small_apply(const double* X, const double* Ri, double* Y, int n, int k) {
    for (long long e = threadIdx.x; e < static_cast<long long>(n) * k; e += kB) {
        const int r = static_cast<int>(e % n), c = static_cast<int>(e / n);
        double s = 0.0;
        for (int p = 0; p <= c; ++p) s = fma(X[r + static_cast<std::size_t>(p) * n], Ri[p + c * kFastK], s);
        Y[e] = s;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kB) basis_products_fast_kernel(const double* __restrict__ W, int n, int k,
                                                                 const double* __restrict__ sig,
                                                                 double* __restrict__ U, double* __restrict__ sv,
                                                                 int* __restrict__ st, int* __restrict__ slow) {
    extern __shared__ double sm[];
    double* X = sm;                                   // n x k
    double* Y = X + static_cast<std::size_t>(n) * k;  // n x k
    __shared__ double C[kFastK * kFastK], Ri[kFastK * kFastK], diag[kFastK], red[32];
    __shared__ int ok, redi[32];
    for (long long e = threadIdx.x; e < static_cast<long long>(n) * k; e += kB) X[e] = W[e];
    __syncthreads();
    small_gram(X, n, k, C, red);
    // rank test on every column (nv_i > sigma1 * floor) before factorising
    const double floor = sig[0] * kRankFloor;
    double nv[kFastK];
    bool pass = true;
    for (int i = 0; i < k; ++i) {
        nv[i] = sqrt(C[i + i * kFastK]);
        pass = pass && nv[i] > floor;
    }
    if (!pass || !small_chol_inv(C, Ri, k, diag, &ok)) {
        if (threadIdx.x == 0) *slow = 1;
        return;
    }
    for (int i = 0; i < k; ++i)
        if (!(diag[i] > kCollapseFloor * nv[i])) {
            if (threadIdx.x == 0) *slow = 1;
            return;
        }
    small_apply(X, Ri, Y, n, k);
    small_gram(Y, n, k, C, red);
    if (!small_chol_inv(C, Ri, k, diag, &ok)) {
        if (threadIdx.x == 0) *slow = 1;
        return;
    }
    small_apply(Y, Ri, X, n, k);
    for (int i = 0; i < k; ++i) cta_canonical_sign(X + static_cast<std::size_t>(i) * n, n, red, redi);
    for (long long e = threadIdx.x; e < static_cast<long long>(n) * k; e += kB) U[e] = X[e];
    if (threadIdx.x < k) sv[threadIdx.x] = sig[threadIdx.x];
    if (threadIdx.x == 0) {
        st[0] = k;
        st[1] = 0;
        st[2] = 0;
        *slow = 0;
    }
}

// Tall version of the fast path (n * k too large for one CTA's shared memory,
// e.g. C4's 65536-row time mode): the k x k Grams on the fp64 tensor cores
// over many CTAs, the small factorisations and tests in one CTA, the row
// updates and the sign vote spread over the grid.  Every kernel after the
// first test is gated on the flag, and the one-CTA Gram-Schmidt kernel runs
// only when a test fails, so the whole chain can sit in a captured graph.
__global__ void __launch_bounds__(kB) tall_chol_kernel(const double* __restrict__ G, int k, const double* __restrict__ sig,
                                                       int first, double* __restrict__ Ri, int* __restrict__ slow) {
    __shared__ double C[kFastK * kFastK], R[kFastK * kFastK], diag[kFastK];
    __shared__ int ok;
    if (!first && slow[0]) return;
    for (int e = threadIdx.x; e < k * k; e += kB) C[(e % k) + (e / k) * kFastK] = G[e];
    __syncthreads();
    if (first) {  // rank floor on every column before factorising (linalg.cpp:66-100)
        const double floor = sig[0] * kRankFloor;
        bool pass = true;
        for (int i = 0; i < k; ++i) pass = pass && sqrt(C[i + i * kFastK]) > floor;
        if (!pass) {
            if (threadIdx.x == 0) slow[0] = 1;
            return;
        }
    }
    double nv[kFastK];
    for (int i = 0; i < k; ++i) nv[i] = sqrt(C[i + i * kFastK]);
    if (!small_chol_inv(C, R, k, diag, &ok)) {
        if (threadIdx.x == 0) slow[0] = 1;
        return;
    }
    if (first)
        for (int i = 0; i < k; ++i)
            if (!(diag[i] > kCollapseFloor * nv[i])) {  // kCollapseFloor (linalg.cpp:37)
                if (threadIdx.x == 0) slow[0] = 1;
                return;
            }
    for (int e = threadIdx.x; e < kFastK * kFastK; e += kB) Ri[e] = R[e];
    if (first && threadIdx.x == 0) slow[0] = 0;
}

// Y (n x k) = X Ri (column-major; Ri upper triangular, ld kFastK), gated
__global__ void tall_apply_kernel(const double* __restrict__ X, int n, int k, const double* __restrict__ Ri,
                                  double* __restrict__ Y, const int* __restrict__ slow) {
    if (slow[0]) return;
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= static_cast<long long>(n) * k) return;
    const int r = static_cast<int>(e % n), c = static_cast<int>(e / n);
    double s = 0.0;
    for (int p = 0; p <= c; ++p) s = fma(X[r + static_cast<std::size_t>(p) * n], Ri[p + c * kFastK], s);
    Y[e] = s;
}

// one CTA per column: canonical sign (largest |u|, lowest row on ties;
// linalg.cpp:18-32), U written; sv / st from CTA 0; gated
__global__ void __launch_bounds__(kB) tall_sign_kernel(const double* __restrict__ X, int n, int k,
                                                       const double* __restrict__ sig, double* __restrict__ U,
                                                       double* __restrict__ sv, int* __restrict__ st,
                                                       const int* __restrict__ slow) {
    if (slow[0]) return;
    __shared__ double redv[32];
    __shared__ int redi[32];
    const int c = blockIdx.x;
    const double* x = X + static_cast<std::size_t>(c) * n;
    const int p = cta_argmax_abs(x, n, redv, redi);
    const double sgn = x[p] < 0.0 ? -1.0 : 1.0;
    for (int r = threadIdx.x; r < n; r += kB) U[r + static_cast<std::size_t>(c) * n] = sgn * x[r];
    if (threadIdx.x == 0) sv[c] = sig[c];
    if (c == 0 && threadIdx.x == 0) { st[0] = k; st[1] = 0; st[2] = 0; }
}

void basis_products_tall(Ctx* ctx, const double* W, int n, int wc, int k, const double* sig, const int* eig_status,
                         double* U, double* sv, int* st) {
    DBuf<double> G(ctx, static_cast<std::size_t>(k) * k), Ri(ctx, kFastK * kFastK), X(ctx, static_cast<std::size_t>(n) * k),
        Y(ctx, static_cast<std::size_t>(n) * k);
    DBuf<int> slow(ctx, 1);
    const long long nk = static_cast<long long>(n) * k;
    gram<double>(ctx, W, 1, n, n, k, G.get());
    MB_LAUNCH(ctx, tall_chol_kernel, 1, kB, 0, G.get(), k, sig, 1, Ri.get(), slow.get());
    MB_LAUNCH(ctx, tall_apply_kernel, ceil_div(nk, 256), 256, 0, W, n, k, Ri.get(), X.get(), slow.get());
    gram<double>(ctx, X.get(), 1, n, n, k, G.get());
    MB_LAUNCH(ctx, tall_chol_kernel, 1, kB, 0, G.get(), k, sig, 0, Ri.get(), slow.get());
    MB_LAUNCH(ctx, tall_apply_kernel, ceil_div(nk, 256), 256, 0, X.get(), n, k, Ri.get(), Y.get(), slow.get());
    MB_LAUNCH(ctx, tall_sign_kernel, k, kB, 0, Y.get(), n, k, sig, U, sv, st, slow.get());
    BasisScratch bs(ctx, n, k);
    MB_LAUNCH_PDL(ctx, basis_from_products_kernel, 1, kB, bs.smem, W, n, wc, k, sig, eig_status, U, sv, st,
                  static_cast<const int*>(slow.get()), bs.g.get());
}

void basis_from_products_gated(Ctx* ctx, const double* W, int n, int wc, int k, const double* sig,
                               const int* eig_status, double* U, double* sv, int* st, const int* need) {
    BasisScratch bs(ctx, n, k);
    MB_LAUNCH_PDL(ctx, basis_from_products_kernel, 1, kB, bs.smem, W, n, wc, k, sig, eig_status, U, sv, st, need,
                  bs.g.get());
}

void basis_from_products(Ctx* ctx, const double* W, int n, int wc, int k, const double* sig, const int* eig_status,
                         double* U, double* sv, int* st) {
    const std::size_t fsm = 2ull * n * k * sizeof(double);
    if (wc >= k && k <= kFastK && fsm <= 200 * 1024) {
        static std::uint64_t attr = 0;  // per-device mask
        if (first_on_device(attr, ctx->device)) {
            MB_CUDA(cudaFuncSetAttribute(basis_products_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        }
        DBuf<int> slow(ctx, 1);
        MB_LAUNCH(ctx, basis_products_fast_kernel, 1, kB, fsm, W, n, k, sig, U, sv, st, slow.get());
        MB_LAUNCH_PDL(ctx, basis_from_products_kernel, 1, kB, basis_smem(n, k), W, n, wc, k, sig, eig_status, U, sv, st,
                  static_cast<const int*>(slow.get()), static_cast<double*>(nullptr));
        return;
    }
    if (wc >= k && k <= kFastK && n <= (1 << 20)) {
        basis_products_tall(ctx, W, n, wc, k, sig, eig_status, U, sv, st);
        return;
    }
    BasisScratch bs(ctx, n, k);
    MB_LAUNCH_PDL(ctx, basis_from_products_kernel, 1, kB, bs.smem, W, n, wc, k, sig, eig_status, U, sv, st,
              static_cast<const int*>(nullptr), bs.g.get());
}

// ---------------------------------------------------------------------------
// identity basis for an exactly-zero matrix (left_singular_basis, linalg.cpp:326-333)
// ---------------------------------------------------------------------------
__global__ void identity_basis_kernel(double* U, int n, int k, double* sv, int* st) {
    for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < static_cast<long long>(n) * k;
         idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(idx / n), r = static_cast<int>(idx % n);
        U[idx] = (r == c) ? 1.0 : 0.0;
    }
    if (blockIdx.x == 0 && threadIdx.x < k) sv[threadIdx.x] = 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0) { st[0] = 0; st[1] = 1; st[2] = 0; }
}

// ---------------------------------------------------------------------------
// core[col + C*alpha] = sum_i U[i, alpha] * Y[i + rows*col]   (U: rows x r)
// i.e. core = Y_(last) x_last U_last^T refolded (tucker.cpp:71-75 via the last
// mode's projection, which already carries every other updated factor).
// ---------------------------------------------------------------------------
template <typename T>
__global__ void core_from_last_kernel(const T* __restrict__ Y, int rows, int C, const double* __restrict__ U, int r,
                                      double* __restrict__ core) {
    pdl_enter();  // programmatic dependent launch: predecessor complete and visible
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= C * r) return;
    const int col = warp % C, alpha = warp / C;
    double s = 0.0;
    for (int i = lane; i < rows; i += 32)
        s += U[i + static_cast<std::size_t>(alpha) * rows] * static_cast<double>(Y[i + static_cast<std::size_t>(col) * rows]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) core[col + static_cast<std::size_t>(C) * alpha] = s;
}

template <typename T>
void core_from_last(Ctx* ctx, const T* Y, int rows, int C, const double* U, int r, double* core) {
    const long long warps = static_cast<long long>(C) * r;
    MB_LAUNCH_PDL(ctx, core_from_last_kernel<T>, ceil_div(warps * 32, 256), 256, 0, Y, rows, C, U, r, core);
}
template void core_from_last<float>(Ctx*, const float*, int, int, const double*, int, double*);
template void core_from_last<double>(Ctx*, const double*, int, int, const double*, int, double*);

// core_from_last and |core|^2 in one launch: each CTA's partial sum of
// squares goes to part[block]; the last CTA to finish (atomic ticket) sums
// the partials in block order (deterministic) and re-arms the ticket.
template <typename T, int WPO>  // WPO warps per output entry (row range split in WPO contiguous parts)
__global__ void __launch_bounds__(256) core_sumsq_kernel(const T* __restrict__ Y, int rows, int C,
                                                         const double* __restrict__ U, int r, double* __restrict__ core,
                                                         double* __restrict__ part, unsigned* __restrict__ ticket,
                                                         double* __restrict__ out) {
    pdl_enter();  // programmatic dependent launch: predecessor complete and visible
    __shared__ double red[8];
    __shared__ double wsum[8];
    __shared__ bool last;
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int entry = blockIdx.x * (8 / WPO) + wib / WPO, sub = wib % WPO;
    double s = 0.0;
    if (entry < C * r) {
        const int col = entry % C, alpha = entry / C;
        // eight independent chains per lane (fixed combination order): a tall
        // last mode (C4: 65536 rows) made the single chain L2-latency-bound
        const double* u = U + static_cast<std::size_t>(alpha) * rows;
        const T* y = Y + static_cast<std::size_t>(col) * rows;
        const int per = ((rows + WPO - 1) / WPO + 31) & ~31;
        const int r0 = sub * per, r1 = min(rows, r0 + per);
        double a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        int i = r0 + lane;
        for (; i + 7 * 32 < r1; i += 256) {
#pragma unroll
            for (int q = 0; q < 8; ++q) a[q] = fma(u[i + 32 * q], static_cast<double>(y[i + 32 * q]), a[q]);
        }
        for (; i < r1; i += 32) a[0] = fma(u[i], static_cast<double>(y[i]), a[0]);
        s = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    }
    if (lane == 0) wsum[wib] = s;
    __syncthreads();
    double sq = 0.0;
    if (lane == 0 && sub == 0 && entry < C * r) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < WPO; ++q) t += wsum[wib + q];  // parts in row order
        core[(entry % C) + static_cast<std::size_t>(C) * (entry / C)] = t;
        sq = t * t;
    }
    if (lane == 0) red[wib] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < 8; ++i) t += red[i];
        part[blockIdx.x] = t;
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        double tot = 0.0;
        for (unsigned b = 0; b < gridDim.x; ++b) tot += const_cast<volatile double*>(part)[b];
        *out = tot;
        *ticket = 0u;
    }
}

int core_sumsq_blocks(int rows, int C, int r) {
    const long long entries = static_cast<long long>(C) * r;
    const int wpo = rows >= 8192 ? 4 : 1;
    return static_cast<int>((entries + (8 / wpo) - 1) / (8 / wpo));
}

template <typename T>
void core_sumsq(Ctx* ctx, const T* Y, int rows, int C, const double* U, int r, double* core, double* part,
                unsigned* ticket, double* out) {
    const int blocks = core_sumsq_blocks(rows, C, r);
    if (rows >= 8192)
        MB_LAUNCH_PDL(ctx, (core_sumsq_kernel<T, 4>), blocks, 256, 0, Y, rows, C, U, r, core, part, ticket, out);
    else
        MB_LAUNCH_PDL(ctx, (core_sumsq_kernel<T, 1>), blocks, 256, 0, Y, rows, C, U, r, core, part, ticket, out);
}
template void core_sumsq<float>(Ctx*, const float*, int, int, const double*, int, double*, double*, unsigned*, double*);
template void core_sumsq<double>(Ctx*, const double*, int, int, const double*, int, double*, double*, unsigned*, double*);

// ---------------------------------------------------------------------------
// deterministic sum of squares: fixed grid, per-block partials, one final block
// ---------------------------------------------------------------------------
constexpr int kRedBlocks = 1024;

template <typename T>
__global__ void __launch_bounds__(256) sumsq_partial_kernel(const T* __restrict__ x, long long n, double* __restrict__ part) {
    pdl_enter();  // programmatic dependent launch: predecessor complete and visible
    __shared__ double red[8];
    double s = 0.0;
    for (long long i = blockIdx.x * 256ll + threadIdx.x; i < n; i += 256ll * kRedBlocks) {
        const double v = static_cast<double>(x[i]);
        s += v * v;
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

__global__ void __launch_bounds__(256) sum_final_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
    pdl_enter();  // programmatic dependent launch: predecessor complete and visible
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

template <typename T>
void sumsq(Ctx* ctx, const T* x, long long n, double* scratch /* >= kRedBlocks */, double* out) {
    MB_LAUNCH_PDL(ctx, sumsq_partial_kernel<T>, kRedBlocks, 256, 0, x, n, scratch);
    MB_LAUNCH_PDL(ctx, sum_final_kernel, 1, 256, 0, scratch, kRedBlocks, out);
}
template void sumsq<float>(Ctx*, const float*, long long, double*, double*);
template void sumsq<double>(Ctx*, const double*, long long, double*, double*);
int sumsq_scratch() { return kRedBlocks; }

// ---------------------------------------------------------------------------
// factor U (fp64, n x r column-major) -> kernel copy (T, row-major, stride rs,
// zero padded to rs columns)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void factor_rowmajor_kernel(const double* __restrict__ U, int n, int r, int rs, T* __restrict__ out,
                                       const int* __restrict__ need) {
    pdl_enter();  // programmatic dependent launch: predecessor complete and visible
    if (need && need[0] == 0) return;
    const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (idx >= static_cast<long long>(n) * rs) return;
    const int i = static_cast<int>(idx / rs), c = static_cast<int>(idx % rs);
    out[idx] = (c < r) ? static_cast<T>(U[i + static_cast<std::size_t>(c) * n]) : T(0);
}

template <typename T>
void factor_rowmajor_gated(Ctx* ctx, const double* U, int n, int r, int rs, T* out, const int* need) {
    const long long tot = static_cast<long long>(n) * rs;
    MB_LAUNCH_PDL(ctx, factor_rowmajor_kernel<T>, ceil_div(tot, 256), 256, 0, U, n, r, rs, out, need);
}
template void factor_rowmajor_gated<float>(Ctx*, const double*, int, int, int, float*, const int*);
template void factor_rowmajor_gated<double>(Ctx*, const double*, int, int, int, double*, const int*);

template <typename T>
void factor_rowmajor(Ctx* ctx, const double* U, int n, int r, int rs, T* out) {
    factor_rowmajor_gated<T>(ctx, U, n, r, rs, out, nullptr);
}
template void factor_rowmajor<float>(Ctx*, const double*, int, int, int, float*);
template void factor_rowmajor<double>(Ctx*, const double*, int, int, int, double*);

void identity_basis(Ctx* ctx, double* U, int n, int k, double* sv, int* st) {
    MB_LAUNCH(ctx, identity_basis_kernel, ceil_div(static_cast<long long>(n) * k + 1, 256), 256, 0, U, n, k, sv, st);
}

}  // namespace machb
