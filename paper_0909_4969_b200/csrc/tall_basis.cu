// Leading left singular basis of a matricization whose column side is too
// wide for a Gram (X_(2) is 65536 x 64000, whose
// column Gram would be 32.8 GB and a dense 64000^2 eigenproblem).
//
// Reference semantics: left_singular_basis / sparse_mode_basis take the
// column side here (sparse_kernels.cpp:82-89: X^T X, then W = X V and
// orthonormal_columns), which is the same left subspace as the rows side.
// This file computes it the way the reference's own subspace_side_basis does
// for large sides (linalg.cpp:128-193), on the rows side and without forming
// any side x side matrix:
//   Q (rows x b, b = k + kOversample) orthonormal, seeded start;
//   repeat:  Z = A^T Q;  T = Z^T Z (= Q^T A A^T Q);  (theta, S) = eig(T);
//            Ritz block R = Q S[:, :k];  converged when every previous Ritz
//            vector with theta_i > theta_1 kDeficiencyFloor^2 lies in span(R)
//            to kSubspaceTol;  else Q = orth(A (Z S) diag(1/theta)).
// then basis_from_side (rank floor, canonical signs, completion) as the
// reference (linalg.cpp:261-276).  A is applied implicitly: sparse A through
// two sorted layouts of the nonzeros (grouped by row for A Z, by column for
// A^T Q), dense A through plain tiled kernels.  Q and Z are row-major with the
// b block columns contiguous, so each gathered operand row is one coalesced
// 8*b-byte read.  All reductions run in a fixed order (deterministic); the
// small b x b eigenproblems run on device (eig_topk), the host only loops and
// reads the convergence test.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>

#include "sparse_ttm.cuh"

namespace machb {

namespace {

constexpr int kOversampleT = 8;          // linalg_internal.hpp:14
constexpr int kMaxItersT = 300;          // linalg_internal.hpp:15
constexpr double kSubspaceTolT = 1e-10;  // linalg_internal.hpp:16
constexpr double kDeficiencyT = 1e-10;   // linalg_internal.hpp:17
constexpr std::uint64_t kSubspaceSeedT = 0x4D414348ull;  // linalg_internal.hpp ("MACH")

__device__ __forceinline__ long long tb_decode(unsigned long long k, const ColDecode& D) {
    long long c = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j)
        if (j < D.nf) c += static_cast<long long>((k >> D.shift[j]) & D.mask[j]) * D.stride[j];
    return c;
}

__device__ __forceinline__ std::uint64_t tb_hash(std::uint64_t seed, std::uint64_t c) {  // internal.hpp:68-73
    std::uint64_t z = seed + (c + 1ull) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// start block: q(r, c) = 2 u(seed, c*side + r) - 1 (linalg.cpp:137-145), row-major
__global__ void tb_start_kernel(double* __restrict__ Q, long long rows, int b) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= rows * b) return;
    const long long r = e / b;
    const int c = static_cast<int>(e - r * b);
    const std::uint64_t h = tb_hash(kSubspaceSeedT, static_cast<std::uint64_t>(c) * rows + r);
    Q[e] = 2.0 * (static_cast<double>(h >> 11) * 0x1.0p-53) - 1.0;
}

// ---- sparse operators (warp per output row; lane j < b owns column j) ----
// out[g(run) * b + j] = sum over the run's nonzeros of v * in[h(key) * b + j]
// where the run is a row of the row-grouped layout (A Z: h = column) or a
// column of the column-grouped layout (A^T Q: h = row, g = decoded column).
template <typename T, typename K, bool COLS>
__global__ void __launch_bounds__(256) tb_spmm_kernel(const K* __restrict__ keys, const T* __restrict__ vals,
                                                      const long long* __restrict__ rs,
                                                      const long long* __restrict__ re, long long nrun, ColDecode D,
                                                      unsigned long long rmask, int b, const double* __restrict__ in,
                                                      double* __restrict__ out) {
    const long long w = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= nrun) return;
    const long long s = rs[w], e1 = COLS ? rs[w + 1] : re[w];
    double acc0 = 0.0, acc1 = 0.0;
    long long oidx = COLS ? 0 : w;
    for (long long base = s; base < e1; base += 32) {
        const long long e = base + lane;
        unsigned long long kk = 0;
        double vv = 0.0;
        if (e < e1) {
            kk = static_cast<unsigned long long>(keys[e]);
            vv = static_cast<double>(vals[e]);
        }
        long long h = COLS ? static_cast<long long>(kk & rmask) : tb_decode(kk, D);
        if (COLS && base == s) oidx = tb_decode(static_cast<unsigned long long>(__shfl_sync(0xffffffffu, kk, 0)), D);
        const int m = static_cast<int>(min(32ll, e1 - base));
        int q = 0;
        for (; q + 2 <= m; q += 2) {  // two gathers in flight, two accumulator chains
            const long long h0 = __shfl_sync(0xffffffffu, h, q), h1 = __shfl_sync(0xffffffffu, h, q + 1);
            const double v0 = __shfl_sync(0xffffffffu, vv, q), v1 = __shfl_sync(0xffffffffu, vv, q + 1);
            if (lane < b) {
                const double g0 = in[h0 * b + lane], g1 = in[h1 * b + lane];
                acc0 = fma(v0, g0, acc0);
                acc1 = fma(v1, g1, acc1);
            }
        }
        if (q < m) {
            const long long h0 = __shfl_sync(0xffffffffu, h, q);
            const double v0 = __shfl_sync(0xffffffffu, vv, q);
            if (lane < b) acc0 = fma(v0, in[h0 * b + lane], acc0);
        }
    }
    if (lane < b && s < e1) out[oidx * b + lane] = acc0 + acc1;
}

// ---- dense operators for a column-major Y (rows x cols) ----
// Z (cols x b) = Y^T Q: warp per column, lanes stride the rows, each lane
// keeps b partial sums, then a fixed-order warp reduction per column j
template <typename T>
__global__ void __launch_bounds__(256) tb_dense_t_kernel(const T* __restrict__ Y, long long rows, long long cols, int b,
                                                         const double* __restrict__ Q, double* __restrict__ Z) {
    const long long c = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (c >= cols) return;
    double acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.0;
    for (long long r = lane; r < rows; r += 32) {
        const double y = static_cast<double>(Y[r + c * rows]);
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (j < b) acc[j] = fma(y, Q[r * b + j], acc[j]);
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        double v = acc[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && j < b) Z[c * b + j] = v;
    }
}

// W (rows x b) = Y Z: thread per (row, j), columns in order
template <typename T>
__global__ void __launch_bounds__(256) tb_dense_n_kernel(const T* __restrict__ Y, long long rows, long long cols, int b,
                                                         const double* __restrict__ Z, double* __restrict__ W) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= rows * b) return;
    const long long r = e % rows;
    const int j = static_cast<int>(e / rows);
    double s = 0.0;
    for (long long c = 0; c < cols; ++c) s = fma(static_cast<double>(Y[r + c * rows]), Z[c * b + j], s);
    W[r * b + j] = s;
}

// ---- small dense steps ----
// out = in (n x bi, row-major) * S (bi x bo, column-major, ld lds) * diag(scale)
// into row-major (ld bo) or column-major (ld n) output
__global__ void tb_rotate_kernel(const double* __restrict__ in, long long n, int bi, const double* __restrict__ S, int lds,
                                 int bo, const double* __restrict__ sig, int col_major, double* __restrict__ out) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= n * bo) return;
    const long long r = e / bo;
    const int j = static_cast<int>(e - r * bo);
    double s = 0.0;
    for (int p = 0; p < bi; ++p) s = fma(in[r * bi + p], S[p + static_cast<long long>(j) * lds], s);
    if (sig) {  // scale by 1 / theta_j = 1 / sig_j^2 (columns of A (Z S) have lengths ~ theta_j)
        const double t = sig[j] * sig[j];
        s = t > 0.0 ? s / t : s;
    }
    if (col_major) out[r + static_cast<long long>(j) * n] = s;
    else out[r * bo + j] = s;
}

// Equilibrated Cholesky: with D = diag(G)^{-1/2}, R = chol(D G D) (upper)
// and Ri = D R^{-1} (column-major b x b), so that W Ri is orthonormal for
// columns of very different lengths (a filtered block).  ok[0] = 0 on a
// non-positive pivot.
__global__ void tb_chol_inv_kernel(const double* __restrict__ G, int b, double* __restrict__ Ri, int* __restrict__ ok) {
    __shared__ double R[32 * 32];
    __shared__ double dsc[32];
    __shared__ int good;
    if (threadIdx.x < b) {
        const double g = G[threadIdx.x + threadIdx.x * b];
        dsc[threadIdx.x] = g > 0.0 ? 1.0 / sqrt(g) : 0.0;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < b * b; e += blockDim.x) R[e] = G[e] * dsc[e % b] * dsc[e / b];
    __syncthreads();
    if (threadIdx.x == 0) {
        good = 1;
        for (int j = 0; j < b && good; ++j) {
            double dj = R[j + j * b];
            for (int p = 0; p < j; ++p) dj -= R[p + j * b] * R[p + j * b];
            if (!(dj > 0.0) || !(dsc[j] > 0.0)) { good = 0; break; }
            const double rjj = sqrt(dj);
            R[j + j * b] = rjj;
            for (int l = j + 1; l < b; ++l) {
                double v = R[j + l * b];
                for (int p = 0; p < j; ++p) v -= R[p + j * b] * R[p + l * b];
                R[j + l * b] = v / rjj;
            }
        }
        ok[0] = good;
    }
    __syncthreads();
    if (!good) return;
    if (threadIdx.x < b) {  // column c of R^{-1} by back substitution, rows scaled by D
        const int c = threadIdx.x;
        double x[32];
        for (int r = b - 1; r >= 0; --r) {
            double v = (r == c) ? 1.0 : 0.0;
            for (int p = r + 1; p <= c; ++p) v -= R[r + p * b] * x[p];
            x[r] = (r <= c) ? v / R[r + r * b] : 0.0;
        }
        for (int r = 0; r < b; ++r) Ri[r + c * b] = dsc[r] * x[r];
    }
}

// out = a * MY + c1 * Y1 + c0 * Y0 (Chebyshev three-term step), elementwise
__global__ void tb_cheb_kernel(const double* __restrict__ MY, const double* __restrict__ Y1, const double* __restrict__ Y0,
                               long long n, double a, double c1, double c0, double* __restrict__ out) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= n) return;
    double v = a * MY[e] + c1 * Y1[e];
    if (Y0) v += c0 * Y0[e];
    out[e] = v;
}

// per column i < k: |prev_i - R C_i|_2 with C = R^T prev (the (k..2k, 0..k)
// block of the Gram of [R | prev]); one CTA per column, fixed-order sum
__global__ void tb_resid_kernel(const double* __restrict__ RP, long long n, int k, const double* __restrict__ G2,
                                double* __restrict__ out) {
    const int i = blockIdx.x;
    const int k2 = 2 * k;
    __shared__ double c[32];
    __shared__ double red[32];
    if (threadIdx.x < k) c[threadIdx.x] = G2[threadIdx.x + static_cast<long long>(k + i) * k2];  // (R^T prev)(p, i)
    __syncthreads();
    double s = 0.0;
    for (long long r = threadIdx.x; r < n; r += blockDim.x) {
        double v = RP[r + static_cast<long long>(k + i) * n];
        for (int p = 0; p < k; ++p) v -= RP[r + static_cast<long long>(p) * n] * c[p];
        s = fma(v, v, s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += red[w];
        out[i] = sqrt(t);
    }
}

struct TallOp {
    long long rows = 0, cols = 0;
    std::function<void(const double*, double*)> At;  // Q (rows x b) -> Z (cols x b), row-major
    std::function<void(const double*, double*)> A;   // Z (cols x b) -> W (rows x b), row-major
};

// Q <- orth(W) by CholQR2 (W's columns are already near-orthogonal: either
// the seeded start or Ritz directions rescaled to unit length)
bool cholqr2(Ctx* ctx, double* W, double* tmp, long long rows, int b, double* G, double* Ri, int* ok) {
    for (int pass = 0; pass < 2; ++pass) {
        gram<double>(ctx, W, b, 1, static_cast<int>(rows), b, G);
        MB_LAUNCH(ctx, tb_chol_inv_kernel, 1, 256, 0, G, b, Ri, ok);
        int h = 0;
        to_host(ctx, &h, ok, 1);
        sync(ctx);
        if (!h) return false;
        MB_LAUNCH(ctx, tb_rotate_kernel, ceil_div(rows * b, 256), 256, 0, W, rows, b, Ri, b, b,
                  static_cast<const double*>(nullptr), 0, tmp);
        MB_CUDA(cudaMemcpyAsync(W, tmp, static_cast<std::size_t>(rows) * b * sizeof(double), cudaMemcpyDeviceToDevice,
                                ctx->stream));
    }
    return true;
}

void tall_iterate(Ctx* ctx, const TallOp& op, int k, double* U, double* sv, int* st, double tol = kSubspaceTolT) {
    const long long rows = op.rows, cols = op.cols;
    if (rows > (1ll << 30) || cols > (1ll << 30)) throw_arg("tall basis: matricization too large");
    const int b = static_cast<int>(std::min<long long>(k + kOversampleT, std::min(rows, cols)));
    if (b > 32) throw Error(MACH_ERR_INTERNAL, "tall basis: rank above 24 not supported");
    const std::size_t rb = static_cast<std::size_t>(rows) * b;
    DBuf<double> Q(ctx, rb), Y0(ctx, rb), Y1(ctx, rb), Y2(ctx, rb), Z(ctx, static_cast<std::size_t>(cols) * b);
    DBuf<double> T(ctx, b * b), S(ctx, b * b), sig(ctx, b), G(ctx, b * b), Ri(ctx, b * b);
    DBuf<double> RP(ctx, static_cast<std::size_t>(rows) * 2 * k), G2(ctx, 4 * k * k), res(ctx, k);
    DBuf<double> work(ctx, eig_work_doubles(b, b));
    DBuf<int> est(ctx, 3), ok(ctx, 1);
    auto apply_M = [&](const double* in, double* out) {  // out = A A^T in
        MB_CUDA(cudaMemsetAsync(Z.get(), 0, static_cast<std::size_t>(cols) * b * sizeof(double), ctx->stream));
        op.At(in, Z.get());
        MB_CUDA(cudaMemsetAsync(out, 0, rb * sizeof(double), ctx->stream));
        op.A(Z.get(), out);
    };
    MB_LAUNCH(ctx, tb_start_kernel, ceil_div(rows * b, 256), 256, 0, Q.get(), rows, b);
    if (!cholqr2(ctx, Q.get(), Y0.get(), rows, b, G.get(), Ri.get(), ok.get()))
        throw Error(MACH_ERR_CONVERGENCE, "subspace iteration start block is rank deficient", 1);
    // Chebyshev degree per outer iteration (1 = the reference's plain
    // subspace iteration); the filter damps [0, theta_b] and amplifies the
    // wanted end, so each outer step costs 2m + 1 operator products
    static const int degree = std::getenv("MACH_TALL_DEGREE") ? std::atoi(std::getenv("MACH_TALL_DEGREE")) : 8;
    static const int maxit = std::getenv("MACH_TALL_MAXIT") ? std::atoi(std::getenv("MACH_TALL_MAXIT")) : kMaxItersT;
    std::vector<double> hsig(static_cast<std::size_t>(b)), hres(static_cast<std::size_t>(k), 1.0);
    bool have_prev = false, conv = false;
    int it = 0;
    for (; it < maxit; ++it) {
        // ---- Rayleigh-Ritz on span(Q) ----
        MB_CUDA(cudaMemsetAsync(Z.get(), 0, static_cast<std::size_t>(cols) * b * sizeof(double), ctx->stream));
        op.At(Q.get(), Z.get());
        gram<double>(ctx, Z.get(), b, 1, static_cast<int>(cols), b, T.get());  // T = Q^T A A^T Q
        eig_topk(ctx, T.get(), b, b, work.get(), S.get(), sig.get(), est.get());
        // Ritz block R = Q S[:, :k] into RP[:, :k] (column-major)
        MB_LAUNCH(ctx, tb_rotate_kernel, ceil_div(rows * k, 256), 256, 0, Q.get(), rows, b, S.get(), b, k,
                  static_cast<const double*>(nullptr), 1, RP.get());
        to_host(ctx, hsig.data(), sig.get(), hsig.size());
        if (have_prev) {
            gram<double>(ctx, RP.get(), 1, rows, static_cast<int>(rows), 2 * k, G2.get());
            MB_LAUNCH(ctx, tb_resid_kernel, k, 256, 0, RP.get(), rows, k, G2.get(), res.get());
            to_host(ctx, hres.data(), res.get(), hres.size());
        }
        sync(ctx);
        if (have_prev) {
            const double t0 = hsig[0] * hsig[0];
            const double floor = t0 * kDeficiencyT * kDeficiencyT;
            conv = true;
            for (int i = 0; i < k && conv; ++i) {
                if (hsig[static_cast<std::size_t>(i)] * hsig[static_cast<std::size_t>(i)] <= floor) continue;
                if (!(hres[static_cast<std::size_t>(i)] <= tol)) conv = false;
            }
            if (std::getenv("MACH_DEBUG_TALL")) {
                double mx = 0.0;
                for (double v : hres) mx = std::max(mx, v);
                std::fprintf(stderr, "[tall] it=%d max resid %.3e sig1 %.4e sig_k %.4e sig_b %.4e\n", it, mx, hsig[0],
                             hsig[static_cast<std::size_t>(k - 1)], hsig[static_cast<std::size_t>(b - 1)]);
            }
            if (conv) break;
        }
        if (std::getenv("MACH_DEBUG_TALL"))
            std::fprintf(stderr, "[tall] it=%d rows=%lld cols=%lld b=%d k=%d sig1 %.4e sig_b %.4e\n", it, rows, cols, b, k,
                         hsig[0], hsig[static_cast<std::size_t>(b - 1)]);
        if (hsig[0] == 0.0) { conv = true; break; }  // A = 0: basis_from_side completes every direction
        MB_CUDA(cudaMemcpyAsync(RP.get() + static_cast<std::size_t>(rows) * k, RP.get(),
                                static_cast<std::size_t>(rows) * k * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
        have_prev = true;
        // ---- filter the Ritz block: Y_m = T_m((M - c) / e) Q S, [0, theta_b] damped ----
        // The degree is capped so that the amplification of the top Ritz
        // direction, T_m(x_1), stays below 1e6: every filtered column then
        // keeps its own directions well above rounding and the equilibrated
        // CholQR2 below resolves them.
        const double cut = hsig[static_cast<std::size_t>(b - 1)] * hsig[static_cast<std::size_t>(b - 1)];
        const double th1 = hsig[0] * hsig[0];
        int m = 1;
        if (degree > 1 && cut > 0.0) {
            const double x1 = (th1 - 0.5 * cut) / (0.5 * cut);
            const double ac = std::acosh(std::max(1.0, x1));
            while (m < degree && std::cosh((m + 1) * ac) <= 1e6) ++m;
        }
        double* y0 = Y0.get();
        double* y1 = Y1.get();
        double* y2 = Y2.get();
        bool orth = false;
        for (int attempt = 0; attempt < 2 && !orth; ++attempt) {
            if (attempt) m = 1;  // a filtered block CholQR2 cannot resolve: plain power step
            y0 = Y0.get();
            y1 = Y1.get();
            y2 = Y2.get();
            MB_LAUNCH(ctx, tb_rotate_kernel, ceil_div(rows * b, 256), 256, 0, Q.get(), rows, b, S.get(), b, b,
                      static_cast<const double*>(nullptr), 0, y0);
            if (m <= 1) {
                apply_M(y0, y1);
                std::swap(y0, y1);
            } else {
                const double e = 0.5 * cut, c = 0.5 * cut;
                apply_M(y0, y2);  // y1 = (M y0 - c y0) / e
                MB_LAUNCH(ctx, tb_cheb_kernel, ceil_div(static_cast<long long>(rb), 256), 256, 0, y2, y0,
                          static_cast<const double*>(nullptr), static_cast<long long>(rb), 1.0 / e, -c / e, 0.0, y1);
                for (int j = 2; j <= m; ++j) {  // y2 = 2 (M y1 - c y1) / e - y0
                    apply_M(y1, y2);
                    MB_LAUNCH(ctx, tb_cheb_kernel, ceil_div(static_cast<long long>(rb), 256), 256, 0, y2, y1, y0,
                              static_cast<long long>(rb), 2.0 / e, -2.0 * c / e, -1.0, y2);
                    std::swap(y0, y1);  // (y0, y1, y2) <- (y1, y2, y0)
                    std::swap(y1, y2);
                }
                std::swap(y0, y1);  // the filtered block is in y0
            }
            orth = cholqr2(ctx, y0, y1, rows, b, G.get(), Ri.get(), ok.get());
            if (!orth && m <= 1) break;
        }
        if (!orth) {
            if (std::getenv("MACH_DEBUG_TALL")) std::fprintf(stderr, "[tall] it=%d orthonormalisation failed (m=%d)\n", it, m);
            // A A^T has rank below b: the current Ritz block is exact
            conv = true;
            break;
        }
        MB_CUDA(cudaMemcpyAsync(Q.get(), y0, rb * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    }
    if (!conv) {
        int first = k;
        for (int i = 0; i < k; ++i)
            if (!(hres[static_cast<std::size_t>(i)] <= tol)) { first = i + 1; break; }
        throw Error(MACH_ERR_CONVERGENCE, "subspace iteration did not converge", first);
    }
    const int hst[3] = {1, 0, it};
    to_device(ctx, est.get(), hst, 3);
    basis_from_side(ctx, RP.get(), sig.get(), static_cast<int>(rows), k, est.get(), U, sv, st);
    sync(ctx);  // the host-side status above is a stack temporary
}

}  // namespace

long long tall_min_cols() {  // read per call: tests lower it to reach the path at small shapes
    const char* e = std::getenv("MACH_TALL_MIN_COLS");
    return e ? std::atoll(e) : 4096;
}

template <typename T>
void sparse_tall_basis(Ctx* ctx, const mach_sparse* X, const ModePlan& P, int k, double* U, double* sv, int* st) {
    const int n = P.mode;
    const long long rows = X->dims[static_cast<std::size_t>(n)];
    const long long cols = X->numel / rows;
    if (X->nnz == 0) {
        identity_basis(ctx, U, static_cast<int>(rows), k, sv, st);
        return;
    }
    auto L = std::make_shared<ColLayout>();
    build_col_layout<T>(ctx, X, n, *L);
    const ColDecode D = plan_col_decode(X->dims, P);
    TallOp op;
    op.rows = rows;
    op.cols = cols;
    const int b = static_cast<int>(std::min<long long>(k + kOversampleT, std::min(rows, cols)));
    const unsigned long long nmask = (1ull << L->bn) - 1ull;
    op.At = [ctx, L, b, nmask](const double* Q, double* Z) {
        if (L->nruns == 0) return;
        const ColDecode& CD = L->dec;
        if (L->key64)
            MB_LAUNCH(ctx, (tb_spmm_kernel<T, unsigned long long, true>), ceil_div(L->nruns * 32, 256), 256, 0,
                      reinterpret_cast<const unsigned long long*>(L->keys.get()), reinterpret_cast<const T*>(L->vals.get()),
                      L->runs.get(), static_cast<const long long*>(nullptr), L->nruns, CD, nmask, b, Q, Z);
        else
            MB_LAUNCH(ctx, (tb_spmm_kernel<T, unsigned int, true>), ceil_div(L->nruns * 32, 256), 256, 0,
                      reinterpret_cast<const unsigned int*>(L->keys.get()), reinterpret_cast<const T*>(L->vals.get()),
                      L->runs.get(), static_cast<const long long*>(nullptr), L->nruns, CD, nmask, b, Q, Z);
    };
    const ModePlan* PP = &P;
    op.A = [ctx, PP, D, b, rows](const double* Z, double* W) {
        if (PP->key64)
            MB_LAUNCH(ctx, (tb_spmm_kernel<T, unsigned long long, false>), ceil_div(rows * 32, 256), 256, 0,
                      reinterpret_cast<const unsigned long long*>(PP->keys.get()), reinterpret_cast<const T*>(PP->vals.get()),
                      PP->row_start.get(), PP->row_end.get(), rows, D, 0ull, b, Z, W);
        else
            MB_LAUNCH(ctx, (tb_spmm_kernel<T, unsigned int, false>), ceil_div(rows * 32, 256), 256, 0,
                      reinterpret_cast<const unsigned int*>(PP->keys.get()), reinterpret_cast<const T*>(PP->vals.get()),
                      PP->row_start.get(), PP->row_end.get(), rows, D, 0ull, b, Z, W);
    };
    // empty rows of X_(n) give zero rows of W (the kernel writes nothing).
    // Stop rule: the reference's 1e-10 Ritz-vector residual (linalg.cpp:170)
    // for fp64 tensors; fp32 tensors carry 6e-8 relative precision and a
    // 1e-3 parity bar, so their subspace is taken at 1e-7
    tall_iterate(ctx, op, k, U, sv, st, sizeof(T) == 4 ? 1e-7 : kSubspaceTolT);
}

template <typename T>
void dense_tall_basis(Ctx* ctx, const T* Y, int rows, long long cols, int k, double* U, double* sv, int* st) {
    TallOp op;
    op.rows = rows;
    op.cols = cols;
    const int b = static_cast<int>(std::min<long long>(k + kOversampleT, std::min<long long>(rows, cols)));
    op.At = [ctx, Y, rows, cols, b](const double* Q, double* Z) {
        MB_LAUNCH(ctx, tb_dense_t_kernel<T>, ceil_div(cols * 32, 256), 256, 0, Y, static_cast<long long>(rows), cols, b, Q, Z);
    };
    op.A = [ctx, Y, rows, cols, b](const double* Z, double* W) {
        MB_LAUNCH(ctx, tb_dense_n_kernel<T>, ceil_div(static_cast<long long>(rows) * b, 256), 256, 0, Y,
                  static_cast<long long>(rows), cols, b, Z, W);
    };
    tall_iterate(ctx, op, k, U, sv, st);
}

template void sparse_tall_basis<float>(Ctx*, const mach_sparse*, const ModePlan&, int, double*, double*, int*);
template void sparse_tall_basis<double>(Ctx*, const mach_sparse*, const ModePlan&, int, double*, double*, int*);
template void dense_tall_basis<float>(Ctx*, const float*, int, long long, int, double*, double*, int*);
template void dense_tall_basis<double>(Ctx*, const double*, int, long long, int, double*, double*, int*);

}  // namespace machb
