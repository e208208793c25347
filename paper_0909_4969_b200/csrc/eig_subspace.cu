// Warm-started, Chebyshev-filtered block subspace eigensolver for the HOOI
// eigen step (reference: gram_side_basis, proj/src/linalg.cpp:106-120 — the
// top-k eigenpairs of the symmetric Gram of Y_(n)).
//
// Why not a full tridiagonal eigensolver per mode: the n sequential Householder
// steps are latency-bound on a GPU (hundreds of microseconds at n = 100),
// while HOOI asks for only k << n eigenvectors of a Gram that barely moves
// between sweeps.  This kernel keeps G in shared memory and runs, in one CTA:
//   X <- previous sweep's Ritz block (or a deterministic random block)
//   repeat: Rayleigh-Ritz (H = X^T G X, one-warp cyclic Jacobi on H),
//           residual test |G x_i - theta_i x_i| <= tol * theta_1 for i < k,
//           degree-m Chebyshev filter damping [0, theta_b], CGS2 orthonormalise
// The residual certificate bounds each Ritz vector's angle to its eigenvector
// by residual / gap, so converged output equals the reference's exact
// eigendecomposition to that precision.  When the residual test is not met
// within max_iters (tiny spectral gaps), status[0] stays 0 and the exact
// selected-eigenpair solver (eig.cu) runs instead — it checks status and is a
// no-op otherwise.
#include "sparse_ttm.cuh"

namespace machb {

namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxB = 32;

__device__ double cta_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < kWarps; ++i) s += red[i];
    return s;
}

__device__ double rnd_unit(unsigned c, unsigned i) {
    unsigned long long z = 0x9E3779B97F4A7C15ULL * (static_cast<unsigned long long>(c) * 0x100000001B3ull + i + 7ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return static_cast<double>(z >> 11) * 0x1.0p-53 * 2.0 - 1.0;
}

// OUT (n x b) = G X, G n x n column-major (smem or global), X/OUT in smem ld n
__device__ void gemm_gx(const double* G, const double* X, double* OUT, int n, int b) {
    const int ncg = (b + 3) / 4;  // column groups of 4
    for (int w = threadIdx.x; w < n * ncg; w += kThreads) {
        const int i = w % n, cg = w / n;
        const int j0 = cg * 4;
        double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
        const double* x0 = X + static_cast<std::size_t>(j0) * n;
        for (int l = 0; l < n; ++l) {
            const double g = G[i + static_cast<std::size_t>(l) * n];
            a0 = fma(g, x0[l], a0);
            if (j0 + 1 < b) a1 = fma(g, x0[l + n], a1);
            if (j0 + 2 < b) a2 = fma(g, x0[l + 2 * n], a2);
            if (j0 + 3 < b) a3 = fma(g, x0[l + 3 * n], a3);
        }
        OUT[i + static_cast<std::size_t>(j0) * n] = a0;
        if (j0 + 1 < b) OUT[i + static_cast<std::size_t>(j0 + 1) * n] = a1;
        if (j0 + 2 < b) OUT[i + static_cast<std::size_t>(j0 + 2) * n] = a2;
        if (j0 + 3 < b) OUT[i + static_cast<std::size_t>(j0 + 3) * n] = a3;
    }
    __syncthreads();
}

// C (b x b) = A^T B for n x b blocks (warp per entry, fixed order)
__device__ void gram_ab(const double* A, const double* B, double* C, int n, int b, bool sym) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int e = warp; e < b * b; e += kWarps) {
        const int i = e % b, j = e / b;
        if (sym && i > j) continue;
        double s = 0.0;
        for (int r = lane; r < n; r += 32) s += A[r + static_cast<std::size_t>(i) * n] * B[r + static_cast<std::size_t>(j) * n];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
            C[i + j * kMaxB] = s;
            if (sym) C[j + i * kMaxB] = s;
        }
    }
    __syncthreads();
}

// classical Gram-Schmidt applied twice (CGS2), column by column; returns
// false if a column collapses (then it is re-randomised once)
__device__ void orthonormalize(double* X, int n, int b, double* coef, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int j = 0; j < b; ++j) {
        double* xj = X + static_cast<std::size_t>(j) * n;
        for (int attempt = 0; attempt < 2; ++attempt) {
            double n0 = 0.0;
            for (int r = threadIdx.x; r < n; r += kThreads) n0 += xj[r] * xj[r];
            n0 = sqrt(cta_sum(n0, red));
            for (int pass = 0; pass < 2 && j > 0; ++pass) {
                for (int c = warp; c < j; c += kWarps) {
                    const double* xc = X + static_cast<std::size_t>(c) * n;
                    double s = 0.0;
                    for (int r = lane; r < n; r += 32) s += xc[r] * xj[r];
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                    if (lane == 0) coef[c] = s;
                }
                __syncthreads();
                for (int r = threadIdx.x; r < n; r += kThreads) {
                    double v = xj[r];
                    for (int c = 0; c < j; ++c) v -= X[r + static_cast<std::size_t>(c) * n] * coef[c];
                    xj[r] = v;
                }
                __syncthreads();
            }
            double nn = 0.0;
            for (int r = threadIdx.x; r < n; r += kThreads) nn += xj[r] * xj[r];
            nn = sqrt(cta_sum(nn, red));
            if (nn > 1e-10 * n0 && nn > 0.0) {
                const double inv = 1.0 / nn;
                for (int r = threadIdx.x; r < n; r += kThreads) xj[r] *= inv;
                __syncthreads();
                break;
            }
            for (int r = threadIdx.x; r < n; r += kThreads) xj[r] = rnd_unit(1000u + j + 97u * attempt, r);
            __syncthreads();
        }
    }
}

// one-warp cyclic Jacobi on H (b x b, ld kMaxB) -> eigenvectors W, values th
// (descending, W columns permuted alike)
__device__ void warp_jacobi(double* H, double* W, double* th, int b, int max_sweeps) {
    const int lane = threadIdx.x & 31;
    __shared__ int jp[kMaxB / 2], jq[kMaxB / 2];
    __shared__ double jc[kMaxB / 2], js[kMaxB / 2];
    const int bp = (b + 1) & ~1;  // even player count (a dummy when b is odd)
    for (int e = lane; e < kMaxB * kMaxB; e += 32) W[e] = ((e % kMaxB) == (e / kMaxB)) ? 1.0 : 0.0;
    __syncwarp();
    double nrm = 0.0;
    for (int e = lane; e < b * b; e += 32) {
        const double h = H[(e % b) + (e / b) * kMaxB];
        nrm += h * h;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
    const int M = bp - 1;
    for (int sweep = 0; sweep < max_sweeps && b > 1; ++sweep) {
        double off = 0.0;
        if (lane < b)
            for (int i = 0; i < lane; ++i) off += H[i + lane * kMaxB] * H[i + lane * kMaxB];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) off += __shfl_xor_sync(0xffffffffu, off, o);
        if (off <= 1e-30 * nrm) break;
        const int np = bp / 2;
        for (int r = 0; r < M; ++r) {
            // pair of this lane (circle method), rotation angle from H
            if (lane < np) {
                int p, q;
                if (lane == 0) { p = 0; q = r + 1; }
                else { p = (r + lane) % M + 1; q = (r - lane + M) % M + 1; }
                if (p > q) { const int t = p; p = q; q = t; }
                double c = 1.0, s = 0.0;
                if (q < b) {
                    const double hpq = H[p + q * kMaxB];
                    if (hpq != 0.0) {
                        const double tau = (H[q + q * kMaxB] - H[p + p * kMaxB]) / (2.0 * hpq);
                        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                        c = 1.0 / sqrt(1.0 + t * t);
                        s = t * c;
                    }
                } else {
                    p = q = 0;
                }
                jp[lane] = p; jq[lane] = q; jc[lane] = c; js[lane] = s;
            }
            __syncwarp();
            // rows p, q of H: lane j owns column j, all pairs (disjoint) in turn
            if (lane < b) {
                const int j = lane;
#pragma unroll 4
                for (int t = 0; t < np; ++t) {
                    const double s = js[t], c = jc[t];
                    const int p = jp[t], q = jq[t];
                    const double a = H[p + j * kMaxB], bq = H[q + j * kMaxB];
                    H[p + j * kMaxB] = c * a - s * bq;
                    H[q + j * kMaxB] = s * a + c * bq;
                }
            }
            __syncwarp();
            // columns p, q of H and W: lane j owns row j
            if (lane < b) {
                const int j = lane;
#pragma unroll 4
                for (int t = 0; t < np; ++t) {
                    const double s = js[t], c = jc[t];
                    const int p = jp[t], q = jq[t];
                    const double a = H[j + p * kMaxB], bq = H[j + q * kMaxB];
                    H[j + p * kMaxB] = c * a - s * bq;
                    H[j + q * kMaxB] = s * a + c * bq;
                    const double wa = W[j + p * kMaxB], wb = W[j + q * kMaxB];
                    W[j + p * kMaxB] = c * wa - s * wb;
                    W[j + q * kMaxB] = s * wa + c * wb;
                }
            }
            __syncwarp();
        }
    }
    // sort descending (selection sort by lane 0 on indices, then permute)
    __shared__ int perm[kMaxB];
    if (lane == 0) {
        for (int i = 0; i < b; ++i) perm[i] = i;
        for (int i = 0; i < b; ++i) {
            int best = i;
            for (int j = i + 1; j < b; ++j)
                if (H[perm[j] + perm[j] * kMaxB] > H[perm[best] + perm[best] * kMaxB]) best = j;
            const int t = perm[i]; perm[i] = perm[best]; perm[best] = t;
        }
    }
    __syncwarp();
    for (int i = lane; i < b; i += 32) th[i] = H[perm[i] + perm[i] * kMaxB];
    __syncwarp();
    // W columns permuted into H's (now free) storage, then copied back
    for (int e = lane; e < b * b; e += 32) {
        const int r = e % b, cidx = e / b;
        H[r + cidx * kMaxB] = W[r + perm[cidx] * kMaxB];
    }
    __syncwarp();
    for (int e = lane; e < b * b; e += 32) W[(e % b) + (e / b) * kMaxB] = H[(e % b) + (e / b) * kMaxB];
    __syncwarp();
}

// X <- X W (n x b) in place using tmp (n x b)
__device__ void rotate(double* X, const double* W, double* tmp, int n, int b) {
    for (int e = threadIdx.x; e < n * b; e += kThreads) {
        const int i = e % n, j = e / n;
        double s = 0.0;
        for (int l = 0; l < b; ++l) s += X[i + static_cast<std::size_t>(l) * n] * W[l + j * kMaxB];
        tmp[e] = s;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n * b; e += kThreads) X[e] = tmp[e];
    __syncthreads();
}

}  // namespace

// status: [0] converged, [1] zero matrix, [2] iterations used
__global__ void __launch_bounds__(kThreads) eig_subspace_kernel(const double* __restrict__ Gin, int n, int k, int b, int m,
                                                                int maxit, double tol, const double* X0,
                                                                int x0_cols, double* Xkeep,  // may alias X0
                                                                double* __restrict__ V, double* __restrict__ sig,
                                                                int* __restrict__ status, int g_in_smem) {
    extern __shared__ double sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* H = sm;                        // kMaxB^2
    double* W = H + kMaxB * kMaxB;         // kMaxB^2
    double* th = W + kMaxB * kMaxB;        // kMaxB
    double* coef = th + kMaxB;             // kMaxB
    double* red = coef + kMaxB;            // 32
    double* X = red + 32;                  // n*b
    double* AX = X + static_cast<std::size_t>(n) * b;
    double* Y0 = AX + static_cast<std::size_t>(n) * b;
    double* Y1 = Y0 + static_cast<std::size_t>(n) * b;
    double* G = g_in_smem ? (Y1 + static_cast<std::size_t>(n) * b) : const_cast<double*>(Gin);

    // ---- load + symmetrise G (linalg.cpp:107), zero test ----
    double fro = 0.0;
    if (g_in_smem) {
        for (int c = warp; c < n; c += kWarps)
            for (int r = lane; r < n; r += 32) {
                const double a = 0.5 * (Gin[r + static_cast<std::size_t>(c) * n] + Gin[c + static_cast<std::size_t>(r) * n]);
                G[r + static_cast<std::size_t>(c) * n] = a;
                fro += a * a;
            }
    } else {
        for (int c = warp; c < n; c += kWarps)
            for (int r = lane; r < n; r += 32) fro += Gin[r + static_cast<std::size_t>(c) * n] * Gin[r + static_cast<std::size_t>(c) * n];
    }
    fro = cta_sum(fro, red);
    if (fro == 0.0) {
        for (int c = warp; c < k; c += kWarps)
            for (int r = lane; r < n; r += 32) V[r + static_cast<std::size_t>(c) * n] = (r == c) ? 1.0 : 0.0;
        if (threadIdx.x < k) sig[threadIdx.x] = 0.0;
        if (threadIdx.x == 0) { status[0] = 1; status[1] = 1; status[2] = 0; }
        return;
    }

    // ---- start block ----
    for (int e = threadIdx.x; e < n * b; e += kThreads) {
        const int r = e % n, c = e / n;
        X[e] = (c < x0_cols && X0) ? X0[r + static_cast<std::size_t>(c) * n] : rnd_unit(static_cast<unsigned>(c), static_cast<unsigned>(r));
    }
    __syncthreads();
    orthonormalize(X, n, b, coef, red);

    int it = 0;
    bool conv = false;
    for (;; ++it) {
        // ---- Rayleigh-Ritz ----
        gemm_gx(G, X, AX, n, b);
        gram_ab(X, AX, H, n, b, true);
        if (warp == 0) warp_jacobi(H, W, th, b, it == 0 ? 10 : 4);
        __syncthreads();
        rotate(X, W, Y0, n, b);
        rotate(AX, W, Y0, n, b);
        // ---- residual certificate for the wanted k ----
        double rmax = 0.0;
        for (int c = warp; c < k; c += kWarps) {
            double s = 0.0;
            for (int r = lane; r < n; r += 32) {
                const double d = AX[r + static_cast<std::size_t>(c) * n] - th[c] * X[r + static_cast<std::size_t>(c) * n];
                s += d * d;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            rmax = fmax(rmax, sqrt(s));
        }
        __syncthreads();
        if (lane == 0) red[warp] = rmax;
        __syncthreads();
        rmax = 0.0;
        for (int i = 0; i < kWarps; ++i) rmax = fmax(rmax, red[i]);
        const double scale = fmax(fabs(th[0]), 1e-300);
        if (rmax <= tol * scale) { conv = true; break; }
        if (it >= maxit) break;
        __syncthreads();
        // ---- Chebyshev filter: damp [lo, cut] = [-|theta_1| 1e-12, theta_b] ----
        const double cut = th[b - 1];
        const double lo = -1e-12 * scale;
        const double e = 0.5 * (cut - lo), cen = 0.5 * (cut + lo);
        if (!(e > 0.0)) {  // degenerate: plain power step
            gemm_gx(G, X, Y0, n, b);
            for (int q = threadIdx.x; q < n * b; q += kThreads) X[q] = Y0[q];
            __syncthreads();
        } else {
            // Y0 = X, Y1 = (G X - c X) / e ; Y_{j+1} = 2 (G Y_j - c Y_j)/e - Y_{j-1}
            gemm_gx(G, X, Y1, n, b);
            for (int q = threadIdx.x; q < n * b; q += kThreads) {
                Y0[q] = X[q];
                Y1[q] = (Y1[q] - cen * X[q]) / e;
            }
            __syncthreads();
            for (int j = 2; j <= m; ++j) {
                gemm_gx(G, Y1, AX, n, b);
                for (int q = threadIdx.x; q < n * b; q += kThreads) {
                    const double y2 = 2.0 * (AX[q] - cen * Y1[q]) / e - Y0[q];
                    Y0[q] = Y1[q];
                    Y1[q] = y2;
                }
                __syncthreads();
                // per-column rescale (keeps the recurrence, avoids overflow)
                for (int c = warp; c < b; c += kWarps) {
                    double mx = 0.0;
                    for (int r = lane; r < n; r += 32) mx = fmax(mx, fabs(Y1[r + static_cast<std::size_t>(c) * n]));
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                    if (mx > 1e100) {
                        const double inv = 1.0 / mx;
                        for (int r = lane; r < n; r += 32) {
                            Y1[r + static_cast<std::size_t>(c) * n] *= inv;
                            Y0[r + static_cast<std::size_t>(c) * n] *= inv;
                        }
                    }
                }
                __syncthreads();
            }
            for (int q = threadIdx.x; q < n * b; q += kThreads) X[q] = Y1[q];
            __syncthreads();
        }
        orthonormalize(X, n, b, coef, red);
    }
    // ---- outputs ----
    for (int e = threadIdx.x; e < n * k; e += kThreads) V[e] = X[e];
    if (Xkeep)
        for (int e = threadIdx.x; e < n * b; e += kThreads) Xkeep[e] = X[e];
    if (threadIdx.x < k) sig[threadIdx.x] = sqrt(fmax(0.0, th[threadIdx.x]));
    if (threadIdx.x == 0) { status[0] = conv ? 1 : 0; status[1] = 0; status[2] = it; }
}

std::size_t subspace_smem(int n, int b, bool g_smem) {
    std::size_t w = 2 * kMaxB * kMaxB + 2 * kMaxB + 32 + 4ull * n * b;
    if (g_smem) w += static_cast<std::size_t>(n) * n;
    return w * sizeof(double);
}

// Returns true when the subspace path applies (else the caller runs eig_topk).
bool eig_subspace(Ctx* ctx, const double* G, int n, int k, const double* X0, int x0_cols, double* Xkeep, int b,
                  double* V, double* sig, int* status) {
    if (b > kMaxB || b >= n) return false;
    bool g_smem = subspace_smem(n, b, true) <= 200 * 1024;
    const std::size_t smem = subspace_smem(n, b, g_smem);
    if (smem > 220 * 1024) return false;
    static bool attr = false;
    if (!attr) {
        MB_CUDA(cudaFuncSetAttribute(eig_subspace_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        attr = true;
    }
    MB_LAUNCH(ctx, eig_subspace_kernel, 1, kThreads, smem, G, n, k, b, 4, 40, 1e-12, X0, x0_cols, Xkeep, V, sig, status,
              g_smem ? 1 : 0);
    return true;
}

}  // namespace machb

namespace machb {

int eig_block(int n, int k) {
    const int p = 4;
    return std::min(n, std::min(kMaxB, k + p));
}

bool eig_select(Ctx* ctx, const double* G, int n, int k, const double* X0, int x0_cols, double* Xkeep, int b,
                double* V, double* sig, int* status) {
    bool launched = false;
    if (n > 48 && b < n && b <= kMaxB)
        launched = eig_subspace(ctx, G, n, k, X0, x0_cols, Xkeep, b, V, sig, status);
    DBuf<double> work(ctx, eig_work_doubles(n, k));
    eig_topk(ctx, G, n, k, work.get(), V, sig, status, launched ? status : nullptr);
    return launched;
}

}  // namespace machb
