// Block subspace eigensolver building blocks shared by the standalone eigen
// kernel (eig_subspace.cu) and the fused mode-basis cluster kernel
// (mode_basis.cu).  See eig_subspace.cu for the method.
#pragma once

#include <cstdio>
#include <cstdlib>

#include "sparse_ttm.cuh"

namespace machb {
namespace {


constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxB = 32;
// smallest n for which the subspace solver (and the fused mode basis) is used
// instead of the exact tridiagonal solver; MACH_SUB_MIN_N overrides for tests
#ifndef MACH_SUB_MIN_N_DEFAULT
#define MACH_SUB_MIN_N_DEFAULT 16
#endif
inline int sub_min_n() {
    static const int v = std::getenv("MACH_SUB_MIN_N") ? std::atoi(std::getenv("MACH_SUB_MIN_N")) : MACH_SUB_MIN_N_DEFAULT;
    return v;
}
#define kSubMinN (::machb::sub_min_n())

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ double cta_sum(double v, double* red) {
    v = warp_sum(v);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < kWarps; ++i) s += red[i];
    return s;
}

__device__ double cta_max(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < kWarps; ++i) s = fmax(s, red[i]);
    return s;
}

__device__ double rnd_unit(unsigned c, unsigned i) {
    unsigned long long z = 0x9E3779B97F4A7C15ULL * (static_cast<unsigned long long>(c) * 0x100000001B3ull + i + 7ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return static_cast<double>(z >> 11) * 0x1.0p-53 * 2.0 - 1.0;
}

// Jacobi rotation annihilating H[p][q]: angle in fp32 (fast SFU), the (c, s)
// pair renormalised in fp64 so the applied rotation is orthogonal to fp64.
__device__ void jacobi_cs(double hpp, double hqq, double hpq, double& c, double& s) {
    c = 1.0;
    s = 0.0;
    const float fpq = static_cast<float>(hpq);
    if (fpq == 0.0f) return;
    const float tau = static_cast<float>(hqq - hpp) / (2.0f * fpq);
    float t;
    if (fabsf(tau) > 1e18f) t = 0.5f / tau;
    else t = copysignf(1.0f, tau) / (fabsf(tau) + sqrtf(1.0f + tau * tau));
    const float c32 = rsqrtf(1.0f + t * t);
    const double cc = c32, ss = static_cast<double>(t) * c32;
    const double delta = cc * cc + ss * ss - 1.0;
    const double sc = 1.0 - 0.5 * delta + 0.375 * delta * delta;
    c = cc * sc;
    s = ss * sc;
}

// D += A B on the fp64 tensor cores (m8n8k4): lane l holds A[l/4][l%4],
// B[l%4][l/4] and D[l/4][2(l%4) + {0,1}].
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

// padded row stride: XS % 16 == 4 makes every 8x4 / 4x8 fragment load of a
// half-warp hit 16 distinct 8-byte bank pairs
__host__ __device__ constexpr int frag_stride(int w) { return w + ((4 - w % 16) + 16) % 16; }

// fine-grained phase stamps inside the small-matrix helpers (debug builds of
// the timing probe only: g_stamp is null unless MACH_DEBUG_EIG_T is set)
__device__ long long* g_stamp = nullptr;
__device__ int g_dbg_eig = 0;  // MACH_DEBUG_EIGC: iteration printouts of the one-CTA solver
__device__ int g_stamp_n = 0;
__device__ __forceinline__ void sub_stamp(int tag) {
    if (g_stamp && threadIdx.x == 0 && g_stamp_n < 100) {
        long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_stamp[2 * g_stamp_n] = tag;
        g_stamp[2 * g_stamp_n + 1] = t;
        ++g_stamp_n;
    }
}

template <int B>
struct Sub {
    static_assert(B % 8 == 0 && B <= kMaxB, "block width must be a multiple of 8");
    static constexpr int XS = frag_stride(B);  // row stride of npad x B row-major blocks (doubles)
    static constexpr int HS = B + 1;           // leading dimension of B x B matrices
    static constexpr int CT = B / 8;           // 8-wide column tiles

    // OUT = a (G IN) + b1 P1 + b2 P2 over npad rows (rows >= n stay zero: G's
    // padding is zero).  Warp per 8-row tile, all column tiles, fp64 MMA.
    // OUT may alias P1 or P2 (a fragment is read and written by one lane).
    // [rt0, rt1): the 8-row tiles this CTA computes (all of them by default;
    // a slice of them in the cluster-distributed solver, where G, OUT, P1, P2
    // are row slices addressed with absolute row indices)
    __device__ static void gemm(const double* G, int ldg, const double* IN, double* OUT, int npad, double a,
                                const double* P1, double b1, const double* P2, double b2, int rt0 = 0, int rt1 = -1) {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const int gr = lane >> 2, tq = lane & 3;
        if (rt1 < 0) rt1 = npad >> 3;
        for (int rt = rt0 + warp; rt < rt1; rt += kWarps) {
            double c[CT][2];
#pragma unroll
            for (int t = 0; t < CT; ++t) c[t][0] = c[t][1] = 0.0;
            const double* ga = G + (rt * 8 + gr) + tq * ldg;
            const double* xb = IN + tq * XS + gr;
            // batches of KB k-steps: all operand loads of a batch are issued
            // before its MMAs (G may live in global memory for large n)
            constexpr int KB = CT <= 2 ? 8 : 4;
            int k0 = 0;
            for (; k0 + 4 * KB <= npad; k0 += 4 * KB) {
                double av[KB], bv[KB][CT];
#pragma unroll
                for (int u = 0; u < KB; ++u) {
                    av[u] = ga[(k0 + 4 * u) * ldg];
#pragma unroll
                    for (int t = 0; t < CT; ++t) bv[u][t] = xb[(k0 + 4 * u) * XS + t * 8];
                }
#pragma unroll
                for (int u = 0; u < KB; ++u)
#pragma unroll
                    for (int t = 0; t < CT; ++t) dmma(c[t][0], c[t][1], av[u], bv[u][t]);
            }
            for (; k0 < npad; k0 += 4) {
                const double av = ga[k0 * ldg];
#pragma unroll
                for (int t = 0; t < CT; ++t) dmma(c[t][0], c[t][1], av, xb[k0 * XS + t * 8]);
            }
            const int off = (rt * 8 + gr) * XS + 2 * tq;
#pragma unroll
            for (int t = 0; t < CT; ++t) {
                double2 v = make_double2(a * c[t][0], a * c[t][1]);
                if (P1) {
                    const double2 p = *reinterpret_cast<const double2*>(P1 + off + t * 8);
                    v.x = fma(b1, p.x, v.x);
                    v.y = fma(b1, p.y, v.y);
                }
                if (P2) {
                    const double2 p = *reinterpret_cast<const double2*>(P2 + off + t * 8);
                    v.x = fma(b2, p.x, v.x);
                    v.y = fma(b2, p.y, v.y);
                }
                *reinterpret_cast<double2*>(OUT + off + t * 8) = v;
            }
        }
        __syncthreads();
    }

    // C (B x B, ld HS) = A^T M over npad rows; 8x8 output tiles on the fp64
    // MMA, the row range split into KG interleaved groups when there are
    // fewer tiles than warps, partials summed in a fixed order.
    // rows [r0, r1) only when given (multiples of 4; the distributed solver's
    // partial Gram over its row slice)
    __device__ static void gram(const double* A, const double* M, double* C, int npad, int r0 = 0, int r1 = -1) {
        constexpr int NT = CT * CT;
        constexpr int KG = (kWarps / NT) > 0 ? kWarps / NT : 1;
        constexpr int TW = kWarps / KG;  // warps per k-group
        __shared__ double part[KG > 1 ? KG * NT * 64 : 1];
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const int gr = lane >> 2, tq = lane & 3;
        const int kg = warp % KG;
        const int KS = (r1 < 0 ? npad : r1) >> 2, KS0 = r0 >> 2;
        for (int t = warp / KG; t < NT; t += TW) {
            const int ti = t % CT, tj = t / CT;
            double c0 = 0.0, c1 = 0.0;
            const double* ap = A + tq * XS + ti * 8 + gr;
            const double* mp = M + tq * XS + tj * 8 + gr;
#pragma unroll 4
            for (int ks = KS0 + kg; ks < KS; ks += KG) dmma(c0, c1, ap[ks * 4 * XS], mp[ks * 4 * XS]);
            if (KG == 1) {
                C[(ti * 8 + gr) + (tj * 8 + 2 * tq) * HS] = c0;
                C[(ti * 8 + gr) + (tj * 8 + 2 * tq + 1) * HS] = c1;
            } else {
                double* p = part + (kg * NT + t) * 64 + gr * 8 + 2 * tq;
                p[0] = c0;
                p[1] = c1;
            }
        }
        if (KG > 1) {
            __syncthreads();
            for (int e = threadIdx.x; e < NT * 64; e += kThreads) {
                double s = 0.0;
#pragma unroll
                for (int g = 0; g < KG; ++g) s += part[g * NT * 64 + e];
                const int t = e >> 6, r = (e >> 3) & 7, cc = e & 7;
                C[((t % CT) * 8 + r) + ((t / CT) * 8 + cc) * HS] = s;
            }
        }
        __syncthreads();
    }

    // OUT = X W (npad x B)(B x B); warp per 8-row tile, fp64 MMA
    __device__ static void rotate(const double* X, const double* W, double* OUT, int npad, int rt0 = 0, int rt1 = -1) {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const int gr = lane >> 2, tq = lane & 3;
        if (rt1 < 0) rt1 = npad >> 3;
        for (int rt = rt0 + warp; rt < rt1; rt += kWarps) {
            double c[CT][2];
#pragma unroll
            for (int t = 0; t < CT; ++t) c[t][0] = c[t][1] = 0.0;
            const double* xa = X + (rt * 8 + gr) * XS + tq;
#pragma unroll
            for (int k0 = 0; k0 < B; k0 += 4) {
                const double av = xa[k0];
#pragma unroll
                for (int t = 0; t < CT; ++t) dmma(c[t][0], c[t][1], av, W[(k0 + tq) + (t * 8 + gr) * HS]);
            }
            const int off = (rt * 8 + gr) * XS + 2 * tq;
#pragma unroll
            for (int t = 0; t < CT; ++t) *reinterpret_cast<double2*>(OUT + off + t * 8) = make_double2(c[t][0], c[t][1]);
        }
        __syncthreads();
    }

    // CholQR: X <- X R^{-1} with S = X^T X = R^T R, the product written to T
    // and the two pointers swapped.  Returns false (X untouched) when S is not
    // numerically positive definite.  S is equilibrated first (D S D, D =
    // diag(1/|x_j|)): a Chebyshev-filtered block has columns of wildly
    // different lengths but nearly orthogonal directions, and only the
    // latter should decide breakdown.
    __device__ static bool cholqr(double*& X, double*& T, double* S, double* Ri, double* rinv, int npad, int* flag,
                                  bool allow_skip = false) {
        sub_stamp(500);
        gram(X, X, S, npad);
        sub_stamp(501);
        bool skip = false;
        if (!chol_factor(S, Ri, rinv, flag, allow_skip, skip)) return false;
        if (skip) return true;
        sub_stamp(504);
        rotate(X, Ri, T, npad);
        sub_stamp(505);
        double* t = X;
        X = T;
        T = t;
        return true;
    }

    // the small part of CholQR on S = X^T X (B x B): equilibration, Cholesky,
    // Ri = D R^{-1}.  False on breakdown; skip = S was already the identity
    // to 1e-14 (with allow_skip).  Uniform across the CTA.
    __device__ static bool chol_factor(double* S, double* Ri, double* rinv, int* flag, bool allow_skip, bool& skip) {
        __shared__ double dn[kMaxB];
        __shared__ int near_identity;
        skip = false;
        if (threadIdx.x == 0) {
            *flag = 1;
            near_identity = 1;
        }
        if (threadIdx.x < B) {
            const double s = S[threadIdx.x + threadIdx.x * HS];
            dn[threadIdx.x] = s > 0.0 ? 1.0 / sqrt(s) : 0.0;
        }
        __syncthreads();
        if (allow_skip) {  // already orthonormal to ~1e-14: leave X as it is
            for (int e = threadIdx.x; e < B * B; e += kThreads) {
                const int l = e % B, m = e / B;
                if (!(fabs(S[l + m * HS] - (l == m ? 1.0 : 0.0)) <= 1e-14)) near_identity = 0;
            }
            __syncthreads();
            if (near_identity) {
                skip = true;
                return true;
            }
        }
        for (int e = threadIdx.x; e < B * B; e += kThreads) {
            const int l = e % B, m = e / B;
            if (l <= m) S[l + m * HS] *= dn[l] * dn[m];
        }
        __syncthreads();
        sub_stamp(502);
        // outer-product Cholesky on the upper triangle, one barrier per step;
        // each thread owns fixed (l, m) entries (l <= m), indices computed once
        constexpr int NI = B * (B + 1) / 2;
        constexpr int PT = (NI + kThreads - 1) / kThreads;  // entries per thread
        int il[PT], im[PT];
#pragma unroll
        for (int q = 0; q < PT; ++q) {
            int e = static_cast<int>(threadIdx.x) + q * kThreads, l = -1, m = -1;
            if (e < NI) {  // column-major upper triangle: column m holds rows 0..m
                m = 0;
                while (e > m) { e -= m + 1; ++m; }
                l = e;
            }
            il[q] = l;
            im[q] = m;
        }
        for (int j = 0; j < B; ++j) {
            const double d = S[j + j * HS];
            // breakdown: the column keeps < ~3e-8 of its length after the
            // projections (CholQR2 is then no longer orthonormal to fp64)
            if (!(d > 1e-15)) {
                if (threadIdx.x == 0) *flag = 0;
                continue;  // uniform: every thread read the same d
            }
            const double inv = 1.0 / d;
#pragma unroll
            for (int q = 0; q < PT; ++q) {
                const int l = il[q], m = im[q];
                if (l > j) S[l + m * HS] -= S[j + l * HS] * S[j + m * HS] * inv;
            }
            __syncthreads();
        }
        __syncthreads();
        sub_stamp(503);
        if (!*flag) return false;
        // R[j][l] = S[j][l] / sqrt(S[j][j])
        if (threadIdx.x < B) rinv[threadIdx.x] = 1.0 / sqrt(S[threadIdx.x + threadIdx.x * HS]);
        __syncthreads();
        for (int e = threadIdx.x; e < B * B; e += kThreads) {
            const int jj = e % B, l = e / B;
            if (jj <= l) S[jj + l * HS] *= rinv[jj];
        }
        __syncthreads();
        // Ri = D R^{-1}: thread c back-substitutes R x = e_c in registers
        if (threadIdx.x < B) {
            const int c = threadIdx.x;
            double x[B];
#pragma unroll
            for (int r = B - 1; r >= 0; --r) {
                double v = (r == c) ? 1.0 : 0.0;
#pragma unroll
                for (int p = r + 1; p < B; ++p) v = fma(-S[r + p * HS], x[p], v);
                x[r] = v * rinv[r];
            }
#pragma unroll
            for (int r = 0; r < B; ++r) Ri[r + c * HS] = x[r] * dn[r];
        }
        __syncthreads();
        return true;
    }

    // classical Gram-Schmidt twice, column by column (fallback of cholqr)
    __device__ static void cgs2(double* X, int n, double* coef, double* red) {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        for (int j = 0; j < B; ++j) {
            for (int attempt = 0; attempt < 2; ++attempt) {
                double n0 = 0.0;
                for (int r = threadIdx.x; r < n; r += kThreads) n0 += X[r * XS + j] * X[r * XS + j];
                n0 = sqrt(cta_sum(n0, red));
                for (int pass = 0; pass < 2 && j > 0; ++pass) {
                    for (int c = warp; c < j; c += kWarps) {
                        double s = 0.0;
                        for (int r = lane; r < n; r += 32) s += X[r * XS + c] * X[r * XS + j];
                        s = warp_sum(s);
                        if (lane == 0) coef[c] = s;
                    }
                    __syncthreads();
                    for (int r = threadIdx.x; r < n; r += kThreads) {
                        double v = X[r * XS + j];
                        for (int c = 0; c < j; ++c) v -= X[r * XS + c] * coef[c];
                        X[r * XS + j] = v;
                    }
                    __syncthreads();
                }
                double nn = 0.0;
                for (int r = threadIdx.x; r < n; r += kThreads) nn += X[r * XS + j] * X[r * XS + j];
                nn = sqrt(cta_sum(nn, red));
                if (nn > 1e-10 * n0 && nn > 0.0) {
                    const double inv = 1.0 / nn;
                    for (int r = threadIdx.x; r < n; r += kThreads) X[r * XS + j] *= inv;
                    __syncthreads();
                    break;
                }
                for (int r = threadIdx.x; r < n; r += kThreads) X[r * XS + j] = rnd_unit(1000u + j + 97u * attempt, r);
                __syncthreads();
            }
        }
    }

    __device__ static void orthonormalize(double*& X, double*& T, int n, int npad, double* S, double* Ri, double* rinv,
                                          double* coef, double* red, int* flag) {
        // CholQR2; the second pass is skipped when the first already left an
        // orthonormal block (its Gram is the identity to 1e-14)
        if (!cholqr(X, T, S, Ri, rinv, npad, flag) || !cholqr(X, T, S, Ri, rinv, npad, flag, true)) cgs2(X, n, coef, red);
    }

    // sort the diagonal of H descending into th, permute W's columns alike
    __device__ static void sort_ritz(double* H, double* W, double* th, double* Z) {
        __shared__ int perm[kMaxB];
        const int tid = threadIdx.x;
        if (tid < B) {
            const double di = H[tid + tid * HS];
            int rank = 0;
#pragma unroll
            for (int q = 0; q < B; ++q) {
                const double dq = H[q + q * HS];
                rank += (dq > di) || (dq == di && q < tid);
            }
            perm[rank] = tid;
        }
        __syncthreads();
        if (tid < B) th[tid] = H[perm[tid] + perm[tid] * HS];
        for (int e = tid; e < B * B; e += kThreads) Z[(e % B) + (e / B) * HS] = W[(e % B) + perm[e / B] * HS];
        __syncthreads();
        for (int e = tid; e < B * B; e += kThreads) W[(e % B) + (e / B) * HS] = Z[(e % B) + (e / B) * HS];
        __syncthreads();
    }

    // C = op(A) M for B x B matrices (ld HS); op = transpose when ta
    __device__ static void mm(const double* A, bool ta, const double* M, double* C) {
        for (int e = threadIdx.x; e < B * B; e += kThreads) {
            const int i = e % B, j = e / B;
            double s = 0.0;
            if (ta) {
#pragma unroll
                for (int l = 0; l < B; ++l) s = fma(A[l + i * HS], M[l + j * HS], s);
            } else {
#pragma unroll
                for (int l = 0; l < B; ++l) s = fma(A[i + l * HS], M[l + j * HS], s);
            }
            C[i + j * HS] = s;
        }
        __syncthreads();
    }

    // Iterated perturbation Rayleigh-Ritz for a nearly diagonal H: each round
    // takes Z_ij = h_ij / (h_jj - h_ii) (antisymmetric), Q = I + Z + Z^2/2
    // made orthogonal to fp64 by Newton-Schulz steps Q <- Q (3I - Q^T Q) / 2,
    // W <- W Q, H <- Q^T H Q; the off-diagonal shrinks quadratically.  Pairs
    // of unwanted (>= k) columns that are not separated are left coupled (they
    // only feed the filter bound).  False when a pair involving a wanted
    // column is not separated or the rounds do not converge: the caller then
    // runs Jacobi on the untouched H.
    __device__ static bool refine_rr(const double* H, double* Hc, double* W, double* Z, double* Q, double* T,
                                     double* th, int k, int* flag) {
        __shared__ unsigned long long zmax_bits;
        const int tid = threadIdx.x;
        for (int e = tid; e < B * B; e += kThreads) {
            const int i = e % B, j = e / B;
            Hc[i + j * HS] = H[i + j * HS];
            W[i + j * HS] = (i == j) ? 1.0 : 0.0;
        }
        bool ok = false;
        for (int round = 0; round < 8; ++round) {
            if (tid == 0) {
                *flag = 1;
                zmax_bits = 0ull;
            }
            __syncthreads();
            for (int e = tid; e < B * B; e += kThreads) {
                const int i = e % B, j = e / B;
                double z = 0.0;
                // guard-guard pairs (both >= k) are left as they are: the guard
                // columns only bound the filter, and nearly degenerate noise
                // pairs there would keep the rounds from converging
                if (i != j && (i < k || j < k)) {
                    const double hij = Hc[i + j * HS];
                    const double gap = Hc[j + j * HS] - Hc[i + i * HS];
                    if (fabs(hij) > 0.25 * fabs(gap)) {
                        if ((i < k || j < k) && hij != 0.0) *flag = 0;
                    } else if (gap != 0.0) {
                        z = hij / gap;
                    }
                }
                Z[i + j * HS] = z;
                if (z != 0.0) atomicMax(&zmax_bits, static_cast<unsigned long long>(__double_as_longlong(fabs(z))));
            }
            __syncthreads();
            if (!*flag) return false;
            const double zmax = __longlong_as_double(static_cast<long long>(zmax_bits));
            if (zmax == 0.0) {
                ok = true;
                break;
            }
            mm(Z, false, Z, T);  // T = Z^2
            for (int e = tid; e < B * B; e += kThreads) {
                const int i = e % B, j = e / B;
                Q[i + j * HS] = (i == j ? 1.0 : 0.0) + Z[i + j * HS] + 0.5 * T[i + j * HS];
            }
            __syncthreads();
            // orthogonality defect of Q is O(zmax^3); each step squares it
            const int ns = zmax > 1e-3 ? 2 : (zmax > 1e-6 ? 1 : 0);
            for (int s = 0; s < ns; ++s) {
                mm(Q, true, Q, T);  // T = Q^T Q
                mm(Q, false, T, Z);  // Z = Q (Q^T Q)
                for (int e = tid; e < B * B; e += kThreads) {
                    const int i = e % B, j = e / B;
                    Q[i + j * HS] = 1.5 * Q[i + j * HS] - 0.5 * Z[i + j * HS];
                }
                __syncthreads();
            }
            mm(W, false, Q, T);  // T = W Q
            mm(Hc, false, Q, Z);  // Z = Hc Q
            for (int e = tid; e < B * B; e += kThreads) W[(e % B) + (e / B) * HS] = T[(e % B) + (e / B) * HS];
            mm(Q, true, Z, Hc);  // Hc = Q^T Hc Q
            if (zmax < 1e-9) {  // the next round's Z would be O(zmax^2)
                ok = true;
                break;
            }
        }
        if (!ok) return false;
        sort_ritz(Hc, W, th, Z);
        return true;
    }

    // CTA-parallel cyclic Jacobi (circle-method rounds, 3 barrier phases each)
    __device__ static int jacobi(double* H, double* W, double* th, int max_sweeps, double* red, double* Z,
                                 bool sort = true) {
        __shared__ int jp[kMaxB / 2], jq[kMaxB / 2];
        __shared__ double jc[kMaxB / 2], js[kMaxB / 2];
        const int tid = threadIdx.x;
        constexpr int NP = B / 2, M = B - 1;
        for (int e = tid; e < B * B; e += kThreads) W[(e % B) + (e / B) * HS] = ((e % B) == (e / B)) ? 1.0 : 0.0;
        double nrm = 0.0;
        for (int e = tid; e < B * B; e += kThreads) nrm += H[(e % B) + (e / B) * HS] * H[(e % B) + (e / B) * HS];
        nrm = cta_sum(nrm, red);
        int sweep = 0;
        for (; sweep < max_sweeps; ++sweep) {
            double off = 0.0;
            for (int e = tid; e < B * B; e += kThreads)
                if ((e % B) < (e / B)) off += H[(e % B) + (e / B) * HS] * H[(e % B) + (e / B) * HS];
            off = cta_sum(off, red);
            if (off <= 1e-30 * nrm) break;
            for (int r = 0; r < M; ++r) {
                if (tid < NP) {
                    int p, q;
                    if (tid == 0) {
                        p = 0;
                        q = r + 1;
                    } else {
                        int x = r + tid;
                        if (x >= M) x -= M;
                        int y = r - tid;
                        if (y < 0) y += M;
                        p = x + 1;
                        q = y + 1;
                    }
                    if (p > q) { const int tt = p; p = q; q = tt; }
                    double c, s;
                    jacobi_cs(H[p + p * HS], H[q + q * HS], H[p + q * HS], c, s);
                    jp[tid] = p; jq[tid] = q; jc[tid] = c; js[tid] = s;
                }
                __syncthreads();
                // (pair t, column j) items: NP * B of them, strided over the CTA
                for (int e = tid; e < NP * B; e += kThreads) {
                    const int t = e / B, j = e - t * B;
                    const double s = js[t];
                    if (s != 0.0) {
                        const double c = jc[t];
                        const int p = jp[t], q = jq[t];
                        const double a = H[p + j * HS], bq = H[q + j * HS];
                        H[p + j * HS] = c * a - s * bq;
                        H[q + j * HS] = s * a + c * bq;
                    }
                }
                __syncthreads();
                for (int e = tid; e < NP * B; e += kThreads) {
                    const int t = e / B, j = e - t * B;
                    const double s = js[t];
                    if (s != 0.0) {
                        const double c = jc[t];
                        const int p = jp[t], q = jq[t];
                        const double a = H[j + p * HS], bq = H[j + q * HS];
                        H[j + p * HS] = c * a - s * bq;
                        H[j + q * HS] = s * a + c * bq;
                        const double wa = W[j + p * HS], wb = W[j + q * HS];
                        W[j + p * HS] = c * wa - s * wb;
                        W[j + q * HS] = s * wa + c * wb;
                    }
                }
                __syncthreads();
            }
        }
        if (sort) sort_ritz(H, W, th, Z);
        return sweep;
    }

    // Rayleigh-Ritz of H when the perturbation rounds do not apply: two
    // Jacobi sweeps bring H close to diagonal, then the perturbation rounds
    // (quadratically convergent) finish; W = W_jacobi W_rounds.  Full Jacobi
    // when the rounds still do not apply.  J7: B x B scratch.
    __device__ static int rr_hybrid(double* H, double* Hc, double* W, double* Z, double* Q, double* S, double* J7,
                                    double* th, int k, int* flag, double* red, int max_sweeps) {
        jacobi(H, W, th, 2, red, Z, false);  // H <- W^T H W (unsorted)
        for (int e = threadIdx.x; e < B * B; e += kThreads) J7[(e % B) + (e / B) * HS] = W[(e % B) + (e / B) * HS];
        __syncthreads();
        int nsw = 2;
        if (!refine_rr(H, Hc, W, Z, Q, S, th, k, flag)) nsw += jacobi(H, W, th, max_sweeps, red, Z);
        mm(J7, false, W, Z);  // Z = W_jacobi W_rest
        for (int e = threadIdx.x; e < B * B; e += kThreads) W[(e % B) + (e / B) * HS] = Z[(e % B) + (e / B) * HS];
        __syncthreads();
        return nsw;
    }

    // th[c] = x_c^T (G x_c) for the B columns (Rayleigh quotients of a block
    // whose columns are orthonormal); warp per column
    __device__ static void rayleigh_diag(const double* X, const double* AX, double* th, int n) {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        for (int c = warp; c < B; c += kWarps) {
            double s = 0.0;
            for (int r = lane; r < n; r += 32) s = fma(X[r * XS + c], AX[r * XS + c], s);
            s = warp_sum(s);
            if (lane == 0) th[c] = s;
        }
        __syncthreads();
    }

    // max over wanted columns c < k of |AX_c - th_c X_c|
    __device__ static double residual(const double* X, const double* AX, const double* th, int n, int k, double* red) {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        double rmax = 0.0;
        for (int c = warp; c < k; c += kWarps) {
            double s = 0.0;
            for (int r = lane; r < n; r += 32) {
                const double d = AX[r * XS + c] - th[c] * X[r * XS + c];
                s = fma(d, d, s);
            }
            rmax = fmax(rmax, sqrt(warp_sum(s)));
        }
        return cta_max(rmax, red);
    }
};

// shared-memory workspace of the solver (npad = n rounded up to 8)
template <int B>
struct SubWs {
    double *H, *W, *S, *Z, *Q, *Hc, *J7, *th, *rinv, *coef, *red, *X, *AX, *Y0, *Y1;
    // blocks: if non-null, the four n x B blocks live there (global memory,
    // for n too large for shared memory) instead of after the small matrices
    __device__ SubWs(double* sm, int npad, double* blocks = nullptr) {
        constexpr int HS = Sub<B>::HS, XS = Sub<B>::XS;
        H = sm;
        W = H + B * HS;
        S = W + B * HS;
        Z = S + B * HS;
        Q = Z + B * HS;
        Hc = Q + B * HS;
        J7 = Hc + B * HS;
        th = J7 + B * HS;
        rinv = th + kMaxB;
        coef = rinv + kMaxB;
        red = coef + kMaxB;
        X = blocks ? blocks : red + 32;
        AX = X + npad * XS;
        Y0 = AX + npad * XS;
        Y1 = Y0 + npad * XS;
    }
    __host__ __device__ static std::size_t doubles(int npad) { return small_doubles() + block_doubles(npad); }
    __host__ __device__ static std::size_t small_doubles() { return 7ull * B * Sub<B>::HS + 3 * kMaxB + 32; }
    __host__ __device__ static std::size_t block_doubles(int npad) { return 4ull * npad * Sub<B>::XS; }
};

#define MB_STAMP(tag)                                                                  \
    do {                                                                               \
        if (tstamp && threadIdx.x == 0 && ns_ < 118) {                                 \
            long long t_;                                                              \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                     \
            tstamp[2 * ns_] = (tag);                                                   \
            tstamp[2 * ns_ + 1] = t_;                                                  \
            ++ns_;                                                                     \
        }                                                                              \
    } while (0)

// Start block into the workspace: X0's columns (column-major n x x0_cols),
// deterministic random columns beyond them; the other three blocks zeroed.
template <int B>
__device__ void load_start_block(SubWs<B>& ws, int n, const double* X0, int x0_cols) {
    constexpr int XS = Sub<B>::XS;
    const int npad = (n + 7) & ~7;
    double *X = ws.X, *AX = ws.AX, *Y0 = ws.Y0, *Y1 = ws.Y1;
    for (int base = threadIdx.x; base < npad * B; base += 8 * kThreads) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {  // batched: eight loads in flight
            const int e = base + u * kThreads;
            const int r = e % npad, c = e / npad;
            v[u] = (e < npad * B && r < n && c < x0_cols && X0) ? X0[r + c * n] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = base + u * kThreads;
            if (e >= npad * B) break;
            const int r = e % npad, c = e / npad;
            if (r < n && !(c < x0_cols && X0)) v[u] = rnd_unit(static_cast<unsigned>(c), static_cast<unsigned>(r));
            X[r * XS + c] = v[u];
            AX[r * XS + c] = 0.0;
            Y0[r * XS + c] = 0.0;
            Y1[r * XS + c] = 0.0;
        }
    }
}

// The solver proper.  G: npad x npad in shared memory (leading dimension ldg,
// exactly symmetric, zero outside n x n).  Returns the final Ritz block (in
// ws, row-major, stride Sub<B>::XS, rows >= n zero); Ritz values in ws.th.
template <int B>
__device__ double* subspace_core(SubWs<B>& ws, const double* G, int ldg, int n, int k, int m, int maxit, double tol,
                                 const double* X0, int x0_cols, bool& conv, int& iters, int* flagp,
                                 long long* tstamp, int& ns_, const double* th0 = nullptr, bool preloaded = false) {
    using SB = Sub<B>;
    constexpr int XS = SB::XS;
    const int npad = (n + 7) & ~7;
    double *H = ws.H, *W = ws.W, *S = ws.S, *Z = ws.Z, *Q = ws.Q, *Hc = ws.Hc, *th = ws.th, *rinv = ws.rinv,
           *coef = ws.coef, *red = ws.red;
    double *X = ws.X, *AX = ws.AX, *Y0 = ws.Y0, *Y1 = ws.Y1;
    int& flag = *flagp;
    // ---- start block (row-major, rows >= n zero in all four blocks) ----
    if (!preloaded) load_start_block<B>(ws, n, X0, x0_cols);
    __syncthreads();
    MB_STAMP(1);
    if (x0_cols < B || !X0) SB::orthonormalize(X, Y0, n, npad, S, Z, rinv, coef, red, &flag);  // a kept Ritz block is orthonormal
    MB_STAMP(2);

    // A warm block that comes with its Ritz values (th0, the previous call's)
    // starts with a filter step: the previous G's spectrum bounds the filter,
    // and one Rayleigh-Ritz pass is saved per call.
    const bool filter_first = X0 && x0_cols >= B && th0;
    if (filter_first && threadIdx.x < B) th[threadIdx.x] = th0[threadIdx.x];
    __syncthreads();
    int it = 0;
    conv = false;
    // AX = G X holds after every Rayleigh-Ritz (rotated with X), so the
    // filter's first product reuses it.  (A warm pre-check of the kept block
    // against the new G was measured: its residual is ~1e-6 theta_1 at steady
    // state, far above the certificate, so it only added a product.)
    bool ax_valid = false;
    for (;; ++it) {
      if (!(filter_first && it == 0)) {
        // ---- Rayleigh-Ritz ----
        SB::gemm(G, ldg, X, AX, npad, 1.0, nullptr, 0.0, nullptr, 0.0);
        MB_STAMP(10);
        SB::gram(X, AX, H, npad);
        MB_STAMP(11);
        int nsw = 99;
        if (!SB::refine_rr(H, Hc, W, Z, Q, S, th, k, &flag))
            nsw = SB::rr_hybrid(H, Hc, W, Z, Q, S, ws.J7, th, k, &flag, red, it == 0 ? 8 : 3);
        MB_STAMP(1000 + nsw);
        SB::rotate(X, W, Y0, npad);
        { double* t = X; X = Y0; Y0 = t; }
        SB::rotate(AX, W, Y0, npad);
        { double* t = AX; AX = Y0; Y0 = t; }
        ax_valid = true;  // AX = G X for the rotated block: the filter's first product
        MB_STAMP(13);
        // ---- residual certificate for the wanted k ----
        const double rmax = SB::residual(X, AX, th, n, k, red);
        const double scale = fmax(fabs(th[0]), 1e-300);
        if (g_dbg_eig && threadIdx.x == 0 && blockIdx.x == 0)
            printf("[eig1] it %d th0 %.6e thB %.6e rmax/scale %.3e\n", it, th[0], th[B - 1], rmax / scale);
        MB_STAMP(14);
        if (rmax <= tol * scale) { conv = true; break; }
        if (it >= maxit) break;
      }
        // ---- Chebyshev filter: damp [lo, cut] = [-|theta_1| 1e-12, theta_B] ----
        const double scale = fmax(fabs(th[0]), 1e-300);
        const double cut = th[B - 1];
        const double lo = -1e-12 * scale;
        const double e = 0.5 * (cut - lo), cen = 0.5 * (cut + lo);
        if (!(e > 0.0)) {  // degenerate spectrum estimate: plain power step
            if (ax_valid) {
                for (int idx = threadIdx.x; idx < npad * XS; idx += kThreads) Y1[idx] = AX[idx];
                __syncthreads();
            } else {
                SB::gemm(G, ldg, X, Y1, npad, 1.0, nullptr, 0.0, nullptr, 0.0);
            }
            ax_valid = false;
            { double* t = X; X = Y1; Y1 = t; }
        } else {
            const double ie = 1.0 / e;
            // Y1 = (G X - c X) / e   (Y0 = X by pointer)
            if (ax_valid) {  // G X from the warm pre-check
                for (int idx = threadIdx.x; idx < npad * XS; idx += kThreads) Y1[idx] = ie * AX[idx] - cen * ie * X[idx];
                __syncthreads();
            } else {
                SB::gemm(G, ldg, X, Y1, npad, ie, X, -cen * ie, nullptr, 0.0);
            }
            ax_valid = false;
            double* y0 = X;
            double* y1 = Y1;
            double* spare = Y0;
            for (int j = 2; j <= m; ++j) {
                // y2 = 2 (G y1 - c y1) / e - y0, written over the spare block
                SB::gemm(G, ldg, y1, spare, npad, 2.0 * ie, y1, -2.0 * cen * ie, y0, -1.0);
                double* t = y0;
                y0 = y1;
                y1 = spare;
                spare = t;
            }
            X = y1;  // growth is ~T_m(theta_1 / e) <= 1e20 at m = 4: no rescale needed in fp64
            Y0 = y0;
            Y1 = spare;
        }
        MB_STAMP(15);
        SB::orthonormalize(X, Y0, n, npad, S, Z, rinv, coef, red, &flag);
        if (g_dbg_eig && threadIdx.x == 0 && blockIdx.x == 0) printf("[eig1] it %d ortho flag %d\n", it, flag);
        MB_STAMP(16);
    }
    MB_STAMP(99);
    iters = it;
    return X;
}

}  // namespace
}  // namespace machb
