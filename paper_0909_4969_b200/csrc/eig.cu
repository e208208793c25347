// On-device symmetric eigensolver for the HOSVD/HOOI eigen step
// (reference: gram_side_basis, proj/src/linalg.cpp:106-120, which runs a full
// Eigen::SelfAdjointEigenSolver and keeps the top k eigenpairs).
//
// Only the top k eigenpairs are needed, so this follows the "selected
// eigenpairs" route (LAPACK dsyevx algorithm class):
//   1. symmetrise A = (G + G^T) / 2                       (linalg.cpp:107)
//   2. Householder tridiagonalisation A = Q T Q^T        (one CTA, smem/L2)
//   3. top-k eigenvalues of T by multisection bisection on Sturm counts
//      (division-free three-term recurrence, one warp per eigenvalue)
//   4. eigenvectors of T by inverse iteration on a pivoted tridiagonal LU,
//      reorthogonalised inside clusters
//   5. back-transformation z = H_0 ... H_{n-3} z_T
// Output: k eigenvectors (n x k, column-major) for eigenvalues in descending
// order and sigma_i = sqrt(max(0, lambda_i)) (linalg.cpp:116-117).
// One thread block of 256 threads does everything; no host round trip.
#include "basis_cta.cuh"
#include "common.cuh"

namespace machb {

namespace {

constexpr int kEigThreads = 256;
constexpr int kEigWarps = kEigThreads / 32;
constexpr int kSmemMatrixN = 150;  // A kept in shared memory up to this n

__device__ double block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < kEigWarps; ++i) s += red[i];  // fixed order: deterministic
    return s;
}

// number of eigenvalues of the (scaled) tridiagonal (d, e2 = e^2) below x:
// sign changes of the leading-minor sequence p_i = det(T_i - x I).
__device__ int sturm_count(const double* d, const double* e2, int n, double x) {
    double pm2 = 0.0, pm1 = 1.0;
    bool neg_prev = false;
    int cnt = 0;
    for (int i = 0; i < n; ++i) {
        double p = (d[i] - x) * pm1;
        if (i > 0) p = fma(-e2[i - 1], pm2, p);
        bool neg;
        if (p == 0.0) {
            neg = !neg_prev;
            ++cnt;
        } else {
            neg = p < 0.0;
            cnt += (neg != neg_prev);
        }
        const double ap = fabs(p);
        if (ap > 1e150) {
            p *= 1e-150;
            pm1 *= 1e-150;
        } else if (ap < 1e-150 && ap != 0.0) {
            p *= 1e150;
            pm1 *= 1e150;
        }
        pm2 = pm1;
        pm1 = p;
        neg_prev = neg;
    }
    return cnt;
}

__device__ double hash_unit(unsigned a, unsigned b) {
    unsigned long long z = 0x9E3779B97F4A7C15ULL * (static_cast<unsigned long long>(a) * 1000003ull + b + 1ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return static_cast<double>(z >> 11) * 0x1.0p-53 * 2.0 - 1.0;
}

}  // namespace

// G: n x n (column-major, ld n).  work: n*n (only used when n > kSmemMatrixN)
// plus per-target scratch 6*n*k.  V: n x k output, sig: k output.
// status[0] = 0 ok; status[1] = 1 if the matrix is exactly zero.
__device__ void eig_topk_cta(const double* __restrict__ G, int n, int k, double* __restrict__ work,
                             double* __restrict__ V, double* __restrict__ sig, int* __restrict__ status, double* sm) {
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    double* sv = sm;            // v (n)
    double* sp = sv + n;        // p / w (n)
    double* sd = sp + n;        // diagonal (n)
    double* se = sd + n;        // off-diagonal (n)
    double* stau = se + n;      // tau (n)
    double* se2 = stau + n;     // e^2 scaled (n)
    double* sdd = se2 + n;      // d scaled (n)
    double* slam = sdd + n;     // eigenvalues (k <= n)
    double* red = slam + n;     // 8*n partials + 32
    double* A = (n <= kSmemMatrixN) ? (red + kEigWarps * n + 32) : work;
    double* scratch = work + static_cast<std::size_t>(n) * n;  // per-target LU + z_T
    double* red_small = red + kEigWarps * n;

    // ---- 1. symmetrise (linalg.cpp:107) ----
    double fro = 0.0;
    for (int c = warp; c < n; c += kEigWarps)
        for (int r = lane; r < n; r += 32) {
            const double a = 0.5 * (G[r + static_cast<std::size_t>(c) * n] + G[c + static_cast<std::size_t>(r) * n]);
            A[r + static_cast<std::size_t>(c) * n] = a;
            fro += a * a;
        }
    fro = block_sum(fro, red_small);
    // exactly-zero Gram (zero matricization): identity basis, flagged
    if (fro == 0.0) {
        if (V)
            for (int c = warp; c < k; c += kEigWarps)
                for (int r = lane; r < n; r += 32) V[r + static_cast<std::size_t>(c) * n] = (r == c) ? 1.0 : 0.0;
        for (int i = t; i < k; i += kEigThreads) sig[i] = 0.0;
        if (t == 0) {
            status[0] = 0;
            status[1] = 1;
        }
        return;
    }
    __syncthreads();

    // ---- 2. Householder tridiagonalisation (lower), reflectors stored in A ----
    for (int j = 0; j + 2 < n; ++j) {
        const int m = n - j - 1;
        double* col = A + static_cast<std::size_t>(j) * n + (j + 1);  // x = A[j+1.., j]
        double s = 0.0;
        for (int i = 1 + t; i < m; i += kEigThreads) s += col[i] * col[i];
        s = block_sum(s, red_small);
        const double alpha = col[0];
        double tau = 0.0, beta = alpha, scale = 0.0;
        if (s != 0.0) {
            beta = -copysign(sqrt(alpha * alpha + s), alpha);
            scale = 1.0 / (alpha - beta);
            tau = (beta - alpha) / beta;
        }
        for (int i = t; i < m; i += kEigThreads) {
            const double vi = (i == 0) ? 1.0 : col[i] * scale;
            sv[i] = vi;
            if (i > 0) col[i] = vi;
        }
        if (t == 0) {
            sd[j] = A[j + static_cast<std::size_t>(j) * n];
            se[j] = beta;
            stau[j] = tau;
        }
        __syncthreads();
        if (tau == 0.0) continue;
        double* Ap = A + static_cast<std::size_t>(j + 1) * n + (j + 1);  // trailing m x m, ld n
        // p = tau * A' v  (2-D split: lanes over rows, warps over columns)
        for (int i = lane; i < m; i += 32) {
            double acc = 0.0;
            for (int c = warp; c < m; c += kEigWarps) acc += Ap[i + static_cast<std::size_t>(c) * n] * sv[c];
            red[warp * n + i] = acc;
        }
        __syncthreads();
        double kp = 0.0;
        for (int i = t; i < m; i += kEigThreads) {
            double s2 = 0.0;
#pragma unroll
            for (int w = 0; w < kEigWarps; ++w) s2 += red[w * n + i];
            s2 *= tau;
            sp[i] = s2;
            kp += s2 * sv[i];
        }
        const double K = 0.5 * tau * block_sum(kp, red_small);
        for (int i = t; i < m; i += kEigThreads) sp[i] -= K * sv[i];
        __syncthreads();
        // A' -= v w^T + w v^T
        for (int c = warp; c < m; c += kEigWarps) {
            const double vc = sv[c], wc = sp[c];
            double* ac = Ap + static_cast<std::size_t>(c) * n;
            for (int i = lane; i < m; i += 32) ac[i] -= sv[i] * wc + sp[i] * vc;
        }
        __syncthreads();
    }
    if (t == 0) {
        if (n >= 2) {
            sd[n - 2] = A[(n - 2) + static_cast<std::size_t>(n - 2) * n];
            se[n - 2] = A[(n - 1) + static_cast<std::size_t>(n - 2) * n];
            stau[n - 2] = 0.0;
        }
        sd[n - 1] = A[(n - 1) + static_cast<std::size_t>(n - 1) * n];
        se[n - 1] = 0.0;
        stau[n - 1] = 0.0;
    }
    __syncthreads();

    // ---- scale T to unit Gershgorin radius ----
    double gmax = 0.0;
    for (int i = t; i < n; i += kEigThreads) {
        const double r = fabs(sd[i]) + fabs(se[i]) + (i > 0 ? fabs(se[i - 1]) : 0.0);
        gmax = fmax(gmax, r);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) gmax = fmax(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
    __syncthreads();
    if (lane == 0) red_small[warp] = gmax;
    __syncthreads();
    gmax = 0.0;
    for (int i = 0; i < kEigWarps; ++i) gmax = fmax(gmax, red_small[i]);
    const double sc = (gmax > 0.0) ? 1.0 / gmax : 1.0;
    for (int i = t; i < n; i += kEigThreads) {
        sdd[i] = sd[i] * sc;
        const double es = se[i] * sc;
        se2[i] = es * es;
    }
    __syncthreads();

    // ---- 3. top-k eigenvalues: 33-way multisection per warp ----
    for (int tk = warp; tk < k; tk += kEigWarps) {
        const int target = n - 1 - tk;  // ascending index
        double a = -1.0 - 1e-12, b = 1.0 + 1e-12;
        for (int round = 0; round < 14; ++round) {
            const double x = a + (b - a) * static_cast<double>(lane + 1) / 33.0;
            const int cnt = sturm_count(sdd, se2, n, x);
            const unsigned above = __ballot_sync(0xffffffffu, cnt > target);
            double na, nb;
            if (above) {
                const int f = __ffs(above) - 1;
                nb = __shfl_sync(0xffffffffu, x, f);
                na = (f == 0) ? a : __shfl_sync(0xffffffffu, x, f - 1);
            } else {
                na = __shfl_sync(0xffffffffu, x, 31);
                nb = b;
            }
            a = na;
            b = nb;
            if (b - a <= 2.2e-16 * fmax(fabs(a), fabs(b)) + 1e-300) break;
        }
        if (lane == 0) slam[tk] = 0.5 * (a + b);
    }
    __syncthreads();
    if (!V) {  // eigenvalues only (the Theorem-1 bound's full spectra, bounds.cu)
        for (int i = t; i < k; i += kEigThreads) sig[i] = sqrt(fmax(0.0, slam[i] * gmax));
        if (t == 0) {
            status[0] = 0;
            status[1] = 0;
        }
        return;
    }

    // ---- 4. inverse iteration (thread per cluster leader) ----
    // scratch layout per target q: U0,U1,U2,mult,swap (5n) ; z_T at scratch + 5nk
    double* zT = scratch + static_cast<std::size_t>(5) * n * k;
    for (int t0 = t; t0 < k; t0 += kEigThreads) {
        const double ortol = 1e-3;  // cluster gap on the unit-scaled spectrum (LAPACK dstein)
        const bool leader = (t0 == 0) || (slam[t0 - 1] - slam[t0] > ortol);
        if (leader) {
            const int t = t0;
            int last = t;
            while (last + 1 < k && slam[last] - slam[last + 1] <= ortol) ++last;
            for (int q = t; q <= last; ++q) {
                double* U0 = scratch + static_cast<std::size_t>(5) * n * q;
                double* U1 = U0 + n;
                double* U2 = U1 + n;
                double* ML = U2 + n;
                double* SW = ML + n;
                double* z = zT + static_cast<std::size_t>(n) * q;
                // perturb coincident shifts inside a cluster slightly (dstein)
                double lam = slam[q];
                if (q > t) {
                    const double prev = slam[q - 1] - 1e-14 * (q - t);
                    if (lam >= prev) lam = prev;
                }
                // pivoted LU of T - lam I; carried row (p, qv, r)
                double p = sdd[0] - lam, qv = (n > 1) ? se[0] * sc : 0.0, r = 0.0;
                for (int i = 0; i + 1 < n; ++i) {
                    const double ei = se[i] * sc;
                    const double dn = sdd[i + 1] - lam;
                    const double en = (i + 2 < n) ? se[i + 1] * sc : 0.0;
                    if (fabs(p) >= fabs(ei)) {
                        const double mlt = (p != 0.0) ? ei / p : 0.0;
                        U0[i] = p; U1[i] = qv; U2[i] = r; ML[i] = mlt; SW[i] = 0.0;
                        p = dn - mlt * qv;
                        qv = en - mlt * r;
                        r = 0.0;
                    } else {
                        const double mlt = p / ei;
                        U0[i] = ei; U1[i] = dn; U2[i] = en; ML[i] = mlt; SW[i] = 1.0;
                        const double np = qv - mlt * dn;
                        const double nq = r - mlt * en;
                        p = np;
                        qv = nq;
                        r = 0.0;
                    }
                }
                U0[n - 1] = p; U1[n - 1] = 0.0; U2[n - 1] = 0.0;
                const double tiny = 2.2e-16;
                for (int i = 0; i < n; ++i)
                    if (fabs(U0[i]) < tiny) U0[i] = (U0[i] < 0.0) ? -tiny : tiny;
                for (int i = 0; i < n; ++i) z[i] = hash_unit(static_cast<unsigned>(q), static_cast<unsigned>(i));
                for (int it = 0; it < 3; ++it) {
                    for (int i = 0; i + 1 < n; ++i) {   // forward: P, L
                        if (SW[i] != 0.0) {
                            const double tmp = z[i];
                            z[i] = z[i + 1];
                            z[i + 1] = tmp;
                        }
                        z[i + 1] -= ML[i] * z[i];
                    }
                    for (int i = n - 1; i >= 0; --i) {  // back: U
                        double s = z[i];
                        if (i + 1 < n) s -= U1[i] * z[i + 1];
                        if (i + 2 < n) s -= U2[i] * z[i + 2];
                        z[i] = s / U0[i];
                    }
                    // reorthogonalise against earlier members of the cluster
                    for (int o = t; o < q; ++o) {
                        const double* zo = zT + static_cast<std::size_t>(n) * o;
                        double dot = 0.0;
                        for (int i = 0; i < n; ++i) dot += zo[i] * z[i];
                        for (int i = 0; i < n; ++i) z[i] -= dot * zo[i];
                    }
                    double nrm = 0.0;
                    for (int i = 0; i < n; ++i) nrm += z[i] * z[i];
                    nrm = sqrt(nrm);
                    const double inv = (nrm > 0.0) ? 1.0 / nrm : 0.0;
                    for (int i = 0; i < n; ++i) z[i] *= inv;
                }
            }
        }
    }
    __syncthreads();

    // ---- 5. back-transformation, one warp per vector ----
    for (int q = warp; q < k; q += kEigWarps) {
        double* z = zT + static_cast<std::size_t>(n) * q;
        for (int j = n - 3; j >= 0; --j) {
            const double tau = stau[j];
            if (tau == 0.0) continue;
            const double* vcol = A + static_cast<std::size_t>(j) * n;  // v[j+1]=1, v[i]=A[i,j] for i>=j+2
            double s = 0.0;
            for (int i = j + 1 + lane; i < n; i += 32) s += ((i == j + 1) ? 1.0 : vcol[i]) * z[i];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            s *= tau;
            for (int i = j + 1 + lane; i < n; i += 32) z[i] -= s * ((i == j + 1) ? 1.0 : vcol[i]);
            __syncwarp();
        }
        for (int i = lane; i < n; i += 32) V[i + static_cast<std::size_t>(q) * n] = z[i];
        if (lane == 0) sig[q] = sqrt(fmax(0.0, slam[q] * gmax));
    }
    if (t == 0) {
        status[0] = 0;
        status[1] = 0;
    }
}

__global__ void __launch_bounds__(kEigThreads) eig_topk_kernel(const double* __restrict__ G, int n, int k,
                                                               double* __restrict__ work, double* __restrict__ V,
                                                               double* __restrict__ sig, int* __restrict__ status,
                                                               const int* __restrict__ skip) {
    pdl_enter();  // programmatic dependent launch: predecessor complete and visible
    if (skip && skip[0] == 1) return;  // the subspace solver already converged
    extern __shared__ double sm[];
    eig_topk_cta(G, n, k, work, V, sig, status, sm);
}

// The fused mode basis's whole fallback chain in one launch (one no-op launch
// on the fast path): the exact eigensolver if the subspace solver was not
// certified (flags[0] == 0), then W = Y V, the basis and the row-major copy
// as flagged (mb_fallback_cta).
template <typename T>
__global__ void __launch_bounds__(kEigThreads) mb_fallback_all_kernel(const double* __restrict__ Gout, int n, int k,
                                                                      double* __restrict__ work, double* __restrict__ V,
                                                                      double* __restrict__ sig, int* __restrict__ est,
                                                                      const T* __restrict__ Y, int rows,
                                                                      double* __restrict__ W, double* __restrict__ U,
                                                                      double* __restrict__ sv, int* __restrict__ st,
                                                                      T* __restrict__ Ur, int rs,
                                                                      const int* __restrict__ flags) {
    pdl_enter();  // programmatic dependent launch: predecessor complete and visible
    const bool eig = flags[0] == 0;
    if (!eig && !flags[1] && !flags[2] && !flags[3]) return;
    extern __shared__ double sm[];
    if (eig) eig_topk_cta(Gout, n, k, work, V, sig, est, sm);
    __syncthreads();
    mb_fallback_cta<T>(Y, rows, n, V, k, W, sig, U, sv, st, Ur, rs, flags, sm);
}

std::size_t eig_smem_bytes(int n) {
    std::size_t words = static_cast<std::size_t>(8) * n + kEigWarps * n + 32;
    if (n <= kSmemMatrixN) words += static_cast<std::size_t>(n) * n;
    return words * sizeof(double);
}

std::size_t eig_work_doubles(int n, int k) {
    return static_cast<std::size_t>(n) * n + static_cast<std::size_t>(6) * n * k;
}

void eig_topk(Ctx* ctx, const double* G, int n, int k, double* work, double* V, double* sig, int* status,
              const int* skip) {
    const std::size_t smem = eig_smem_bytes(n);
    static std::uint64_t attr_set = 0;  // per-device mask
    if (first_on_device(attr_set, ctx->device)) {
        MB_CUDA(cudaFuncSetAttribute(eig_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    }
    if (smem > 227 * 1024) throw Error(MACH_ERR_INTERNAL, "eigen step too large for one CTA (n=" + std::to_string(n) + ")");
    MB_LAUNCH_PDL(ctx, eig_topk_kernel, 1, kEigThreads, smem, G, n, k, work, V, sig, status, skip);
}

template <typename T>
void mb_fallback_all(Ctx* ctx, const double* Gout, int n, int k, double* work, double* V, double* sig, int* est,
                     const T* Y, int rows, double* W, double* U, double* sv, int* st, T* Ur, int rs, const int* flags) {
    const std::size_t smem = std::max(eig_smem_bytes(n), basis_smem(rows, k));
    static std::uint64_t attr_set = 0;  // per-device mask
    if (first_on_device(attr_set, ctx->device)) {
        MB_CUDA(cudaFuncSetAttribute(mb_fallback_all_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    }
    if (smem > 227 * 1024) throw Error(MACH_ERR_INTERNAL, "eigen step too large for one CTA (n=" + std::to_string(n) + ")");
    MB_LAUNCH_PDL(ctx, mb_fallback_all_kernel<T>, 1, kEigThreads, smem, Gout, n, k, work, V, sig, est, Y, rows, W, U, sv,
                  st, Ur, rs, flags);
}
template void mb_fallback_all<float>(Ctx*, const double*, int, int, double*, double*, double*, int*, const float*, int,
                                     double*, double*, double*, int*, float*, int, const int*);
template void mb_fallback_all<double>(Ctx*, const double*, int, int, double*, double*, double*, int*, const double*, int,
                                      double*, double*, double*, int*, double*, int, const int*);

}  // namespace machb
