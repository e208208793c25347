// Cluster-distributed version of the warm-started subspace eigensolver
// (eig_sub.cuh / eig_subspace.cu) for Grams too large for one CTA's shared
// memory (n up to ~256: C5's 256 x 256 column Gram, C3's 256 x 256 row Gram),
// where the one-CTA kernel has to stream G and its blocks from L2 with a few
// KB of loads in flight (~1 ms per call at C5).
//
// CL CTAs of a thread-block cluster each own a slice of 8-row tiles: their
// rows of G (column-major, resident in shared memory for the whole solve) and
// of the n x B blocks.  Block products G X need all of X: before each, the
// slices are gathered over distributed shared memory into a local full copy.
// B x B Grams are partial sums over the slice, reduced over DSMEM in a fixed
// rank order, so every CTA holds the same small matrices and runs the same
// small-matrix steps (Rayleigh-Ritz rotations, Cholesky, filter bounds) —
// identical inputs, identical results, uniform control flow across the
// cluster.  The algorithm is the one-CTA solver's, step for step (same
// filter, certificate and tolerances, CholQR2 with the twice-Gram-Schmidt
// fallback); an uncertified solve leaves the exact selected-eigenpair solver
// to run next, as there.
#pragma once

#include <cooperative_groups.h>

#include "eig_sub.cuh"

namespace machb {
namespace {

namespace cgc = cooperative_groups;

constexpr int kECL = 8;  // cluster size

template <int B>
struct ClusterLayout {
    static constexpr int XS = Sub<B>::XS;
    int npad, rpc, r0, r1, ldl;
    __host__ __device__ ClusterLayout(int n, int rank) {
        npad = (n + 7) & ~7;
        rpc = ((npad + kECL - 1) / kECL + 7) & ~7;  // rows per CTA, whole 8-row tiles
        r0 = min(npad, rank * rpc);
        r1 = min(npad, r0 + rpc);
        ldl = frag_stride(rpc);
    }
    // doubles: small matrices | G slice (ldl x npad) | full gather copy (npad x XS) | 4 local blocks (rpc x XS) | partials
    __host__ __device__ static std::size_t doubles(int n) {
        ClusterLayout L(n, 0);
        return SubWs<B>::small_doubles() + static_cast<std::size_t>(L.ldl) * L.npad +
               static_cast<std::size_t>(L.npad) * XS + 4ull * L.rpc * XS + static_cast<std::size_t>(B) * Sub<B>::HS + 64;
    }
};

template <int B>
struct Dist {
    using SB = Sub<B>;
    static constexpr int XS = SB::XS, HS = SB::HS;
    cgc::cluster_group cl;
    int rank, CL;
    ClusterLayout<B> L;
    double* F;     // full gather copy (npad x XS)
    double* Cp;    // B x B partial (ld HS)
    double* colp;  // per-column partials (B)
    double* red_;  // CTA reduction scratch (32)
    __device__ Dist(cgc::cluster_group c, int n, double* f, double* cp, double* cols, double* red)
        : cl(c), rank(static_cast<int>(c.block_rank())), CL(static_cast<int>(c.num_blocks())), L(n, rank), F(f),
          Cp(cp), colp(cols), red_(red) {}

    // all slices of block P (absolute rows, each CTA's slice at the same smem
    // offset) into F.  The two cluster barriers: writers done / readers done.
    __device__ void gather(const double* P) {
        cl.sync();
        // P is an absolute-row view; its slice storage starts at P + r0 XS,
        // at the same shared-memory offset in every CTA
        double* base = const_cast<double*>(P) + static_cast<std::ptrdiff_t>(L.r0) * XS;
        for (int q = 0; q < CL; ++q) {
            const int q0 = min(L.npad, q * L.rpc), q1 = min(L.npad, q0 + L.rpc);
            const double* src = cl.map_shared_rank(base, q);
            for (int e = threadIdx.x; e < (q1 - q0) * XS; e += kThreads) F[q0 * XS + e] = src[e];
        }
        cl.sync();
    }
    // C (B x B, ld HS) = A^T M over all rows: slice partials, fixed-order DSMEM sum
    __device__ void gram(const double* A, const double* M, double* C) {
        SB::gram(A, M, Cp, L.npad, L.r0, L.r1);  // ends with __syncthreads
        cl.sync();
        for (int e = threadIdx.x; e < B * B; e += kThreads) {
            const int i = e % B, j = e / B;
            double s = 0.0;
            for (int q = 0; q < CL; ++q) s += cl.map_shared_rank(Cp, q)[i + j * HS];
            C[i + j * HS] = s;
        }
        cl.sync();  // partials may be overwritten after this
    }
    // max over wanted columns of |AX_c - th_c X_c| (sums of squares reduced over the cluster)
    __device__ double residual(const double* X, const double* AX, const double* th, int n, int k, double* red) {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const int rn = min(L.r1, n);
        for (int c = warp; c < k; c += kWarps) {
            double s = 0.0;
            for (int r = L.r0 + lane; r < rn; r += 32) {
                const double d = AX[r * XS + c] - th[c] * X[r * XS + c];
                s = fma(d, d, s);
            }
            s = warp_sum(s);
            if (lane == 0) colp[c] = s;
        }
        cl.sync();
        double rmax = 0.0;
        for (int c = 0; c < k; ++c) {
            double s = 0.0;
            for (int q = 0; q < CL; ++q) s += cl.map_shared_rank(colp, q)[c];
            rmax = fmax(rmax, sqrt(s));
        }
        cl.sync();
        (void)red;
        return rmax;
    }
    // OUT = a G IN + b1 P1 + b2 P2 on this CTA's rows (IN gathered into F first)
    __device__ void gemm(const double* Gv, const double* IN, double* OUT, double a, const double* P1, double b1,
                         const double* P2, double b2) {
        gather(IN);
        SB::gemm(Gv, L.ldl, F, OUT, L.npad, a, P1, b1, P2, b2, L.r0 >> 3, L.r1 >> 3);
    }
    __device__ void rotate(const double* X, const double* W, double* OUT) {
        SB::rotate(X, W, OUT, L.npad, L.r0 >> 3, L.r1 >> 3);
    }
    // CholQR on the distributed block (X <- X R^{-1}, pointers swapped)
    __device__ bool cholqr(double*& X, double*& T, double* S, double* Ri, double* rinv, int* flag, bool allow_skip) {
        gram(X, X, S);
        bool skip = false;
        if (!SB::chol_factor(S, Ri, rinv, flag, allow_skip, skip)) return false;
        if (skip) return true;
        rotate(X, Ri, T);
        double* t = X;
        X = T;
        T = t;
        return true;
    }
    // sum over the cluster of per-CTA values v[0..cnt) (cnt <= B), fixed rank order
    __device__ void reduce_cols(double* out, int cnt) {
        cl.sync();
        for (int c = threadIdx.x; c < cnt; c += kThreads) {
            double s = 0.0;
            for (int q = 0; q < CL; ++q) s += cl.map_shared_rank(colp, q)[c];
            out[c] = s;
        }
        cl.sync();
    }
    // classical Gram-Schmidt twice, column by column, collapsed columns
    // replaced by the same deterministic random vectors as Sub::cgs2
    __device__ void cgs2(double* X, int n, double* coef) {
        __shared__ double nrm[2];
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const int rn = min(L.r1, n);
        auto colnorm = [&](int j) -> double {
            double s = 0.0;
            for (int r = L.r0 + static_cast<int>(threadIdx.x); r < rn; r += kThreads) s += X[r * XS + j] * X[r * XS + j];
            __shared__ double rd[kWarps];
            s = warp_sum(s);
            if (lane == 0) rd[warp] = s;
            __syncthreads();
            if (threadIdx.x == 0) {
                double t = 0.0;
                for (int w = 0; w < kWarps; ++w) t += rd[w];
                colp[0] = t;
            }
            reduce_cols(nrm, 1);
            __syncthreads();
            return sqrt(nrm[0]);
        };
        for (int j = 0; j < B; ++j) {
            for (int attempt = 0; attempt < 2; ++attempt) {
                const double n0 = colnorm(j);
                for (int pass = 0; pass < 2 && j > 0; ++pass) {
                    for (int c = warp; c < j; c += kWarps) {
                        double s = 0.0;
                        for (int r = L.r0 + lane; r < rn; r += 32) s += X[r * XS + c] * X[r * XS + j];
                        s = warp_sum(s);
                        if (lane == 0) colp[c] = s;
                    }
                    reduce_cols(coef, j);
                    __syncthreads();
                    for (int r = L.r0 + static_cast<int>(threadIdx.x); r < rn; r += kThreads) {
                        double v = X[r * XS + j];
                        for (int c = 0; c < j; ++c) v -= X[r * XS + c] * coef[c];
                        X[r * XS + j] = v;
                    }
                    __syncthreads();
                }
                const double nn = colnorm(j);
                if (nn > 1e-10 * n0 && nn > 0.0) {
                    const double inv = 1.0 / nn;
                    for (int r = L.r0 + static_cast<int>(threadIdx.x); r < rn; r += kThreads) X[r * XS + j] *= inv;
                    __syncthreads();
                    break;
                }
                for (int r = L.r0 + static_cast<int>(threadIdx.x); r < rn; r += kThreads)
                    X[r * XS + j] = rnd_unit(1000u + j + 97u * attempt, r);
                __syncthreads();
            }
        }
    }
    __device__ void orthonormalize(double*& X, double*& T, double* S, double* Ri, double* rinv, double* coef, int n,
                                   int* flag) {
        if (!cholqr(X, T, S, Ri, rinv, flag, false) || !cholqr(X, T, S, Ri, rinv, flag, true)) {
            if (rank == 0) sub_stamp(600);
            // the Gram-Schmidt fallback on a gathered full copy, run by every
            // CTA (identical results), each keeping its own rows: one gather
            // instead of ~8 cluster barriers per column
            gather(X);
            SB::cgs2(F, n, coef, red_);
            for (int e = threadIdx.x; e < (L.r1 - L.r0) * XS; e += kThreads) X[L.r0 * XS + e] = F[L.r0 * XS + e];
            __syncthreads();
        }
    }
};

template <int B>
__global__ void __launch_bounds__(kThreads, 1)
    eig_cluster_kernel(const double* __restrict__ Gin, int n, int k, const double* X0, int x0_cols, const double* th0,
                       double* Xkeep, double* __restrict__ V, double* __restrict__ sig, int* __restrict__ status, int m,
                       int maxit, double tol, int dbg) {
    using SB = Sub<B>;
    constexpr int XS = SB::XS, HS = SB::HS;
    cgc::cluster_group cl = cgc::this_cluster();
    extern __shared__ __align__(16) double sm[];
    __shared__ int flag;
    const int rank = static_cast<int>(cl.block_rank());
    ClusterLayout<B> L(n, rank);
    SubWs<B> ws(sm, L.npad, sm);  // small matrices only (the blocks are laid out below)
    double* Gl = sm + SubWs<B>::small_doubles();
    double* F = Gl + static_cast<std::size_t>(L.ldl) * L.npad;
    double* blk = F + static_cast<std::size_t>(L.npad) * XS;
    double* Cp = blk + 4ull * L.rpc * XS;
    double* colp = Cp + B * HS;
    Dist<B> D(cl, n, F, Cp, colp, ws.red);
    // absolute-row views of the local slices
    double* Gv = Gl - L.r0;
    double* X = blk - static_cast<std::ptrdiff_t>(L.r0) * XS;
    double* AX = X + static_cast<std::ptrdiff_t>(L.rpc) * XS;
    double* Y0 = AX + static_cast<std::ptrdiff_t>(L.rpc) * XS;
    double* Y1 = Y0 + static_cast<std::ptrdiff_t>(L.rpc) * XS;
    double *H = ws.H, *W = ws.W, *S = ws.S, *Z = ws.Z, *Q = ws.Q, *Hc = ws.Hc, *th = ws.th, *rinv = ws.rinv,
           *red = ws.red;

    // ---- G slice (rows [r0, r1), all columns; zero padding) and start block ----
    for (int e = threadIdx.x; e < (L.r1 - L.r0) * L.npad; e += kThreads) {
        const int rl = e % (L.r1 - L.r0), c = e / (L.r1 - L.r0), r = L.r0 + rl;
        Gl[rl + static_cast<std::size_t>(c) * L.ldl] = (r < n && c < n) ? Gin[r + static_cast<std::size_t>(c) * n] : 0.0;
    }
    for (int e = threadIdx.x; e < (L.r1 - L.r0) * B; e += kThreads) {
        const int r = L.r0 + e / B, c = e % B;
        double v = 0.0;
        if (r < n) v = (X0 && c < x0_cols) ? X0[r + static_cast<std::size_t>(c) * n] : rnd_unit(static_cast<unsigned>(c), static_cast<unsigned>(r));
        X[r * XS + c] = v;
        AX[r * XS + c] = 0.0;
        Y0[r * XS + c] = 0.0;
        Y1[r * XS + c] = 0.0;
    }
    // trace of G on the whole cluster: zero matrix?
    double tr = 0.0;
    for (int r = L.r0 + static_cast<int>(threadIdx.x); r < min(L.r1, n); r += kThreads) tr += Gl[(r - L.r0) + static_cast<std::size_t>(r) * L.ldl];
    tr = cta_sum(tr, red);
    if (threadIdx.x == 0) colp[0] = tr;
    cl.sync();
    double trace = 0.0;
    for (int q = 0; q < static_cast<int>(cl.num_blocks()); ++q) trace += cl.map_shared_rank(colp, q)[0];
    cl.sync();
    if (trace == 0.0) {
        for (int e = threadIdx.x; e < (L.r1 - L.r0) * k; e += kThreads) {
            const int r = L.r0 + e / k, c = e % k;
            if (r < n) V[r + static_cast<std::size_t>(c) * n] = (r == c) ? 1.0 : 0.0;
        }
        if (rank == 0 && threadIdx.x < k) sig[threadIdx.x] = 0.0;
        if (rank == 0 && threadIdx.x == 0) { status[0] = 1; status[1] = 1; status[2] = 0; }
        cl.sync();
        return;
    }
    auto stamp = [&](int tag) {
        if (rank == 0) sub_stamp(tag);
    };
    stamp(1);
    bool ok = true;
    if (x0_cols < B || !X0) D.orthonormalize(X, Y0, S, Z, rinv, ws.coef, n, &flag);
    stamp(2);
    const bool filter_first = X0 && x0_cols >= B && th0;
    if (filter_first && threadIdx.x < B) th[threadIdx.x] = th0[threadIdx.x];
    __syncthreads();
    bool conv = false, ax_valid = false, guards_saved = false;
    int it = 0;
    for (;; ++it) {
        if (!(filter_first && it == 0)) {
            D.gemm(Gv, X, AX, 1.0, nullptr, 0.0, nullptr, 0.0);
            stamp(10);
            D.gram(X, AX, H);
            stamp(11);
            int nsw = 99;
            if (!SB::refine_rr(H, Hc, W, Z, Q, S, th, k, &flag)) nsw = SB::rr_hybrid(H, Hc, W, Z, Q, S, ws.J7, th, k, &flag, red, it == 0 ? 8 : 3);
            stamp(1000 + nsw);
            D.rotate(X, W, Y0);
            { double* t = X; X = Y0; Y0 = t; }
            D.rotate(AX, W, Y0);
            { double* t = AX; AX = Y0; Y0 = t; }
            ax_valid = true;
            stamp(13);
            const double rmax = D.residual(X, AX, th, n, k, red);
            stamp(14);
            const double scale = fmax(fabs(th[0]), 1e-300);
            if (dbg && rank == 0 && threadIdx.x == 0)
                printf("[eigc] it %d th0 %.6e thB %.6e rmax/scale %.3e flag %d\n", it, th[0], th[B - 1], rmax / scale, flag);
            if (rmax <= tol * scale) { conv = true; break; }
            if (it >= maxit) break;
        }
        // ---- Chebyshev filter on [-|theta_1| 1e-12, theta_B] (as subspace_core) ----
        const double scale = fmax(fabs(th[0]), 1e-300);
        const double cut = th[B - 1];
        const double lo = -1e-12 * scale;
        const double e = 0.5 * (cut - lo), cen = 0.5 * (cut + lo);
        const int lr0 = L.r0, lr1 = L.r1;
        (void)lr0;
        if (!(e > 0.0)) {
            if (ax_valid) {
                for (int idx = lr0 * XS + static_cast<int>(threadIdx.x); idx < lr1 * XS; idx += kThreads) Y1[idx] = AX[idx];
                __syncthreads();
            } else {
                D.gemm(Gv, X, Y1, 1.0, nullptr, 0.0, nullptr, 0.0);
            }
            ax_valid = false;
            { double* t = X; X = Y1; Y1 = t; }
        } else {
            const double ie = 1.0 / e;
            guards_saved = false;
            if (ax_valid) {
                for (int idx = lr0 * XS + static_cast<int>(threadIdx.x); idx < lr1 * XS; idx += kThreads)
                    Y1[idx] = ie * AX[idx] - cen * ie * X[idx];
                __syncthreads();
                // keep the pre-filter guard columns (AX is free until the next
                // Rayleigh-Ritz): if the filter's gain lifts traces of the
                // leading directions in them above the guards themselves, the
                // CholQR retries with them instead of falling back to
                // Gram-Schmidt
                for (int e = threadIdx.x; e < (lr1 - lr0) * (B - k); e += kThreads) {
                    const int r = lr0 + e / (B - k), c = k + e % (B - k);
                    AX[r * XS + c] = X[r * XS + c];
                }
                __syncthreads();
                guards_saved = true;
            } else {
                D.gemm(Gv, X, Y1, ie, X, -cen * ie, nullptr, 0.0);
                for (int e = threadIdx.x; e < (lr1 - lr0) * (B - k); e += kThreads) {
                    const int r = lr0 + e / (B - k), c = k + e % (B - k);
                    AX[r * XS + c] = X[r * XS + c];
                }
                __syncthreads();
                guards_saved = true;
            }
            ax_valid = false;
            double* y0 = X;
            double* y1 = Y1;
            double* spare = Y0;
            for (int j = 2; j <= m; ++j) {
                D.gemm(Gv, y1, spare, 2.0 * ie, y1, -2.0 * cen * ie, y0, -1.0);
                double* t = y0;
                y0 = y1;
                y1 = spare;
                spare = t;
            }
            X = y1;
            Y0 = y0;
            Y1 = spare;
        }
        stamp(15);
        if (guards_saved && !D.cholqr(X, Y0, S, Z, rinv, &flag, false)) {
            stamp(601);
            for (int e = threadIdx.x; e < (lr1 - lr0) * (B - k); e += kThreads) {
                const int r = lr0 + e / (B - k), c = k + e % (B - k);
                X[r * XS + c] = AX[r * XS + c];
            }
            __syncthreads();
        } else if (guards_saved) {
            // first pass done: the second (usually skipped) below
            if (!D.cholqr(X, Y0, S, Z, rinv, &flag, true)) D.orthonormalize(X, Y0, S, Z, rinv, ws.coef, n, &flag);
            stamp(16);
            continue;
        }
        D.orthonormalize(X, Y0, S, Z, rinv, ws.coef, n, &flag);
        stamp(16);
    }
    // ---- outputs (column-major, absolute rows of this slice) ----
    const int rn = min(L.r1, n);
    for (int e = threadIdx.x; e < (rn - L.r0) * k; e += kThreads) {
        const int r = L.r0 + e / k, c = e % k;
        V[r + static_cast<std::size_t>(c) * n] = X[r * XS + c];
    }
    if (Xkeep) {
        for (int e = threadIdx.x; e < (rn - L.r0) * B; e += kThreads) {
            const int r = L.r0 + e / B, c = e % B;
            Xkeep[r + static_cast<std::size_t>(c) * n] = X[r * XS + c];
        }
        if (rank == 0 && threadIdx.x < B) Xkeep[static_cast<std::size_t>(n) * B + threadIdx.x] = th[threadIdx.x];
    }
    if (rank == 0 && threadIdx.x < k) sig[threadIdx.x] = sqrt(fmax(0.0, th[threadIdx.x]));
    if (rank == 0 && threadIdx.x == 0) { status[0] = (conv && ok) ? 1 : 0; status[1] = 0; status[2] = it; }
    cl.sync();  // no CTA leaves while its shared memory may still be read
}

}  // namespace
}  // namespace machb
