// Subspace eigensolver for large Grams (n too big for one CTA's shared memory,
// e.g. the 512 x 512 row Grams of the C2 HOSVD): the same method as
// eig_sub.cuh (Rayleigh-Ritz with a residual certificate, Chebyshev filter,
// CholQR2), but the O(n^2 B) products G X run on many CTAs and the O(n B^2)
// steps on one CTA per job, as a fixed sequence of launches whose kernels
// return immediately once the job is certified (or handed to the exact
// solver).  G and the four n x B blocks live in global memory (L2-resident);
// a small per-job state record carries the block roles between launches.
//
// Per iteration: gemm (AX = G X) -> rr (Rayleigh-Ritz, rotation, residual
// test, filter bounds) -> m filter gemms -> orth.  Several jobs (the modes of
// one HOSVD) share every launch.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "eig_sub.cuh"

namespace machb {

namespace {

constexpr int kLJobs = 8;

struct LState {
    int roles[4];  // block index of X, AX, Y0, Y1
    int conv, fail, it, zero;
    double ie, cen;  // filter: 1 / half-width, centre
    double th[kMaxB];
};

struct LJob {
    const double* Gin;
    int n, k;
    double* Gp;       // npad x ldg, zero padded
    double* blk;      // four npad x XS blocks
    LState* st;
    const double* X0;
    int x0_cols;
    double* Xkeep;
    double* V;
    double* sig;
    int* status;
};

struct LJobs {
    LJob j[kLJobs];
};

template <int B>
__device__ __forceinline__ double* block(const LJob& J, int npad, int role) {
    return J.blk + static_cast<std::size_t>(role) * npad * Sub<B>::XS;
}

// ---- G padded (zeros outside n x n), many CTAs; grid (slabs, jobs) ----
__global__ void lg_pad_kernel(const LJobs J) {
    const LJob& jb = J.j[blockIdx.y];
    const int n = jb.n, npad = (n + 7) & ~7, ldg = frag_stride(npad);
    const long long tot = static_cast<long long>(npad) * npad;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < tot;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(e % npad), c = static_cast<int>(e / npad);
        jb.Gp[r + static_cast<std::size_t>(c) * ldg] = (r < n && c < n) ? jb.Gin[r + static_cast<std::size_t>(c) * n] : 0.0;
    }
}

// ---- start block + orthonormalisation, one CTA per job ----
template <int B>
__global__ void __launch_bounds__(kThreads, 1) lg_init_kernel(const LJobs J) {
    using SB = Sub<B>;
    constexpr int XS = SB::XS;
    const LJob& jb = J.j[blockIdx.x];
    extern __shared__ __align__(16) double sm[];
    __shared__ int flag;
    const int n = jb.n, npad = (n + 7) & ~7, ldg = frag_stride(npad);
    SubWs<B> ws(sm, npad, block<B>(jb, npad, 0));
    LState* st = jb.st;
    // zero test by the trace (G is a Gram: zero iff its trace is)
    double tr = 0.0;
    for (int i = threadIdx.x; i < n; i += kThreads) tr += jb.Gp[i + static_cast<std::size_t>(i) * ldg];
    tr = cta_sum(tr, ws.red);
    if (threadIdx.x == 0) {
        st->roles[0] = 0; st->roles[1] = 1; st->roles[2] = 2; st->roles[3] = 3;
        st->conv = 0; st->fail = 0; st->it = 0; st->zero = tr == 0.0 ? 1 : 0;
    }
    if (tr == 0.0) return;
    double* X = ws.X;
    for (int e = threadIdx.x; e < npad * B; e += kThreads) {
        const int r = e % npad, c = e / npad;
        double v = 0.0;
        if (r < n) v = (c < jb.x0_cols && jb.X0) ? jb.X0[r + c * n] : rnd_unit(static_cast<unsigned>(c), static_cast<unsigned>(r));
        X[r * XS + c] = v;
        ws.AX[r * XS + c] = 0.0;
        ws.Y0[r * XS + c] = 0.0;
        ws.Y1[r * XS + c] = 0.0;
    }
    __syncthreads();
    double* Xp = ws.X;
    double* T = ws.Y0;
    SB::orthonormalize(Xp, T, n, npad, ws.S, ws.Z, ws.rinv, ws.coef, ws.red, &flag);
    if (threadIdx.x == 0 && Xp != ws.X) {  // CholQR swapped X and Y0
        st->roles[0] = 2;
        st->roles[2] = 0;
    }
}

// ---- OUT = a (G IN) + b1 P1 + b2 P2 on row slabs; grid (slabs, jobs) ----
// step 0: AX = G X; step s >= 1: filter recurrence step s (roles rotate
// y0 <- y1 <- spare <- y0 as in subspace_core)
template <int B>
__global__ void __launch_bounds__(kThreads) lg_gemm_kernel(const LJobs J, int step) {
    constexpr int XS = Sub<B>::XS, CT = Sub<B>::CT;
    const LJob& jb = J.j[blockIdx.y];
    const LState* st = jb.st;
    if (st->conv || st->fail || st->zero) return;
    const int n = jb.n, npad = (n + 7) & ~7, ldg = frag_stride(npad);
    const int row0 = blockIdx.x * 8;
    if (row0 >= npad) return;
    int rX = st->roles[0], rAX = st->roles[1], rY0 = st->roles[2], rY1 = st->roles[3];
    const double* IN;
    double* OUT;
    const double *P1 = nullptr, *P2 = nullptr;
    double a = 1.0, b1 = 0.0, b2 = 0.0;
    if (step == 0) {
        IN = block<B>(jb, npad, rX);
        OUT = block<B>(jb, npad, rAX);
    } else {
        // (y0, y1, spare) before step s: s = 1: (X, -, -) -> Y1; s >= 2 after rotations
        int y0 = rX, y1 = rY1, spare = rY0;
        for (int s = 2; s < step; ++s) {
            const int t = y0;
            y0 = y1;
            y1 = spare;
            spare = t;
        }
        if (step == 1) {
            IN = block<B>(jb, npad, rX);
            OUT = block<B>(jb, npad, rY1);
            P1 = IN;
            a = st->ie;
            b1 = -st->cen * st->ie;
        } else {
            IN = block<B>(jb, npad, y1);
            OUT = block<B>(jb, npad, spare);
            P1 = IN;
            P2 = block<B>(jb, npad, y0);
            a = 2.0 * st->ie;
            b1 = -2.0 * st->cen * st->ie;
            b2 = -1.0;
        }
    }
    // one 8-row tile per CTA; the k range is split over the warps (k-steps
    // of 4 interleaved), partial tiles summed in a fixed order
    __shared__ double part[kThreads / 32][CT * 64];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gr = lane >> 2, tq = lane & 3;
    double c[CT][2];
#pragma unroll
    for (int t = 0; t < CT; ++t) c[t][0] = c[t][1] = 0.0;
    const double* ga = jb.Gp + (row0 + gr) + static_cast<std::size_t>(tq) * ldg;
    const double* xb = IN + tq * XS + gr;
    const int KS = npad >> 2;
#pragma unroll 4
    for (int ks = warp; ks < KS; ks += kThreads / 32) {
        const double av = ga[static_cast<std::size_t>(4 * ks) * ldg];
        double bv[CT];
#pragma unroll
        for (int t = 0; t < CT; ++t) bv[t] = xb[4 * ks * XS + t * 8];
#pragma unroll
        for (int t = 0; t < CT; ++t) dmma(c[t][0], c[t][1], av, bv[t]);
    }
#pragma unroll
    for (int t = 0; t < CT; ++t) {
        part[warp][t * 64 + gr * 8 + 2 * tq] = c[t][0];
        part[warp][t * 64 + gr * 8 + 2 * tq + 1] = c[t][1];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < CT * 64; e += kThreads) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < kThreads / 32; ++w) s += part[w][e];
        const int t = e >> 6, r = (e >> 3) & 7, cc = e & 7;
        const int off = (row0 + r) * XS + t * 8 + cc;
        double v = a * s;
        if (P1) v = fma(b1, P1[off], v);
        if (P2) v = fma(b2, P2[off], v);
        OUT[off] = v;
    }
}

// ---- Rayleigh-Ritz + residual test + filter bounds, one CTA per job ----
template <int B>
__global__ void __launch_bounds__(kThreads, 1) lg_rr_kernel(const LJobs J, int maxit, double tol) {
    using SB = Sub<B>;
    const LJob& jb = J.j[blockIdx.x];
    LState* st = jb.st;
    if (st->conv || st->fail || st->zero) return;
    extern __shared__ __align__(16) double sm[];
    __shared__ int flag;
    const int n = jb.n, k = jb.k, npad = (n + 7) & ~7;
    SubWs<B> ws(sm, npad, jb.blk);
    double* X = block<B>(jb, npad, st->roles[0]);
    double* AX = block<B>(jb, npad, st->roles[1]);
    double* Y0 = block<B>(jb, npad, st->roles[2]);
    const int it = st->it;
    SB::gram(X, AX, ws.H, npad);
    if (!SB::refine_rr(ws.H, ws.Hc, ws.W, ws.Z, ws.Q, ws.S, ws.th, k, &flag))
        SB::rr_hybrid(ws.H, ws.Hc, ws.W, ws.Z, ws.Q, ws.S, ws.J7, ws.th, k, &flag, ws.red, it == 0 ? 8 : 4);
    SB::rotate(X, ws.W, Y0, npad);
    SB::rotate(AX, ws.W, X, npad);  // X is free again: AX' lands there
    // roles: X' = old Y0, AX' = old X, Y0' = old AX
    const int rX = st->roles[2], rAX = st->roles[0], rY0 = st->roles[1];
    const double rmax = SB::residual(block<B>(jb, npad, rX), block<B>(jb, npad, rAX), ws.th, n, k, ws.red);
    const double scale = fmax(fabs(ws.th[0]), 1e-300);
    __syncthreads();
    if (threadIdx.x < B) st->th[threadIdx.x] = ws.th[threadIdx.x];
    if (threadIdx.x == 0) {
        st->roles[0] = rX;
        st->roles[1] = rAX;
        st->roles[2] = rY0;
        if (rmax <= tol * scale) {
            st->conv = 1;
        } else if (it >= maxit) {
            st->fail = 1;  // the exact solver takes over
        } else {
            const double cut = ws.th[B - 1], lo = -1e-12 * scale;
            const double e = 0.5 * (cut - lo);
            st->ie = e > 0.0 ? 1.0 / e : 0.0;
            st->cen = 0.5 * (cut + lo);
            if (!(e > 0.0)) st->fail = 1;
            st->it = it + 1;
        }
    }
}

// ---- orthonormalise the filtered block, one CTA per job ----
template <int B>
__global__ void __launch_bounds__(kThreads, 1) lg_orth_kernel(const LJobs J, int m) {
    using SB = Sub<B>;
    const LJob& jb = J.j[blockIdx.x];
    LState* st = jb.st;
    if (st->conv || st->fail || st->zero) return;
    extern __shared__ __align__(16) double sm[];
    __shared__ int flag;
    const int n = jb.n, npad = (n + 7) & ~7;
    SubWs<B> ws(sm, npad, jb.blk);
    // roles after m filter steps (see lg_gemm_kernel)
    int y0 = st->roles[0], y1 = st->roles[3], spare = st->roles[2];
    for (int s = 2; s <= m; ++s) {
        const int t = y0;
        y0 = y1;
        y1 = spare;
        spare = t;
    }
    double* X = block<B>(jb, npad, y1);
    double* T = block<B>(jb, npad, y0);
    double* X0p = X;
    SB::orthonormalize(X, T, n, npad, ws.S, ws.Z, ws.rinv, ws.coef, ws.red, &flag);
    if (threadIdx.x == 0) {
        const bool swapped = X != X0p;
        st->roles[0] = swapped ? y0 : y1;  // X
        st->roles[2] = swapped ? y1 : y0;  // Y0
        st->roles[3] = spare;              // Y1
        // roles[1] (AX) is unchanged
    }
}

// ---- outputs, one CTA per job ----
template <int B>
__global__ void lg_final_kernel(const LJobs J) {
    constexpr int XS = Sub<B>::XS;
    const LJob& jb = J.j[blockIdx.x];
    const LState* st = jb.st;
    const int n = jb.n, k = jb.k, npad = (n + 7) & ~7;
    if (st->zero) {
        for (int e = threadIdx.x; e < n * k; e += blockDim.x) jb.V[e] = ((e % n) == (e / n)) ? 1.0 : 0.0;
        if (threadIdx.x < k) jb.sig[threadIdx.x] = 0.0;
        if (threadIdx.x == 0) { jb.status[0] = 1; jb.status[1] = 1; jb.status[2] = 0; }
        return;
    }
    const double* X = block<B>(jb, npad, st->roles[0]);
    for (int e = threadIdx.x; e < n * k; e += blockDim.x) jb.V[e] = X[(e % n) * XS + e / n];
    if (jb.Xkeep) {
        for (int e = threadIdx.x; e < n * B; e += blockDim.x) jb.Xkeep[e] = X[(e % n) * XS + e / n];
        if (threadIdx.x < B) jb.Xkeep[n * B + threadIdx.x] = st->th[threadIdx.x];
    }
    if (threadIdx.x < k) jb.sig[threadIdx.x] = sqrt(fmax(0.0, st->th[threadIdx.x]));
    if (threadIdx.x == 0) { jb.status[0] = st->conv ? 1 : 0; jb.status[1] = 0; jb.status[2] = st->it; }
}

template <int B>
bool run_large(Ctx* ctx, const std::vector<EigJob>& jobs) {
    if (jobs.empty() || jobs.size() > static_cast<std::size_t>(kLJobs)) return false;
    LJobs L{};
    std::vector<DBuf<double>> bufs;
    bufs.reserve(2 * jobs.size());
    DBuf<LState> st(ctx, jobs.size());
    int npmax = 0;
    for (std::size_t i = 0; i < jobs.size(); ++i) {
        const EigJob& e = jobs[i];
        const int npad = (e.n + 7) & ~7;
        npmax = std::max(npmax, npad);
        bufs.emplace_back(ctx, static_cast<std::size_t>(npad) * frag_stride(npad));
        double* gp = bufs.back().get();
        bufs.emplace_back(ctx, static_cast<std::size_t>(4) * npad * Sub<B>::XS);
        double* blk = bufs.back().get();
        L.j[i] = LJob{e.G, e.n, e.k, gp, blk, st.get() + i, e.X0, e.x0_cols, e.Xkeep, e.V, e.sig, e.status};
    }
    const unsigned nj = static_cast<unsigned>(jobs.size());
    const std::size_t smem = SubWs<B>::small_doubles() * sizeof(double);
    const int slabs = npmax / 8;  // one 8-row tile of G per gemm CTA
    // filter degree 6 from the cold random block (growth T_6(theta_1 / e) stays
    // far inside fp64 range; the equilibrated CholQR2 absorbs the column scales)
    static const int kM = std::getenv("MACH_LG_M") ? std::atoi(std::getenv("MACH_LG_M")) : 6;
    static const int kMaxIt = std::getenv("MACH_LG_IT") ? std::atoi(std::getenv("MACH_LG_IT")) : 16;
    static std::uint64_t attr = 0;  // per-device mask
    if (first_on_device(attr, ctx->device)) {
        MB_CUDA(cudaFuncSetAttribute(lg_init_kernel<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        MB_CUDA(cudaFuncSetAttribute(lg_rr_kernel<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        MB_CUDA(cudaFuncSetAttribute(lg_orth_kernel<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    }
    MB_LAUNCH(ctx, lg_pad_kernel, dim3(64, nj), 256, 0, L);
    MB_LAUNCH(ctx, lg_init_kernel<B>, nj, kThreads, smem, L);
    // Eager (not under stream capture): iterations in batches, polling the
    // per-job state between batches so no launches are spent after every job
    // is certified.  Captured: the fixed sequence (finished jobs no-op).
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    MB_CUDA(cudaStreamIsCapturing(ctx->stream, &cs));
    const bool poll = cs == cudaStreamCaptureStatusNone;
    std::vector<LState> hs(jobs.size());
    int next_poll = 5;
    for (int it = 0; it <= kMaxIt; ++it) {
        MB_LAUNCH(ctx, lg_gemm_kernel<B>, dim3(slabs, nj), kThreads, 0, L, 0);
        MB_LAUNCH(ctx, lg_rr_kernel<B>, nj, kThreads, smem, L, kMaxIt, 1e-12);
        if (it == kMaxIt) break;
        if (poll && it + 1 == next_poll) {
            to_host(ctx, hs.data(), st.get(), jobs.size());
            sync(ctx);
            bool done = true;
            for (const LState& q : hs) done = done && (q.conv || q.fail || q.zero);
            if (done) break;
            next_poll += 2;
        }
        for (int s = 1; s <= kM; ++s) MB_LAUNCH(ctx, lg_gemm_kernel<B>, dim3(slabs, nj), kThreads, 0, L, s);
        MB_LAUNCH(ctx, lg_orth_kernel<B>, nj, kThreads, smem, L, kM);
    }
    MB_LAUNCH(ctx, lg_final_kernel<B>, nj, 256, 0, L);
    static const bool dbg = std::getenv("MACH_DEBUG_EIG_T") != nullptr;
    if (dbg) {
        std::vector<LState> h(jobs.size());
        to_host(ctx, h.data(), st.get(), jobs.size());
        sync(ctx);
        for (std::size_t i = 0; i < jobs.size(); ++i)
            std::fprintf(stderr, "[eig-large] job %zu n=%d B=%d it=%d conv=%d fail=%d zero=%d\n", i, jobs[i].n, B,
                         h[i].it, h[i].conv, h[i].fail, h[i].zero);
    }
    return true;
}

}  // namespace

// Large-n eigenproblems (same block size b for all jobs).  False when not
// applicable (the caller keeps its other path).  Uncertified jobs keep
// status[0] = 0 so the exact solver that follows in the stream takes over.
bool eig_large_batched(Ctx* ctx, const std::vector<EigJob>& jobs, int b) {
    switch (b) {
        case 8: return run_large<8>(ctx, jobs);
        case 16: return run_large<16>(ctx, jobs);
        case 24: return run_large<24>(ctx, jobs);
        case 32: return run_large<32>(ctx, jobs);
        default: return false;
    }
}

}  // namespace machb
