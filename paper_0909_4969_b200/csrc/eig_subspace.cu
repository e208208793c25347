// Warm-started, Chebyshev-filtered block subspace eigensolver for the HOOI
// eigen step (reference: gram_side_basis, proj/src/linalg.cpp:106-120 — the
// top-k eigenpairs of the symmetric Gram of Y_(n)).
//
// Why not a full tridiagonal eigensolver per mode: the n sequential Householder
// steps are latency-bound on a GPU (hundreds of microseconds at n = 100),
// while HOOI asks for only k << n eigenvectors of a Gram that barely moves
// between sweeps.  One CTA keeps G and the n x B block in shared memory and
// runs:
//   X <- previous sweep's Ritz block (or a deterministic random block)
//   repeat: Rayleigh-Ritz (H = X^T G X; second-order perturbation rotation
//           when H is nearly diagonal, CTA-parallel cyclic Jacobi otherwise),
//           residual test |G x_i - theta_i x_i| <= tol * theta_1 for i < k,
//           degree-m Chebyshev filter damping [0, theta_B], CholQR2
// The residual certificate bounds each Ritz vector's angle to its eigenvector
// by residual / gap, so converged output equals the reference's exact
// eigendecomposition to that precision.  Unconverged calls (tiny gaps) leave
// status[0] = 0 and the exact selected-eigenpair solver (eig.cu) runs next in
// the stream — it checks status and is a no-op otherwise.
//
// Layout: the block size B is a template parameter (multiple of 4, <= 32);
// n x B blocks are row-major with a padded row stride (B + 2 doubles) so a
// row is two-to-eight 128-bit loads and different rows hit different banks;
// B x B matrices use an odd leading dimension (B + 1).
#include <algorithm>
#include <vector>

#include "eig_cluster.cuh"
#include "eig_sub.cuh"

namespace machb {

namespace {

// status: [0] converged, [1] zero matrix, [2] iterations used.  Gw: global
// workspace (npad x ldg doubles) for G when it does not fit shared memory.
constexpr int kMaxJobs = 8;
struct EigJobs {  // by value (kernel parameter): no host->device copy, graph-capturable
    EigJob j[kMaxJobs];
};

template <int B>
__global__ void __launch_bounds__(kThreads, 1) eig_subspace_kernel(const EigJobs jobs, int m, int maxit, double tol,
                                                                long long* __restrict__ tstamp) {
    // one CTA per job (independent eigenproblems, e.g. the d modes of HOSVD)
    const EigJob J = jobs.j[blockIdx.x];
    const double* __restrict__ Gin = J.G;
    const int n = J.n, k = J.k, x0_cols = J.x0_cols;
    const double* X0 = J.X0;
    double* Xkeep = J.Xkeep;  // may alias X0
    double* __restrict__ V = J.V;
    double* __restrict__ sig = J.sig;
    int* __restrict__ status = J.status;
    double* Gw = J.Gw;
    double* Bw = J.Bw;
    if (blockIdx.x > 0) tstamp = nullptr;
    using SB = Sub<B>;
    constexpr int XS = SB::XS;
    extern __shared__ __align__(16) double sm[];
    int ns_ = 0;
    if (tstamp && threadIdx.x == 0) tstamp[239] = clock64();
    MB_STAMP(0);
    __shared__ int flag;
    const int npad = (n + 7) & ~7;
    const int ldg = frag_stride(npad);
    // shared memory: [small matrices][blocks unless Bw][G unless Gw]
    const std::size_t blk_sm = Bw ? 0 : SubWs<B>::block_doubles(npad);
    double* G = Gw ? Gw : (sm + SubWs<B>::small_doubles() + blk_sm);
    double* red = SubWs<B>(sm, npad, Bw).red;

    // ---- load G padded to npad x npad (zeros outside n x n).  Every
    // producer of G (gram_mma_kernel, the fixed-point sparse Grams) writes it
    // exactly symmetric, so the symmetrisation of linalg.cpp:107 is a no-op. ----
    double fro = 0.0;
    {
        constexpr int U = 8;  // eight independent global loads in flight per thread
        const int nn = n * n;
        for (int base = threadIdx.x; base < nn; base += U * kThreads) {
            double v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int e = base + u * kThreads;
                v[u] = e < nn ? Gin[e] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int e = base + u * kThreads;
                if (e < nn) {
                    G[(e % n) + (e / n) * ldg] = v[u];
                    fro = fma(v[u], v[u], fro);
                }
            }
        }
    }
    for (int e = threadIdx.x; e < (npad - n) * npad; e += kThreads) {
        const int r = n + e % (npad - n), c = e / (npad - n);
        G[r + c * ldg] = 0.0;
    }
    for (int e = threadIdx.x; e < n * (npad - n); e += kThreads) {
        const int r = e % n, c = n + e / n;
        G[r + c * ldg] = 0.0;
    }
    fro = cta_sum(fro, red);  // its barriers also publish G
    if (fro == 0.0) {
        for (int e = threadIdx.x; e < n * k; e += kThreads) V[e] = ((e % n) == (e / n)) ? 1.0 : 0.0;
        if (threadIdx.x < k) sig[threadIdx.x] = 0.0;
        if (threadIdx.x == 0) { status[0] = 1; status[1] = 1; status[2] = 0; }
        return;
    }

    int it = 0;
    bool conv = false;
    SubWs<B> ws(sm, npad, Bw);
    const double* th0 = (X0 && x0_cols >= B) ? J.th0 : nullptr;
    double* X = subspace_core<B>(ws, G, ldg, n, k, m, maxit, tol, X0, x0_cols, conv, it, &flag, tstamp, ns_, th0);
    const double* th = ws.th;
    if (tstamp && threadIdx.x == 0) tstamp[238] = clock64();
    // ---- outputs (column-major) ----
    for (int e = threadIdx.x; e < n * k; e += kThreads) V[e] = X[(e % n) * XS + e / n];
    if (Xkeep) {
        for (int e = threadIdx.x; e < n * B; e += kThreads) Xkeep[e] = X[(e % n) * XS + e / n];
        if (threadIdx.x < B) Xkeep[n * B + threadIdx.x] = th[threadIdx.x];  // Ritz values travel with the block
    }
    if (threadIdx.x < k) sig[threadIdx.x] = sqrt(fmax(0.0, th[threadIdx.x]));
    if (threadIdx.x == 0) { status[0] = conv ? 1 : 0; status[1] = 0; status[2] = it; }
}

std::size_t g_doubles(int n) {
    const int npad = (n + 7) & ~7;
    return static_cast<std::size_t>(npad) * frag_stride(npad);
}

template <int B>
std::size_t subspace_smem(int n, bool g_smem, bool b_smem) {
    const int npad = (n + 7) & ~7;
    std::size_t w = SubWs<B>::small_doubles();
    if (b_smem) w += SubWs<B>::block_doubles(npad);
    if (g_smem) w += g_doubles(n);
    return w * sizeof(double);
}

constexpr std::size_t kSmemCap = 200 * 1024;

// shared-memory layout decision for one job
template <int B>
std::size_t job_plan(int n, bool& g_smem, bool& b_smem) {
    // shared memory first for G and the blocks; what does not fit lives in
    // global memory (L2-resident at these sizes): G first, then the blocks
    g_smem = true;
    b_smem = true;
    if (subspace_smem<B>(n, true, true) > kSmemCap) g_smem = false;
    if (subspace_smem<B>(n, g_smem, true) > kSmemCap) b_smem = false;
    return subspace_smem<B>(n, g_smem, b_smem);
}

// Launch the jobs (all with block size B) as one grid, one CTA each.
template <int B>
bool launch_subspace_jobs(Ctx* ctx, std::vector<EigJob>& jobs, std::vector<DBuf<double>>& ws) {
    std::size_t smem = 0;
    for (auto& J : jobs) {
        bool gs, bs;
        const std::size_t sm = job_plan<B>(J.n, gs, bs);
        if (sm > kSmemCap) return false;
        smem = std::max(smem, sm);
        if (!gs) {
            ws.emplace_back(ctx, g_doubles(J.n));
            J.Gw = ws.back().get();
        }
        if (!bs) {
            ws.emplace_back(ctx, SubWs<B>::block_doubles((J.n + 7) & ~7));
            J.Bw = ws.back().get();
        }
    }
    static std::uint64_t attr = 0;  // per-device mask
    if (first_on_device(attr, ctx->device)) {
        MB_CUDA(cudaFuncSetAttribute(eig_subspace_kernel<B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kSmemCap)));
    }
    if (jobs.size() > static_cast<std::size_t>(kMaxJobs)) return false;
    EigJobs dj{};
    for (std::size_t i = 0; i < jobs.size(); ++i) dj.j[i] = jobs[i];
    static const bool dbg = std::getenv("MACH_DEBUG_EIG_T") != nullptr;
    static const int dbgc = std::getenv("MACH_DEBUG_EIGC") ? 1 : 0;
    if (dbgc) MB_CUDA(cudaMemcpyToSymbolAsync(g_dbg_eig, &dbgc, sizeof(int), 0, cudaMemcpyHostToDevice, ctx->stream));
    DBuf<long long> ts;
    if (dbg) {
        ts.alloc(ctx, 240);
        ts.zero(ctx);
    }
    MB_LAUNCH(ctx, eig_subspace_kernel<B>, static_cast<unsigned>(jobs.size()), kThreads, smem, dj, 4, 40, 1e-12,
              dbg ? ts.get() : nullptr);
    if (dbg) {
        long long h[240];
        to_host(ctx, h, ts.get(), 240);
        sync(ctx);
        std::fprintf(stderr, "[eig-t] n=%d B=%d jobs=%d gsmem=%d bsmem=%d:", jobs[0].n, B, static_cast<int>(jobs.size()),
                     jobs[0].Gw ? 0 : 1, jobs[0].Bw ? 0 : 1);
        long long t_end = h[1];
        for (int i = 1; i < 118 && h[2 * i + 1]; ++i) {
            std::fprintf(stderr, " %lld:%.1f", h[2 * i], (h[2 * i + 1] - h[2 * i - 1]) * 1e-3);
            t_end = h[2 * i + 1];
        }
        const double us = (t_end - h[1]) * 1e-3;
        std::fprintf(stderr, " total=%.1fus cycles=%lld\n", us, h[238] - h[239]);
    }
    return true;
}

template <int B>
bool launch_subspace(Ctx* ctx, const double* G, int n, int k, const double* X0, int x0_cols, double* Xkeep, double* V,
                     double* sig, int* status) {
    std::vector<EigJob> jobs(1);
    jobs[0] = EigJob{G, n, k, X0, x0_cols, Xkeep, V, sig, status, nullptr, nullptr};
    if (X0 && x0_cols >= B) jobs[0].th0 = X0 + static_cast<std::size_t>(n) * B;  // a kept warm block
    std::vector<DBuf<double>> ws;
    ws.reserve(2);
    return launch_subspace_jobs<B>(ctx, jobs, ws);
}

}  // namespace

// Returns true when the subspace path applies (else the caller runs eig_topk).
bool eig_subspace(Ctx* ctx, const double* G, int n, int k, const double* X0, int x0_cols, double* Xkeep, int b,
                  double* V, double* sig, int* status) {
    if (b >= n || k > b - 2) return false;
    switch (b) {
        case 8: return launch_subspace<8>(ctx, G, n, k, X0, x0_cols, Xkeep, V, sig, status);
        case 16: return launch_subspace<16>(ctx, G, n, k, X0, x0_cols, Xkeep, V, sig, status);
        case 24: return launch_subspace<24>(ctx, G, n, k, X0, x0_cols, Xkeep, V, sig, status);
        case 32: return launch_subspace<32>(ctx, G, n, k, X0, x0_cols, Xkeep, V, sig, status);
        default: return false;
    }
}

int eig_block(int n, int k) {
    int b = ((k + 4 + 7) / 8) * 8;  // >= k + 4 oversampling, multiple of 8 (MMA tiles)
    if (b > kMaxB) b = kMaxB;
    return std::min(n, b);
}

bool subspace_applies(int n, int k) {
    const int b = eig_block(n, k);
    return n > kSubMinN && b < n && b <= kMaxB && (b % 8) == 0 && k <= b - 2;
}

// Cluster-distributed solver (eig_cluster.cuh) for a G that does not fit one
// CTA; false when it does not apply either.
template <int B>
bool launch_cluster(Ctx* ctx, const double* G, int n, int k, const double* X0, int x0_cols, double* Xkeep, double* V,
                    double* sig, int* status) {
    static const bool off = std::getenv("MACH_NO_EIG_CLUSTER") != nullptr;
    if (off) return false;
    const std::size_t smem = ClusterLayout<B>::doubles(n) * sizeof(double);
    static int optin = 0;
    static std::uint64_t attr = 0;
    auto kern = eig_cluster_kernel<B>;
    if (first_on_device(attr, ctx->device)) {
        cudaFuncAttributes fa{};
        MB_CUDA(cudaFuncGetAttributes(&fa, kern));
        int mx = 0;
        MB_CUDA(cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
        optin = mx - static_cast<int>(fa.sharedSizeBytes);
        MB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    }
    if (smem > static_cast<std::size_t>(optin)) return false;
    const double* th0 = (X0 && x0_cols >= B) ? X0 + static_cast<std::size_t>(n) * B : nullptr;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(kECL, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kECL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    static const int dbg = std::getenv("MACH_DEBUG_EIGC") ? 1 : 0;
    static const bool tdbg = std::getenv("MACH_DEBUG_EIG_T") != nullptr;
    DBuf<long long> sb;
    if (tdbg) {  // phase stamps of rank 0 (sub_stamp)
        sb.alloc(ctx, 200);
        sb.zero(ctx);
        long long* p = sb.get();
        int z = 0;
        MB_CUDA(cudaMemcpyToSymbolAsync(g_stamp, &p, sizeof(p), 0, cudaMemcpyHostToDevice, ctx->stream));
        MB_CUDA(cudaMemcpyToSymbolAsync(g_stamp_n, &z, sizeof(z), 0, cudaMemcpyHostToDevice, ctx->stream));
    }
    MB_LAUNCH_EX(ctx, "eig_cluster_kernel<B>", &cfg, kern, G, n, k, X0, x0_cols, th0, Xkeep, V, sig, status, 4, 40,
                 1e-12, dbg);
    if (tdbg) {
        long long f[200];
        to_host(ctx, f, sb.get(), 200);
        sync(ctx);
        std::fprintf(stderr, "[eigc-t] n=%d:", n);
        for (int i = 1; i < 100 && f[2 * i + 1]; ++i) std::fprintf(stderr, " %lld:%.1f", f[2 * i], (f[2 * i + 1] - f[2 * i - 1]) * 1e-3);
        std::fprintf(stderr, "\n");
        long long* np = nullptr;
        cudaMemcpyToSymbol(g_stamp, &np, sizeof(np));
    }
    return true;
}

bool eig_select(Ctx* ctx, const double* G, int n, int k, const double* X0, int x0_cols, double* Xkeep, int b,
                double* V, double* sig, int* status) {
    bool launched = false;
    if (n > kSubMinN && b < n && b <= kMaxB && (b % 8) == 0 && k <= b - 2) {
        bool gs = true, bs = true;
        switch (b) {
            case 8: job_plan<8>(n, gs, bs); break;
            case 16: job_plan<16>(n, gs, bs); break;
            case 24: job_plan<24>(n, gs, bs); break;
            default: job_plan<32>(n, gs, bs); break;
        }
        if (!gs || !bs) {  // G or the blocks would live in L2: the cluster solver instead
            switch (b) {
                case 8: launched = launch_cluster<8>(ctx, G, n, k, X0, x0_cols, Xkeep, V, sig, status); break;
                case 16: launched = launch_cluster<16>(ctx, G, n, k, X0, x0_cols, Xkeep, V, sig, status); break;
                case 24: launched = launch_cluster<24>(ctx, G, n, k, X0, x0_cols, Xkeep, V, sig, status); break;
                case 32: launched = launch_cluster<32>(ctx, G, n, k, X0, x0_cols, Xkeep, V, sig, status); break;
                default: break;
            }
        }
    }
    if (launched) {
        DBuf<double> work(ctx, eig_work_doubles(n, k));
        eig_topk(ctx, G, n, k, work.get(), V, sig, status, status);
        return true;
    }
    if (n > kSubMinN && b < n && b <= kMaxB && (b % 8) == 0 && k <= b - 2)
        launched = eig_subspace(ctx, G, n, k, X0, x0_cols, Xkeep, b, V, sig, status);
    DBuf<double> work(ctx, eig_work_doubles(n, k));
    eig_topk(ctx, G, n, k, work.get(), V, sig, status, launched ? status : nullptr);
    return launched;
}

// Several independent eigenproblems (same k): subspace solver CTAs in one
// launch when they share a block size, then each exact fallback in the
// stream (no-ops where certified).
void eig_select_batched(Ctx* ctx, std::vector<EigJob> jobs) {
    bool same = !jobs.empty();
    int b = 0;
    for (auto& J : jobs) {
        const int bj = eig_block(J.n, J.k);
        const bool ok = J.n > kSubMinN && bj < J.n && bj <= kMaxB && (bj % 8) == 0 && J.k <= bj - 2;
        if (!ok || (b && bj != b)) same = false;
        b = bj;
    }
    bool launched = false;
    std::vector<DBuf<double>> ws;
    ws.reserve(2 * jobs.size());
    if (same && !std::getenv("MACH_EIG_LARGE_OFF")) {
        // G beyond one CTA's shared memory: the multi-kernel solver spreads
        // the G X products over many SMs
        bool big = true;
        for (auto& J : jobs) {
            bool gs = true, bs = true;
            switch (b) {
                case 8: job_plan<8>(J.n, gs, bs); break;
                case 16: job_plan<16>(J.n, gs, bs); break;
                case 24: job_plan<24>(J.n, gs, bs); break;
                default: job_plan<32>(J.n, gs, bs); break;
            }
            if (gs) big = false;
        }
        static const int bf = std::getenv("MACH_LG_B") ? std::atoi(std::getenv("MACH_LG_B")) : 0;
        if (big) launched = eig_large_batched(ctx, jobs, bf ? bf : b);
    }
    if (same && !launched) {
        switch (b) {
            case 8: launched = launch_subspace_jobs<8>(ctx, jobs, ws); break;
            case 16: launched = launch_subspace_jobs<16>(ctx, jobs, ws); break;
            case 24: launched = launch_subspace_jobs<24>(ctx, jobs, ws); break;
            case 32: launched = launch_subspace_jobs<32>(ctx, jobs, ws); break;
            default: break;
        }
    }
    for (auto& J : jobs) {
        if (!launched) {
            eig_select(ctx, J.G, J.n, J.k, J.X0, J.x0_cols, J.Xkeep, eig_block(J.n, J.k), J.V, J.sig, J.status);
            continue;
        }
        DBuf<double> work(ctx, eig_work_doubles(J.n, J.k));
        eig_topk(ctx, J.G, J.n, J.k, work.get(), J.V, J.sig, J.status, J.status);
    }
}

}  // namespace machb
