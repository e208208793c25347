// Theorem-1 reconstruction bound on the device (reference
// proj/src/bounds.cpp:152-184).
//
// Per mode the bound needs the FULL sigma^2 spectrum of the mode unfolding of
// the original dense tensor and of the sampled tensor, split at the rank into
// a head (|X_(i),r|) and a tail (|X_(i) - X_(i),r|) norm.  The reference takes
// the shorter side's Gram and a full symmetric eigensolver
// (bounds.cpp:41-66, sparse_kernels.cpp:92-101); here the Grams come from the
// kernels the HOSVD already uses (fp64-accumulating DMMA Gram for the dense
// tensor — the TF32 tensor-core Gram's 1e-3 entry error would swamp the tail
// sums — and the deterministic fixed-point sparse row / column Gram), and the
// spectrum from the exact tridiagonal solver in eigenvalues-only mode
// (eig.cu).  The amplitude b = max |x| is one reduction pass.  The closed-form
// parts (p_min, success probability, condition flags) are scalar host code.
#include <algorithm>
#include <cmath>

#include "sparse_ttm.cuh"

namespace machb {

namespace {

template <typename T>
__global__ void maxabs_kernel(const T* __restrict__ x, long long n, double* __restrict__ part) {
    double m = 0.0;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        m = fmax(m, fabs(static_cast<double>(x[i])));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    __shared__ double red[32];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) red[w] = m;
    __syncthreads();
    if (w == 0) {
        m = l < (blockDim.x >> 5) ? red[l] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (l == 0) part[blockIdx.x] = m;
    }
}

constexpr int kMaxSpectrumN = 1700;  // one-CTA tridiagonal solver's shared-memory limit (eig.cu)

void check_spectrum_side(long long n) {
    if (n > kMaxSpectrumN)
        throw Error(MACH_ERR_INTERNAL, "full mode spectrum: shorter side " + std::to_string(n) + " exceeds " +
                                           std::to_string(kMaxSpectrumN));
}

// descending sigma^2 (clamped at 0) of the symmetric n x n Gram G (device)
std::vector<double> gram_spectrum(Ctx* ctx, const double* G, int n) {
    check_spectrum_side(n);
    DBuf<double> work(ctx, eig_work_doubles(n, 1) + static_cast<std::size_t>(8) * n);
    DBuf<double> sig(ctx, static_cast<std::size_t>(n));
    DBuf<int> est(ctx, 3);
    eig_topk(ctx, G, n, n, work.get(), nullptr, sig.get(), est.get());
    std::vector<double> s(static_cast<std::size_t>(n));
    to_host(ctx, s.data(), sig.get(), s.size());
    sync(ctx);
    for (double& v : s) v = v * v;  // sigma -> sigma^2 (sigma = sqrt(max(0, lambda)))
    return s;
}

template <typename T>
std::vector<double> dense_mode_spectrum(Ctx* ctx, const mach_dense* t, int mode) {
    const int rows = t->dims[static_cast<std::size_t>(mode)];
    const long long cols = t->numel / rows;
    if (std::max<long long>(rows, cols) > (1ll << 31) - 1) throw_shape("mode unfolding too wide for the Gram kernel");
    const bool row_side = rows <= cols;
    const int n = row_side ? rows : static_cast<int>(cols);
    check_spectrum_side(n);
    DBuf<T> xm(ctx, static_cast<std::size_t>(t->numel));
    dense_matricize<T, T>(ctx, static_cast<const T*>(t->data), t->dims, mode, xm.get());
    DBuf<double> G(ctx, static_cast<std::size_t>(n) * n);
    if (row_side) gram<T>(ctx, xm.get(), rows, 1, static_cast<int>(cols), rows, G.get());
    else gram<T>(ctx, xm.get(), 1, rows, rows, n, G.get());
    return gram_spectrum(ctx, G.get(), n);
}

template <typename T>
std::vector<double> sparse_mode_spectrum(Ctx* ctx, mach_sparse* X, int mode, const std::vector<int>& ranks,
                                         double normX2) {
    const int rows = X->dims[static_cast<std::size_t>(mode)];
    const long long cols = X->numel / rows;
    const bool row_side = rows <= cols;
    const int n = row_side ? rows : static_cast<int>(std::min<long long>(cols, 1 << 30));
    check_spectrum_side(n);
    DBuf<double> G(ctx, static_cast<std::size_t>(n) * n);
    if (X->nnz == 0) {
        G.zero(ctx);
    } else if (row_side) {
        sparse_row_gram<T>(ctx, X, mode, normX2, G.get());
    } else {
        auto P = get_plan<T>(X, mode, ranks);
        sparse_col_gram<T>(ctx, X, *P, cols, normX2, G.get());
    }
    return gram_spectrum(ctx, G.get(), n);
}

// bounds.cpp:75-88: head / tail norms, both sums smallest-first
void split_spectrum(const std::vector<double>& s2, int r, double* lowrank, double* residual) {
    const int n = static_cast<int>(s2.size());
    const int head = std::min(r, n);
    double acc = 0.0;
    for (int l = n - 1; l >= head; --l) acc += s2[static_cast<std::size_t>(l)];
    *residual = std::sqrt(acc);
    acc = 0.0;
    for (int l = head - 1; l >= 0; --l) acc += s2[static_cast<std::size_t>(l)];
    *lowrank = std::sqrt(acc);
}

double min_probability_core(const std::vector<int>& dims) {  // bounds.cpp:20-35
    double worst = 0.0;
    for (std::size_t j = 0; j < dims.size(); ++j) {
        double log_sum = 0.0, prod = 1.0;
        for (std::size_t k = 0; k < dims.size(); ++k) {
            if (k == j) continue;
            log_sum += std::log(static_cast<double>(dims[k]));
            prod *= static_cast<double>(dims[k]);
        }
        const double base = 8.0 * log_sum;
        worst = std::max(worst, base * base * base * base / prod);
    }
    return worst;
}

}  // namespace

void bound_conditions(const std::vector<int>& dims, double p, mach_bound_report* rep) {  // bounds.cpp:91-116
    *rep = mach_bound_report{};
    rep->p = p;
    rep->p_min = min_probability_core(dims);
    rep->success_probability = 1.0;
    const int d = static_cast<int>(dims.size());
    for (int i = 0; i < d; ++i) {
        double log_sum = 0.0;
        for (int k = 0; k < d; ++k)
            if (k != i) log_sum += std::log(static_cast<double>(dims[static_cast<std::size_t>(k)]));
        rep->success_probability *= 1.0 - std::exp(-19.0 * log_sum);
    }
    double total = 1.0;
    for (int n : dims) total *= static_cast<double>(n);
    rep->dims_large_enough = 1;
    rep->dims_balanced = 1;
    for (int n : dims) {
        if (n < 76) rep->dims_large_enough = 0;
        if (static_cast<double>(n) * static_cast<double>(n) > total) rep->dims_balanced = 0;
    }
    rep->p_above_min = p >= rep->p_min ? 1 : 0;
    rep->conditions_met = (rep->dims_large_enough && rep->dims_balanced && rep->p_above_min) ? 1 : 0;
}

double bound_min_probability(const std::vector<int>& dims) {  // bounds.cpp:145-150
    if (dims.size() < 2) throw_arg("at least two modes required");
    for (int d : dims)
        if (d < 2) throw_arg("every dimension must be >= 2");
    return min_probability_core(dims);
}

template <typename T>
static double maxabs(Ctx* ctx, const T* x, long long n) {
    if (n <= 0) return 0.0;
    const int blocks = static_cast<int>(std::min<long long>(148 * 8, (n + 255) / 256));
    DBuf<double> part(ctx, static_cast<std::size_t>(blocks));
    MB_LAUNCH(ctx, maxabs_kernel<T>, blocks, 256, 0, x, n, part.get());
    std::vector<double> h(static_cast<std::size_t>(blocks));
    to_host(ctx, h.data(), part.get(), h.size());
    sync(ctx);
    return *std::max_element(h.begin(), h.end());
}

template <typename T>
static double sparse_norm2(Ctx* ctx, mach_sparse* X) {
    if (X->norm2 >= 0.0) return X->norm2;
    if (X->nnz == 0) return X->norm2 = 0.0;
    DBuf<double> red(ctx, sumsq_scratch());
    DBuf<double> out(ctx, 1);
    sumsq<T>(ctx, static_cast<const T*>(X->val), X->nnz, red.get(), out.get());
    double v = 0.0;
    to_host(ctx, &v, out.get(), 1);
    sync(ctx);
    return X->norm2 = v;
}

// theorem1_bound (bounds.cpp:152-184); per_mode holds order entries
void theorem1_bound_dev(Ctx* ctx, const mach_dense* x, mach_sparse* xhat, const std::vector<int>& ranks, double p,
                        mach_bound_report* rep, mach_bound_mode* per_mode) {
    if (x->dims != xhat->dims) throw_shape("x and xhat must share dims");  // bounds.cpp:118-130
    if (ranks.size() != x->dims.size()) throw_arg("ranks must name one rank per mode");
    for (std::size_t m = 0; m < ranks.size(); ++m)
        if (ranks[m] < 1 || ranks[m] > x->dims[m])
            throw_arg("rank for mode " + std::to_string(m + 1) + " must be in [1, " + std::to_string(x->dims[m]) + "]");
    if (!(p > 0.0 && p <= 1.0)) throw_arg("p must be in (0, 1]");
    if (x->dtype != xhat->dtype) throw_arg("x and xhat must share a value type");
    const int d = static_cast<int>(x->dims.size());
    bound_conditions(x->dims, p, rep);
    const bool f32 = x->dtype == MACH_F32;
    rep->b = f32 ? maxabs<float>(ctx, static_cast<const float*>(x->data), x->numel)
                 : maxabs<double>(ctx, static_cast<const double*>(x->data), x->numel);
    const double nx2 = f32 ? sparse_norm2<float>(ctx, xhat) : sparse_norm2<double>(ctx, xhat);
    for (int i = 0; i < d; ++i) {
        mach_bound_mode& mode = per_mode[i];
        mode = mach_bound_mode{};
        mode.rank = ranks[static_cast<std::size_t>(i)];
        const std::vector<double> xs = f32 ? dense_mode_spectrum<float>(ctx, x, i) : dense_mode_spectrum<double>(ctx, x, i);
        split_spectrum(xs, mode.rank, &mode.x_lowrank_norm, &mode.x_residual);
        const std::vector<double> hs =
            f32 ? sparse_mode_spectrum<float>(ctx, xhat, i, ranks, nx2) : sparse_mode_spectrum<double>(ctx, xhat, i, ranks, nx2);
        double low = 0.0;
        split_spectrum(hs, mode.rank, &low, &mode.xhat_residual);
    }
    for (int i = 0; i < d; ++i) {
        mach_bound_mode& mode = per_mode[i];
        double others = 1.0, cross = 0.0;
        for (int j = 0; j < d; ++j) {
            if (j == i) continue;
            others *= static_cast<double>(x->dims[static_cast<std::size_t>(j)]);
            cross += per_mode[j].xhat_residual;
        }
        const double ratio = static_cast<double>(mode.rank) / p * others;
        mode.t_i = mode.x_residual + 4.0 * rep->b * std::sqrt(ratio) +
                   4.0 * std::sqrt(mode.x_lowrank_norm * rep->b) * std::pow(ratio, 0.25) + cross;
        rep->t = i == 0 ? mode.t_i : std::min(rep->t, mode.t_i);
    }
}

}  // namespace machb
