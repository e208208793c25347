// Host orchestration of the device Tucker pipeline (reference:
// proj/src/tucker.cpp:18-217 and sampling.cpp:33-47).  All tensors, factors,
// Grams and projections live in HBM; the host only decides dispatch (the
// reference's branch structure) and reads back, once per sweep, the fit and
// the per-mode basis status needed for the stop rule (tucker.cpp:102) and the
// completion warnings (tucker.cpp:34-38).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "sparse_ttm.cuh"

namespace machb {

mach_sparse* sample_dense(const mach_dense* x, double p, std::uint64_t seed);
int core_sumsq_blocks(int rows, int C, int r);  // linalg.cu: grid of core_sumsq (must fit the sumsq_scratch() partials)

std::int64_t checked_size(const std::vector<int>& dims) {
    if (dims.empty()) throw_arg("tensor must have at least one mode");
    std::int64_t n = 1;
    for (int d : dims) {
        if (d < 1) throw_arg("every dimension must be >= 1");
        if (n > INT64_MAX / d) throw_arg("shape product overflows");
        n *= d;
    }
    return n;
}

Split split_at(const std::vector<int>& dims, int mode) {
    if (mode < 0 || mode >= static_cast<int>(dims.size())) throw_arg("mode out of range");
    Split s;
    for (int m = 0; m < mode; ++m) s.inner *= dims[static_cast<std::size_t>(m)];
    for (int m = mode + 1; m < static_cast<int>(dims.size()); ++m) s.outer *= dims[static_cast<std::size_t>(m)];
    s.len = dims[static_cast<std::size_t>(mode)];
    return s;
}

namespace {

constexpr double kDensifyThreshold = 0.25;  // tucker.cpp:69

void check_ranks(const std::vector<int>& dims, const std::vector<int>& ranks) {  // tucker.cpp:20-27
    if (ranks.size() != dims.size()) throw_arg("ranks must name one rank per mode");
    for (std::size_t m = 0; m < dims.size(); ++m)
        if (ranks[m] < 1 || ranks[m] > dims[m])
            throw_arg("rank for mode " + std::to_string(m + 1) + " must be in [1, " + std::to_string(dims[m]) + "]");
}

void check_hooi_config(int max_it, double tol) {  // tucker.cpp:29-32
    if (max_it < 1) throw_arg("max_iterations must be >= 1");
    if (!(tol >= 0.0)) throw_arg("fit_tolerance must be >= 0");
}

std::string completion_warning(int mode, int nr, int requested) {  // tucker.cpp:34-38
    return "mode " + std::to_string(mode + 1) + " matricization has numerical rank " + std::to_string(nr) +
           " below requested rank " + std::to_string(requested) + "; remaining directions were basis-completed";
}

struct Timer {
    Ctx* ctx;
    cudaEvent_t a, b;
    explicit Timer(Ctx* c) : ctx(c) {
        MB_CUDA(cudaEventCreate(&a));
        MB_CUDA(cudaEventCreate(&b));
    }
    ~Timer() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
    void start() { MB_CUDA(cudaEventRecord(a, ctx->stream)); }
    float stop_ms() {
        MB_CUDA(cudaEventRecord(b, ctx->stream));
        MB_CUDA(cudaEventSynchronize(b));
        float ms = 0;
        MB_CUDA(cudaEventElapsedTime(&ms, a, b));
        return ms;
    }
};

// Device state shared by both routes: fp64 factors, basis status per mode,
// scalar slots.
struct FactorSet {
    std::vector<DBuf<double>> U;
    DBuf<double> sv;         // sum of ranks
    DBuf<int> st;            // 3 ints per mode: numerical rank, completed, completion failure
    DBuf<double> scal;       // [0] |X|^2, [1] |G|^2, [2] residual^2
    DBuf<double> red;        // reduction scratch
    void init(Ctx* ctx, const std::vector<int>& dims, const std::vector<int>& ranks) {
        const int d = static_cast<int>(dims.size());
        U.resize(static_cast<std::size_t>(d));
        int rs = 0;
        for (int m = 0; m < d; ++m) {
            U[static_cast<std::size_t>(m)].alloc(ctx, static_cast<std::size_t>(dims[m]) * ranks[m]);
            rs += ranks[m];
        }
        sv.alloc(ctx, rs);
        st.alloc(ctx, 3 * d);
        st.zero(ctx);
        scal.alloc(ctx, 4);
        scal.zero(ctx);
        red.alloc(ctx, sumsq_scratch());
    }
};

// left_singular_basis (linalg.cpp:319-353) of Y (rows x cols, column-major,
// device) into U (rows x k).  Dispatch follows the reference: rows side when
// rows <= cols and k <= cols, otherwise the columns side plus products.  The
// reference switches to subspace iteration above 512; the device Gram +
// selected-eigenpair solver returns the same subspace, so one path serves.
// Warm start (HOOI): per-mode Ritz block kept across sweeps; on the first
// sweep the row side starts from the current factor and the column side from
// Y^T U (one power step from the current factor).
struct Warm {
    DBuf<double> X;   // side x b
    int cols = 0;     // valid warm columns (0 = none)
    int b = 0;
};

// out (C x k) = Y^T U: one warp per entry, lanes over the rows (fixed-order shuffle reduction)
template <typename T>
__global__ void yt_u_kernel(const T* __restrict__ Y, int rows, int C, const double* __restrict__ U, int k,
                            double* __restrict__ out) {
    const long long idx = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (idx >= static_cast<long long>(C) * k) return;
    const int c = static_cast<int>(idx % C), j = static_cast<int>(idx / C);
    const T* y = Y + static_cast<std::size_t>(c) * rows;
    const double* u = U + static_cast<std::size_t>(j) * rows;
    double s = 0.0;
    for (int i = lane; i < rows; i += 32) s += static_cast<double>(y[i]) * u[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[idx] = s;
}

template <typename T>
void lsb_device(Ctx* ctx, const T* Y, int rows, long long cols, int k, double* U, double* sv, int* st,
                Warm* warm = nullptr, const double* Uprev = nullptr) {
    if (rows < 1 || cols < 1) throw_arg("matrix must be nonempty");
    if (k < 1 || k > rows) throw_arg("k must satisfy 1 <= k <= rows");
    const bool row_side = rows <= cols && k <= cols;
    if (!row_side && cols > tall_min_cols() && k <= 24) {
        // column side too wide for a Gram: implicit subspace iteration (tall_basis.cu)
        dense_tall_basis<T>(ctx, Y, rows, cols, k, U, sv, st);
        if (warm) warm->cols = 0;
        return;
    }
    if (!row_side && cols > 16384)
        throw Error(MACH_ERR_INTERNAL, "column-side eigen step wider than 16384 with rank above 24 is not supported");
    const int side = row_side ? rows : static_cast<int>(std::min<long long>(cols, 1 << 30));
    const int kk = row_side ? k : static_cast<int>(std::min<long long>(k, cols));
    DBuf<double> G(ctx, static_cast<std::size_t>(side) * side);
    DBuf<double> V(ctx, static_cast<std::size_t>(side) * kk);
    DBuf<double> sig(ctx, kk);
    DBuf<int> est(ctx, 3);
    if (row_side)
        gram<T>(ctx, Y, rows, 1, static_cast<int>(cols), rows, G.get());
    else
        gram<T>(ctx, Y, 1, rows, rows, side, G.get());
    const int b = eig_block(side, kk);
    const double* X0 = nullptr;
    int x0c = 0;
    DBuf<double> seed;
    if (warm) {
        if (warm->X.n != warm_doubles(side, b)) {
            warm->X.alloc(ctx, warm_doubles(side, b));
            warm->cols = 0;
        }
        warm->b = b;
        if (warm->cols > 0) {
            X0 = warm->X.get();
            x0c = warm->cols;
        } else if (Uprev && subspace_applies(side, kk)) {  // (the exact solver takes no start block)
            if (row_side) {
                X0 = Uprev;
                x0c = kk;
            } else {
                seed.alloc(ctx, static_cast<std::size_t>(side) * kk);
                MB_LAUNCH(ctx, yt_u_kernel<T>, ceil_div(static_cast<long long>(side) * kk * 32, 256), 256, 0, Y, rows, side, Uprev,
                          kk, seed.get());
                X0 = seed.get();
                x0c = kk;
            }
        }
    }
    const bool sub = eig_select(ctx, G.get(), side, kk, X0, x0c, warm ? warm->X.get() : nullptr, b, V.get(), sig.get(),
                                est.get());
    if (warm) warm->cols = sub ? b : 0;
    if (std::getenv("MACH_DEBUG_EIG")) {
        int h[3] = {0, 0, 0};
        to_host(ctx, h, est.get(), 3);
        sync(ctx);
        std::fprintf(stderr, "[eig] side=%d k=%d b=%d subspace=%d converged=%d iters=%d warm=%d\n", side, kk, b,
                     sub ? 1 : 0, h[0], h[2], x0c);
    }
    if (row_side) {
        basis_from_side(ctx, V.get(), sig.get(), rows, k, est.get(), U, sv, st);
    } else {
        DBuf<double> W(ctx, static_cast<std::size_t>(rows) * kk);
        matmul_yv<T>(ctx, Y, rows, side, V.get(), kk, W.get());
        basis_from_products(ctx, W.get(), rows, kk, k, sig.get(), est.get(), U, sv, st);
    }
}

// Row-side left_singular_basis of a dense tensor's mode-m unfolding with the
// Gram formed on the tensor cores (gram_tc.cu) — the dense HOSVD's step
// (tucker.cpp:135-150 -> linalg.cpp:319-353 row side).
inline void lsb_from_gram(Ctx* ctx, const float* x, const std::vector<int>& dims, int m, int k, double* U, double* sv,
                          int* st) {
    const int rows = dims[static_cast<std::size_t>(m)];
    DBuf<double> G(ctx, static_cast<std::size_t>(rows) * rows);
    gram_tc(ctx, x, dims, m, G.get());
    DBuf<double> V(ctx, static_cast<std::size_t>(rows) * k);
    DBuf<double> sig(ctx, k);
    DBuf<int> est(ctx, 3);
    const int b = eig_block(rows, k);
    eig_select(ctx, G.get(), rows, k, nullptr, 0, nullptr, b, V.get(), sig.get(), est.get());
    basis_from_side(ctx, V.get(), sig.get(), rows, k, est.get(), U, sv, st);
}

// Column-side factor update through the fused cluster kernel (mode_basis.cu),
// including the TTM kernel's row-major factor copy.  False when the fused
// route does not apply (the caller then runs lsb_device + the copy).
template <typename T>
bool lsb_fused(Ctx* ctx, const T* Y, int rows, long long cols, int k, double* U, double* sv, int* st, Warm* warm,
               const double* Uprev, T* Ur, int rs) {
    if (!warm || rows < 1 || cols < 1 || k < 1 || k > rows) return false;
    const bool row_side = rows <= cols && k <= cols;
    if (row_side || cols > 4096 || k > cols) return false;
    const int side = static_cast<int>(cols);
    const int b = eig_block(side, k);
    if (warm->X.n != warm_doubles(side, b)) {
        warm->X.alloc(ctx, warm_doubles(side, b));
        warm->cols = 0;
    }
    warm->b = b;
    const double* X0 = nullptr;
    int x0c = 0;
    DBuf<double> seed;
    if (warm->cols > 0) {
        X0 = warm->X.get();
        x0c = warm->cols;
    } else if (Uprev) {
        seed.alloc(ctx, static_cast<std::size_t>(side) * k);
        MB_LAUNCH(ctx, yt_u_kernel<T>, ceil_div(static_cast<long long>(side) * k * 32, 256), 256, 0, Y, rows, side, Uprev, k,
                  seed.get());
        X0 = seed.get();
        x0c = k;
    }
    if (!mode_basis_fused<T>(ctx, Y, rows, side, k, X0, x0c, warm->X.get(), b, U, sv, st, Ur, rs)) return false;
    warm->cols = b;
    return true;
}

// core x_1 U_1 ... x_d U_d into a fresh fp64 dense buffer (tucker.cpp:204-209)
DBuf<double> reconstruct_dev(Ctx* ctx, const double* core, const std::vector<int>& ranks, const std::vector<int>& dims,
                             const std::vector<DBuf<double>>& U) {
    const int d = static_cast<int>(dims.size());
    std::vector<int> cur = ranks;
    DBuf<double> y(ctx, static_cast<std::size_t>(checked_size(ranks)));
    MB_CUDA(cudaMemcpyAsync(y.get(), core, y.n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    for (int m = 0; m < d; ++m) {
        std::vector<int> nd = cur;
        nd[static_cast<std::size_t>(m)] = dims[static_cast<std::size_t>(m)];
        DBuf<double> z(ctx, static_cast<std::size_t>(checked_size(nd)));
        dense_mode_product<double>(ctx, y.get(), cur, m, U[static_cast<std::size_t>(m)].get(), dims[static_cast<std::size_t>(m)],
                                   false, z.get());
        y = std::move(z);
        cur = nd;
    }
    return y;
}

// t x_1 U_1^T ... (skipping `skip`) for a dense device tensor (tucker.cpp:109-118,
// :195-202).  Returns fp64 buffer and its dims.
template <typename T>
DBuf<double> project_dense(Ctx* ctx, const T* x, const std::vector<int>& dims, const std::vector<int>& ranks,
                           const std::vector<DBuf<double>>& U, int skip, std::vector<int>& out_dims) {
    const int d = static_cast<int>(dims.size());
    std::vector<int> cur = dims;
    DBuf<double> y;
    bool first = true;
    for (int m = 0; m < d; ++m) {
        if (m == skip) continue;
        std::vector<int> nd = cur;
        nd[static_cast<std::size_t>(m)] = ranks[static_cast<std::size_t>(m)];
        DBuf<double> z(ctx, static_cast<std::size_t>(checked_size(nd)));
        if (first)
            dense_mode_product<T>(ctx, x, cur, m, U[static_cast<std::size_t>(m)].get(), ranks[static_cast<std::size_t>(m)], true,
                                  z.get());
        else
            dense_mode_product<double>(ctx, y.get(), cur, m, U[static_cast<std::size_t>(m)].get(),
                                       ranks[static_cast<std::size_t>(m)], true, z.get());
        y = std::move(z);
        cur = nd;
        first = false;
    }
    if (first) {  // order-1 tensor: project_except returns t itself
        y.alloc(ctx, static_cast<std::size_t>(checked_size(dims)));
        dense_matricize<T, double>(ctx, x, dims, 0, y.get());
    }
    out_dims = cur;
    return y;
}

// Continue a projection chain: contract y (dims cur, fp64) over every mode
// not in `done` and != skip, ascending (products commute: equal to the
// reference's project_except order up to rounding).
// y0 is read, not consumed (it may be a buffer reused across modes).
DBuf<double> chain_rest(Ctx* ctx, const double* y0, std::vector<int> cur, const std::vector<int>& ranks,
                        const std::vector<DBuf<double>>& U, int skip, const std::vector<bool>& done,
                        std::vector<int>& out_dims) {
    const int d = static_cast<int>(cur.size());
    DBuf<double> y;
    const double* src = y0;
    for (int m = 0; m < d; ++m) {
        if (m == skip || done[static_cast<std::size_t>(m)]) continue;
        std::vector<int> nd = cur;
        nd[static_cast<std::size_t>(m)] = ranks[static_cast<std::size_t>(m)];
        DBuf<double> z(ctx, static_cast<std::size_t>(checked_size(nd)));
        dense_mode_product<double>(ctx, src, cur, m, U[static_cast<std::size_t>(m)].get(),
                                   ranks[static_cast<std::size_t>(m)], true, z.get());
        y = std::move(z);
        src = y.get();
        cur = nd;
    }
    if (src == y0) {  // nothing left to contract: a copy
        y.alloc(ctx, static_cast<std::size_t>(checked_size(cur)));
        MB_CUDA(cudaMemcpyAsync(y.get(), y0, y.n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    }
    out_dims = cur;
    return y;
}

std::vector<double> download(Ctx* ctx, const DBuf<double>& b) {
    std::vector<double> h(b.n);
    to_host(ctx, h.data(), b.get(), b.n);
    return h;
}

// read the per-mode basis status, raise on completion failure, collect warnings
std::vector<std::string> warnings_from(const std::vector<int>& h, const std::vector<int>& ranks,
                                       const std::vector<int>& modes) {
    std::vector<std::string> w;
    for (int m : modes) {
        const int nr = h[3 * m], comp = h[3 * m + 1], fail = h[3 * m + 2];
        if (fail) throw Error(MACH_ERR_CONVERGENCE, "orthonormal completion found no free direction (singular index " +
                                                         std::to_string(fail) + ")", fail);
        if (comp) w.push_back(completion_warning(m, nr, ranks[static_cast<std::size_t>(m)]));
    }
    return w;
}

std::vector<std::string> read_warnings(Ctx* ctx, const DBuf<int>& st, const std::vector<int>& ranks,
                                       const std::vector<int>& modes) {
    const int d = static_cast<int>(ranks.size());
    std::vector<int> h(static_cast<std::size_t>(3 * d));
    to_host(ctx, h.data(), st.get(), h.size());
    sync(ctx);
    return warnings_from(h, ranks, modes);
}

double fit_from(double normX2, double err2) {
    if (normX2 == 0.0) return 1.0;
    return 1.0 - std::sqrt(std::max(0.0, err2)) / std::sqrt(normX2);
}

// ============================================================================
// Sessions: begin() = setup + HOSVD (tucker.cpp:135-169), step() = HOOI sweeps
// with the reference stop rule (hooi_loop, tucker.cpp:80-106), snapshot() =
// TuckerModel.  One-shot hosvd/hooi are thin loops over a session.
// ============================================================================
struct SessionBase {
    Ctx* ctx = nullptr;
    std::vector<int> dims, ranks;
    int d = 0;
    FactorSet fs;
    std::vector<Warm> warm;  // per-mode Ritz blocks carried across sweeps
    std::vector<int> all;
    int iterations = 0;
    double fit = 0.0, prev_fit = 0.0;
    bool stopped = false;
    std::vector<double> sweep_fits, sweep_ms;
    std::vector<std::string> warnings;
    double setup_ms = 0, hosvd_ms = 0, sample_ms = 0;
    virtual ~SessionBase() = default;
    virtual void sweep() = 0;                       // one sweep: all modes, core, fit
    virtual long long ttm_bytes(int) const { return -1; }  // algorithmic bytes of one mode-n TTM launch
    // split sweep for an external reduction between the TTM and the basis
    // (time-slab sharding): Y_(m) of the local nonzeros, then the update
    virtual void* ext_mode_y(int, int*, int*) { throw Error(MACH_ERR_ARGUMENT, "split sweeps need a sparse session"); }
    virtual void ext_mode_update(int) { throw Error(MACH_ERR_ARGUMENT, "split sweeps need a sparse session"); }
    virtual void ext_core_fit() { throw Error(MACH_ERR_ARGUMENT, "split sweeps need a sparse session"); }
    // the starting fit (sweep_fits[0]) from the last mode's Y as it stands
    // (after an external reduction): a shard session started from factors
    void ext_refresh_fit() {
        ext_core_fit();
        prev_fit = fit;
        sweep_fits.assign(1, fit);
    }
    virtual void set_norm2(double) { throw Error(MACH_ERR_ARGUMENT, "split sweeps need a sparse session"); }
    virtual void shard() { throw Error(MACH_ERR_ARGUMENT, "sharded sweeps need a sparse session"); }
    int ext_sweep_end(double tol) {
        ext_core_fit();
        sweep_ms.push_back(0.0);
        sweep_fits.push_back(fit);
        ++iterations;
        if (tol >= 0.0 && fit - prev_fit < (tol < stop_guard ? tol - stop_guard : tol)) stopped = true;  // see step()
        prev_fit = fit;
        return stopped ? 1 : 0;
    }
    virtual const double* core_dev() const = 0;
    double* sv_at(int m) {
        int o = 0;
        for (int q = 0; q < m; ++q) o += ranks[static_cast<std::size_t>(q)];
        return fs.sv.get() + o;
    }
    void init_common(Ctx* c, const std::vector<int>& dm, const std::vector<int>& rk) {
        ctx = c;
        dims = dm;
        ranks = rk;
        d = static_cast<int>(dims.size());
        fs.init(ctx, dims, ranks);
        warm.resize(static_cast<std::size_t>(d));
        all.resize(static_cast<std::size_t>(d));
        for (int m = 0; m < d; ++m) all[static_cast<std::size_t>(m)] = m;
    }
    // run up to n sweeps; returns the number run (stops on the tolerance rule)
    // tol < 0 (session extension, e.g. fixed-length benchmarks) disables the rule
    double stop_guard = 0.0;  // set by the fp32 sessions (1e-6)
    int step(int n, double tol) {
        if (std::isnan(tol)) throw_arg("fit_tolerance must be >= 0");
        const bool rule = tol >= 0.0;
        if (!rule) stopped = false;
        Timer tm(ctx);
        int done = 0;
        for (int s = 0; s < n && !stopped; ++s) {
            tm.start();
            sweep();
            sweep_ms.push_back(tm.stop_ms());
            sweep_fits.push_back(fit);
            ++iterations;
            ++done;
            // tucker.cpp:102 stops on fit - prev < tol.  The fit of an fp32
            // tensor moves by ~1e-8 from rounding once converged, which at
            // tol = 0 stopped runs a sweep before the fp64 reference (whose
            // fit is monotone); tolerances below that noise floor therefore
            // ignore decreases smaller than stop_guard (0 for fp64 tensors).
            const double thr = tol < stop_guard ? tol - stop_guard : tol;
            if (rule && fit - prev_fit < thr) stopped = true;
            prev_fit = fit;
        }
        return done;
    }
    mach_model* snapshot() const {
        auto m = std::make_unique<mach_model>();
        m->order = d;
        m->dims = dims;
        m->ranks = ranks;
        m->core.resize(static_cast<std::size_t>(checked_size(ranks)));
        to_host(ctx, m->core.data(), core_dev(), m->core.size());
        for (int q = 0; q < d; ++q) {
            std::vector<double> f(fs.U[static_cast<std::size_t>(q)].n);
            to_host(ctx, f.data(), fs.U[static_cast<std::size_t>(q)].get(), f.size());
            m->factors.push_back(std::move(f));
        }
        sync(ctx);
        m->iterations = iterations;
        m->fit = fit;
        m->sweep_fits = sweep_fits;
        m->warnings = warnings;
        m->sample_ms = sample_ms;
        m->setup_ms = setup_ms;
        m->hosvd_ms = hosvd_ms;
        m->sweep_ms = sweep_ms;
        return m.release();
    }
};

// ---- dense route: hosvd/hooi(DenseTensor) (tucker.cpp:135-150, :171-180) ----
template <typename T>
struct DenseSession : SessionBase {
    const T* x = nullptr;
    DBuf<T> owned;  // densified copy when coming from a sparse tensor
    long long numel = 0;
    DBuf<double> core;

    // fp32 tensors of supported shape: the streaming first contraction of each
    // projection runs on the tensor cores (ttm_tc.cu, 3xTF32), and the mode-0
    // projection Z0 = X x_0 U_0^T is formed once per sweep (right after U_0's
    // update) and reused by every later mode and the core — a dimension tree
    // with two passes over X per sweep instead of d + 1.
    bool tc0 = false, tc1 = false;
    DBuf<double> z0;
    std::vector<int> z0dims;
    bool z0_valid = false;  // Z0 formed with the current U_0
    void form_z0() {
        z0_valid = true;
        z0dims = dims;
        z0dims[0] = ranks[0];
        z0.alloc(ctx, static_cast<std::size_t>(checked_size(z0dims)));
        if constexpr (std::is_same_v<T, float>) ttm_tc(ctx, x, dims, 0, fs.U[0].get(), ranks[0], z0.get());
    }
    DBuf<double> project_tc(int skip, std::vector<int>& od) {
        std::vector<bool> done(static_cast<std::size_t>(d), false);
        if (skip != 0) {  // from Z0
            done[0] = true;
            return chain_rest(ctx, z0.get(), z0dims, ranks, fs.U, skip, done, od);
        }
        // mode 0's update: contract mode 1 first on the tensor cores
        std::vector<int> cur = dims;
        cur[1] = ranks[1];
        DBuf<double> y(ctx, static_cast<std::size_t>(checked_size(cur)));
        if constexpr (std::is_same_v<T, float>) ttm_tc(ctx, x, dims, 1, fs.U[1].get(), ranks[1], y.get());
        done[1] = true;
        return chain_rest(ctx, y.get(), cur, ranks, fs.U, 0, done, od);
    }
    double core_and_fit() {
        std::vector<int> cd;
        if (tc0) {
            if (!z0_valid) form_z0();  // HOSVD: U_0 final now (a sweep formed it after U_0's update)
            std::vector<bool> done(static_cast<std::size_t>(d), false);
            done[0] = true;
            core = chain_rest(ctx, z0.get(), z0dims, ranks, fs.U, -1, done, cd);
            // |X - X_hat|^2 = |X|^2 - |G|^2 (orthonormal factors, G the projection
            // by the final factors; every term fp64 from exactly represented fp32
            // data and ~2^-22-accurate products); the reference's entrywise form
            // (tucker.cpp:47-50) only when the model is near exact (the
            // difference then cancels: residual below 1e-3 of |X|)
            sumsq<double>(ctx, core.get(), static_cast<long long>(core.n), fs.red.get(), fs.scal.get() + 1);
            double sc[2];
            to_host(ctx, sc, fs.scal.get(), 2);
            sync(ctx);
            const double e2 = sc[0] - sc[1];
            if (e2 > 1e-6 * sc[0]) return fit_from(sc[0], e2);
        } else {
            core = project_dense<T>(ctx, x, dims, ranks, fs.U, -1, cd);
        }
        DBuf<double> rec = reconstruct_dev(ctx, core.get(), ranks, dims, fs.U);
        sumsq_diff<T>(ctx, x, rec.get(), numel, fs.red.get(), fs.scal.get() + 2);
        double sc[3];
        to_host(ctx, sc, fs.scal.get(), 3);
        sync(ctx);
        return fit_from(sc[0], sc[2]);
    }
    void begin(Ctx* c, const T* data, const std::vector<int>& dm, const std::vector<int>& rk) {
        stop_guard = sizeof(T) == 4 ? 1e-6 : 0.0;
        init_common(c, dm, rk);
        x = data;
        numel = checked_size(dims);
        if constexpr (std::is_same_v<T, float>) {
            tc0 = d >= 2 && ttm_tc_applies(dims, 0, ranks[0]);
            tc1 = tc0 && ttm_tc_applies(dims, 1, ranks[1]);
        }
        Timer tm(ctx);
        tm.start();
        sumsq<T>(ctx, x, numel, fs.red.get(), fs.scal.get());
        for (int m = 0; m < d; ++m) {
            const int rows = dims[static_cast<std::size_t>(m)];
            const long long cols = numel / rows;
            if constexpr (std::is_same_v<T, float>) {
                // row side (rows <= cols) with the Gram on the tensor cores,
                // straight from the tensor (no matricised copy)
                if (rows <= cols && ranks[static_cast<std::size_t>(m)] <= cols && gram_tc_applies(dims, m)) {
                    lsb_from_gram(ctx, x, dims, m, ranks[static_cast<std::size_t>(m)], fs.U[static_cast<std::size_t>(m)].get(),
                                  sv_at(m), fs.st.get() + 3 * m);
                    continue;
                }
            }
            if (m == 0) {
                lsb_device<T>(ctx, x, rows, cols, ranks[0], fs.U[0].get(), sv_at(0), fs.st.get());
            } else {
                DBuf<T> xm(ctx, static_cast<std::size_t>(numel));
                dense_matricize<T, T>(ctx, x, dims, m, xm.get());
                lsb_device<T>(ctx, xm.get(), rows, cols, ranks[static_cast<std::size_t>(m)],
                              fs.U[static_cast<std::size_t>(m)].get(), sv_at(m), fs.st.get() + 3 * m);
            }
        }
        warnings = read_warnings(ctx, fs.st, ranks, all);
        fit = prev_fit = core_and_fit();
        hosvd_ms = tm.stop_ms();
        sweep_fits.assign(1, fit);
    }
    void sweep() override {
        z0_valid = false;
        for (int i = 0; i < d; ++i) {
            std::vector<int> yd;
            DBuf<double> y = (tc0 && (i > 0 || tc1)) ? project_tc(i, yd) : project_dense<T>(ctx, x, dims, ranks, fs.U, i, yd);
            const int rows = dims[static_cast<std::size_t>(i)];
            const long long cols = checked_size(yd) / rows;
            DBuf<double> ym(ctx, y.n);
            dense_matricize<double, double>(ctx, y.get(), yd, i, ym.get());
            lsb_device<double>(ctx, ym.get(), rows, cols, ranks[static_cast<std::size_t>(i)],
                               fs.U[static_cast<std::size_t>(i)].get(), sv_at(i), fs.st.get() + 3 * i,
                               &warm[static_cast<std::size_t>(i)], fs.U[static_cast<std::size_t>(i)].get());
            if (i == 0 && tc0) form_z0();  // reused by modes 1.. and the core
        }
        warnings = read_warnings(ctx, fs.st, ranks, all);
        fit = core_and_fit();
    }
    const double* core_dev() const override { return core.get(); }
};

// ---- sparse route: hosvd/hooi(SparseTensor) (tucker.cpp:152-169, :182-193) ----
template <typename T>
struct SparseSession : SessionBase {
    mach_sparse* X = nullptr;
    std::vector<std::shared_ptr<ModePlan>> plans;
    std::vector<DBuf<T>> Ur;
    std::vector<const T*> Urp;
    std::vector<int> C;
    DBuf<T> one, Pbuf, Y;
    DBuf<double> core;
    double normX2 = 0.0;

    void refresh(int m) {
        factor_rowmajor<T>(ctx, fs.U[static_cast<std::size_t>(m)].get(), dims[static_cast<std::size_t>(m)],
                           ranks[static_cast<std::size_t>(m)], ttm_stride(ranks[static_cast<std::size_t>(m)], sizeof(T)),
                           Ur[static_cast<std::size_t>(m)].get());
    }
    // Fibre-sum reuse (d = 3): when mode m's layout has b = m + 1, its TTM
    // also writes every segment's fibre sum F = X x_a U_a, and Y_(m+1) is
    // formed from F and the freshly updated U_m instead of a second pass over
    // X.  F stays valid while U_a is unchanged: a != m, m + 1, and mode a is
    // not updated between the two projections of a sweep.
    DBuf<T> fseg;
    int fseg_for = -1;  // mode whose Y_(.) the current fibre sums give (-1: none)

    // Overlapped sweep (d = 3; MACH_NO_OVERLAP=1 disables).  Mode n's layout
    // takes a = n + 1 and b = n + 2 (mod 3), so its TTM splits into stage 1,
    // F = X x_a U_a (the gathers: ~all the TTM's time), which needs only
    // factors settled before mode n - 1's update, and a short stage 2,
    // Y_(n) = sum F (x) U_b, which needs the U_{n-1} just computed.  Stage 1 of
    // mode n is launched right behind mode n - 1's basis kernel and runs on
    // the SMs that kernel's 16-CTA cluster leaves idle.
    // One fibre-sum buffer per mode: stage 1 of mode n (next sweep) may run
    // before stage 2 of mode n - 1 has finished reading its own buffer
    // (stage 1 does not wait at entry), so the buffers must be distinct; the
    // strict launch order of the stage-2 kernels (pdl_enter_strict) keeps
    // every stage 1 behind the completion of the stage 2 two modes back.
    std::vector<DBuf<T>> Fov;
    bool overlap = false;
    bool split4 = false;    // order 4: stage 1 + the dimension-tree stage 2 (stage2_4way_kernel)
    bool f0_ready = false;  // Fov[0] holds mode 0's stage 1 for the current factors
    // order 4: Fov[m] already holds mode m's stage 1 for the current factors
    // (launched beside the previous mode's unfused basis chain, sweep_body)
    std::vector<char> s1_ready;
    bool prefetch4(int i, int nx) const {
        static const bool off = std::getenv("MACH_NO_SIDE_STAGE1") != nullptr;
        if (off || !split4 || (sharded && !comm_shard)) return false;
        if (plans[static_cast<std::size_t>(nx)]->a == i) return false;  // stage 1 of nx gathers the factor being updated
        const long long rows = dims[static_cast<std::size_t>(i)], cols = C[static_cast<std::size_t>(i)];
        const bool row_side = rows <= cols && ranks[static_cast<std::size_t>(i)] <= cols;
        return row_side || cols > 4096;  // the update is the unfused chain (lsb_fused declines these)
    }
    bool overlap_ok() const { return overlap && (!sharded || comm_shard); }
    // one shard of a time-slab partition with the library's NCCL communicator:
    // every mode's partial Y_(n) is all-reduced in stream before its update
    bool comm_shard = false;
    void reduce_y(int m) {
        if (!comm_shard) return;
        comm_allreduce_sum(ctx, Y.get(), static_cast<std::size_t>(dims[static_cast<std::size_t>(m)]) * C[static_cast<std::size_t>(m)],
                           sizeof(T) == 8);
    }
    bool stage1_waits = false;  // side-stream launch beside an unfused basis chain: wait at entry
    void stage1(int m) {
        // SMs left to the concurrent basis work: the fused 16-CTA cluster is
        // already resident when stage 1 starts (16); the unfused chain's
        // kernels arrive later and its 8-CTA cluster solver needs 8 free SMs
        // inside one GPC (measured at C5: 16 or 32 free SMs leave the cluster
        // waiting for stage 1 to drain, 1.7 ms instead of 0.43; 40 and more do not)
        static const int reserve = std::getenv("MACH_OV_RESERVE") ? std::atoi(std::getenv("MACH_OV_RESERVE")) : 16;
        static const int reserve_side =
            std::getenv("MACH_OV_RESERVE_SIDE") ? std::atoi(std::getenv("MACH_OV_RESERVE_SIDE")) : 40;
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
        sparse_mode_stage1<T>(ctx, *plans[static_cast<std::size_t>(m)], dims, ranks, Urp,
                              Fov[static_cast<std::size_t>(m)].get(),
                              std::max(8, sms - (stage1_waits ? reserve_side : reserve)), !stage1_waits);
    }
    void stage2(int m) {
        auto& P = *plans[static_cast<std::size_t>(m)];
        sparse_mode_stage2<T>(ctx, P, dims, ranks, Fov[static_cast<std::size_t>(m)].get(),
                              Urp[static_cast<std::size_t>(P.b)], Y.get());
    }
    bool fseg_use(int m) const {
        const bool off = std::getenv("MACH_NO_FIBRE_REUSE") != nullptr;
        if (off || d != 3 || m + 1 >= d) return false;
        return plans[static_cast<std::size_t>(m)]->b == m + 1;
    }
    void mode_y(int m) {
        const std::size_t sm = static_cast<std::size_t>(m);
        if (split4) {  // order 4: fibre sums (waiting launch), then the two-level stage 2
            if (!s1_ready[sm]) {  // not prefetched beside the previous mode's basis chain
                int sms = 148;
                cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
                sparse_mode_stage1<T>(ctx, *plans[sm], dims, ranks, Urp, Fov[sm].get(), sms, false);
            }
            s1_ready[sm] = 0;
            sparse_mode_stage2_4way<T>(ctx, *plans[sm], dims, ranks, Fov[sm].get(), Urp, Y.get());
            return;
        }
        if (m >= 1 && fseg_for == m) {
            y_from_segments<T>(ctx, *plans[sm - 1], dims, ranks, fseg.get(), Urp[sm - 1], Y.get());
            return;
        }
        T* fs_out = nullptr;
        const int* fpos = nullptr;
        if (fseg_use(m)) {
            auto& P = *plans[sm];
            build_segment_groups(ctx, P, dims[static_cast<std::size_t>(P.b)]);
            const std::size_t need = static_cast<std::size_t>(P.n_task) * 32 * ranks[static_cast<std::size_t>(P.a)];
            if (fseg.n < need + 16) fseg.alloc(ctx, need + 16);  // slack: bulk copies read aligned supersets
            fs_out = fseg.get();
            fpos = P.seg_pos.get();
        }
        sparse_mode_ttm<T>(ctx, *plans[sm], dims, ranks, Urp, one.get(), Pbuf.get(), Y.get(), fs_out, fpos);
        fseg_for = fs_out ? m + 1 : -1;
    }
    // core from the last mode's projection (which already carries every other
    // updated factor), then fit = 1 - sqrt(|X|^2 - |G|^2)/|X| (orthonormal
    // factors).  Near-exact models take the reference's entrywise residual
    // (tucker.cpp:47-64) instead of the cancelling identity.
    DBuf<unsigned> ticket;  // core_sumsq's last-block ticket (zeroed once)
    void core_device() {
        const int last = d - 1;
        const int rows = dims[static_cast<std::size_t>(last)], cols = C[static_cast<std::size_t>(last)];
        const int r = ranks[static_cast<std::size_t>(last)];
        const long long blocks = core_sumsq_blocks(rows, cols, r);
        if (blocks <= sumsq_scratch()) {  // one launch: core + |core|^2
            if (!ticket.get()) {
                ticket.alloc(ctx, 1);
                ticket.zero(ctx);
            }
            core_sumsq<T>(ctx, Y.get(), rows, cols, fs.U[static_cast<std::size_t>(last)].get(), r, core.get(), fs.red.get(),
                          ticket.get(), fs.scal.get() + 1);
            return;
        }
        core_from_last<T>(ctx, Y.get(), rows, cols, fs.U[static_cast<std::size_t>(last)].get(), r, core.get());
        sumsq<double>(ctx, core.get(), static_cast<long long>(core.n), fs.red.get(), fs.scal.get() + 1);
    }
    double core_and_fit() {
        core_device();
        return fit_host();
    }
    // st_out: if given, the per-mode basis status is read back with the same
    // synchronisation (one host round trip per sweep)
    double fit_host(std::vector<int>* st_out = nullptr) {
        double sc[2];
        to_host(ctx, sc, fs.scal.get(), 2);
        if (st_out) {
            st_out->resize(static_cast<std::size_t>(3 * d));
            to_host(ctx, st_out->data(), fs.st.get(), st_out->size());
        }
        sync(ctx);
        const double e2 = sc[0] - sc[1];
        const double guard = std::is_same<T, double>::value ? 1e-6 : 1e-3;
        if (!sharded && sc[0] > 0.0 && e2 <= guard * sc[0]) {
            DBuf<double> rec = reconstruct_dev(ctx, core.get(), ranks, dims, fs.U);
            scatter_sub<T>(ctx, X, rec.get());
            sumsq<double>(ctx, rec.get(), static_cast<long long>(rec.n), fs.red.get(), fs.scal.get() + 2);
            double ex = 0.0;
            to_host(ctx, &ex, fs.scal.get() + 2, 1);
            sync(ctx);
            return fit_from(sc[0], ex);
        }
        return fit_from(sc[0], e2);
    }
    bool sharded = false;  // |X|^2 set externally; no local entrywise residual guard
    void begin(mach_sparse* sp, const std::vector<int>& rk) {
        want_hosvd = true;
        setup(sp, rk);
        hosvd_init();
    }
    // HOSVD's row-side sparse Grams (atomic-throughput-bound, independent of
    // the TTM layouts) run on a side stream while setup builds the layouts
    // (small kernels and host syncs that leave the GPU mostly idle).
    bool want_hosvd = false;
    std::vector<DBuf<double>> preG;
    cudaStream_t side = nullptr;
    cudaEvent_t grams_done = nullptr;
    // Row Gram X_(m) X_(m)^T of the sampled tensor (sparse_kernels.cpp:60-63).
    // The nonzero route forms every pair of a mode-m fibre (p^2 I_m / 2 pair
    // products per element of the tensor); when that exceeds the dense
    // contraction's work by a margin (C5 p = 0.1: 5.5e9 pairs per mode, 27 ms)
    // the fp32 tensor is densified once (values rounded to TF32 to nearest,
    // so the tensor core's operand truncation is exact and unbiased) and the
    // Gram runs on tcgen05 (gram_tc.cu), read in place for every mode.
    DBuf<float> xdense;
    bool dense_gram_pays(int m) const {
        if constexpr (!std::is_same_v<T, float>) return false;
        const char* e = std::getenv("MACH_SPARSE_GRAM_TC_MIN");  // read per session (tests toggle it); <= 0: off
        const double thr = e ? std::atof(e) : 1.5;
        if (thr <= 0.0 || !gram_tc_applies(dims, m)) return false;
        const double dens = static_cast<double>(X->nnz) / static_cast<double>(X->numel);
        return 0.5 * dens * dens * dims[static_cast<std::size_t>(m)] >= thr;
    }
    void row_gram(int m, double* G) {
        if constexpr (std::is_same_v<T, float>) {
            if (dense_gram_pays(m)) {
                if (!xdense.get()) {
                    xdense.alloc(ctx, static_cast<std::size_t>(X->numel));
                    densify_tf32(ctx, X, xdense.get());
                }
                gram_tc(ctx, xdense.get(), dims, m, G);
                return;
            }
        }
        sparse_row_gram<T>(ctx, X, m, normX2, G);
    }
    void launch_row_grams() {
        if (std::getenv("MACH_NO_ASYNC_GRAMS")) return;  // read per session (tests toggle it)
        preG.clear();
        preG.resize(static_cast<std::size_t>(d));
        bool any = false;
        for (int m = 0; m < d; ++m) {
            const int rows = dims[static_cast<std::size_t>(m)];
            if (static_cast<long long>(rows) <= X->numel / rows) any = true;
        }
        if (!any) return;
        if (!side) MB_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
        if (!grams_done) MB_CUDA(cudaEventCreateWithFlags(&grams_done, cudaEventDisableTiming));
        cudaEvent_t ready;
        MB_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
        MB_CUDA(cudaEventRecord(ready, ctx->stream));  // the sampled tensor and |X|^2 are ready
        MB_CUDA(cudaStreamWaitEvent(side, ready, 0));
        cudaEventDestroy(ready);
        cudaStream_t main = ctx->stream;
        ctx->stream = side;
        try {
            for (int m = 0; m < d; ++m) {
                const int rows = dims[static_cast<std::size_t>(m)];
                if (static_cast<long long>(rows) > X->numel / rows) continue;  // column side: needs the layouts
                preG[static_cast<std::size_t>(m)].alloc(ctx, static_cast<std::size_t>(rows) * rows);
                row_gram(m, preG[static_cast<std::size_t>(m)].get());
            }
            xdense.release();  // (stream-ordered: after the last tensor-core Gram on this stream)
        } catch (...) {
            ctx->stream = main;
            throw;
        }
        ctx->stream = main;
        MB_CUDA(cudaEventRecord(grams_done, side));
    }

    // start from given factors (a replicated HOSVD) instead of computing them
    void begin_from(mach_sparse* sp, const std::vector<int>& rk, const mach_model* init) {
        setup(sp, rk);
        if (init->order != d || init->ranks != ranks || init->dims != dims)
            throw Error(MACH_ERR_SHAPE, "initial model does not match the tensor and ranks");
        for (int m = 0; m < d; ++m) {
            to_device(ctx, fs.U[static_cast<std::size_t>(m)].get(), init->factors[static_cast<std::size_t>(m)].data(),
                      init->factors[static_cast<std::size_t>(m)].size());
            refresh(m);
        }
        fit = prev_fit = init->fit;
        sweep_fits.assign(1, fit);
        warnings = init->warnings;
        fseg_for = -1;
        f0_ready = false;
        std::fill(s1_ready.begin(), s1_ready.end(), 0);
    }
    void setup(mach_sparse* sp, const std::vector<int>& rk) {
        stop_guard = sizeof(T) == 4 ? 1e-6 : 0.0;
        X = sp;
        init_common(sp->ctx, sp->dims, rk);
        Timer tm(ctx);
        // ---- setup: layouts, |X|^2, kernel factor copies, buffers ----
        tm.start();
        plans.resize(static_cast<std::size_t>(d));
        const bool no_overlap = std::getenv("MACH_NO_OVERLAP") != nullptr;  // read per session (tests toggle it)
        overlap = d == 3 && !no_overlap;
        if (overlap) {
            // the overlapped sweep fixes mode n's inner mode to n + 1; when that
            // costs far more than the best inner mode (C4's host mode: 31M
            // one-nonzero fibres over the 64 metrics instead of 64K time
            // fibres), the unconstrained plans run without the overlap
            for (int m = 0; m < d && overlap; ++m) {
                double best = -1.0;
                for (int a = 0; a < d; ++a)
                    if (a != m) {
                        const double c = inner_cost(sp, m, rk, a);
                        if (best < 0 || c < best) best = c;
                    }
                if (inner_cost(sp, m, rk, (m + 1) % 3) > 2.0 * best) overlap = false;
            }
            if (std::getenv("MACH_DEBUG_SETUP")) std::fprintf(stderr, "[setup] overlap %d\n", overlap ? 1 : 0);
        }
        split4 = d == 4;
        sumsq<T>(ctx, static_cast<const T*>(X->val), X->nnz, fs.red.get(), fs.scal.get());
        to_host(ctx, &normX2, fs.scal.get(), 1);
        sync(ctx);
        X->norm2 = normX2;
        if (want_hosvd) launch_row_grams();
        for (int m = 0; m < d; ++m)
            plans[static_cast<std::size_t>(m)] = get_plan<T>(X, m, ranks, overlap ? (m + 1) % 3 : -1);
        Ur.resize(static_cast<std::size_t>(d));
        Urp.resize(static_cast<std::size_t>(d));
        for (int m = 0; m < d; ++m) {
            Ur[static_cast<std::size_t>(m)].alloc(ctx, static_cast<std::size_t>(dims[static_cast<std::size_t>(m)]) *
                                                           ttm_stride(ranks[static_cast<std::size_t>(m)], sizeof(T)));
            Urp[static_cast<std::size_t>(m)] = Ur[static_cast<std::size_t>(m)].get();
        }
        one.alloc(ctx, 16 / sizeof(T));  // one 16-byte unit (bulk-copy granule)
        const T h1[2] = {T(1), T(0)};
        one.zero(ctx);
        to_device(ctx, one.get(), h1, 1);
        long long maxP = 1, maxY = 1;
        C.resize(static_cast<std::size_t>(d));
        for (int m = 0; m < d; ++m) {
            const auto& P = *plans[static_cast<std::size_t>(m)];
            int c = 1;  // Y_(m) columns: product of the other ranks
            for (int q = 0; q < d; ++q)
                if (q != m) c *= ranks[static_cast<std::size_t>(q)];
            C[static_cast<std::size_t>(m)] = c;
            if (!split4) maxP = std::max(maxP, P.n_task * c);
            maxY = std::max(maxY, static_cast<long long>(dims[static_cast<std::size_t>(m)]) * c);
        }
        Pbuf.alloc(ctx, maxP);
        Y.alloc(ctx, maxY);
        if (overlap || split4) {
            Fov.clear();
            Fov.resize(static_cast<std::size_t>(d));  // one fibre-sum buffer per mode (3-way overlap, 4-way prefetch)
            s1_ready.assign(static_cast<std::size_t>(d), 0);
            for (int m = 0; m < d; ++m) {
                const std::size_t need = static_cast<std::size_t>(plans[static_cast<std::size_t>(m)]->n_task) * 32 *
                                             ranks[static_cast<std::size_t>(plans[static_cast<std::size_t>(m)]->a)] + 16;
                auto& B = Fov[static_cast<std::size_t>(m)];  // slack: stage 2 bulk-copies aligned supersets
                if (B.n < need) B.alloc(ctx, need);
            }
        }
        core.alloc(ctx, static_cast<std::size_t>(checked_size(ranks)));
        setup_ms = tm.stop_ms();
    }
    void hosvd_init() {
        Timer tm(ctx);
        // ---- HOSVD: sparse_mode_basis per mode (sparse_kernels.cpp:82-90) ----
        tm.start();
        const long long numel = X->numel;
        // all modes' Grams first, then their eigenproblems in one launch (one
        // CTA each: independent, latency-bound), then the bases
        struct ModeWork {
            bool row = false, tall = false;
            int n, kc;
            DBuf<double> G, V, sig;
            DBuf<int> est;
        };
        std::vector<ModeWork> mw(static_cast<std::size_t>(d));
        std::vector<EigJob> jobs;
        for (int m = 0; m < d; ++m) {
            ModeWork& w = mw[static_cast<std::size_t>(m)];
            const int rows = dims[static_cast<std::size_t>(m)];
            const long long cols = numel / rows;
            const int k = ranks[static_cast<std::size_t>(m)];
            w.row = rows <= cols;
            w.tall = !w.row && cols > tall_min_cols() && k <= 24;
            if (!w.row && !w.tall && cols > 16384)
                throw Error(MACH_ERR_INTERNAL, "column-side sparse HOSVD wider than 16384 with rank above 24 is not supported");
            if (w.tall) continue;  // implicit subspace iteration below, no Gram
            w.n = w.row ? rows : static_cast<int>(cols);
            w.kc = w.row ? k : static_cast<int>(std::min<long long>(k, cols));
            if (w.row && m < static_cast<int>(preG.size()) && preG[static_cast<std::size_t>(m)].get()) {
                w.G = std::move(preG[static_cast<std::size_t>(m)]);  // computed on the side stream during setup
                w.G.s = ctx->stream;  // released in this stream's order, after its last use here
            } else {
                w.G.alloc(ctx, static_cast<std::size_t>(w.n) * w.n);
                if (w.row) row_gram(m, w.G.get());
                else sparse_col_gram<T>(ctx, X, *plans[static_cast<std::size_t>(m)], cols, normX2, w.G.get());
            }
            w.V.alloc(ctx, static_cast<std::size_t>(w.n) * w.kc);
            w.sig.alloc(ctx, w.kc);
            w.est.alloc(ctx, 3);
            jobs.push_back(EigJob{w.G.get(), w.n, w.kc, nullptr, 0, nullptr, w.V.get(), w.sig.get(), w.est.get(),
                                  nullptr, nullptr});
        }
        xdense.release();
        if (grams_done) MB_CUDA(cudaStreamWaitEvent(ctx->stream, grams_done, 0));  // join the side stream's Grams
        if (!jobs.empty()) eig_select_batched(ctx, jobs);
        for (int m = 0; m < d; ++m) {
            ModeWork& w = mw[static_cast<std::size_t>(m)];
            const int rows = dims[static_cast<std::size_t>(m)];
            const int k = ranks[static_cast<std::size_t>(m)];
            if (w.tall) {
                sparse_tall_basis<T>(ctx, X, *plans[static_cast<std::size_t>(m)], k, fs.U[static_cast<std::size_t>(m)].get(),
                                     sv_at(m), fs.st.get() + 3 * m);
            } else if (w.row) {
                basis_from_side(ctx, w.V.get(), w.sig.get(), rows, k, w.est.get(), fs.U[static_cast<std::size_t>(m)].get(),
                                sv_at(m), fs.st.get() + 3 * m);
            } else {
                DBuf<double> W(ctx, static_cast<std::size_t>(rows) * w.kc);
                sparse_times<T>(ctx, X, *plans[static_cast<std::size_t>(m)], w.V.get(), w.n, w.kc, W.get());
                basis_from_products(ctx, W.get(), rows, w.kc, k, w.sig.get(), w.est.get(),
                                    fs.U[static_cast<std::size_t>(m)].get(), sv_at(m), fs.st.get() + 3 * m);
            }
            refresh(m);
        }
        warnings = read_warnings(ctx, fs.st, ranks, all);
        fseg_for = -1;
        f0_ready = false;
        std::fill(s1_ready.begin(), s1_ready.end(), 0);
        mode_y(d - 1);
        fit = prev_fit = core_and_fit();
        hosvd_ms = tm.stop_ms();
        sweep_fits.assign(1, fit);
    }
    // factor update of mode i from Y (tucker.cpp:182-193)
    void mode_update(int i) {
        static const bool nofuse = std::getenv("MACH_NO_FUSED_BASIS") != nullptr;
        const std::size_t si = static_cast<std::size_t>(i);
        if (fseg_for >= 1 && plans[static_cast<std::size_t>(fseg_for - 1)]->a == i) fseg_for = -1;  // F used U_i
        if (plans[0]->a == i) f0_ready = false;  // the prefetched mode-0 stage 1 used U_i
        for (std::size_t m = 0; m < s1_ready.size(); ++m)
            if (plans[m]->a == i) s1_ready[m] = 0;
        if (!nofuse && lsb_fused<T>(ctx, Y.get(), dims[si], C[si], ranks[si], fs.U[si].get(), sv_at(i),
                                    fs.st.get() + 3 * i, &warm[si], fs.U[si].get(), Ur[si].get(),
                                    ttm_stride(ranks[si], sizeof(T))))
            return;
        // Unfused basis chain (Grams too large for the fused cluster: C5's 256
        // columns): the next mode's stage 1, queued in after_basis, needs only
        // factors this update does not touch, so it runs beside the chain on
        // the side stream (fork / join by events: a parallel branch of the
        // sweep graph), on the SMs stage1() does not reserve.
        bool forked = false;
        static const bool no_side = std::getenv("MACH_NO_SIDE_STAGE1") != nullptr;
        if (ctx->after_basis && !no_side) {
            auto cb = std::move(ctx->after_basis);
            ctx->after_basis = nullptr;
            if (!side) MB_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
            if (!ev_fork) MB_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
            if (!ev_join) MB_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
            MB_CUDA(cudaEventRecord(ev_fork, ctx->stream));
            MB_CUDA(cudaStreamWaitEvent(side, ev_fork, 0));
            cudaStream_t main = ctx->stream;
            ctx->stream = side;
            stage1_waits = true;
            try {
                cb();
            } catch (...) {
                ctx->stream = main;
                stage1_waits = false;
                throw;
            }
            ctx->stream = main;
            stage1_waits = false;
            MB_CUDA(cudaEventRecord(ev_join, side));
            forked = true;
        }
        lsb_device<T>(ctx, Y.get(), dims[si], C[si], ranks[si], fs.U[si].get(), sv_at(i), fs.st.get() + 3 * i,
                      &warm[si], fs.U[si].get());
        refresh(i);
        if (forked) MB_CUDA(cudaStreamWaitEvent(ctx->stream, ev_join, 0));
    }
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // Steady-state sweeps (every mode warm-started) are captured once into a
    // CUDA graph and replayed: one launch per sweep instead of ~40 host
    // submissions.  Only the fit read-back (and its rare entrywise-residual
    // guard) stays outside the graph.
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t graph_exec = nullptr;
    std::int64_t graph_launches = 0;
    ~SparseSession() override {
        if (graph_exec) cudaGraphExecDestroy(graph_exec);
        if (graph) cudaGraphDestroy(graph);
        if (grams_done) cudaEventDestroy(grams_done);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
        if (side) cudaStreamDestroy(side);
    }
    bool graph_ok() const {
        static const bool off = std::getenv("MACH_NO_GRAPH") || std::getenv("MACH_DEBUG_EIG") ||
                                std::getenv("MACH_DEBUG_EIG_T") || std::getenv("MACH_TTM_TS");
        if (off || ctx->profile || (sharded && !comm_shard)) return false;
        // the first sweep seeds the warm blocks of the modes that keep them;
        // from the second on every sweep issues the same launches
        return iterations >= 1;
    }
    void sweep_body() {
        if (overlap_ok()) {
            // the next sweep's stage 1 of mode 0 (it needs U_1 of this sweep)
            // runs behind this sweep's last basis kernel
            if (!f0_ready) stage1(0);
            for (int i = 0; i < d; ++i) {
                stage2(i);
                reduce_y(i);
                if (i + 1 < d) ctx->after_basis = [this, i]() { stage1(i + 1); };
                else ctx->after_basis = [this]() { stage1(0); };
                mode_update(i);
                if (ctx->after_basis) {  // the unfused basis path ran: launch it now
                    auto cb = std::move(ctx->after_basis);
                    ctx->after_basis = nullptr;
                    cb();
                }
            }
            f0_ready = true;
            core_device();
            return;
        }
        for (int i = 0; i < d; ++i) {
            mode_y(i);
            reduce_y(i);
            const int nx = (i + 1) % d;
            if (prefetch4(i, nx))  // order 4: the next mode's stage 1 beside this mode's basis chain (side stream)
                ctx->after_basis = [this, nx]() {
                    stage1(nx);
                    s1_ready[static_cast<std::size_t>(nx)] = 1;
                };
            mode_update(i);
            ctx->after_basis = nullptr;  // not taken (side launches off): mode_y runs it in line
        }
        core_device();
    }
    void sweep() override {
        if (graph_ok()) {
            if (!graph_exec) {
                const std::int64_t l0 = ctx->launches;
                MB_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
                try {
                    sweep_body();
                } catch (...) {
                    cudaGraph_t g = nullptr;
                    cudaStreamEndCapture(ctx->stream, &g);
                    if (g) cudaGraphDestroy(g);
                    throw;
                }
                MB_CUDA(cudaStreamEndCapture(ctx->stream, &graph));
                MB_CUDA(cudaGraphInstantiate(&graph_exec, graph, 0));
                graph_launches = ctx->launches - l0;
                ctx->launches = l0;
            }
            MB_CUDA(cudaGraphLaunch(graph_exec, ctx->stream));
            ctx->launches += graph_launches;
        } else {
            sweep_body();
        }
        std::vector<int> st;
        fit = fit_host(&st);
        warnings = warnings_from(st, ranks, all);
    }
    void* ext_mode_y(int m, int* rows, int* cols) override {
        if (m < 0 || m >= d) throw_arg("mode out of range");
        mode_y(m);
        *rows = dims[static_cast<std::size_t>(m)];
        *cols = C[static_cast<std::size_t>(m)];
        return Y.get();
    }
    void ext_mode_update(int m) override {
        if (m < 0 || m >= d) throw_arg("mode out of range");
        mode_update(m);
    }
    void ext_core_fit() override {
        fit = core_and_fit();
        warnings = read_warnings(ctx, fs.st, ranks, all);
    }
    void shard() override {
        if (!ctx->comm) throw Error(MACH_ERR_NCCL, "no communicator on this context (mach_ctx_comm_init)");
        // |X|^2 of this shard's nonzeros, summed over the shards
        DBuf<double> n2(ctx, 1);
        sumsq<T>(ctx, static_cast<const T*>(X->val), X->nnz, fs.red.get(), n2.get());
        comm_allreduce_sum(ctx, n2.get(), 1, true);
        double v = 0.0;
        to_host(ctx, &v, n2.get(), 1);
        sync(ctx);
        set_norm2(v);
        comm_shard = true;
        // the sweep graph (if any) was captured without the exchange
        if (graph_exec) { cudaGraphExecDestroy(graph_exec); graph_exec = nullptr; }
        if (graph) { cudaGraphDestroy(graph); graph = nullptr; }
        f0_ready = false;
        std::fill(s1_ready.begin(), s1_ready.end(), 0);
    }
    void set_norm2(double v) override {
        if (!(v >= 0.0)) throw_arg("norm2 must be >= 0");
        normX2 = v;
        sharded = true;
        to_device(ctx, fs.scal.get(), &v, 1);
    }
    const double* core_dev() const override { return core.get(); }
    // bytes one mode-n TTM launch must move: per nonzero the inner index and
    // the value, per task its record and descriptor, per task the partial
    // row block it writes (the factor rows come from L2, not counted)
    // algorithmic bytes of mode m's TTM launch in a steady sweep; -1 when the
    // mode runs no TTM (its Y_(m) comes from the previous mode's fibre sums)
    long long ttm_bytes(int m) const override {
        if (m < 0 || m >= d || !plans[static_cast<std::size_t>(m)]) return -1;
        const ModePlan& P = *plans[static_cast<std::size_t>(m)];
        const long long nnz = X->nnz;
        if (overlap_ok() || split4)  // stage 1: nonzeros + task records in, fibre sums (every segment slot) out
            return nnz * ((P.ia16 ? 2 : 4) + static_cast<long long>(sizeof(T))) +
                   P.n_task * (static_cast<long long>(kDesc * sizeof(int2) + sizeof(TtmTask)) +
                               32 * ranks[static_cast<std::size_t>(P.a)] * static_cast<long long>(sizeof(T)));
        if (m >= 1 && fseg_use(m - 1)) return -1;
        long long b = nnz * ((P.ia16 ? 2 : 4) + static_cast<long long>(sizeof(T))) +
                      P.n_task * (static_cast<long long>(kDesc * sizeof(int2) + sizeof(TtmTask)) +
                                  static_cast<long long>(C[static_cast<std::size_t>(m)]) * static_cast<long long>(sizeof(T)));
        if (fseg_use(m) && P.n_seg > 0)  // + the fibre sums written (and their positions read)
            b += P.n_task * 32 * static_cast<long long>(sizeof(int)) +
                 P.n_seg * ranks[static_cast<std::size_t>(P.a)] * static_cast<long long>(sizeof(T));
        return b;
    }
};

}  // namespace

// ---- session factory + one-shot entry points used by the C ABI ------------
void* session_sparse(mach_sparse* X, const std::vector<int>& ranks) {
    check_ranks(X->dims, ranks);
    Ctx* ctx = X->ctx;
    const bool dense_enough = static_cast<double>(X->nnz) >= kDensifyThreshold * static_cast<double>(X->numel);
    if (dense_enough || !sparse_fast_path_ok(X->dims, ranks)) {
        // tucker.cpp:154-155 / :185-186 densify switch; also the general-shape route
        if (X->dtype == MACH_F32) {
            auto s = std::make_unique<DenseSession<float>>();
            s->owned.alloc(ctx, static_cast<std::size_t>(X->numel));
            densify<float>(ctx, X, s->owned.get());
            s->begin(ctx, s->owned.get(), X->dims, ranks);
            return static_cast<SessionBase*>(s.release());
        }
        auto s = std::make_unique<DenseSession<double>>();
        s->owned.alloc(ctx, static_cast<std::size_t>(X->numel));
        densify<double>(ctx, X, s->owned.get());
        s->begin(ctx, s->owned.get(), X->dims, ranks);
        return static_cast<SessionBase*>(s.release());
    }
    if (X->dtype == MACH_F32) {
        auto s = std::make_unique<SparseSession<float>>();
        s->begin(X, ranks);
        return static_cast<SessionBase*>(s.release());
    }
    auto s = std::make_unique<SparseSession<double>>();
    s->begin(X, ranks);
    return static_cast<SessionBase*>(s.release());
}

void* session_sparse_from(mach_sparse* X, const std::vector<int>& ranks, const mach_model* init) {
    check_ranks(X->dims, ranks);
    if (!sparse_fast_path_ok(X->dims, ranks))
        throw Error(MACH_ERR_ARGUMENT, "split sweeps need the sparse route (order <= 4, ranks <= 32)");
    if (X->dtype == MACH_F32) {
        auto s = std::make_unique<SparseSession<float>>();
        s->begin_from(X, ranks, init);
        return static_cast<SessionBase*>(s.release());
    }
    auto s = std::make_unique<SparseSession<double>>();
    s->begin_from(X, ranks, init);
    return static_cast<SessionBase*>(s.release());
}

void* session_dense(const mach_dense* X, const std::vector<int>& ranks) {
    check_ranks(X->dims, ranks);
    if (X->dtype == MACH_F32) {
        auto s = std::make_unique<DenseSession<float>>();
        s->begin(X->ctx, static_cast<const float*>(X->data), X->dims, ranks);
        return static_cast<SessionBase*>(s.release());
    }
    auto s = std::make_unique<DenseSession<double>>();
    s->begin(X->ctx, static_cast<const double*>(X->data), X->dims, ranks);
    return static_cast<SessionBase*>(s.release());
}

static SessionBase* S(void* p) { return static_cast<SessionBase*>(p); }
int session_step(void* s, int n, double tol) { return S(s)->step(n, tol); }
mach_model* session_snapshot(void* s) { return S(s)->snapshot(); }
void session_free(void* s) { delete S(s); }
void session_set_sample_ms(void* s, double ms) { S(s)->sample_ms = ms; }
int session_iterations(void* s) { return S(s)->iterations; }
double session_fit(void* s) { return S(s)->fit; }
bool session_stopped(void* s) { return S(s)->stopped; }
long long session_ttm_bytes(void* s, int m) { return S(s)->ttm_bytes(m); }
void* session_mode_y(void* s, int m, int* rows, int* cols) { return S(s)->ext_mode_y(m, rows, cols); }
void session_mode_update(void* s, int m) { S(s)->ext_mode_update(m); }
int session_sweep_end(void* s, double tol) { return S(s)->ext_sweep_end(tol); }
void session_set_norm2(void* s, double v) { S(s)->set_norm2(v); }
void session_shard(void* s) { S(s)->shard(); }

void session_refresh_fit(void* s) { S(s)->ext_refresh_fit(); }

// Row Gram X_(n) X_(n)^T of a sampled tensor into host memory (n x n,
// column-major).  With time-slab shards the columns of X_(n), n != last, are
// partitioned by the slabs, so the shards' Grams add up to the full one
// (partial Grams + all-reduce).
void sparse_row_gram_host(Ctx* ctx, const mach_sparse* X, int n, double* host) {
    if (n < 0 || n >= static_cast<int>(X->dims.size())) throw_arg("mode out of range");
    const int rows = X->dims[static_cast<std::size_t>(n)];
    if (static_cast<long long>(rows) > X->numel / rows) throw_arg("the row Gram needs rows <= columns of the unfolding");
    DBuf<double> G(ctx, static_cast<std::size_t>(rows) * rows);
    if (X->nnz == 0) {
        G.zero(ctx);
    } else {
        DBuf<double> red(ctx, sumsq_scratch()), n2(ctx, 1);
        double norm2 = 0.0;
        if (X->dtype == MACH_F32) sumsq<float>(ctx, static_cast<const float*>(X->val), X->nnz, red.get(), n2.get());
        else sumsq<double>(ctx, static_cast<const double*>(X->val), X->nnz, red.get(), n2.get());
        to_host(ctx, &norm2, n2.get(), 1);
        sync(ctx);
        if (X->dtype == MACH_F32) sparse_row_gram<float>(ctx, X, n, norm2, G.get());
        else sparse_row_gram<double>(ctx, X, n, norm2, G.get());
    }
    to_host(ctx, host, G.get(), static_cast<std::size_t>(rows) * rows);
    sync(ctx);
}

// HOSVD factors from full row Grams (host, one per mode): the eigen step and
// the basis of sparse_mode_basis's row side (sparse_kernels.cpp:82-84 ->
// linalg.cpp:106-120).  The model carries the factors and warnings; its core
// and fit are left to the caller (mach_hooi_begin_from + mach_hooi_refresh_fit).
mach_model* hosvd_from_grams(Ctx* ctx, const std::vector<int>& dims, const std::vector<int>& ranks,
                             const double* const* grams) {
    check_ranks(dims, ranks);
    const int d = static_cast<int>(dims.size());
    FactorSet fs;
    fs.init(ctx, dims, ranks);
    struct ModeWork {
        DBuf<double> G, V, sig;
        DBuf<int> est;
    };
    std::vector<ModeWork> mw(static_cast<std::size_t>(d));
    std::vector<EigJob> jobs;
    for (int m = 0; m < d; ++m) {
        const int n = dims[static_cast<std::size_t>(m)], k = ranks[static_cast<std::size_t>(m)];
        if (!grams[m]) throw_arg("a Gram is missing");
        ModeWork& w = mw[static_cast<std::size_t>(m)];
        w.G.alloc(ctx, static_cast<std::size_t>(n) * n);
        to_device(ctx, w.G.get(), grams[m], static_cast<std::size_t>(n) * n);
        w.V.alloc(ctx, static_cast<std::size_t>(n) * k);
        w.sig.alloc(ctx, k);
        w.est.alloc(ctx, 3);
        jobs.push_back(EigJob{w.G.get(), n, k, nullptr, 0, nullptr, w.V.get(), w.sig.get(), w.est.get(), nullptr, nullptr});
    }
    eig_select_batched(ctx, jobs);
    int so = 0;
    for (int m = 0; m < d; ++m) {
        ModeWork& w = mw[static_cast<std::size_t>(m)];
        basis_from_side(ctx, w.V.get(), w.sig.get(), dims[static_cast<std::size_t>(m)], ranks[static_cast<std::size_t>(m)],
                        w.est.get(), fs.U[static_cast<std::size_t>(m)].get(), fs.sv.get() + so, fs.st.get() + 3 * m);
        so += ranks[static_cast<std::size_t>(m)];
    }
    auto out = std::make_unique<mach_model>();
    out->order = d;
    out->dims = dims;
    out->ranks = ranks;
    out->core.assign(static_cast<std::size_t>(checked_size(ranks)), 0.0);
    for (int m = 0; m < d; ++m) {
        std::vector<double> f(fs.U[static_cast<std::size_t>(m)].n);
        to_host(ctx, f.data(), fs.U[static_cast<std::size_t>(m)].get(), f.size());
        out->factors.push_back(std::move(f));
    }
    std::vector<int> all(static_cast<std::size_t>(d));
    for (int m = 0; m < d; ++m) all[static_cast<std::size_t>(m)] = m;
    out->warnings = read_warnings(ctx, fs.st, ranks, all);
    sync(ctx);
    out->sweep_fits.assign(1, 0.0);
    return out.release();
}

mach_model* tucker_sparse(mach_sparse* X, const std::vector<int>& ranks, bool do_hooi, int max_it, double tol) {
    check_ranks(X->dims, ranks);
    if (do_hooi) check_hooi_config(max_it, tol);
    std::unique_ptr<SessionBase> s(S(session_sparse(X, ranks)));
    if (do_hooi) s->step(max_it, tol);
    return s->snapshot();
}

mach_model* tucker_dense(const mach_dense* X, const std::vector<int>& ranks, bool do_hooi, int max_it, double tol) {
    check_ranks(X->dims, ranks);
    if (do_hooi) check_hooi_config(max_it, tol);
    std::unique_ptr<SessionBase> s(S(session_dense(X, ranks)));
    if (do_hooi) s->step(max_it, tol);
    return s->snapshot();
}


// accuracy (tucker.cpp:211-217) against a device tensor
double accuracy_dev(const mach_dense* t, const mach_model* m) {
    Ctx* ctx = t->ctx;
    const int d = m->order;
    DBuf<double> red(ctx, sumsq_scratch()), scal(ctx, 2);
    if (t->dtype == MACH_F32) sumsq<float>(ctx, static_cast<const float*>(t->data), t->numel, red.get(), scal.get());
    else sumsq<double>(ctx, static_cast<const double*>(t->data), t->numel, red.get(), scal.get());
    double n2 = 0;
    to_host(ctx, &n2, scal.get(), 1);
    sync(ctx);
    if (n2 == 0.0) throw_arg("accuracy needs a reference tensor with nonzero norm");
    if (m->dims != t->dims) throw_shape("model reconstructs to a different shape");
    std::vector<DBuf<double>> U(static_cast<std::size_t>(d));
    for (int q = 0; q < d; ++q) {
        U[static_cast<std::size_t>(q)].alloc(ctx, m->factors[static_cast<std::size_t>(q)].size());
        to_device(ctx, U[static_cast<std::size_t>(q)].get(), m->factors[static_cast<std::size_t>(q)].data(),
                  m->factors[static_cast<std::size_t>(q)].size());
    }
    DBuf<double> core(ctx, m->core.size());
    to_device(ctx, core.get(), m->core.data(), m->core.size());
    // fused reconstruct-and-compare (metrics.cu): no dense reconstruction
    std::vector<const double*> up;
    for (auto& u : U) up.push_back(u.get());
    const double e2 = t->dtype == MACH_F32
                          ? residual2_fused<float>(ctx, static_cast<const float*>(t->data), t->dims, m->ranks, core.get(), up)
                          : residual2_fused<double>(ctx, static_cast<const double*>(t->data), t->dims, m->ranks, core.get(), up);
    return 1.0 - std::sqrt(e2) / std::sqrt(n2);
}

mach_dense* reconstruct_model(Ctx* ctx, const mach_model* m) {
    const int d = m->order;
    std::vector<DBuf<double>> U(static_cast<std::size_t>(d));
    for (int q = 0; q < d; ++q) {
        U[static_cast<std::size_t>(q)].alloc(ctx, m->factors[static_cast<std::size_t>(q)].size());
        to_device(ctx, U[static_cast<std::size_t>(q)].get(), m->factors[static_cast<std::size_t>(q)].data(),
                  m->factors[static_cast<std::size_t>(q)].size());
    }
    DBuf<double> core(ctx, m->core.size());
    to_device(ctx, core.get(), m->core.data(), m->core.size());
    DBuf<double> rec = reconstruct_dev(ctx, core.get(), m->ranks, m->dims, U);
    auto out = std::make_unique<mach_dense>();
    out->ctx = ctx;
    out->dtype = MACH_F64;
    out->dims = m->dims;
    out->numel = checked_size(m->dims);
    out->data = rec.p;
    out->owns = true;
    rec.p = nullptr;
    rec.n = 0;
    return out.release();
}

// left_singular_basis on a host matrix (linalg.cpp:319-353)
void lsb_host(Ctx* ctx, int rows, int cols, const double* a, int k, double* basis, double* sv, int* nr, int* completed) {
    if (rows < 1 || cols < 1) throw_arg("matrix must be nonempty");
    if (k < 1 || k > rows) throw_arg("k must satisfy 1 <= k <= rows");
    DBuf<double> A(ctx, static_cast<std::size_t>(rows) * cols), U(ctx, static_cast<std::size_t>(rows) * k), s(ctx, k);
    DBuf<int> st(ctx, 3);
    st.zero(ctx);
    to_device(ctx, A.get(), a, A.n);
    lsb_device<double>(ctx, A.get(), rows, cols, k, U.get(), s.get(), st.get());
    int h[3];
    to_host(ctx, basis, U.get(), U.n);
    to_host(ctx, sv, s.get(), s.n);
    to_host(ctx, h, st.get(), 3);
    sync(ctx);
    if (h[2]) throw Error(MACH_ERR_CONVERGENCE, "orthonormal completion found no free direction (singular index " +
                                                    std::to_string(h[2]) + ")", h[2]);
    *nr = h[0];
    *completed = h[1];
}

// mode_product (tensor.cpp:224-259) with a host matrix m (rows x cols = J x len)
mach_dense* mode_product_dev(Ctx* ctx, const mach_dense* t, const mach_sparse* s, int rows, int cols, const double* m,
                             int mode) {
    const std::vector<int>& dims = t ? t->dims : s->dims;
    const Split sp = split_at(dims, mode);
    if (cols != sp.len) throw_shape("mode_product inner dimensions disagree");
    std::vector<int> od = dims;
    od[static_cast<std::size_t>(mode)] = rows;
    // device M as U (len x J) so that M(q, r) = U[r + len*q] = m(q, r) with transpose=true
    std::vector<double> ut(static_cast<std::size_t>(rows) * cols);
    for (int q = 0; q < rows; ++q)
        for (int r = 0; r < cols; ++r) ut[static_cast<std::size_t>(r) + static_cast<std::size_t>(cols) * q] = m[q + static_cast<std::size_t>(rows) * r];
    DBuf<double> U(ctx, ut.size());
    to_device(ctx, U.get(), ut.data(), ut.size());
    auto out = std::make_unique<mach_dense>();
    out->ctx = ctx;
    out->dtype = MACH_F64;
    out->dims = od;
    out->numel = checked_size(od);
    DBuf<double> y(ctx, static_cast<std::size_t>(out->numel));
    if (t) {
        // fp32 tensors stream through the tensor cores (3xTF32, ~1e-7 relative)
        if (t->dtype == MACH_F32 && ttm_tc_applies(dims, mode, rows))
            ttm_tc(ctx, static_cast<const float*>(t->data), dims, mode, U.get(), rows, y.get());
        else if (t->dtype == MACH_F32) dense_mode_product<float>(ctx, static_cast<const float*>(t->data), dims, mode, U.get(), rows, true, y.get());
        else dense_mode_product<double>(ctx, static_cast<const double*>(t->data), dims, mode, U.get(), rows, true, y.get());
    } else {
        // straight from the nonzeros (sparse_mode_product.cu), no densified copy
        DBuf<double> Md(ctx, static_cast<std::size_t>(rows) * cols);
        to_device(ctx, Md.get(), m, Md.n);
        sparse_mode_product(ctx, s, mode, Md.get(), rows, y.get());
    }
    sync(ctx);
    out->data = y.p;
    y.p = nullptr;
    y.n = 0;
    return out.release();
}

}  // namespace machb
