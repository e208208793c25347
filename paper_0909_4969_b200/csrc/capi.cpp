// C ABI of libmach_b200 (include/mach_b200.h).  Every entry point catches,
// maps the error to a mach_status and stores the message thread-locally; no
// exception crosses the boundary.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "common.cuh"
#include "sparse_ttm.cuh"

namespace machb {
mach_sparse* sample_dense(const mach_dense* x, double p, std::uint64_t seed);
mach_sparse* sample_slab(const mach_dense* x, const std::vector<int>& gdims, std::int64_t offset, double p,
                         std::uint64_t seed);
mach_model* tucker_sparse(mach_sparse* X, const std::vector<int>& ranks, bool do_hooi, int max_it, double tol);
mach_model* tucker_dense(const mach_dense* X, const std::vector<int>& ranks, bool do_hooi, int max_it, double tol);
double accuracy_dev(const mach_dense* t, const mach_model* m);
mach_dense* reconstruct_model(Ctx* ctx, const mach_model* m);
void lsb_host(Ctx* ctx, int rows, int cols, const double* a, int k, double* basis, double* sv, int* nr, int* completed);
mach_dense* mode_product_dev(Ctx* ctx, const mach_dense* t, const mach_sparse* s, int rows, int cols, const double* m,
                             int mode);
mach_sparse* sparse_from_host(Ctx* ctx, int dtype, const std::vector<int>& dims, std::int64_t nnz, const std::int64_t* idx,
                              const double* vals);
void sparse_to_host(const mach_sparse* s, std::int64_t* idx, double* vals);
void check_finite_upload(Ctx* ctx, int dtype, const void* dev, std::int64_t n);
}  // namespace machb

using namespace machb;

namespace {
thread_local std::string g_err;
thread_local int g_err_index = 0;

template <typename F>
mach_status guard(F&& f) {
    try {
        f();
        return MACH_OK;
    } catch (const Error& e) {
        g_err = e.what();
        g_err_index = e.index;
        return static_cast<mach_status>(e.code);
    } catch (const std::bad_alloc& e) {
        g_err = e.what();
        return MACH_ERR_OOM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return MACH_ERR_INTERNAL;
    }
}

std::vector<int> dims_of(int order, const int* dims) {
    if (order < 1 || !dims) throw_arg("tensor must have at least one mode");
    return std::vector<int>(dims, dims + order);
}

void need(const void* p, const char* what) {
    if (!p) throw_arg(std::string(what) + " must not be null");
}

// Makes the handle's device current for the call and restores the caller's
// afterwards: handles on different GPUs can be used from one thread, and a
// caller (e.g. torch) may have switched devices in between.
struct DevGuard {
    int prev = -1, dev = -1;
    explicit DevGuard(int d) : dev(d) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) MB_CUDA(cudaSetDevice(dev));
    }
    ~DevGuard() {
        if (prev >= 0 && prev != dev) cudaSetDevice(prev);
    }
};
}  // namespace

extern "C" {

const char* mach_last_error(void) { return g_err.c_str(); }
int mach_last_error_index(void) { return g_err_index; }
const char* mach_version(void) { return "mach-b200 0.1 (sm_100a)"; }

mach_status mach_ctx_create(int device, mach_ctx** out) {
    return guard([&] {
        need(out, "out");
        auto c = std::make_unique<mach_ctx>();
        c->c.device = device;
        MB_CUDA(cudaSetDevice(device));
        MB_CUDA(cudaStreamCreateWithFlags(&c->c.stream, cudaStreamNonBlocking));
        c->c.own_stream = true;
        // keep freed stream-ordered allocations cached in the device pool
        // (the default threshold returns them to the driver at every sync,
        // so each job would pay for fresh allocations)
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            std::uint64_t keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        *out = c.release();
    });
}

mach_status mach_ctx_destroy(mach_ctx* ctx) {
    return guard([&] {
        if (!ctx) return;
        cudaStreamSynchronize(ctx->c.stream);
        comm_destroy(&ctx->c);
        if (ctx->c.own_stream) cudaStreamDestroy(ctx->c.stream);
        delete ctx;
    });
}

mach_status mach_ctx_set_stream(mach_ctx* ctx, void* stream) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        MB_CUDA(cudaStreamSynchronize(ctx->c.stream));
        if (ctx->c.own_stream) cudaStreamDestroy(ctx->c.stream);
        if (stream) {
            ctx->c.stream = static_cast<cudaStream_t>(stream);
            ctx->c.own_stream = false;
        } else {
            MB_CUDA(cudaStreamCreateWithFlags(&ctx->c.stream, cudaStreamNonBlocking));
            ctx->c.own_stream = true;
        }
    });
}

mach_status mach_ctx_synchronize(mach_ctx* ctx) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        sync(&ctx->c);
    });
}

mach_status mach_ctx_launch_count(mach_ctx* ctx, int64_t* out) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        *out = ctx->c.launches;
    });
}

// ---- dense ----
mach_status mach_dense_upload(mach_ctx* ctx, mach_dtype dtype, int order, const int* dims, const void* host,
                              mach_dense** out) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(out, "out");
        auto t = std::make_unique<mach_dense>();
        t->ctx = &ctx->c;
        t->dtype = dtype;
        t->dims = dims_of(order, dims);
        t->numel = checked_size(t->dims);
        need(host, "host");
        const std::size_t bytes = static_cast<std::size_t>(t->numel) * dtype_size(dtype);
        MB_CUDA(cudaMallocAsync(&t->data, bytes, ctx->c.stream));
        MB_CUDA(cudaMemcpyAsync(t->data, host, bytes, cudaMemcpyHostToDevice, ctx->c.stream));
        t->owns = true;
        check_finite_upload(&ctx->c, dtype, t->data, t->numel);
        *out = t.release();
    });
}

mach_status mach_dense_wrap(mach_ctx* ctx, mach_dtype dtype, int order, const int* dims, void* dev, mach_dense** out) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(out, "out");
        need(dev, "device_ptr");
        auto t = std::make_unique<mach_dense>();
        t->ctx = &ctx->c;
        t->dtype = dtype;
        t->dims = dims_of(order, dims);
        t->numel = checked_size(t->dims);
        t->data = dev;
        t->owns = false;
        *out = t.release();
    });
}

mach_status mach_dense_download(const mach_dense* t, void* host) {
    return guard([&] {
        need(t, "tensor");
        DevGuard dg_(t->ctx->device);
        need(host, "host");
        MB_CUDA(cudaMemcpyAsync(host, t->data, static_cast<std::size_t>(t->numel) * dtype_size(t->dtype),
                                cudaMemcpyDeviceToHost, t->ctx->stream));
        sync(t->ctx);
    });
}

mach_status mach_dense_free(mach_dense* t) {
    return guard([&] {
        if (!t) return;
        if (t->owns && t->data) cudaFreeAsync(t->data, t->ctx->stream);
        delete t;
    });
}

// ---- sampler ----
mach_status mach_sparsify(mach_ctx* ctx, const mach_dense* x, double p, uint64_t seed, mach_sparse** out) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(x, "tensor");
        need(out, "out");
        *out = sample_dense(x, p, seed);
    });
}

mach_status mach_sparsify_slab(mach_ctx* ctx, const mach_dense* slab, int order, const int* global_dims,
                               int64_t offset, double p, uint64_t seed, mach_sparse** out) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(slab, "slab");
        need(out, "out");
        *out = sample_slab(slab, dims_of(order, global_dims), offset, p, seed);
    });
}

mach_status mach_sparse_device_view(const mach_sparse* s, void** idx, void** vals, int* idx_bytes) {
    return guard([&] {
        need(s, "tensor");
        DevGuard dg_(s->ctx->device);
        if (idx) *idx = s->idx;
        if (vals) *vals = s->val;
        if (idx_bytes) *idx_bytes = s->idx64 ? 8 : 4;
    });
}

mach_status mach_sparse_from_device(mach_ctx* ctx, mach_dtype dtype, int order, const int* dims, int64_t nnz,
                                    const void* idx, const void* vals, mach_sparse** out) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(out, "out");
        if (nnz < 0) throw_arg("nnz must be >= 0");
        auto t = std::make_unique<mach_sparse>();
        t->ctx = &ctx->c;
        t->dtype = dtype;
        t->dims = dims_of(order, dims);
        t->numel = checked_size(t->dims);
        t->idx64 = t->numel > 0xFFFFFFFFll;
        t->nnz = nnz;
        if (nnz > 0) {
            need(idx, "idx");
            need(vals, "vals");
            const std::size_t ib = static_cast<std::size_t>(nnz) * (t->idx64 ? 8 : 4);
            const std::size_t vb = static_cast<std::size_t>(nnz) * (dtype == MACH_F32 ? 4 : 8);
            MB_CUDA(cudaMallocAsync(&t->idx, ib, ctx->c.stream));
            MB_CUDA(cudaMallocAsync(&t->val, vb, ctx->c.stream));
            MB_CUDA(cudaMemcpyAsync(t->idx, idx, ib, cudaMemcpyDeviceToDevice, ctx->c.stream));
            MB_CUDA(cudaMemcpyAsync(t->val, vals, vb, cudaMemcpyDeviceToDevice, ctx->c.stream));
        }
        *out = t.release();
    });
}

mach_status mach_sparsify_host(mach_ctx* ctx, mach_dtype dtype, int order, const int* dims, const void* host_x, double p,
                               uint64_t seed, int64_t* nnz_out, int64_t** idx_out, double** val_out) {
    mach_dense* x = nullptr;
    mach_sparse* s = nullptr;
    mach_status st = mach_dense_upload(ctx, dtype, order, dims, host_x, &x);
    if (st != MACH_OK) return st;
    st = mach_sparsify(ctx, x, p, seed, &s);
    if (st == MACH_OK) {
        st = guard([&] {
            *nnz_out = s->nnz;
            *idx_out = static_cast<int64_t*>(std::malloc(static_cast<std::size_t>(std::max<int64_t>(1, s->nnz)) * 8));
            *val_out = static_cast<double*>(std::malloc(static_cast<std::size_t>(std::max<int64_t>(1, s->nnz)) * 8));
            sparse_to_host(s, *idx_out, *val_out);
        });
    }
    mach_sparse_free(s);
    mach_dense_free(x);
    return st;
}

void mach_free_host(void* p) { std::free(p); }

// ---- sparse ----
mach_status mach_sparse_upload(mach_ctx* ctx, mach_dtype dtype, int order, const int* dims, int64_t nnz,
                               const int64_t* idx, const double* vals, mach_sparse** out) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(out, "out");
        if (nnz < 0) throw_arg("nnz must be >= 0");
        if (nnz > 0) {
            need(idx, "idx");
            need(vals, "vals");
        }
        *out = sparse_from_host(&ctx->c, dtype, dims_of(order, dims), nnz, idx, vals);
    });
}

mach_status mach_sparse_nnz(const mach_sparse* s, int64_t* nnz) {
    return guard([&] {
        need(s, "tensor");
        DevGuard dg_(s->ctx->device);
        *nnz = s->nnz;
    });
}

mach_status mach_sparse_download(const mach_sparse* s, int64_t* idx, double* vals) {
    return guard([&] {
        need(s, "tensor");
        DevGuard dg_(s->ctx->device);
        sparse_to_host(s, idx, vals);
    });
}

mach_status mach_sparse_norm(const mach_sparse* s, double* out);

mach_status mach_sparse_free(mach_sparse* s) {
    return guard([&] { delete s; });
}

// ---- decompositions ----
static std::vector<int> ranks_of(int order, const int* ranks) {
    need(ranks, "ranks");
    return std::vector<int>(ranks, ranks + order);
}

mach_status mach_hosvd_sparse(mach_ctx* ctx, const mach_sparse* t, const int* ranks, mach_model** out) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(t, "tensor");
        need(out, "out");
        *out = tucker_sparse(const_cast<mach_sparse*>(t), ranks_of(static_cast<int>(t->dims.size()), ranks), false, 1, 0.0);
    });
}

mach_status mach_hosvd_dense(mach_ctx* ctx, const mach_dense* t, const int* ranks, mach_model** out) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(t, "tensor");
        need(out, "out");
        *out = tucker_dense(t, ranks_of(static_cast<int>(t->dims.size()), ranks), false, 1, 0.0);
    });
}

mach_status mach_hooi_sparse(mach_ctx* ctx, const mach_sparse* t, const int* ranks, int max_iterations,
                             double fit_tolerance, mach_model** out) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(t, "tensor");
        need(out, "out");
        *out = tucker_sparse(const_cast<mach_sparse*>(t), ranks_of(static_cast<int>(t->dims.size()), ranks), true,
                             max_iterations, fit_tolerance);
    });
}

mach_status mach_hooi_dense(mach_ctx* ctx, const mach_dense* t, const int* ranks, int max_iterations,
                            double fit_tolerance, mach_model** out) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(t, "tensor");
        need(out, "out");
        *out = tucker_dense(t, ranks_of(static_cast<int>(t->dims.size()), ranks), true, max_iterations, fit_tolerance);
    });
}

static mach_status mach_pipeline(mach_ctx* ctx, const mach_dense* t, const int* ranks, double p, uint64_t seed,
                                 bool do_hooi, int max_it, double tol, mach_model** out, mach_sparse** sampled) {
    return guard([&] {
        need(ctx, "ctx");
        need(t, "tensor");
        need(out, "out");
        cudaEvent_t a, b;
        MB_CUDA(cudaEventCreate(&a));
        MB_CUDA(cudaEventCreate(&b));
        MB_CUDA(cudaEventRecord(a, ctx->c.stream));
        std::unique_ptr<mach_sparse> s(sample_dense(t, p, seed));
        MB_CUDA(cudaEventRecord(b, ctx->c.stream));
        MB_CUDA(cudaEventSynchronize(b));
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        // p == 1 keeps every nonzero entry unchanged: the densified sample (the
        // densify switch, tucker.cpp:154-155) is the input itself, so the dense
        // route reads t in place instead of a scattered copy
        // (only when the sample is dense enough for that switch: a mostly-zero
        // input keeps the sparse route)
        const bool in_place = p == 1.0 && static_cast<double>(s->nnz) >= 0.25 * static_cast<double>(s->numel);
        mach_model* m = in_place
                            ? tucker_dense(t, ranks_of(static_cast<int>(t->dims.size()), ranks), do_hooi, max_it, tol)
                            : tucker_sparse(s.get(), ranks_of(static_cast<int>(t->dims.size()), ranks), do_hooi, max_it, tol);
        m->sample_ms = ms;
        *out = m;
        if (sampled) *sampled = s.release();
    });
}

mach_status mach_mach_hooi(mach_ctx* ctx, const mach_dense* t, const int* ranks, double p, uint64_t seed,
                           int max_iterations, double fit_tolerance, mach_model** out, mach_sparse** sampled) {
    return mach_pipeline(ctx, t, ranks, p, seed, true, max_iterations, fit_tolerance, out, sampled);
}

mach_status mach_mach_hosvd(mach_ctx* ctx, const mach_dense* t, const int* ranks, double p, uint64_t seed,
                            mach_model** out, mach_sparse** sampled) {
    return mach_pipeline(ctx, t, ranks, p, seed, false, 1, 0.0, out, sampled);
}

// ---- model ----
mach_status mach_model_info(const mach_model* m, int* order, int* iterations, double* fit, int* n_sweep_fits,
                            int* n_warnings) {
    return guard([&] {
        need(m, "model");
        if (order) *order = m->order;
        if (iterations) *iterations = m->iterations;
        if (fit) *fit = m->fit;
        if (n_sweep_fits) *n_sweep_fits = static_cast<int>(m->sweep_fits.size());
        if (n_warnings) *n_warnings = static_cast<int>(m->warnings.size());
    });
}

mach_status mach_model_dims(const mach_model* m, int* dims, int* ranks) {
    return guard([&] {
        need(m, "model");
        for (int i = 0; i < m->order; ++i) {
            if (dims) dims[i] = m->dims[static_cast<std::size_t>(i)];
            if (ranks) ranks[i] = m->ranks[static_cast<std::size_t>(i)];
        }
    });
}

mach_status mach_model_core(const mach_model* m, double* host) {
    return guard([&] {
        need(m, "model");
        std::memcpy(host, m->core.data(), m->core.size() * sizeof(double));
    });
}

mach_status mach_model_factor(const mach_model* m, int mode, double* host) {
    return guard([&] {
        need(m, "model");
        if (mode < 0 || mode >= m->order) throw_arg("mode out of range");
        const auto& f = m->factors[static_cast<std::size_t>(mode)];
        std::memcpy(host, f.data(), f.size() * sizeof(double));
    });
}

mach_status mach_model_sweep_fits(const mach_model* m, double* host) {
    return guard([&] {
        need(m, "model");
        std::memcpy(host, m->sweep_fits.data(), m->sweep_fits.size() * sizeof(double));
    });
}

mach_status mach_model_warning(const mach_model* m, int i, char* buf, size_t len) {
    return guard([&] {
        need(m, "model");
        if (i < 0 || i >= static_cast<int>(m->warnings.size())) throw_arg("warning index out of range");
        if (len == 0) return;
        std::strncpy(buf, m->warnings[static_cast<std::size_t>(i)].c_str(), len - 1);
        buf[len - 1] = 0;
    });
}

mach_status mach_model_times(const mach_model* m, double* sample_ms, double* setup_ms, double* hosvd_ms, double* sweep_ms,
                             int max_sweeps) {
    return guard([&] {
        need(m, "model");
        if (sample_ms) *sample_ms = m->sample_ms;
        if (setup_ms) *setup_ms = m->setup_ms;
        if (hosvd_ms) *hosvd_ms = m->hosvd_ms;
        for (int i = 0; sweep_ms && i < max_sweeps && i < static_cast<int>(m->sweep_ms.size()); ++i)
            sweep_ms[i] = m->sweep_ms[static_cast<std::size_t>(i)];
    });
}

mach_status mach_model_free(mach_model* m) {
    return guard([&] { delete m; });
}

mach_status mach_accuracy(mach_ctx* ctx, const mach_dense* t, const mach_model* m, double* out) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(t, "tensor");
        need(m, "model");
        *out = accuracy_dev(t, m);
    });
}

mach_status mach_reconstruct(mach_ctx* ctx, const mach_model* m, mach_dense** out) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(m, "model");
        *out = reconstruct_model(&ctx->c, m);
    });
}

mach_status mach_left_singular_basis(mach_ctx* ctx, int rows, int cols, const double* a, int k, double* basis, double* sv,
                                     int* numerical_rank, int* completed) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        lsb_host(&ctx->c, rows, cols, a, k, basis, sv, numerical_rank, completed);
    });
}

mach_status mach_model_accuracy(mach_ctx* ctx, const mach_dense* t, const int* ranks, const double* core,
                                const double* const* factors, double* out) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(t, "tensor");
        need(ranks, "ranks");
        need(core, "core");
        need(factors, "factors");
        need(out, "out");
        Ctx* c = &ctx->c;
        const int d = static_cast<int>(t->dims.size());
        std::vector<int> rk(ranks, ranks + d);
        std::int64_t cn = 1;
        for (int m = 0; m < d; ++m) {
            if (rk[static_cast<std::size_t>(m)] < 1) throw_arg("ranks must be >= 1");
            cn *= rk[static_cast<std::size_t>(m)];
        }
        DBuf<double> red(c, sumsq_scratch()), scal(c, 1), G(c, static_cast<std::size_t>(cn));
        if (t->dtype == MACH_F32) sumsq<float>(c, static_cast<const float*>(t->data), t->numel, red.get(), scal.get());
        else sumsq<double>(c, static_cast<const double*>(t->data), t->numel, red.get(), scal.get());
        double n2 = 0.0;
        to_host(c, &n2, scal.get(), 1);
        sync(c);
        if (n2 == 0.0) throw_arg("accuracy needs a reference tensor with nonzero norm");
        to_device(c, G.get(), core, G.n);
        std::vector<DBuf<double>> U(static_cast<std::size_t>(d));
        std::vector<const double*> up;
        for (int m = 0; m < d; ++m) {
            need(factors[m], "factor");
            const std::size_t n = static_cast<std::size_t>(t->dims[static_cast<std::size_t>(m)]) * rk[static_cast<std::size_t>(m)];
            U[static_cast<std::size_t>(m)].alloc(c, n);
            to_device(c, U[static_cast<std::size_t>(m)].get(), factors[m], n);
            up.push_back(U[static_cast<std::size_t>(m)].get());
        }
        const double e2 = t->dtype == MACH_F32
                              ? residual2_fused<float>(c, static_cast<const float*>(t->data), t->dims, rk, G.get(), up)
                              : residual2_fused<double>(c, static_cast<const double*>(t->data), t->dims, rk, G.get(), up);
        *out = 1.0 - std::sqrt(e2) / std::sqrt(n2);
    });
}

mach_status mach_subspace_sin(mach_ctx* ctx, int n, int r, const double* a, const double* b, double* out) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(a, "a");
        need(b, "b");
        need(out, "out");
        if (n < 1 || r < 1 || r > n) throw_arg("subspace_sin needs 1 <= r <= n");
        Ctx* c = &ctx->c;
        DBuf<double> A(c, static_cast<std::size_t>(n) * r), B(c, static_cast<std::size_t>(n) * r);
        to_device(c, A.get(), a, A.n);
        to_device(c, B.get(), b, B.n);
        *out = subspace_sin_dev(c, A.get(), B.get(), n, r);
    });
}

mach_status mach_truncated_svd(mach_ctx* ctx, int rows, int cols, const double* a, int k, double* left, double* sv,
                               double* right) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(a, "matrix");
        need(left, "left");
        need(sv, "singular_values");
        need(right, "right");
        if (rows < 1 || cols < 1) throw_arg("matrix must be nonempty");
        if (k < 1 || k > std::min(rows, cols)) throw_arg("k must satisfy 1 <= k <= min(rows, cols)");
        Ctx* c = &ctx->c;
        DBuf<double> A(c, static_cast<std::size_t>(rows) * cols), L(c, static_cast<std::size_t>(rows) * k),
            S(c, static_cast<std::size_t>(k)), R(c, static_cast<std::size_t>(cols) * k);
        to_device(c, A.get(), a, A.n);
        truncated_svd_dev(c, A.get(), rows, cols, k, L.get(), S.get(), R.get());
        to_host(c, left, L.get(), L.n);
        to_host(c, sv, S.get(), S.n);
        to_host(c, right, R.get(), R.n);
        sync(c);
    });
}

mach_status mach_low_rank_approx(mach_ctx* ctx, int rows, int cols, const double* a, int k, double* out) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(a, "matrix");
        need(out, "out");
        if (rows < 1 || cols < 1) throw_arg("matrix must be nonempty");
        if (k < 1 || k > std::min(rows, cols)) throw_arg("k must satisfy 1 <= k <= min(rows, cols)");
        Ctx* c = &ctx->c;
        DBuf<double> A(c, static_cast<std::size_t>(rows) * cols), L(c, static_cast<std::size_t>(rows) * k),
            S(c, static_cast<std::size_t>(k)), R(c, static_cast<std::size_t>(cols) * k);
        to_device(c, A.get(), a, A.n);
        truncated_svd_dev(c, A.get(), rows, cols, k, L.get(), S.get(), R.get());
        low_rank_dev(c, L.get(), S.get(), R.get(), rows, cols, k, A.get());
        to_host(c, out, A.get(), A.n);
        sync(c);
    });
}

mach_status mach_mode_product_dense(mach_ctx* ctx, const mach_dense* t, int rows, int cols, const double* m, int mode,
                                    mach_dense** out) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(t, "tensor");
        *out = mode_product_dev(&ctx->c, t, nullptr, rows, cols, m, mode);
    });
}

mach_status mach_mode_product_sparse(mach_ctx* ctx, const mach_sparse* t, int rows, int cols, const double* m, int mode,
                                     mach_dense** out) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(t, "tensor");
        *out = mode_product_dev(&ctx->c, nullptr, t, rows, cols, m, mode);
    });
}

mach_status mach_dense_mode_gram(mach_ctx* ctx, const mach_dense* t, int mode, double* host, int* tensor_cores) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(t, "tensor");
        need(host, "host");
        if (mode < 0 || mode >= static_cast<int>(t->dims.size())) throw_arg("mode out of range");
        Ctx* c = &ctx->c;
        const int R = t->dims[static_cast<std::size_t>(mode)];
        const long long K = t->numel / std::max(1, R);
        DBuf<double> G(c, static_cast<std::size_t>(R) * R);
        int tc = 0;
        if (t->dtype == MACH_F32 && gram_tc_applies(t->dims, mode)) {
            gram_tc(c, static_cast<const float*>(t->data), t->dims, mode, G.get());
            tc = 1;
        } else if (K <= (1ll << 31) - 1) {
            if (t->dtype == MACH_F32) {
                DBuf<float> xm(c, static_cast<std::size_t>(t->numel));
                dense_matricize<float, float>(c, static_cast<const float*>(t->data), t->dims, mode, xm.get());
                gram<float>(c, xm.get(), R, 1, static_cast<int>(K), R, G.get());
            } else {
                DBuf<double> xm(c, static_cast<std::size_t>(t->numel));
                dense_matricize<double, double>(c, static_cast<const double*>(t->data), t->dims, mode, xm.get());
                gram<double>(c, xm.get(), R, 1, static_cast<int>(K), R, G.get());
            }
        } else {
            throw_shape("mode unfolding too wide for the CUDA-core Gram");
        }
        to_host(c, host, G.get(), static_cast<std::size_t>(R) * R);
        sync(c);
        if (tensor_cores) *tensor_cores = tc;
    });
}

}  // extern "C"

// ---- sessions + profiling ----
namespace machb {
void* session_sparse(mach_sparse* X, const std::vector<int>& ranks);
void* session_dense(const mach_dense* X, const std::vector<int>& ranks);
int session_step(void* s, int n, double tol);
mach_model* session_snapshot(void* s);
void session_free(void* s);
int session_iterations(void* s);
double session_fit(void* s);
bool session_stopped(void* s);
long long session_ttm_bytes(void* s, int m);
void* session_sparse_from(mach_sparse* X, const std::vector<int>& ranks, const mach_model* init);
void* session_mode_y(void* s, int m, int* rows, int* cols);
void session_mode_update(void* s, int m);
int session_sweep_end(void* s, double tol);
void session_set_norm2(void* s, double v);
void session_shard(void* s);
void session_refresh_fit(void* s);
void sparse_row_gram_host(Ctx* ctx, const mach_sparse* X, int n, double* host);
mach_model* hosvd_from_grams(Ctx* ctx, const std::vector<int>& dims, const std::vector<int>& ranks,
                             const double* const* grams);
}  // namespace machb

struct mach_session {
    void* s = nullptr;
};

extern "C" {

mach_status mach_hooi_begin(mach_ctx* ctx, const mach_sparse* t, const int* ranks, mach_session** out) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(t, "tensor");
        need(out, "out");
        auto h = std::make_unique<mach_session>();
        h->s = session_sparse(const_cast<mach_sparse*>(t), ranks_of(static_cast<int>(t->dims.size()), ranks));
        *out = h.release();
    });
}

mach_status mach_hooi_begin_dense(mach_ctx* ctx, const mach_dense* t, const int* ranks, mach_session** out) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(t, "tensor");
        need(out, "out");
        auto h = std::make_unique<mach_session>();
        h->s = session_dense(t, ranks_of(static_cast<int>(t->dims.size()), ranks));
        *out = h.release();
    });
}

mach_status mach_hooi_step(mach_session* s, int n, double tol, int* done, int* stopped) {
    return guard([&] {
        need(s, "session");
        if (n < 0) throw_arg("n must be >= 0");
        const int k = session_step(s->s, n, tol);
        if (done) *done = k;
        if (stopped) *stopped = session_stopped(s->s) ? 1 : 0;
    });
}

mach_status mach_hooi_state(mach_session* s, double* fit, int* iterations) {
    return guard([&] {
        need(s, "session");
        if (fit) *fit = session_fit(s->s);
        if (iterations) *iterations = session_iterations(s->s);
    });
}

mach_status mach_hooi_begin_from(mach_ctx* ctx, const mach_sparse* t, const int* ranks, const mach_model* init,
                                 mach_session** out) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(t, "tensor");
        need(init, "init");
        need(out, "out");
        auto h = std::make_unique<mach_session>();
        h->s = session_sparse_from(const_cast<mach_sparse*>(t), ranks_of(static_cast<int>(t->dims.size()), ranks), init);
        *out = h.release();
    });
}

mach_status mach_comm_unique_id(unsigned char* out) {
    return guard([&] {
        need(out, "out");
        comm_unique_id(out);
    });
}

mach_status mach_ctx_comm_init(mach_ctx* ctx, int world, int rank, const unsigned char* id) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(id, "id");
        comm_init(&ctx->c, world, rank, id);
    });
}

mach_status mach_hooi_shard(mach_session* s) {
    return guard([&] {
        need(s, "session");
        session_shard(s->s);
    });
}

mach_status mach_hooi_set_norm2(mach_session* s, double norm2) {
    return guard([&] {
        need(s, "session");
        session_set_norm2(s->s, norm2);
    });
}

mach_status mach_hooi_mode_y(mach_session* s, int mode, void** y, int* rows, int* cols) {
    return guard([&] {
        need(s, "session");
        need(y, "y");
        need(rows, "rows");
        need(cols, "cols");
        *y = session_mode_y(s->s, mode, rows, cols);
    });
}

mach_status mach_hooi_mode_update(mach_session* s, int mode) {
    return guard([&] {
        need(s, "session");
        session_mode_update(s->s, mode);
    });
}

mach_status mach_hooi_sweep_end(mach_session* s, double fit_tolerance, int* stopped) {
    return guard([&] {
        need(s, "session");
        if (std::isnan(fit_tolerance)) throw_arg("fit_tolerance must be a number");
        const int st = session_sweep_end(s->s, fit_tolerance);
        if (stopped) *stopped = st;
    });
}

mach_status mach_hooi_ttm_bytes(mach_session* s, int mode, long long* bytes) {
    return guard([&] {
        need(s, "session");
        need(bytes, "bytes");
        *bytes = session_ttm_bytes(s->s, mode);
    });
}

mach_status mach_hooi_model(mach_session* s, mach_model** out) {
    return guard([&] {
        need(s, "session");
        need(out, "out");
        *out = session_snapshot(s->s);
    });
}

mach_status mach_hooi_refresh_fit(mach_session* s) {
    return guard([&] {
        need(s, "session");
        session_refresh_fit(s->s);
    });
}

mach_status mach_sparse_row_gram(mach_ctx* ctx, const mach_sparse* t, int mode, double* host) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(t, "tensor");
        need(host, "host");
        sparse_row_gram_host(&ctx->c, t, mode, host);
    });
}

mach_status mach_hosvd_from_grams(mach_ctx* ctx, int order, const int* dims, const int* ranks,
                                  const double* const* grams, mach_model** out) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(grams, "grams");
        need(out, "out");
        *out = hosvd_from_grams(&ctx->c, dims_of(order, dims), ranks_of(order, ranks), grams);
    });
}

mach_status mach_session_free(mach_session* s) {
    return guard([&] {
        if (!s) return;
        session_free(s->s);
        delete s;
    });
}

mach_status mach_ctx_profile(mach_ctx* ctx, int enable) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        ctx->c.resolve();
        ctx->c.profile = enable != 0;
        if (enable) ctx->c.stats.clear();
    });
}

mach_status mach_ctx_kernel_stat(mach_ctx* ctx, int i, char* name, size_t len, int64_t* launches, double* total_ms) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        ctx->c.resolve();
        if (i < 0 || i >= static_cast<int>(ctx->c.stats.size())) throw_arg("kernel index out of range");
        auto it = ctx->c.stats.begin();
        std::advance(it, i);
        if (name && len) {
            std::strncpy(name, it->first.c_str(), len - 1);
            name[len - 1] = 0;
        }
        if (launches) *launches = it->second.launches;
        if (total_ms) *total_ms = it->second.ms;
    });
}

}  // extern "C"

// ---- Theorem-1 bound, streaming ingest, binary files ----
namespace machb {
void bound_conditions(const std::vector<int>& dims, double p, mach_bound_report* rep);
double bound_min_probability(const std::vector<int>& dims);
void theorem1_bound_dev(Ctx* ctx, const mach_dense* x, mach_sparse* xhat, const std::vector<int>& ranks, double p,
                        mach_bound_report* rep, mach_bound_mode* per_mode);
mach_stream* stream_begin(Ctx* ctx, int dtype, const std::vector<int>& dims, double p, std::uint64_t seed);
void stream_append(mach_stream* s, const mach_dense* slab);
void stream_append_host(mach_stream* s, const void* host, int ticks);
void stream_append_records(mach_stream* s, std::int64_t n, const std::int32_t* machine, const std::int32_t* metric,
                           const std::int32_t* tick, const double* value, int ticks, bool carry);
void stream_state(mach_stream* s, std::int64_t* ticks, std::int64_t* nnz);
mach_sparse* stream_tensor(mach_stream* s);
mach_dense* stream_last_slab(mach_stream* s);
void stream_free(mach_stream* s);
int stream_device(const mach_stream* s);
void dense_save(const mach_dense* t, const char* path);
mach_dense* dense_load(Ctx* ctx, const char* path);
void sparse_save(const mach_sparse* t, const char* path);
mach_sparse* sparse_load(Ctx* ctx, const char* path);
void tensor_file_kind(const char* path, int* kind, int* dtype, int* order, int* dims, std::int64_t* count);
}  // namespace machb

extern "C" {

mach_status mach_achlioptas_bounds(double b, int64_t n, int64_t k, double p, double* two_norm, double* frobenius) {
    return guard([&] {  // bounds.cpp:132-143
        if (!(b >= 0.0)) throw_arg("b must be >= 0");
        if (n < 1) throw_arg("n must be >= 1");
        if (k < 1) throw_arg("k must be >= 1");
        if (!(p > 0.0 && p <= 1.0)) throw_arg("p must be in (0, 1]");
        const double nd = static_cast<double>(n), kd = static_cast<double>(k);
        if (two_norm) *two_norm = 4.0 * b * std::sqrt(nd / p);
        if (frobenius) *frobenius = 4.0 * b * std::sqrt(nd * kd / p);
    });
}

mach_status mach_min_sampling_probability(int order, const int* dims, double* out) {
    return guard([&] {
        need(out, "out");
        *out = bound_min_probability(order > 0 && dims ? std::vector<int>(dims, dims + order) : std::vector<int>());
    });
}

mach_status mach_theorem1_conditions(int order, const int* dims, double p, mach_bound_report* rep) {
    return guard([&] {  // bounds.cpp:152-158
        need(rep, "rep");
        const std::vector<int> d = order > 0 && dims ? std::vector<int>(dims, dims + order) : std::vector<int>();
        bound_min_probability(d);  // the same shape checks
        if (!(p > 0.0 && p <= 1.0)) throw_arg("p must be in (0, 1]");
        bound_conditions(d, p, rep);
    });
}

mach_status mach_theorem1_bound(mach_ctx* ctx, const mach_dense* x, const mach_sparse* xhat, const int* ranks, double p,
                                mach_bound_report* rep, mach_bound_mode* per_mode) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(x, "x");
        need(xhat, "xhat");
        need(ranks, "ranks");
        need(rep, "rep");
        need(per_mode, "per_mode");
        theorem1_bound_dev(&ctx->c, x, const_cast<mach_sparse*>(xhat),
                           std::vector<int>(ranks, ranks + x->dims.size()), p, rep, per_mode);
    });
}

mach_status mach_stream_begin(mach_ctx* ctx, mach_dtype dtype, int order, const int* dims, double p, uint64_t seed,
                              mach_stream** out) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(out, "out");
        *out = stream_begin(&ctx->c, dtype, dims_of(order, dims), p, seed);
    });
}

mach_status mach_stream_append(mach_stream* s, const mach_dense* slab) {
    return guard([&] {
        need(s, "stream");
        DevGuard dg_(stream_device(s));
        need(slab, "slab");
        stream_append(s, slab);
    });
}

mach_status mach_stream_append_host(mach_stream* s, const void* host, int ticks) {
    return guard([&] {
        need(s, "stream");
        DevGuard dg_(stream_device(s));
        stream_append_host(s, host, ticks);
    });
}

mach_status mach_stream_append_records(mach_stream* s, int64_t n, const int32_t* machine, const int32_t* metric,
                                       const int32_t* tick, const double* value, int ticks, int carry_forward) {
    return guard([&] {
        need(s, "stream");
        DevGuard dg_(stream_device(s));
        stream_append_records(s, n, machine, metric, tick, value, ticks, carry_forward != 0);
    });
}

mach_status mach_stream_state(mach_stream* s, int64_t* ticks, int64_t* nnz) {
    return guard([&] {
        need(s, "stream");
        DevGuard dg_(stream_device(s));
        std::int64_t t = 0, z = 0;
        stream_state(s, &t, &z);
        if (ticks) *ticks = t;
        if (nnz) *nnz = z;
    });
}

mach_status mach_stream_tensor(mach_stream* s, mach_sparse** out) {
    return guard([&] {
        need(s, "stream");
        DevGuard dg_(stream_device(s));
        need(out, "out");
        *out = stream_tensor(s);
    });
}

mach_status mach_stream_last_slab(mach_stream* s, mach_dense** out) {
    return guard([&] {
        need(s, "stream");
        DevGuard dg_(stream_device(s));
        need(out, "out");
        *out = stream_last_slab(s);
    });
}

mach_status mach_stream_free(mach_stream* s) {
    return guard([&] {
        if (!s) return;
        DevGuard dg_(stream_device(s));
        stream_free(s);
    });
}

mach_status mach_dense_save(const mach_dense* t, const char* path) {
    return guard([&] {
        need(t, "tensor");
        DevGuard dg_(t->ctx->device);
        dense_save(t, path);
    });
}

mach_status mach_dense_load(mach_ctx* ctx, const char* path, mach_dense** out) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(out, "out");
        *out = dense_load(&ctx->c, path);
    });
}

mach_status mach_sparse_save(const mach_sparse* t, const char* path) {
    return guard([&] {
        need(t, "tensor");
        DevGuard dg_(t->ctx->device);
        sparse_save(t, path);
    });
}

mach_status mach_sparse_load(mach_ctx* ctx, const char* path, mach_sparse** out) {
    return guard([&] {
        need(ctx, "ctx");
        DevGuard dg_(ctx->c.device);
        need(out, "out");
        *out = sparse_load(&ctx->c, path);
    });
}

mach_status mach_tensor_file_kind(const char* path, int* kind, mach_dtype* dtype, int* order, int* dims, int64_t* nnz) {
    return guard([&] {
        int dt = 0;
        std::int64_t c = 0;
        tensor_file_kind(path, kind, &dt, order, dims, &c);
        if (dtype) *dtype = static_cast<mach_dtype>(dt);
        if (nnz) *nnz = c;
    });
}

}  // extern "C"
