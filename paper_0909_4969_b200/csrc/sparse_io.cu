// Sparse tensor upload/download and input validation.
// mach_sparse_upload canonicalises on the device exactly like the reference's
// SparseTensor constructor (proj/src/tensor.cpp:78-96): sort by flat index,
// merge duplicates by summation, drop exact zeros.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_select.cuh>

#include <cmath>

#include "sparse_ttm.cuh"

namespace machb {

namespace {

template <typename T, typename IdxT>
__global__ void narrow_kernel(const unsigned long long* __restrict__ ki, const double* __restrict__ vi, const int* __restrict__ nsel,
                              IdxT* __restrict__ ko, T* __restrict__ vo) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= *nsel) return;
    ko[i] = static_cast<IdxT>(ki[i]);
    vo[i] = static_cast<T>(vi[i]);
}

template <typename T, typename IdxT>
__global__ void widen_kernel(const IdxT* __restrict__ ki, const T* __restrict__ vi, long long n,
                             long long* __restrict__ ko, double* __restrict__ vo) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    ko[i] = static_cast<long long>(ki[i]);
    vo[i] = static_cast<double>(vi[i]);
}

template <typename T>
__global__ void finite_kernel(const T* __restrict__ x, long long n, int* __restrict__ bad) {
    int b = 0;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        b |= !isfinite(static_cast<double>(x[i]));
    if (__syncthreads_or(b) && threadIdx.x == 0) atomicOr(bad, 1);
}

// values whose kept pairs are (idx, val) pairs where val != 0 after merging
__global__ void flag_nonzero_kernel(const double* __restrict__ v, const int* __restrict__ nrun, char* __restrict__ f) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i < *nrun) f[i] = v[i] != 0.0;
}

}  // namespace

void check_finite_upload(Ctx* ctx, int dtype, const void* dev, std::int64_t n) {
    if (n == 0) return;
    DBuf<int> bad(ctx, 1);
    bad.zero(ctx);
    const int blocks = static_cast<int>(std::min<long long>(148 * 16, (n + 255) / 256));
    if (dtype == MACH_F32) MB_LAUNCH(ctx, finite_kernel<float>, blocks, 256, 0, static_cast<const float*>(dev), n, bad.get());
    else MB_LAUNCH(ctx, finite_kernel<double>, blocks, 256, 0, static_cast<const double*>(dev), n, bad.get());
    int h = 0;
    to_host(ctx, &h, bad.get(), 1);
    sync(ctx);
    if (h) throw_arg("tensor values must be finite");
}

mach_sparse* sparse_from_host(Ctx* ctx, int dtype, const std::vector<int>& dims, std::int64_t nnz, const std::int64_t* idx,
                              const double* vals) {
    const std::int64_t total = checked_size(dims);
    for (std::int64_t i = 0; i < nnz; ++i) {  // tensor.cpp:80-84 validation
        if (idx[i] < 0 || idx[i] >= total) throw_arg("sparse entry index out of bounds");
        if (!std::isfinite(vals[i])) throw_arg("tensor values must be finite");
    }
    auto out = std::make_unique<mach_sparse>();
    out->ctx = ctx;
    out->dtype = dtype;
    out->dims = dims;
    out->numel = total;
    out->idx64 = total > 0xFFFFFFFFll;
    if (nnz == 0) return out.release();
    DBuf<unsigned long long> k0(ctx, nnz), k1(ctx, nnz), kr(ctx, nnz), ks(ctx, nnz);
    DBuf<double> v0(ctx, nnz), v1(ctx, nnz), vr(ctx, nnz), vs(ctx, nnz);
    DBuf<int> nrun(ctx, 1), nsel(ctx, 1);
    DBuf<char> flags(ctx, nnz);
    to_device(ctx, k0.get(), reinterpret_cast<const unsigned long long*>(idx), nnz);
    to_device(ctx, v0.get(), vals, nnz);
    int bits = 1;
    while ((1ll << bits) < total && bits < 64) ++bits;
    std::size_t tmp = 0, t2 = 0, t3 = 0;
    MB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0.get(), k1.get(), v0.get(), v1.get(), nnz, 0, bits, ctx->stream));
    MB_CUDA(cub::DeviceReduce::ReduceByKey(nullptr, t2, k1.get(), kr.get(), v1.get(), vr.get(), nrun.get(), ::cuda::std::plus<double>(),
                                           nnz, ctx->stream));
    MB_CUDA(cub::DeviceSelect::Flagged(nullptr, t3, kr.get(), flags.get(), ks.get(), nsel.get(), nnz, ctx->stream));
    DBuf<unsigned char> t(ctx, std::max(tmp, std::max(t2, t3)));
    MB_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, k0.get(), k1.get(), v0.get(), v1.get(), nnz, 0, bits, ctx->stream));
    MB_CUDA(cub::DeviceReduce::ReduceByKey(t.get(), t2, k1.get(), kr.get(), v1.get(), vr.get(), nrun.get(),
                                           ::cuda::std::plus<double>(), nnz, ctx->stream));
    MB_LAUNCH(ctx, flag_nonzero_kernel, ceil_div(nnz, 256), 256, 0, vr.get(), nrun.get(), flags.get());
    int hrun = 0;
    to_host(ctx, &hrun, nrun.get(), 1);
    sync(ctx);
    MB_CUDA(cub::DeviceSelect::Flagged(t.get(), t3, kr.get(), flags.get(), ks.get(), nsel.get(), hrun, ctx->stream));
    MB_CUDA(cub::DeviceSelect::Flagged(t.get(), t3, vr.get(), flags.get(), vs.get(), nsel.get(), hrun, ctx->stream));
    ctx->launches += 8;
    int hsel = 0;
    to_host(ctx, &hsel, nsel.get(), 1);
    sync(ctx);
    out->nnz = hsel;
    const int isz = out->idx64 ? 8 : 4;
    if (hsel > 0) {
        MB_CUDA(cudaMallocAsync(&out->idx, static_cast<std::size_t>(hsel) * isz, ctx->stream));
        MB_CUDA(cudaMallocAsync(&out->val, static_cast<std::size_t>(hsel) * dtype_size(dtype), ctx->stream));
        const int blocks = ceil_div(hsel, 256);
#define MB_NARROW(T, I) \
    MB_LAUNCH(ctx, (narrow_kernel<T, I>), blocks, 256, 0, ks.get(), vs.get(), nsel.get(), static_cast<I*>(out->idx), static_cast<T*>(out->val))
        if (dtype == MACH_F32) {
            if (out->idx64) MB_NARROW(float, unsigned long long); else MB_NARROW(float, unsigned int);
        } else {
            if (out->idx64) MB_NARROW(double, unsigned long long); else MB_NARROW(double, unsigned int);
        }
#undef MB_NARROW
    }
    sync(ctx);
    return out.release();
}

void sparse_to_host(const mach_sparse* s, std::int64_t* idx, double* vals) {
    Ctx* ctx = s->ctx;
    if (s->nnz == 0) return;
    DBuf<long long> ko(ctx, s->nnz);
    DBuf<double> vo(ctx, s->nnz);
    const int blocks = ceil_div(s->nnz, 256);
#define MB_WIDEN(T, I) \
    MB_LAUNCH(ctx, (widen_kernel<T, I>), blocks, 256, 0, static_cast<const I*>(s->idx), static_cast<const T*>(s->val), s->nnz, ko.get(), vo.get())
    if (s->dtype == MACH_F32) {
        if (s->idx64) MB_WIDEN(float, unsigned long long); else MB_WIDEN(float, unsigned int);
    } else {
        if (s->idx64) MB_WIDEN(double, unsigned long long); else MB_WIDEN(double, unsigned int);
    }
#undef MB_WIDEN
    if (idx) to_host(ctx, reinterpret_cast<long long*>(idx), ko.get(), s->nnz);
    if (vals) to_host(ctx, vals, vo.get(), s->nnz);
    sync(ctx);
}

}  // namespace machb

extern "C" mach_status mach_sparse_norm(const mach_sparse* s, double* out) {
    try {
        using namespace machb;
        if (!s || !out) throw_arg("null argument");
        Ctx* ctx = s->ctx;
        DBuf<double> red(ctx, sumsq_scratch()), r(ctx, 1);
        if (s->nnz == 0) {
            *out = 0.0;
            return MACH_OK;
        }
        if (s->dtype == MACH_F32) sumsq<float>(ctx, static_cast<const float*>(s->val), s->nnz, red.get(), r.get());
        else sumsq<double>(ctx, static_cast<const double*>(s->val), s->nnz, red.get(), r.get());
        double h = 0;
        to_host(ctx, &h, r.get(), 1);
        sync(ctx);
        *out = std::sqrt(h);
        return MACH_OK;
    } catch (const machb::Error& e) {
        return static_cast<mach_status>(e.code);
    } catch (...) {
        return MACH_ERR_INTERNAL;
    }
}
