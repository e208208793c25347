// Standalone sparse mode product Y = X x_m M (reference: mode_product(const
// SparseTensor&, const Matrix&, int), proj/src/tensor.cpp:241-259): for each
// nonzero (a, r, c) of the split (inner, len, outer) at mode m,
// y[a, q, c] += v * M(q, r).  No densified copy of X.
//
// The reference walks the entries in ascending flat index, so every output
// element receives its terms in ascending r.  Here the nonzeros are stably
// sorted by the output fibre key c * inner + a (the stable radix sort keeps
// ascending r inside a fibre), and one thread per (fibre, q) accumulates its
// fibre's terms in that same order with unfused multiply and add — the
// reference's rounding sequence, so the result is bit-identical to it.
// Fibres with no nonzeros stay zero.
#include <cub/cub.cuh>

#include "common.cuh"
#include "sparse_ttm.cuh"

namespace machb {

namespace {

template <typename IdxT>
__global__ void fibre_key_kernel(const IdxT* __restrict__ idx, long long nnz, long long inner, long long len,
                                 unsigned long long* __restrict__ key, unsigned* __restrict__ pos) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= nnz) return;
    const unsigned long long f = static_cast<unsigned long long>(idx[i]);
    const unsigned long long a = f % static_cast<unsigned long long>(inner);
    const unsigned long long c = f / static_cast<unsigned long long>(inner * len);
    key[i] = c * static_cast<unsigned long long>(inner) + a;
    pos[i] = static_cast<unsigned>(i);
}

// one thread per (run, q): runs of equal key are consecutive in the sorted order
template <typename T, typename IdxT>
__global__ void fibre_accumulate_kernel(const unsigned long long* __restrict__ ukey, const int* __restrict__ start,
                                        const int* __restrict__ count, const int* __restrict__ nrun,
                                        const unsigned* __restrict__ pos, const IdxT* __restrict__ idx,
                                        const T* __restrict__ val, long long inner, long long len, int J,
                                        const double* __restrict__ M, double* __restrict__ y) {
    const long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    const long long runs = *nrun;
    if (t >= runs * J) return;
    const long long run = t / J;
    const int q = static_cast<int>(t - run * J);
    const int s0 = start[run], n = count[run];
    double acc = 0.0;
    for (int j = 0; j < n; ++j) {
        const unsigned p = pos[s0 + j];
        const unsigned long long f = static_cast<unsigned long long>(idx[p]);
        const long long r = static_cast<long long>((f / static_cast<unsigned long long>(inner)) % static_cast<unsigned long long>(len));
        acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(val[p]), M[q + static_cast<long long>(J) * r]));
    }
    const unsigned long long k = ukey[run];
    const long long a = static_cast<long long>(k % static_cast<unsigned long long>(inner));
    const long long c = static_cast<long long>(k / static_cast<unsigned long long>(inner));
    y[a + inner * (q + static_cast<long long>(J) * c)] = acc;
}

template <typename T, typename IdxT>
void run(Ctx* ctx, const mach_sparse* s, int mode, const double* M, int J, double* y) {
    const Split sp = split_at(s->dims, mode);
    const long long nnz = s->nnz;
    const long long total = sp.inner * J * sp.outer;
    MB_CUDA(cudaMemsetAsync(y, 0, static_cast<std::size_t>(total) * sizeof(double), ctx->stream));
    if (nnz == 0) return;
    if (nnz >= (1ll << 31)) throw Error(MACH_ERR_INTERNAL, "sparse mode_product: more than 2^31 nonzeros");
    const IdxT* idx = static_cast<const IdxT*>(s->idx);
    const T* val = static_cast<const T*>(s->val);
    DBuf<unsigned long long> k0(ctx, nnz), k1(ctx, nnz), uk(ctx, nnz);
    DBuf<unsigned> p0(ctx, nnz), p1(ctx, nnz);
    DBuf<int> cnt(ctx, nnz), st(ctx, nnz), nrun(ctx, 1);
    MB_LAUNCH(ctx, (fibre_key_kernel<IdxT>), ceil_div(nnz, 256), 256, 0, idx, nnz, sp.inner, static_cast<long long>(sp.len),
              k0.get(), p0.get());
    const unsigned long long maxkey = static_cast<unsigned long long>(sp.outer) * static_cast<unsigned long long>(sp.inner);
    int bits = 1;
    while (bits < 64 && (1ull << bits) < maxkey) ++bits;
    std::size_t t1 = 0, t2 = 0, t3 = 0;
    MB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t1, k0.get(), k1.get(), p0.get(), p1.get(), static_cast<int>(nnz), 0, bits,
                                            ctx->stream));
    MB_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, t2, k1.get(), uk.get(), cnt.get(), nrun.get(), static_cast<int>(nnz),
                                               ctx->stream));
    MB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t3, cnt.get(), st.get(), static_cast<int>(nnz), ctx->stream));
    DBuf<unsigned char> tmp(ctx, std::max(t1, std::max(t2, t3)));
    MB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), t1, k0.get(), k1.get(), p0.get(), p1.get(), static_cast<int>(nnz), 0, bits,
                                            ctx->stream));
    MB_CUDA(cub::DeviceRunLengthEncode::Encode(tmp.get(), t2, k1.get(), uk.get(), cnt.get(), nrun.get(), static_cast<int>(nnz),
                                               ctx->stream));
    // counts past the last run are never read by the accumulate kernel; the
    // scan runs over nnz entries so it needs no host read of the run count
    MB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), t3, cnt.get(), st.get(), static_cast<int>(nnz), ctx->stream));
    MB_LAUNCH(ctx, (fibre_accumulate_kernel<T, IdxT>), ceil_div(nnz * J, 256), 256, 0, uk.get(), st.get(), cnt.get(),
              nrun.get(), p1.get(), idx, val, sp.inner, static_cast<long long>(sp.len), J, M, y);
}

}  // namespace

// M: J x len column-major (the reference's Matrix), on the device
void sparse_mode_product(Ctx* ctx, const mach_sparse* s, int mode, const double* M, int J, double* y) {
    if (s->dtype == MACH_F32) {
        if (s->idx64) run<float, unsigned long long>(ctx, s, mode, M, J, y);
        else run<float, unsigned>(ctx, s, mode, M, J, y);
    } else {
        if (s->idx64) run<double, unsigned long long>(ctx, s, mode, M, J, y);
        else run<double, unsigned>(ctx, s, mode, M, J, y);
    }
}

}  // namespace machb
