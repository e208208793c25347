// MACH Bernoulli sampler (reference: proj/src/sampling.cpp:21-31 with the
// counter RNG of proj/src/internal.hpp:68-77).
//
// One streaming pass over the dense tensor in HBM.  Each element i is kept iff
// x_i != 0 and SplitMix64(seed, i) >> 11 < ceil(p * 2^53), which is exactly the
// reference's  counter_uniform01(seed, i) < p  (the top 53 bits of the hash are
// an integer u53 and u53 * 2^-53 < p  <=>  u53 < ceil(p * 2^53)).  Kept values
// are x_i / p computed as a correctly rounded fp64 division (the reference's
// v[i] / cfg.p) and rounded to the tensor dtype.
//
// Compaction is order preserving (ascending flat index, the canonical order of
// SparseTensor, tensor.cpp:78-96) with a single-pass decoupled look-back scan:
// tiles of 4096 (fp32) / 2048 (fp64) elements are claimed in order through an
// atomic ticket, each tile publishes its kept count, and the tile's outputs
// are staged in shared memory and written back coalesced.  The input is read
// exactly once.
#include <cub/block/block_scan.cuh>

#include <cmath>

#include "common.cuh"

namespace machb {

namespace {

constexpr int kThreads = 256;
constexpr std::uint64_t kFlagAgg = 1ull << 62;
constexpr std::uint64_t kFlagPre = 2ull << 62;
constexpr std::uint64_t kValMask = (1ull << 62) - 1;

__device__ __forceinline__ std::uint64_t splitmix_finalize(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

template <typename T>
struct Vec;
// per thread and vector: one 16-byte load (4 fp32 / 2 fp64 elements)
template <>
struct Vec<float> {
    using type = float4;
    static constexpr int per = 4;
    static constexpr int n = 4;
    __device__ static void unpack(const float4& v, float* o) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
};
template <>
struct Vec<double> {
    using type = double2;
    static constexpr int per = 2;
    static constexpr int n = 2;
    __device__ static void unpack(const double2& v, double* o) { o[0] = v.x; o[1] = v.y; }
};

__device__ __forceinline__ bool is_finite_bits(float x) { return (__float_as_uint(x) & 0x7f800000u) != 0x7f800000u; }
__device__ __forceinline__ bool is_finite_bits(double x) {
    return (static_cast<unsigned long long>(__double_as_longlong(x)) & 0x7ff0000000000000ull) != 0x7ff0000000000000ull;
}

// Tile = kThreads threads x NV vector loads x VEC elements.  Element order in
// the tile is (v, thread, j) which is ascending flat index, so an exclusive
// scan of the per-(v, thread) kept counts in that order gives each kept
// element its output slot.  The NV counts of a thread are packed into one u64
// (16-bit fields; a block-wide per-v total is <= kThreads * VEC <= 2048).
template <typename T, typename IdxT>
__global__ void __launch_bounds__(kThreads, 4) sample_kernel(const T* __restrict__ x, std::int64_t numel,
                                                          std::int64_t gofs,  // global flat index of x[0]
                                                          std::uint64_t seed, std::uint64_t thr_shift,
                                                          int keep_all, double p, IdxT* __restrict__ out_idx,
                                                          T* __restrict__ out_val, std::int64_t capacity,
                                                          unsigned long long* __restrict__ status,
                                                          unsigned int* __restrict__ ticket,
                                                          long long* __restrict__ total_out,
                                                          int* __restrict__ flags) {
    using V = Vec<T>;
    constexpr int VEC = V::n;
    constexpr int NV = 4;
    constexpr int TILE = kThreads * NV * VEC;
    using BlockScan = cub::BlockScan<unsigned long long, kThreads>;

    __shared__ typename BlockScan::TempStorage scan_tmp;
    extern __shared__ __align__(16) unsigned char s_dyn[];
    IdxT* s_idx = reinterpret_cast<IdxT*>(s_dyn);
    T* s_val = reinterpret_cast<T*>(s_dyn + TILE * sizeof(IdxT));
    __shared__ unsigned int s_tile;
    __shared__ long long s_excl;

    const int tid = threadIdx.x;
    if (tid == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const std::int64_t tile = s_tile;
    const std::int64_t base = tile * TILE;

    // ---- load (all vectors in flight first) + hash ----
    T vals[NV][VEC];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const std::int64_t e0 = base + (static_cast<std::int64_t>(v) * kThreads + tid) * VEC;
        if (e0 + VEC <= numel) {
#pragma unroll
            for (int l = 0; l < VEC / V::per; ++l) {
                const auto raw = __ldcs(reinterpret_cast<const typename V::type*>(x + e0) + l);
                V::unpack(raw, vals[v] + l * V::per);
            }
        } else {
#pragma unroll
            for (int j = 0; j < VEC; ++j) vals[v][j] = (e0 + j < numel) ? x[e0 + j] : T(0);
        }
    }
    unsigned keep_bits = 0;  // bit (v*VEC + j)
    unsigned tie_bits = 0;   // high word of the hash equal to the threshold's (exact check below)
    T nanacc = T(0);         // x * 0 is NaN exactly for inf / NaN inputs
    const unsigned thr_hi = static_cast<unsigned>(thr_shift >> 32);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const std::int64_t e0 = base + (static_cast<std::int64_t>(v) * kThreads + tid) * VEC;
        const std::int64_t rem = numel - e0;
        const int lim = rem >= VEC ? VEC : (rem > 0 ? static_cast<int>(rem) : 0);
        // z_j = seed + (i + 1) * golden for consecutive i: incremental adds.
        std::uint64_t z = seed + (static_cast<std::uint64_t>(gofs + e0) + 1ull) * 0x9E3779B97F4A7C15ULL;
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
            const T xv = vals[v][j];
            nanacc = fma(xv, T(0), nanacc);
            // keep iff hash < thr_shift.  The final xor-shift's high word needs
            // only the high word of the last product; the low words matter
            // only on a high-word tie (probability 2^-32), handled after.
            std::uint64_t y = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
            y ^= y >> 27;
            const unsigned ylo = static_cast<unsigned>(y), yhi = static_cast<unsigned>(y >> 32);
            const unsigned zhi = __umulhi(ylo, 0x133111EBu) + ylo * 0x94D049BBu + yhi * 0x133111EBu;
            const unsigned hhi = zhi ^ (zhi >> 31);
            const bool live = (xv != T(0)) & (j < lim);
            keep_bits |= static_cast<unsigned>(live & (keep_all | (hhi < thr_hi))) << (v * VEC + j);
            tie_bits |= static_cast<unsigned>(live & (hhi == thr_hi)) << (v * VEC + j);
            z += 0x9E3779B97F4A7C15ULL;
        }
    }
    if (tie_bits && !keep_all) {  // exact 64-bit comparison for the (rare) ties
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const std::int64_t e0 = base + (static_cast<std::int64_t>(v) * kThreads + tid) * VEC;
#pragma unroll
            for (int j = 0; j < VEC; ++j)
                if ((tie_bits >> (v * VEC + j)) & 1u) {
                    const std::uint64_t z = seed + (static_cast<std::uint64_t>(gofs + e0 + j) + 1ull) * 0x9E3779B97F4A7C15ULL;
                    if (splitmix_finalize(z) < thr_shift) keep_bits |= 1u << (v * VEC + j);
                }
        }
    }
    if (nanacc != nanacc) atomicOr(flags, 1);

    unsigned long long packed = 0;
#pragma unroll
    for (int v = 0; v < NV; ++v)
        packed |= static_cast<unsigned long long>(__popc((keep_bits >> (v * VEC)) & ((1u << VEC) - 1u))) << (16 * v);
    unsigned long long excl_packed, tot_packed;
    BlockScan(scan_tmp).ExclusiveSum(packed, excl_packed, tot_packed);

    unsigned offv[NV];
    unsigned run = 0;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        offv[v] = run + static_cast<unsigned>((excl_packed >> (16 * v)) & 0xFFFFu);
        run += static_cast<unsigned>((tot_packed >> (16 * v)) & 0xFFFFu);
    }
    const unsigned tile_total = run;
    // publish this tile's aggregate as early as possible (successors' look-back)
    if (tid == 0 && tile > 0) atomicExch(&status[tile], kFlagAgg | tile_total);

    // ---- stage kept entries (raw values) in shared memory in tile order ----
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        unsigned o = offv[v];
        const std::int64_t e0 = base + (static_cast<std::int64_t>(v) * kThreads + tid) * VEC;
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
            if ((keep_bits >> (v * VEC + j)) & 1u) {
                s_idx[o] = static_cast<IdxT>(gofs + e0 + j);
                s_val[o] = vals[v][j];
                ++o;
            }
        }
    }
    __syncthreads();

    if (tid < 32) {
        // ---- decoupled look-back (warp 0) ----
        const int lane = tid;
        long long excl = 0;
        if (tile == 0) {
            if (lane == 0) atomicExch(&status[0], kFlagPre | tile_total);
        } else {
            std::int64_t look = tile - 1;
            while (true) {
                const std::int64_t j = look - lane;
                unsigned long long s = kFlagPre | 0ull;
                if (j >= 0) asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(s) : "l"(status + j) : "memory");
                const bool unset = (s >> 62) == 0;
                if (__any_sync(0xffffffffu, unset)) continue;
                const unsigned pmask = __ballot_sync(0xffffffffu, (s & ~kValMask) == kFlagPre);
                long long mine = static_cast<long long>(s & kValMask);
                if (pmask) {
                    const int first = __ffs(pmask) - 1;
                    if (lane > first) mine = 0;
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, off);
                excl += mine;
                if (pmask) break;
                look -= 32;
            }
            if (lane == 0) atomicExch(&status[tile], kFlagPre | static_cast<unsigned long long>(excl + tile_total));
        }
        if (lane == 0) {
            s_excl = excl;
            const std::int64_t ntiles = (numel + TILE - 1) / TILE;
            if (tile == ntiles - 1) *total_out = excl + tile_total;
        }
    } else {
        // ---- meanwhile the other warps form x / p (correctly rounded fp64
        // division, sampling.cpp:28) for the staged entries, coalesced ----
        for (unsigned k = tid - 32; k < tile_total; k += kThreads - 32)
            s_val[k] = static_cast<T>(__ddiv_rn(static_cast<double>(s_val[k]), p));
    }
    __syncthreads();

    // ---- coalesced write-back ----
    const long long g0 = s_excl;
    if (g0 + tile_total > capacity) {
        if (tid == 0 && tile_total) atomicOr(flags, 2);
        return;
    }
    for (unsigned k = tid; k < tile_total; k += kThreads) {
        out_idx[g0 + k] = s_idx[k];
        out_val[g0 + k] = s_val[k];
    }
}

template <typename T, typename IdxT>
std::int64_t launch_sample(Ctx* ctx, const T* x, std::int64_t numel, std::int64_t gofs, std::uint64_t seed, double p,
                           std::int64_t capacity, IdxT* out_idx, T* out_val, int* flags_host) {
    constexpr int VEC = Vec<T>::n;
    constexpr int TILE = kThreads * 4 * VEC;  // NV = 4
    const std::int64_t ntiles = (numel + TILE - 1) / TILE;
    // threshold: keep iff (h >> 11) < ceil(p * 2^53)  <=>  h < ceil(p*2^53) << 11
    const double t53 = std::ceil(std::ldexp(p, 53));
    const bool keep_all = t53 >= 9007199254740992.0;  // p == 1
    const std::uint64_t thr = keep_all ? 0 : (static_cast<std::uint64_t>(t53) << 11);

    // scratch: status[ntiles] + ticket + total + flags, one allocation
    const std::size_t words = static_cast<std::size_t>(ntiles) + 4;
    DBuf<unsigned long long> scratch(ctx, words);
    scratch.zero(ctx);
    unsigned long long* status = scratch.get();
    unsigned int* ticket = reinterpret_cast<unsigned int*>(status + ntiles);
    long long* total = reinterpret_cast<long long*>(status + ntiles + 1);
    int* flags = reinterpret_cast<int*>(status + ntiles + 2);
    const std::size_t smem = static_cast<std::size_t>(TILE) * (sizeof(IdxT) + sizeof(T));
    static bool attr = false;
    if (!attr) {
        MB_CUDA(cudaFuncSetAttribute(sample_kernel<T, IdxT>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        attr = true;
    }
    if (ntiles > 0)
        MB_LAUNCH(ctx, (sample_kernel<T, IdxT>), static_cast<unsigned>(ntiles), kThreads, smem, x, numel, gofs, seed, thr,
                  keep_all ? 1 : 0, p, out_idx, out_val, capacity, status, ticket, total, flags);
    long long tot = 0;
    int fl = 0;
    to_host(ctx, &tot, total, 1);
    to_host(ctx, &fl, flags, 1);
    sync(ctx);
    *flags_host = fl;
    return tot;
}

}  // namespace

// Host entry: returns a new canonical sparse tensor in HBM.  With a slab, x
// holds the flat range [offset, offset + x->numel) of a tensor of dims gdims
// (a time slab under first-mode-fastest layout): the RNG counter and the
// stored index are the global flat index, so the kept set is exactly the
// full tensor's restricted to the slab.
mach_sparse* sample_slab(const mach_dense* x, const std::vector<int>& gdims, std::int64_t offset, double p,
                         std::uint64_t seed) {
    if (!(p > 0.0 && p <= 1.0)) throw_arg("p must be in (0, 1]");
    Ctx* ctx = x->ctx;
    auto out = std::make_unique<mach_sparse>();
    out->ctx = ctx;
    out->dtype = x->dtype;
    out->dims = gdims;
    out->numel = checked_size(gdims);
    if (offset < 0 || offset + x->numel > out->numel) throw Error(MACH_ERR_SHAPE, "slab exceeds the global tensor");
    out->idx64 = out->numel > 0xFFFFFFFFll;
    const int isz = out->idx64 ? 8 : 4;
    const int vsz = dtype_size(x->dtype);
    const double mean = p * static_cast<double>(x->numel);
    std::int64_t cap = static_cast<std::int64_t>(mean + 12.0 * std::sqrt(mean + 1.0) + 8192.0);
    if (cap > x->numel) cap = x->numel;
    for (int attempt = 0; attempt < 2; ++attempt) {
        void *di = nullptr, *dv = nullptr;
        if (cap > 0) {
            MB_CUDA(cudaMallocAsync(&di, static_cast<std::size_t>(cap) * isz, ctx->stream));
            MB_CUDA(cudaMallocAsync(&dv, static_cast<std::size_t>(cap) * vsz, ctx->stream));
        }
        int flags = 0;
        std::int64_t nnz = 0;
        if (x->dtype == MACH_F32) {
            if (out->idx64)
                nnz = launch_sample<float, unsigned long long>(ctx, static_cast<const float*>(x->data), x->numel, offset,
                                                               seed, p, cap, static_cast<unsigned long long*>(di),
                                                               static_cast<float*>(dv), &flags);
            else
                nnz = launch_sample<float, unsigned int>(ctx, static_cast<const float*>(x->data), x->numel, offset, seed,
                                                         p, cap, static_cast<unsigned int*>(di), static_cast<float*>(dv),
                                                         &flags);
        } else {
            if (out->idx64)
                nnz = launch_sample<double, unsigned long long>(ctx, static_cast<const double*>(x->data), x->numel,
                                                                offset, seed, p, cap,
                                                                static_cast<unsigned long long*>(di),
                                                                static_cast<double*>(dv), &flags);
            else
                nnz = launch_sample<double, unsigned int>(ctx, static_cast<const double*>(x->data), x->numel, offset,
                                                          seed, p, cap, static_cast<unsigned int*>(di),
                                                          static_cast<double*>(dv), &flags);
        }
        if (flags & 1) {
            if (di) cudaFreeAsync(di, ctx->stream);
            if (dv) cudaFreeAsync(dv, ctx->stream);
            throw_arg("tensor values must be finite");
        }
        if ((flags & 2) || nnz > cap) {
            if (di) cudaFreeAsync(di, ctx->stream);
            if (dv) cudaFreeAsync(dv, ctx->stream);
            cap = x->numel;  // rare: binomial tail beyond 12 sigma; retry with the hard bound
            continue;
        }
        out->nnz = nnz;
        out->idx = di;
        out->val = dv;
        return out.release();
    }
    throw Error(MACH_ERR_INTERNAL, "sampler capacity retry failed");
}

mach_sparse* sample_dense(const mach_dense* x, double p, std::uint64_t seed) { return sample_slab(x, x->dims, 0, p, seed); }

}  // namespace machb
