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

// One CTA per tile of kThreads x NV vectors x VEC elements; element order in
// the tile is (v, thread, j) = ascending flat index, so the exclusive scan of
// the per-(v, thread) kept counts gives every kept element its output slot.
// The design is latency hiding by occupancy (measured best on B200: a plain
// streaming hash reaches ~0.52 of HBM only with 6-8 resident CTAs per SM):
// few registers, no shared-memory staging, no per-tile pipeline state.
//   - a ticket orders the tiles (the look-back only waits on tiles that
//     started earlier);
//   - all NV 16-byte vectors are loaded first, then the SplitMix64 rounds run
//     on 32-bit halves; keep iff the hash's high word is below the
//     threshold's, with an exact 64-bit compare on a high-word tie
//     (probability 2^-32 per element);
//   - packed per-v counts (16-bit fields) are scanned with warp shuffles and
//     one pass over the warp totals; the tile's aggregate is published and
//     warp 0 runs the decoupled look-back (relaxed polls: the status word
//     carries its own payload);
//   - each thread writes its kept (index, x / p) straight from registers:
//     for one v the warp's kept entries are contiguous in the output.
// x / p is the reference's correctly rounded fp64 division (sampling.cpp:28):
// for fp32 data through Markstein's correction (y = RN(1/p), q = RN(x y),
// r = x - q p exactly by FMA, RN(q + r y) = RN(x / p) for these ranges),
// for fp64 data through __ddiv_rn.
template <typename T>
__device__ __forceinline__ T scaled(T xv, double p, double inv_p) {
    if constexpr (sizeof(T) == 4) {
        const double xd = static_cast<double>(xv);
        const double q = xd * inv_p;
        const double r = fma(-q, p, xd);
        return static_cast<T>(fma(r, inv_p, q));
    } else {
        return __ddiv_rn(xv, p);
    }
}

template <typename T, typename IdxT>
__global__ void __launch_bounds__(kThreads, 5) sample_kernel(const T* __restrict__ x, std::int64_t numel,
                                                          std::int64_t gofs,  // global flat index of x[0]
                                                          std::uint64_t seed, std::uint64_t thr_shift,
                                                          int keep_all, double p, double inv_p,
                                                          IdxT* __restrict__ out_idx, T* __restrict__ out_val,
                                                          std::int64_t capacity,
                                                          unsigned long long* __restrict__ status,
                                                          unsigned int* __restrict__ ticket,
                                                          long long* __restrict__ total_out,
                                                          int* __restrict__ flags) {
    using V = Vec<T>;
    constexpr int VEC = V::n;
    constexpr int NV = 4;
    constexpr int TILE = kThreads * NV * VEC;
    constexpr int NW = kThreads / 32;
    __shared__ unsigned long long s_wtot[NW];
    __shared__ long long s_excl;
    __shared__ unsigned s_tile;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const std::int64_t tile = s_tile;
    const std::int64_t base = tile * TILE;
    const bool full = base + TILE <= numel;
    T vals[NV][VEC];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const std::int64_t e0 = base + (static_cast<std::int64_t>(v) * kThreads + tid) * VEC;
        if (full) {
            V::unpack(__ldcs(reinterpret_cast<const typename V::type*>(x + e0)), vals[v]);
        } else {
#pragma unroll
            for (int j = 0; j < VEC; ++j) vals[v][j] = (e0 + j < numel) ? x[e0 + j] : T(0);
        }
    }
    const unsigned thr_hi = static_cast<unsigned>(thr_shift >> 32);
    unsigned keep = 0;  // bit v * VEC + j
    bool tie = false;
    T nanacc = T(0);  // x * 0 is NaN exactly for inf / NaN inputs
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const std::int64_t e0 = base + (static_cast<std::int64_t>(v) * kThreads + tid) * VEC;
        // z_j = seed + (i + 1) * golden for consecutive i
        const std::uint64_t z0 = seed + (static_cast<std::uint64_t>(gofs + e0) + 1ull) * 0x9E3779B97F4A7C15ULL;
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
            const T xv = vals[v][j];
            nanacc = fma(xv, T(0), nanacc);
            const std::uint64_t z = z0 + static_cast<std::uint64_t>(j) * 0x9E3779B97F4A7C15ULL;
            const unsigned zl = static_cast<unsigned>(z), zh = static_cast<unsigned>(z >> 32);
            const unsigned al = zl ^ __funnelshift_r(zl, zh, 30), ah = zh ^ (zh >> 30);
            const std::uint64_t pm = static_cast<std::uint64_t>(al) * 0x1CE4E5B9u;
            const unsigned yl = static_cast<unsigned>(pm);
            const unsigned yh = static_cast<unsigned>(pm >> 32) + al * 0xBF58476Du + ah * 0x1CE4E5B9u;
            const unsigned bl = yl ^ __funnelshift_r(yl, yh, 27), bh = yh ^ (yh >> 27);
            const unsigned zhi = __umulhi(bl, 0x133111EBu) + bl * 0x94D049BBu + bh * 0x133111EBu;
            const unsigned hhi = zhi ^ (zhi >> 31);
            const bool live = (xv != T(0)) & (full || e0 + j < numel);
            if (live & (keep_all | (hhi < thr_hi))) keep |= 1u << (v * VEC + j);
            tie |= live & (hhi == thr_hi);
        }
    }
    if (tie && !keep_all) {  // exact 64-bit comparison for the rare high-word ties
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const std::int64_t e0 = base + (static_cast<std::int64_t>(v) * kThreads + tid) * VEC;
#pragma unroll
            for (int j = 0; j < VEC; ++j) {
                if (vals[v][j] == T(0) || !(full || e0 + j < numel)) continue;
                const std::uint64_t h = splitmix_finalize(seed + (static_cast<std::uint64_t>(gofs + e0 + j) + 1ull) * 0x9E3779B97F4A7C15ULL);
                if (h < thr_shift) keep |= 1u << (v * VEC + j);
            }
        }
    }
    if (nanacc != nanacc) atomicOr(flags, 1);
    // ---- per-v counts (16-bit fields), warp scan, warp totals ----
    unsigned long long packed = 0;
#pragma unroll
    for (int v = 0; v < NV; ++v)
        packed |= static_cast<unsigned long long>(__popc((keep >> (v * VEC)) & ((1u << VEC) - 1u))) << (16 * v);
    unsigned long long inc = packed;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) s_wtot[warp] = inc;
    __syncthreads();
    unsigned long long before = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        const unsigned long long t = s_wtot[w];
        before += (w < warp) ? t : 0ull;
        tot += t;
    }
    const unsigned long long excl_packed = before + inc - packed;
    unsigned tile_total = 0;
#pragma unroll
    for (int v = 0; v < NV; ++v) tile_total += static_cast<unsigned>((tot >> (16 * v)) & 0xFFFFull);
    if (tid < 32) {
        // ---- decoupled look-back (warp 0) ----
        long long excl = 0;
        if (tile == 0) {
            if (lane == 0) atomicExch(&status[0], kFlagPre | tile_total);
        } else {
            if (lane == 0) atomicExch(&status[tile], kFlagAgg | tile_total);
            std::int64_t look = tile - 1;
            while (true) {
                const std::int64_t j = look - lane;
                unsigned long long st = kFlagPre | 0ull;
                if (j >= 0) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(st) : "l"(status + j) : "memory");
                const bool unset = (st >> 62) == 0;
                if (__any_sync(0xffffffffu, unset)) continue;
                const unsigned pmask = __ballot_sync(0xffffffffu, (st & ~kValMask) == kFlagPre);
                long long mine = static_cast<long long>(st & kValMask);
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
    }
    __syncthreads();
    // ---- write kept (index, x / p) straight from registers ----
    const long long g0 = s_excl;
    if (g0 + tile_total > capacity) {
        if (tid == 0 && tile_total) atomicOr(flags, 2);
        return;
    }
    if (!keep) return;
    unsigned run = 0;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        unsigned o = run + static_cast<unsigned>((excl_packed >> (16 * v)) & 0xFFFFull);
        run += static_cast<unsigned>((tot >> (16 * v)) & 0xFFFFull);
        const std::int64_t e0 = base + (static_cast<std::int64_t>(v) * kThreads + tid) * VEC;
#pragma unroll
        for (int j = 0; j < VEC; ++j)
            if ((keep >> (v * VEC + j)) & 1u) {
                out_idx[g0 + o] = static_cast<IdxT>(gofs + e0 + j);
                out_val[g0 + o] = scaled<T>(vals[v][j], p, inv_p);
                ++o;
            }
    }
}

template <typename T, typename IdxT>
std::int64_t launch_sample(Ctx* ctx, const T* x, std::int64_t numel, std::int64_t gofs, std::uint64_t seed, double p,
                           std::int64_t capacity, IdxT* out_idx, T* out_val, int* flags_host) {
    constexpr int TILE = kThreads * 4 * Vec<T>::n;
    const std::int64_t ntiles = (numel + TILE - 1) / TILE;
    // threshold: keep iff (h >> 11) < ceil(p * 2^53)  <=>  h < ceil(p*2^53) << 11
    const double t53 = std::ceil(std::ldexp(p, 53));
    const bool keep_all = t53 >= 9007199254740992.0;  // p == 1
    const std::uint64_t thr = keep_all ? 0 : (static_cast<std::uint64_t>(t53) << 11);
    if (ntiles > 0x7fffffffll) throw_arg("tensor too large for one sampler launch");
    // scratch: status[ntiles] + ticket + total + flags, one allocation
    const std::size_t words = static_cast<std::size_t>(ntiles) + 4;
    DBuf<unsigned long long> scratch(ctx, words);
    scratch.zero(ctx);
    unsigned long long* status = scratch.get();
    unsigned int* ticket = reinterpret_cast<unsigned int*>(status + ntiles);
    long long* total = reinterpret_cast<long long*>(status + ntiles + 1);
    int* flags = reinterpret_cast<int*>(status + ntiles + 2);
    if (ntiles > 0)
        MB_LAUNCH(ctx, (sample_kernel<T, IdxT>), static_cast<unsigned>(ntiles), kThreads, 0, x, numel, gofs, seed, thr,
                  keep_all ? 1 : 0, p, 1.0 / p, out_idx, out_val, capacity, status, ticket, total, flags);
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
