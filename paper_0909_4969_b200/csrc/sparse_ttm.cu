// Sparse route of the Tucker sweep: per-mode sorted layouts (built once per
// sampled tensor), the fused mode-n TTM chain, and the sparse HOSVD Grams.
//
// Reference path replaced (proj/src):
//   project_except(SparseTensor)   tucker.cpp:120-131  (sparse TTM tensor.cpp:241-259
//                                                      + dense TTM tensor.cpp:224-239
//                                                      + matricize tensor.cpp:180-200)
//   sparse_core                    tucker.cpp:71-75
//   sparse_row_gram / col_gram     sparse_kernels.cpp:21-67
//   sparse_matricization_times     sparse_kernels.cpp:69-80
//
// Layout for mode n (order d <= 3; a 2-way tensor gets a dummy mode of size 1):
// every nonzero carries a packed key  row | i_b | i_a  (row = i_n most
// significant, i_a least), sorted ascending, so one output row of Y_(n) is a
// contiguous run and, inside it, each mode-a fibre (fixed i_n, i_b) is a
// contiguous run.  Rows are cut into warp sub-tiles of <= 32*seg nonzeros.
//
// Kernel (one warp per sub-tile, no atomics, fixed summation order):
//   stage 1  each lane streams `seg` consecutive nonzeros from shared memory and
//            accumulates the fibre sum f = sum v * U_a[i_a, :]   (r_a FMAs/nnz)
//   stage 2  finished fibres are queued per lane; the warp drains the queue
//            collectively, accumulating f (x) U_b[i_b, :] into the row block
//   output   one partial row (C = r_a * r_b values) per sub-tile; a second tiny
//            kernel sums a row's partials in sub-tile order and writes Y_(n)
//            (I_n x C, column-major) directly in matricised layout.
#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "sparse_ttm.cuh"

namespace cg = cooperative_groups;

namespace machb {

namespace {


int bits_for(int n) {
    int b = 0;
    while ((1ll << b) < n) ++b;
    return b;
}

struct KeyFields {
    int nf = 0;
    int mode[4];
    int shift[4];
};

struct DimArr {
    int d;
    int dims[8];
};

// per-mode shift of the coordinate in the packed key (-1: not in the key)
struct ModeShift {
    int sh[8];
};

inline ModeShift mode_shift(const KeyFields& kf) {
    ModeShift ms;
    for (int m = 0; m < 8; ++m) ms.sh[m] = -1;
    for (int j = 0; j < kf.nf; ++j) ms.sh[kf.mode[j]] = kf.shift[j];
    return ms;
}

template <typename IdxT, typename K>
__global__ void build_keys_kernel(const IdxT* __restrict__ idx, long long nnz, DimArr da, ModeShift ms,
                                  K* __restrict__ out) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= nnz) return;
    unsigned long long key = 0;
    if (sizeof(IdxT) == 4) {  // 32-bit mixed-radix decode
        unsigned f = static_cast<unsigned>(idx[i]);
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            if (m >= da.d) break;
            const unsigned q = f / static_cast<unsigned>(da.dims[m]);
            const unsigned c = f - q * static_cast<unsigned>(da.dims[m]);
            f = q;
            if (ms.sh[m] >= 0) key |= static_cast<unsigned long long>(c) << ms.sh[m];
        }
    } else {
        unsigned long long f = static_cast<unsigned long long>(idx[i]);
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            if (m >= da.d) break;
            const unsigned long long q = f / static_cast<unsigned long long>(da.dims[m]);
            const unsigned long long c = f - q * static_cast<unsigned long long>(da.dims[m]);
            f = q;
            if (ms.sh[m] >= 0) key |= c << ms.sh[m];
        }
    }
    out[i] = static_cast<K>(key);
}

template <typename K>
__global__ void row_bounds_kernel(const K* __restrict__ keys, long long nnz, int shift, long long* __restrict__ rs,
                                  long long* __restrict__ re) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= nnz) return;
    const long long r = static_cast<long long>(static_cast<unsigned long long>(keys[i]) >> shift);
    if (i == 0 || (static_cast<unsigned long long>(keys[i - 1]) >> shift) != static_cast<unsigned long long>(r)) rs[r] = i;
    if (i == nnz - 1 || (static_cast<unsigned long long>(keys[i + 1]) >> shift) != static_cast<unsigned long long>(r))
        re[r] = i + 1;
}

// ---- TTM task layout -------------------------------------------------------
// fibre = run of equal key >> ba (row, i_b); each fibre is cut into
// ceil(len / kSegMax) balanced segments; a row's segments are grouped 32 to a
// task; inside a task the nonzeros are re-laid in jagged-diagonal order.
template <typename K>
__global__ void fibre_flag_kernel(const K* __restrict__ keys, long long nnz, int ba, unsigned char* __restrict__ flag) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= nnz) return;
    flag[i] = (i == 0 || (static_cast<unsigned long long>(keys[i]) >> ba) != (static_cast<unsigned long long>(keys[i - 1]) >> ba))
                  ? 1 : 0;
}

__global__ void piece_count_kernel(const long long* __restrict__ fs, long long F, long long nnz, long long* __restrict__ cnt) {
    const long long f = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (f > F) return;
    if (f == F) { cnt[f] = 0; return; }
    const long long len = (f + 1 < F ? fs[f + 1] : nnz) - fs[f];
    cnt[f] = (len + kSegMax - 1) / kSegMax;
}

template <typename K>
__global__ void piece_fill_kernel(const K* __restrict__ keys, const long long* __restrict__ fs, long long F, long long nnz,
                                  const long long* __restrict__ pbase, int ba, int bb, long long* __restrict__ pstart,
                                  int* __restrict__ plen, int* __restrict__ prow, int* __restrict__ pib) {
    const long long f = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (f >= F) return;
    const long long s = fs[f];
    const long long len = (f + 1 < F ? fs[f + 1] : nnz) - s;
    const unsigned long long key = static_cast<unsigned long long>(keys[s]);
    const int row = static_cast<int>(key >> (ba + bb));
    const int ib = static_cast<int>((key >> ba) & ((1ull << bb) - 1ull));
    const long long m = pbase[f + 1] - pbase[f];
    const long long q = len / m, r = len % m;
    long long off = s;
    for (long long k = 0; k < m; ++k) {
        const long long pl = q + (k < r ? 1 : 0);
        const long long p = pbase[f] + k;
        pstart[p] = off;
        plen[p] = static_cast<int>(pl);
        prow[p] = row;
        pib[p] = ib;
        off += pl;
    }
}

__global__ void piece_row_bounds_kernel(const int* __restrict__ prow, long long np, long long* __restrict__ rs,
                                        long long* __restrict__ re) {
    const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (p >= np) return;
    const int r = prow[p];
    if (p == 0 || prow[p - 1] != r) rs[r] = p;
    if (p == np - 1 || prow[p + 1] != r) re[r] = p + 1;
}

__global__ void task_counts_kernel(const long long* __restrict__ rs, const long long* __restrict__ re, int rows,
                                   int* __restrict__ cnt) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r > rows) return;
    cnt[r] = (r < rows) ? static_cast<int>((re[r] - rs[r] + 31) / 32) : 0;
}

__global__ void task_first_kernel(const int* __restrict__ prow, long long np, const long long* __restrict__ rs,
                                  const long long* __restrict__ re, const int* __restrict__ st_base,
                                  long long* __restrict__ first, TtmTask* __restrict__ tasks) {
    const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (p >= np) return;
    const int r = prow[p];
    const long long rank = p - rs[r];
    if (rank % 32) return;
    const long long t = st_base[r] + rank / 32;
    first[t] = p;
    TtmTask tk{};
    tk.row = r;
    tk.nseg = static_cast<int>(min(32ll, re[r] - p));
    tasks[t] = tk;
}

// One warp per task: sort the segments by length (descending, stable) so the
// running lanes of every step are a prefix, then write the jagged-diagonal
// layout.  The order inside each segment is free (a fibre sum), so each step
// is scheduled to keep the TTM kernel's factor-row gathers bank-conflict free:
// rows start at 16-byte unit 3*i_a mod 8 (48-byte stride for r <= 12 fp32), a
// 128-bit shared load is served per group of 8 lanes, and within a group the
// lanes greedily pick elements whose i_a mod 8 differ.
template <typename K, typename IA, typename T>
__global__ void jds_kernel(const K* __restrict__ keys, const T* __restrict__ vals, long long n_task,
                           const long long* __restrict__ first, const long long* __restrict__ pstart,
                           const int* __restrict__ plen, const int* __restrict__ pib, unsigned long long maska,
                           TtmTask* __restrict__ tasks, IA* __restrict__ ia_out, T* __restrict__ v_out,
                           int2* __restrict__ desc, int* __restrict__ pslot) {
    const long long t = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= n_task) return;
    TtmTask tk = tasks[t];
    const long long p0 = first[t];
    long long st0 = 0;
    int len0 = 0, ib0 = 0;
    if (lane < tk.nseg) {
        st0 = pstart[p0 + lane];
        len0 = plen[p0 + lane];
        ib0 = pib[p0 + lane];
    }
    int rank = 0;
    for (int o = 0; o < 32; ++o) {
        const int lo = __shfl_sync(0xffffffffu, len0, o);
        rank += (lo > len0) || (lo == len0 && o < lane);
    }
    if (pslot && lane < tk.nseg) pslot[p0 + lane] = static_cast<int>(t * 32 + rank);  // piece (key order) -> slot
    const long long base = __shfl_sync(0xffffffffu, st0, 0);
    // lane l takes the segment of rank l
    long long st = 0;
    int len = 0, ib = 0;
    for (int o = 0; o < 32; ++o) {
        const int ro = __shfl_sync(0xffffffffu, rank, o);
        const long long so = __shfl_sync(0xffffffffu, st0, o);
        const int lo = __shfl_sync(0xffffffffu, len0, o);
        const int bo = __shfl_sync(0xffffffffu, ib0, o);
        if (ro == lane) { st = so; len = lo; ib = bo; }
    }
    int maxlen = len, total = len;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
        total += __shfl_xor_sync(0xffffffffu, total, o);
    }
    unsigned cm[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) cm[c] = 0u;
    for (int e = 0; e < len; ++e) {
        const unsigned r = static_cast<unsigned>(static_cast<unsigned long long>(keys[st + e]) & maska);
#pragma unroll
        for (int c = 0; c < 8; ++c)
            if ((r & 7u) == static_cast<unsigned>(c)) cm[c] |= 1u << e;
    }
    unsigned rem = len >= 32 ? 0xffffffffu : ((1u << len) - 1u);
    long long ptr = base;
    const int grp = lane & ~7;
    unsigned short* joff = reinterpret_cast<unsigned short*>(desc + t * kDesc + 32);
    joff[lane] = static_cast<unsigned short>(total);  // positions >= maxlen: never read
    __syncwarp();
    for (int j = 0; j < maxlen; ++j) {
        const int aj = __popc(__ballot_sync(0xffffffffu, j < len));
        if (lane == 0) joff[j] = static_cast<unsigned short>(ptr - base);
        // which running lanes still hold a row of each residue: a lane takes,
        // among the residues still free in its group, the one fewest of the
        // lanes after it could use (then the one it holds most of) — the
        // plain first-free choice left the last lanes of a group without a
        // free residue twice as often (simulated on Poisson fibres: 0.60 ->
        // 0.42 extra wavefronts per gather wavefront; a per-step maximum
        // matching reaches 0.38)
        const bool run = j < len;
        const unsigned later = ((0xFEu << (lane & 7)) & 0xFFu) << grp;  // the lanes that lose ties to this one
        int key[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const unsigned mine = cm[c] & rem;
            const unsigned avc = __ballot_sync(0xffffffffu, run && mine != 0u);
            key[c] = mine ? __popc(avc & later) * 64 - __popc(mine) : (1 << 30);
        }
        // Rounds of propose / resolve inside each quarter instead of a
        // lane-after-lane pass: every unplaced lane proposes its best free
        // residue, the lowest lane among equal proposals wins, losers retry
        // against the updated free set (2-3 rounds as a rule); a lane with no
        // free residue left takes its first remaining element and conflicts.
        unsigned taken = 0u;
        int pick = 0;
        bool placed = !run;
        while (__any_sync(0xffffffffu, !placed)) {
            int bestkey = 1 << 30, prop = 8;
            unsigned pref = 0u;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                if (!((taken >> c) & 1u) && key[c] < bestkey) {
                    bestkey = key[c];
                    pref = cm[c] & rem;
                    prop = c;
                }
            }
            // lanes that are placed already, or have nothing free, do not compete
            const bool compete = !placed && prop < 8;
            const unsigned same = __match_any_sync(0xffffffffu, compete ? (grp | prop) : (0x100 | lane));
            const bool win = compete && (__ffs(static_cast<int>(same)) - 1) == lane;
            const bool forced = !placed && prop == 8;  // conflict: first remaining element
            if (win || forced) {
                const unsigned choose = win ? pref : rem;
                pick = __ffs(static_cast<int>(choose)) - 1;
                rem &= ~(1u << pick);
                placed = true;
            }
            unsigned won = win ? (1u << prop) : 0u;
            won |= __shfl_xor_sync(0xffffffffu, won, 1);
            won |= __shfl_xor_sync(0xffffffffu, won, 2);
            won |= __shfl_xor_sync(0xffffffffu, won, 4);
            taken |= won;
        }
        if (j < len) {
            const long long dst = ptr + lane;
            ia_out[dst] = static_cast<IA>(static_cast<unsigned long long>(keys[st + pick]) & maska);
            v_out[dst] = vals[st + pick];
        }
        ptr += aj;
    }
    desc[t * kDesc + lane] = make_int2(ib, len);
    if (lane == 0) {
        tk.base = base;
        tk.len = total;
        tk.maxlen = maxlen;
        tasks[t] = tk;
    }
}

}  // namespace
}  // namespace machb

#include "ttm_kernel.cuh"

namespace machb {
namespace {

template <typename T>
__global__ void reduce_partials_kernel(const T* __restrict__ P, const int* __restrict__ st_base, int rows, int C,
                                       T* __restrict__ Y) {
    pdl_enter();  // programmatic dependent launch: predecessor complete and visible
    // consecutive threads take consecutive columns of one row: the task
    // partials P[q][:] are read coalesced (the Y stores are strided)
    const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (idx >= static_cast<long long>(rows) * C) return;
    const int col = static_cast<int>(idx % C), row = static_cast<int>(idx / C);
    T s = T(0);
    for (int q = st_base[row]; q < st_base[row + 1]; ++q) s += P[static_cast<long long>(q) * C + col];
    Y[row + static_cast<long long>(col) * rows] = s;
}

// ---------------------------------------------------------------------------
// sparse Grams with deterministic 64-bit fixed-point accumulation
// ---------------------------------------------------------------------------
// row Gram: keys sorted with i_n in the low `bn` bits; a fibre is a run of
// equal key >> bn.  Pair (y <= x) of one fibre adds v_y v_x to G[i_y, i_x].
template <typename T, typename K>
__global__ void row_gram_kernel(const K* __restrict__ keys, const T* __restrict__ vals, long long nnz, int bn,
                                double scale, int n, unsigned long long* __restrict__ G) {
    const long long x = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (x >= nnz) return;
    const unsigned long long kx = static_cast<unsigned long long>(keys[x]);
    const unsigned long long up = kx >> bn;
    const int ix = static_cast<int>(kx & ((1ull << bn) - 1ull));
    const double vx = static_cast<double>(vals[x]);
    for (long long y = x; y >= 0; --y) {
        const unsigned long long ky = static_cast<unsigned long long>(keys[y]);
        if ((ky >> bn) != up) break;
        const int iy = static_cast<int>(ky & ((1ull << bn) - 1ull));
        const long long q = __double2ll_rn(static_cast<double>(vals[y]) * vx * scale);
        atomicAdd(&G[iy + static_cast<long long>(ix) * n], static_cast<unsigned long long>(q));
    }
}

__device__ __forceinline__ long long decode_col(unsigned long long k, const ColDecode& D) {
    long long c = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j)
        if (j < D.nf) c += static_cast<long long>((k >> D.shift[j]) & D.mask[j]) * D.stride[j];
    return c;
}

// column Gram: entries of one row of X_(n) are a run of equal key >> rsh in
// the mode-n TTM layout; the column comes from the other fields (ColDecode).
template <typename T, typename K>
__global__ void col_gram_kernel(const K* __restrict__ keys, const T* __restrict__ vals, long long nnz, int rsh,
                                ColDecode D, double scale, long long n, unsigned long long* __restrict__ G) {
    const long long x = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (x >= nnz) return;
    const unsigned long long kx = static_cast<unsigned long long>(keys[x]);
    const unsigned long long row = kx >> rsh;
    const long long cx = decode_col(kx, D);
    const double vx = static_cast<double>(vals[x]);
    for (long long y = x; y >= 0; --y) {
        const unsigned long long ky = static_cast<unsigned long long>(keys[y]);
        if ((ky >> rsh) != row) break;
        const long long cy = decode_col(ky, D);
        const long long lo = cx < cy ? cx : cy, hi = cx < cy ? cy : cx;
        const long long q = __double2ll_rn(static_cast<double>(vals[y]) * vx * scale);
        atomicAdd(&G[lo + hi * n], static_cast<unsigned long long>(q));
    }
}

__global__ void fixed_to_double_kernel(const unsigned long long* __restrict__ Gi, long long n, double inv_scale,
                                       double* __restrict__ G) {
    const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (idx >= n * n) return;
    const long long c = idx / n, r = idx - c * n;
    const long long lo = r < c ? r : c, hi = r < c ? c : r;
    G[idx] = static_cast<double>(static_cast<long long>(Gi[lo + hi * n])) * inv_scale;
}

// W = X_(n) V for the column-side HOSVD basis (sparse_kernels.cpp:69-80):
// one warp per row of X_(n), fixed-order reduction.
template <typename T, typename K, int KC>
__global__ void sparse_times_kernel(const K* __restrict__ keys, const T* __restrict__ vals,
                                    const long long* __restrict__ rs, const long long* __restrict__ re, int rows,
                                    ColDecode D, const double* __restrict__ V, long long vld, int kc,
                                    double* __restrict__ W) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= rows) return;
    double acc[KC];
#pragma unroll
    for (int c = 0; c < KC; ++c) acc[c] = 0.0;
    for (long long e = rs[warp] + lane; e < re[warp]; e += 32) {
        const long long col = decode_col(static_cast<unsigned long long>(keys[e]), D);
        const double v = static_cast<double>(vals[e]);
#pragma unroll
        for (int c = 0; c < KC; ++c)
            if (c < kc) acc[c] += v * V[col + c * vld];
    }
#pragma unroll
    for (int c = 0; c < KC; ++c) {
        double s = acc[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0 && c < kc) W[warp + static_cast<long long>(c) * rows] = s;
    }
}

template <typename K, typename T>
void sort_pairs(Ctx* ctx, const K* kin, K* kout, const T* vin, T* vout, long long n, int bits) {
    std::size_t tmp = 0;
    MB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, n, 0, bits, ctx->stream));
    DBuf<unsigned char> t(ctx, tmp);
    MB_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, kin, kout, vin, vout, n, 0, bits, ctx->stream));
    ctx->launches += 4;
}

DimArr dimarr(const std::vector<int>& dims) {
    DimArr da{};
    da.d = static_cast<int>(dims.size());
    for (int m = 0; m < da.d; ++m) da.dims[m] = dims[m];
    return da;
}

// Build packed keys for `fields` (least significant first) and sort (key, value)
// pairs.  Returns key width.
template <typename T>
void build_sorted(Ctx* ctx, const mach_sparse* X, const KeyFields& kf, int total_bits, bool key64, DBuf<unsigned char>& keys,
                  DBuf<unsigned char>& vals, bool need_sort) {
    const long long nnz = X->nnz;
    const DimArr da = dimarr(X->dims);
    const int ks = key64 ? 8 : 4;
    DBuf<unsigned char> kraw(ctx, static_cast<std::size_t>(nnz) * ks + 32);
    const int blocks = ceil_div(nnz, 256);
    const ModeShift ms = mode_shift(kf);
    if (nnz > 0) {
        if (X->idx64) {
            if (key64) MB_LAUNCH(ctx, (build_keys_kernel<unsigned long long, unsigned long long>), blocks, 256, 0,
                                 static_cast<const unsigned long long*>(X->idx), nnz, da, ms,
                                 reinterpret_cast<unsigned long long*>(kraw.get()));
            else MB_LAUNCH(ctx, (build_keys_kernel<unsigned long long, unsigned int>), blocks, 256, 0,
                           static_cast<const unsigned long long*>(X->idx), nnz, da, ms,
                           reinterpret_cast<unsigned int*>(kraw.get()));
        } else {
            if (key64) MB_LAUNCH(ctx, (build_keys_kernel<unsigned int, unsigned long long>), blocks, 256, 0,
                                 static_cast<const unsigned int*>(X->idx), nnz, da, ms,
                                 reinterpret_cast<unsigned long long*>(kraw.get()));
            else MB_LAUNCH(ctx, (build_keys_kernel<unsigned int, unsigned int>), blocks, 256, 0,
                           static_cast<const unsigned int*>(X->idx), nnz, da, ms,
                           reinterpret_cast<unsigned int*>(kraw.get()));
        }
    }
    vals.alloc(ctx, static_cast<std::size_t>(nnz) * sizeof(T) + 32);
    if (!need_sort || nnz == 0) {
        keys = std::move(kraw);
        if (nnz) MB_CUDA(cudaMemcpyAsync(vals.get(), X->val, nnz * sizeof(T), cudaMemcpyDeviceToDevice, ctx->stream));
        return;
    }
    keys.alloc(ctx, static_cast<std::size_t>(nnz) * ks + 32);
    const T* vin = static_cast<const T*>(X->val);
    T* vout = reinterpret_cast<T*>(vals.get());
    if (key64)
        sort_pairs(ctx, reinterpret_cast<const unsigned long long*>(kraw.get()), reinterpret_cast<unsigned long long*>(keys.get()),
                   vin, vout, nnz, total_bits);
    else
        sort_pairs(ctx, reinterpret_cast<const unsigned int*>(kraw.get()), reinterpret_cast<unsigned int*>(keys.get()), vin,
                   vout, nnz, total_bits);
}

int ra_bucket(int r) {
    if (r <= 4) return 4;
    if (r <= 8) return 8;
    if (r <= 10) return 10;
    if (r <= 12) return 12;
    if (r <= 16) return 16;
    if (r <= 20) return 20;
    if (r <= 24) return 24;
    return 32;
}

}  // namespace

int ttm_ra_bucket(int r) { return ra_bucket(r); }
int ttm_stride(int r, int elem_bytes) {
    const int vn = 16 / elem_bytes;
    const int rs = ((ra_bucket(r) + vn - 1) / vn) * vn;
    return ((rs / vn) & 1) ? rs : rs + vn;  // odd number of 16-byte units (bank spread)
}

bool sparse_fast_path_ok(const std::vector<int>& dims, const std::vector<int>& ranks) {
    const int d = static_cast<int>(dims.size());
    if (d < 2 || d > 4) return false;
    int bits = 0;
    for (int m = 0; m < d; ++m) {
        if (ranks[m] > 32) return false;
        bits += bits_for(dims[m]);
    }
    if (bits > 64) return false;
    if (d == 4) {
        // every mode's stage 2 (any choice of inner mode) must fit: the
        // composite i_b in an int and the per-row Z block in shared memory
        for (int n = 0; n < 4; ++n)
            for (int a = 0; a < 4; ++a) {
                if (a == n) continue;
                int r[2], k = 0;
                for (int m = 0; m < 4; ++m)
                    if (m != n && m != a) r[k++] = m;
                if (bits_for(dims[r[0]]) + bits_for(dims[r[1]]) > 30) return false;
                const int b1 = dims[r[0]] >= dims[r[1]] ? r[0] : r[1], b2 = b1 == r[0] ? r[1] : r[0];
                if (!stage2_4way_ok(dims, ranks, n, a, b1, b2)) return false;
            }
    }
    return true;
}

// Choose the innermost contracted mode for mode n by a FMA cost model:
// nnz * RA(r_a) for the fibre sums + expected fibres * r_a * r_b for stage 2
// (order 4: r_b = the larger rank of the two composite modes; the outer one
// is contracted once per (row, i_b2) group, see stage2_4way_kernel).
// Work model of mode n's TTM with inner (gathered) mode a: the nonzero
// stream's gathers plus the fibre sums' expansion (expected fibre count at
// the tensor's density).
double inner_cost(const mach_sparse* X, int n, const std::vector<int>& ranks, int a) {
    const int d = static_cast<int>(X->dims.size());
    const double dens = X->numel ? static_cast<double>(X->nnz) / static_cast<double>(X->numel) : 0.0;
    int rb = 1;
    for (int m = 0; m < d; ++m)
        if (m != n && m != a) rb = std::max(rb, ranks[m]);
    const double Ia = X->dims[a];
    const double fibres = (static_cast<double>(X->numel) / Ia) * (1.0 - std::pow(1.0 - dens, Ia));
    return static_cast<double>(X->nnz) * ra_bucket(ranks[a]) + fibres * ranks[a] * rb;
}

static int choose_inner(const mach_sparse* X, int n, const std::vector<int>& ranks, int avoid) {
    const int d = static_cast<int>(X->dims.size());
    if (d == 2) return 1 - n;
    int best = -1;
    double best_cost = 0;
    for (int a = 0; a < d; ++a) {
        if (a == n || a == avoid) continue;
        const double cost = inner_cost(X, n, ranks, a);
        if (best < 0 || cost < best_cost - 1e-9) { best = a; best_cost = cost; }
    }
    return best;
}

// TTM task layout of a sorted mode plan (see the kernels above).
template <typename T, typename K>
void build_ttm_layout_k(Ctx* ctx, long long nnz, ModePlan& P) {
    const K* keys = reinterpret_cast<const K*>(P.keys.get());
    const T* vals = reinterpret_cast<const T*>(P.vals.get());
    const int rows = P.rows;
    P.ia16 = P.ba <= 16;
    const std::size_t isz = P.ia16 ? 2 : 4;
    P.ia.alloc(ctx, static_cast<std::size_t>(nnz) * isz + 32);
    P.jv.alloc(ctx, static_cast<std::size_t>(nnz) * sizeof(T) + 32);
    P.st_base.alloc(ctx, rows + 1);
    if (nnz == 0) {
        P.st_base.zero(ctx);
        P.n_task = 0;
        P.tasks.alloc(ctx, 1);
        P.desc.alloc(ctx, kDesc);
        return;
    }
    // fibre starts
    DBuf<unsigned char> flag(ctx, nnz);
    MB_LAUNCH(ctx, fibre_flag_kernel<K>, ceil_div(nnz, 256), 256, 0, keys, nnz, P.ba, flag.get());
    DBuf<long long> fs(ctx, nnz);
    DBuf<long long> nf_d(ctx, 1);
    {
        thrust::counting_iterator<long long> cnt_it(0);
        std::size_t tmp = 0;
        MB_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, cnt_it, flag.get(), fs.get(), nf_d.get(), nnz, ctx->stream));
        DBuf<unsigned char> t(ctx, tmp);
        MB_CUDA(cub::DeviceSelect::Flagged(t.get(), tmp, cnt_it, flag.get(), fs.get(), nf_d.get(), nnz, ctx->stream));
        ctx->launches += 1;
    }
    long long F = 0;
    to_host(ctx, &F, nf_d.get(), 1);
    sync(ctx);
    // segments (pieces) of <= kSegMax nonzeros
    DBuf<long long> pc(ctx, F + 1), pbase(ctx, F + 1);
    MB_LAUNCH(ctx, piece_count_kernel, ceil_div(F + 1, 256), 256, 0, fs.get(), F, nnz, pc.get());
    {
        std::size_t tmp = 0;
        MB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, pc.get(), pbase.get(), F + 1, ctx->stream));
        DBuf<unsigned char> t(ctx, tmp);
        MB_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, pc.get(), pbase.get(), F + 1, ctx->stream));
        ctx->launches += 1;
    }
    long long NP = 0;
    to_host(ctx, &NP, pbase.get() + F, 1);
    sync(ctx);
    DBuf<long long> pstart(ctx, NP);
    DBuf<int> plen(ctx, NP), prow(ctx, NP), pib(ctx, NP);
    // (order 4 keeps pib: moved into the plan below, after the layout is built)
    MB_LAUNCH(ctx, piece_fill_kernel<K>, ceil_div(F, 256), 256, 0, keys, fs.get(), F, nnz, pbase.get(), P.ba, P.bb,
              pstart.get(), plen.get(), prow.get(), pib.get());
    // tasks: 32 consecutive segments of one row
    DBuf<long long> prs(ctx, rows), pre(ctx, rows);
    prs.zero(ctx);
    pre.zero(ctx);
    MB_LAUNCH(ctx, piece_row_bounds_kernel, ceil_div(NP, 256), 256, 0, prow.get(), NP, prs.get(), pre.get());
    if (P.keep_pieces) {  // order 4: the key-ordered piece list drives stage 2 (stage2_4way_kernel)
        P.n_piece = NP;
        P.pslot.alloc(ctx, std::max<long long>(1, NP));
        P.piece_rs.alloc(ctx, rows);
        P.piece_re.alloc(ctx, rows);
        MB_CUDA(cudaMemcpyAsync(P.piece_rs.get(), prs.get(), rows * sizeof(long long), cudaMemcpyDeviceToDevice, ctx->stream));
        MB_CUDA(cudaMemcpyAsync(P.piece_re.get(), pre.get(), rows * sizeof(long long), cudaMemcpyDeviceToDevice, ctx->stream));
    }
    DBuf<int> tc(ctx, rows + 1);
    MB_LAUNCH(ctx, task_counts_kernel, ceil_div(rows + 1, 256), 256, 0, prs.get(), pre.get(), rows, tc.get());
    {
        std::size_t tmp = 0;
        MB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, tc.get(), P.st_base.get(), rows + 1, ctx->stream));
        DBuf<unsigned char> t(ctx, tmp);
        MB_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, tc.get(), P.st_base.get(), rows + 1, ctx->stream));
        ctx->launches += 1;
    }
    int nt = 0;
    to_host(ctx, &nt, P.st_base.get() + rows, 1);
    sync(ctx);
    P.n_task = nt;
    P.tasks.alloc(ctx, std::max(1, nt));
    P.desc.alloc(ctx, static_cast<std::size_t>(std::max(1, nt)) * kDesc);
    DBuf<long long> first(ctx, std::max(1, nt));
    MB_LAUNCH(ctx, task_first_kernel, ceil_div(NP, 256), 256, 0, prow.get(), NP, prs.get(), pre.get(), P.st_base.get(),
              first.get(), P.tasks.get());
    const unsigned long long maska = (1ull << P.ba) - 1ull;
    if (P.ia16)
        MB_LAUNCH(ctx, (jds_kernel<K, unsigned short, T>), ceil_div(static_cast<long long>(nt) * 32, 256), 256, 0, keys, vals,
                  static_cast<long long>(nt), first.get(), pstart.get(), plen.get(), pib.get(), maska, P.tasks.get(),
                  reinterpret_cast<unsigned short*>(P.ia.get()), reinterpret_cast<T*>(P.jv.get()), P.desc.get(),
                  P.pslot.get());
    else
        MB_LAUNCH(ctx, (jds_kernel<K, unsigned int, T>), ceil_div(static_cast<long long>(nt) * 32, 256), 256, 0, keys, vals,
                  static_cast<long long>(nt), first.get(), pstart.get(), plen.get(), pib.get(), maska, P.tasks.get(),
                  reinterpret_cast<unsigned int*>(P.ia.get()), reinterpret_cast<T*>(P.jv.get()), P.desc.get(),
                  P.pslot.get());
    if (P.keep_pieces) P.pib = std::move(pib);
}

template <typename T>
void build_ttm_layout(Ctx* ctx, long long nnz, ModePlan& P) {
    if (P.key64) build_ttm_layout_k<T, unsigned long long>(ctx, nnz, P);
    else build_ttm_layout_k<T, unsigned int>(ctx, nnz, P);
}

template <typename T>
std::shared_ptr<ModePlan> get_plan(mach_sparse* X, int n, const std::vector<int>& ranks, int force_a) {
    Ctx* ctx = X->ctx;
    if (X->plans.size() != X->dims.size()) X->plans.assign(X->dims.size(), nullptr);
    const int d = static_cast<int>(X->dims.size());
    // force_a >= 0 fixes the inner mode; force_a <= -2 excludes mode -force_a - 2
    const int avoid = force_a <= -2 ? -force_a - 2 : -1;
    const int a = (force_a >= 0 && force_a < d && force_a != n) ? force_a : choose_inner(X, n, ranks, avoid);
    // composite i_b: the remaining modes, inner first.  Order 4: the mode
    // with the smaller extent is outer (b2: its per-row partial block is
    // staged in shared memory by stage 2)
    std::vector<int> rest;
    for (int m = 0; m < d; ++m)
        if (m != n && m != a) rest.push_back(m);
    if (rest.size() == 2 && X->dims[rest[0]] < X->dims[rest[1]]) std::swap(rest[0], rest[1]);
    const int b = rest.empty() ? -1 : rest[0];
    auto& slot = X->plans[static_cast<std::size_t>(n)];
    if (slot && slot->a == a) return slot;
    auto P = std::make_shared<ModePlan>();
    P->mode = n;
    P->a = a;
    P->b = b;
    P->bmodes = rest;
    P->ba = bits_for(X->dims[a]);
    P->bb = 0;
    for (int m : rest) P->bb += bits_for(X->dims[m]);
    const int bn = bits_for(X->dims[n]);
    const int total = P->ba + P->bb + bn;
    P->key64 = total > 32;
    KeyFields kf{};
    kf.nf = 0;
    kf.mode[kf.nf] = a; kf.shift[kf.nf++] = 0;
    int sh = P->ba;
    for (int m : rest) { kf.mode[kf.nf] = m; kf.shift[kf.nf++] = sh; sh += bits_for(X->dims[m]); }
    kf.mode[kf.nf] = n; kf.shift[kf.nf++] = P->ba + P->bb;
    P->nf = kf.nf;
    for (int j = 0; j < kf.nf; ++j) { P->fmode[j] = kf.mode[j]; P->fshift[j] = kf.shift[j]; }
    P->keep_pieces = d == 4;
    // the sampler's flat order already is (i_{d-1}, ..., i_0) lexicographic
    bool natural = true;
    for (int j = 0; j < kf.nf; ++j) natural = natural && kf.mode[j] == j;
    static const bool tdbg = std::getenv("MACH_DEBUG_SETUP") != nullptr;
    auto tnow = [&]() {
        if (!tdbg) return 0.0;
        sync(ctx);
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
    };
    const double t0 = tnow();
    build_sorted<T>(ctx, X, kf, total, P->key64, P->keys, P->vals, !natural);
    const double t1 = tnow();

    const int rows = X->dims[n];
    P->rows = rows;
    P->row_start.alloc(ctx, rows);
    P->row_end.alloc(ctx, rows);
    P->row_start.zero(ctx);
    P->row_end.zero(ctx);
    const long long nnz = X->nnz;
    if (nnz > 0) {
        if (P->key64) MB_LAUNCH(ctx, row_bounds_kernel<unsigned long long>, ceil_div(nnz, 256), 256, 0,
                                reinterpret_cast<const unsigned long long*>(P->keys.get()), nnz, P->ba + P->bb,
                                P->row_start.get(), P->row_end.get());
        else MB_LAUNCH(ctx, row_bounds_kernel<unsigned int>, ceil_div(nnz, 256), 256, 0,
                       reinterpret_cast<const unsigned int*>(P->keys.get()), nnz, P->ba + P->bb, P->row_start.get(),
                       P->row_end.get());
    }
    const double t2 = tnow();
    build_ttm_layout<T>(ctx, nnz, *P);
    const double t3 = tnow();
    if (tdbg) std::fprintf(stderr, "[setup] mode %d a=%d: sort %.3f ms, bounds %.3f ms, layout %.3f ms\n", n, a, t1 - t0,
                           t2 - t1, t3 - t2);
    slot = P;
    return P;
}

template <typename T, typename IA, int RA>
static void launch_ttm(Ctx* ctx, TtmArgs<T, IA> A, int max_ctas) {
    constexpr int VN = 16 / static_cast<int>(sizeof(T));
    constexpr int RS = ((RA + VN - 1) / VN) * VN;
    constexpr int RSS = ((RS / VN) & 1) ? RS : RS + VN;
    using L = ttm::RingLayout<T, IA, RS>;
    const std::size_t budget = 227 * 1024;
    std::size_t fac = ttm::al16(static_cast<std::size_t>(A.ua_rows * RSS + A.ub_elems) * sizeof(T));
    A.fac_smem = L::bytes(fac, 6, 4) <= budget ? 1 : 0;
    if (!A.fac_smem) fac = 0;
    A.fac_bytes = fac;
    // consumer warps W and ring slots S: S is a multiple of W (>= 2W) so slot
    // q is always drained by warp q mod W, which takes its rounds in order and
    // so never waits on a parity two phases ahead; S <= 32 (one producer lane
    // per slot).  Defaults favour the most warps that fit.
    static const int wmax = std::getenv("MACH_TTM_W") ? std::atoi(std::getenv("MACH_TTM_W")) : 16;
    int W = std::max(1, std::min(16, wmax)), S = 0;
    for (; W >= 1; --W) {
        S = (32 / W) * W;
        while (S >= 2 * W && L::bytes(fac, S, W) > budget) S -= W;
        if (S >= 2 * W && L::bytes(fac, S, W) <= budget) break;
    }
    A.n_cons = W;
    A.n_slot = S;
    static const int dbg = std::getenv("MACH_TTM_DBG") ? std::atoi(std::getenv("MACH_TTM_DBG")) : 0;
    A.dbg = dbg;
    const std::size_t smem = L::bytes(fac, S, W);
    auto kern = A.fac_smem ? ttm::ttm_mode_kernel<T, IA, RA, true> : ttm::ttm_mode_kernel<T, IA, RA, false>;
    MB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int sms = 148;
    MB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    const long long blocks = std::min<long long>(A.n_task, max_ctas > 0 ? std::min(max_ctas, sms) : sms);
    if (blocks <= 0) return;
    static const bool tsdbg = std::getenv("MACH_TTM_TS") != nullptr;
    DBuf<unsigned long long> tsb;
    if (tsdbg) {
        tsb.alloc(ctx, 8 * blocks);
        tsb.zero(ctx);
        A.ts = tsb.get();
    }
    if (A.fac_smem)
        MB_LAUNCH_PDL(ctx, (ttm::ttm_mode_kernel<T, IA, RA, true>), static_cast<unsigned>(blocks), (W + 1) * 32, smem, A);
    else
        MB_LAUNCH_PDL(ctx, (ttm::ttm_mode_kernel<T, IA, RA, false>), static_cast<unsigned>(blocks), (W + 1) * 32, smem, A);
    if (tsdbg) {
        std::vector<unsigned long long> h(8 * blocks);
        to_host(ctx, h.data(), tsb.get(), h.size());
        sync(ctx);
        unsigned long long t0 = ~0ull;
        for (long long b = 0; b < blocks; ++b) t0 = std::min(t0, h[8 * b]);
        double mean[5] = {0, 0, 0, 0, 0}, mx[5] = {0, 0, 0, 0, 0};
        for (long long b = 0; b < blocks; ++b)
            for (int k = 0; k < 5; ++k) {
                const double v = (h[8 * b + k] - t0) * 1e-3;
                mean[k] += v / blocks;
                mx[k] = std::max(mx[k], v);
            }
        std::fprintf(stderr, "[ttm-ts] W=%d S=%d tasks=%lld  mean/max us: entry %.1f/%.1f init %.1f/%.1f prod %.1f/%.1f "
                     "fac %.1f/%.1f cons %.1f/%.1f\n", W, S, A.n_task, mean[0], mx[0], mean[1], mx[1], mean[2], mx[2],
                     mean[3], mx[3], mean[4], mx[4]);
    }
}

template <typename T, typename IA>
static void dispatch_ttm(Ctx* ctx, const TtmArgs<T, IA>& A, int rab, int max_ctas = 0) {
    switch (rab) {
        case 4: launch_ttm<T, IA, 4>(ctx, A, max_ctas); break;
        case 8: launch_ttm<T, IA, 8>(ctx, A, max_ctas); break;
        case 10: launch_ttm<T, IA, 10>(ctx, A, max_ctas); break;
        case 12: launch_ttm<T, IA, 12>(ctx, A, max_ctas); break;
        case 16: launch_ttm<T, IA, 16>(ctx, A, max_ctas); break;
        case 20: launch_ttm<T, IA, 20>(ctx, A, max_ctas); break;
        case 24: launch_ttm<T, IA, 24>(ctx, A, max_ctas); break;
        default: launch_ttm<T, IA, 32>(ctx, A, max_ctas); break;
    }
}

// Y_(n) (I_n x C, column-major, T) for the current factors.  Ur[m] are the
// row-major kernel copies (stride ttm_stride(r_m, sizeof(T))).
template <typename T>
void sparse_mode_ttm(Ctx* ctx, const ModePlan& P, const std::vector<int>& dims, const std::vector<int>& ranks,
                     const std::vector<const T*>& Ur, const T* one, T* Pbuf, T* Y, T* fseg, const int* fpos) {
    const int n = P.mode, a = P.a, b = P.b;
    const int ra = ranks[a];
    const int rb = (b >= 0) ? ranks[b] : 1;
    const int C = ra * rb;
    int sa, sb;
    if (b < 0) { sa = 1; sb = 0; }
    else if (a < b) { sa = 1; sb = ra; }
    else { sb = 1; sa = rb; }
    const int rab = ra_bucket(ra);
    auto fill = [&](auto& A) {
        A.vals = reinterpret_cast<const T*>(P.jv.get());
        A.tasks = P.tasks.get();
        A.desc = P.desc.get();
        A.n_task = P.n_task;
        A.Ua = Ur[a]; A.ra = ra;
        A.Ub = (b >= 0) ? Ur[b] : one; A.rb = rb; A.rbs = (b >= 0) ? ttm_stride(rb, sizeof(T)) : 1;
        A.sa = sa; A.sb = sb; A.C = C; A.P = Pbuf;
        A.ua_rows = dims[a];
        A.ub_elems = (b >= 0) ? static_cast<long long>(dims[b]) * A.rbs : 16 / static_cast<long long>(sizeof(T));
        A.fseg = fseg;
        A.fpos = fpos;
    };
    if (P.ia16) {
        TtmArgs<T, unsigned short> A{};
        A.ia = reinterpret_cast<const unsigned short*>(P.ia.get());
        fill(A);
        dispatch_ttm(ctx, A, rab);
    } else {
        TtmArgs<T, unsigned int> A{};
        A.ia = reinterpret_cast<const unsigned int*>(P.ia.get());
        fill(A);
        dispatch_ttm(ctx, A, rab);
    }
    const long long tot = static_cast<long long>(dims[n]) * C;
    MB_LAUNCH_PDL(ctx, reduce_partials_kernel<T>, ceil_div(tot, 256), 256, 0, Pbuf, P.st_base.get(), dims[n], C, Y);
}

// ---- Y_(b) from the previous mode's fibre sums ------------------------------
namespace {

__global__ void seg_keys_kernel(const TtmTask* __restrict__ tasks, const int2* __restrict__ desc, long long n_task,
                                int sentinel, int* __restrict__ key, int* __restrict__ id) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= n_task * 32) return;
    const long long t = i >> 5;
    const int lane = static_cast<int>(i & 31);
    key[i] = lane < tasks[t].nseg ? desc[t * kDesc + lane].x : sentinel;
    id[i] = static_cast<int>(i);
}

// ptr[r] = first position with key >= r (r = 0 .. rows)
__global__ void seg_bounds_kernel(const int* __restrict__ key, long long n, int rows, int* __restrict__ ptr) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r > rows) return;
    long long lo = 0, hi = n;
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (key[mid] < r) lo = mid + 1;
        else hi = mid;
    }
    ptr[r] = static_cast<int>(lo);
}

// inverse permutation (segment -> position) and each position's i_n
__global__ void seg_pos_kernel(const int* __restrict__ ids, long long n, const TtmTask* __restrict__ tasks,
                               int* __restrict__ pos, int* __restrict__ row) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const int s = ids[i];
    pos[s] = static_cast<int>(i);
    row[i] = tasks[s >> 5].row;
}

// One CTA per output row i_b.  The row's fibre sums and their i_n are
// contiguous (the TTM wrote them in i_b order) and U_n is small: all three
// arrive by 1-D TMA bulk copies (16-byte-aligned supersets of the ranges),
// chunk by chunk.  Thread t = g * ra + r_a (g < G groups) keeps the RN
// accumulators of Y_(b)[i_b, (r_a, 0 .. rn)] in registers and takes the
// chunk's segments j = g mod G (one fibre-sum value times one U_n row each);
// the G partial rows are summed in group order at the end (deterministic).
template <typename T, int RN>
__global__ void __launch_bounds__(512, 3) y_from_segments_kernel(const int* __restrict__ seg_ptr,
                                                              const int* __restrict__ seg_row, const T* __restrict__ fseg,
                                                              int ra, const T* __restrict__ Un, int rns, int rn, int sa,
                                                              int sn, int rows, int un_rows, int chunk, int ptr_mul,
                                                              int nbuf, T* __restrict__ Y) {
    // wait, then trigger: the overlapped stage 1 launched two kernels later
    // (which does not wait at entry) then starts only after this grid's
    // predecessors are complete: it cannot overwrite fibre sums or factor
    // copies still being read (see SparseSession::sweep_body)
    pdl_enter_strict();
    extern __shared__ __align__(128) unsigned char ysm[];
    __shared__ __align__(8) std::uint64_t bar[2];
    const int G = blockDim.x / ra;
    const int tid = threadIdx.x;
    const int g = tid / ra, r_a = tid - (tid / ra) * ra;
    const bool on = g < G;
    const std::size_t ub = static_cast<std::size_t>(un_rows) * rns * sizeof(T);  // multiple of 16
    // [U][nbuf fibre-sum chunks, later the group partials][nbuf i_n chunks]; nbuf = 2: the next chunk's bulk copies
    // fly while the current one is consumed (persistent CTAs with a large staged U: one CTA per SM)
    const std::size_t fcap = (static_cast<std::size_t>(chunk) * ra * sizeof(T) + 16 + 15) & ~std::size_t(15);
    const std::size_t rcap = (static_cast<std::size_t>(chunk) * sizeof(int) + 16 + 15) & ~std::size_t(15);
    T* sU = reinterpret_cast<T*>(ysm);
    unsigned char* sFb0 = ysm + ub;
    unsigned char* sRb0 = sFb0 + max(static_cast<std::size_t>(nbuf) * fcap,
                                     (static_cast<std::size_t>(G) * ra * rn * sizeof(T) + 15) & ~std::size_t(15));
    T* part = reinterpret_cast<T*>(sFb0);  // the group partials reuse the fibre-sum chunks once they are consumed
    if (tid == 0) {
        ttm::mbar_init(&bar[0], 1);
        ttm::mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    std::uint32_t phase[2] = {0u, 0u};
    bool ustaged = false;
    for (int row = blockIdx.x; row < rows; row += gridDim.x) {  // rows share the staged U
    const int s0 = seg_ptr[row] * ptr_mul, s1 = seg_ptr[row + 1] * ptr_mul;
    T acc[RN];
#pragma unroll
    for (int q = 0; q < RN; ++q) acc[q] = T(0);
    // chunk c of this row covers segments [s0 + c * chunk, ...); its copies are 16-byte-aligned supersets
    auto issue = [&](int base, int buf, bool with_u) {
        const int m = max(0, min(chunk, s1 - base));
        const unsigned char* fsrc = reinterpret_cast<const unsigned char*>(fseg + static_cast<long long>(base) * ra);
        const unsigned char* rsrc = reinterpret_cast<const unsigned char*>(seg_row + base);
        const unsigned char* f0 = reinterpret_cast<const unsigned char*>(reinterpret_cast<std::uintptr_t>(fsrc) & ~std::uintptr_t(15));
        const unsigned char* r0 = reinterpret_cast<const unsigned char*>(reinterpret_cast<std::uintptr_t>(rsrc) & ~std::uintptr_t(15));
        const std::uint32_t fb = static_cast<std::uint32_t>(((fsrc - f0) + static_cast<std::size_t>(m) * ra * sizeof(T) + 15) & ~std::size_t(15));
        const std::uint32_t rb = static_cast<std::uint32_t>(((rsrc - r0) + static_cast<std::size_t>(m) * sizeof(int) + 15) & ~std::size_t(15));
        const std::uint32_t ubytes = with_u && un_rows > 0 ? static_cast<std::uint32_t>(ub) : 0u;
        ttm::mbar_expect_tx(&bar[buf], ubytes + (m ? fb + rb : 0u));
        if (ubytes) ttm::bulk_g2s(sU, Un, ubytes, &bar[buf]);
        if (m) {
            ttm::bulk_g2s(sFb0 + buf * fcap, f0, fb, &bar[buf]);
            ttm::bulk_g2s(sRb0 + buf * rcap, r0, rb, &bar[buf]);
        }
    };
    if (tid == 0) issue(s0, 0, !ustaged);
    int buf = 0;
    for (int base = s0, first = 1; base < s1 || first; base += chunk, first = 0) {
        const int m = max(0, min(chunk, s1 - base));
        if (nbuf == 2 && tid == 0 && base + chunk < s1) issue(base + chunk, buf ^ 1, false);  // (its last readers passed the barrier below)
        ttm::mbar_wait(&bar[buf], phase[buf]);
        phase[buf] ^= 1u;
        ustaged = true;
        const unsigned char* fsrc = reinterpret_cast<const unsigned char*>(fseg + static_cast<long long>(base) * ra);
        const unsigned char* rsrc = reinterpret_cast<const unsigned char*>(seg_row + base);
        const T* sF = reinterpret_cast<const T*>(sFb0 + buf * fcap + (reinterpret_cast<std::uintptr_t>(fsrc) & 15));
        const int* sR = reinterpret_cast<const int*>(sRb0 + buf * rcap + (reinterpret_cast<std::uintptr_t>(rsrc) & 15));
        // two copies of the loop so the staged case compiles to shared-memory loads
        auto run = [&](const T* U) {
            for (int j = g; j < m; j += G) {
                const T fv = sF[j * ra + r_a];
                const T* ur = U + sR[j] * rns;
                if constexpr (sizeof(T) == 4 && RN % 4 == 0) {
                    // 128-bit row loads (rows are whole 16-byte units, zero padded)
#pragma unroll
                    for (int q = 0; q < RN; q += 4) {
                        if (q < rn) {
                            const float4 u4 = *reinterpret_cast<const float4*>(ur + q);
                            acc[q] = fmaf(fv, u4.x, acc[q]);
                            acc[q + 1] = fmaf(fv, u4.y, acc[q + 1]);
                            acc[q + 2] = fmaf(fv, u4.z, acc[q + 2]);
                            acc[q + 3] = fmaf(fv, u4.w, acc[q + 3]);
                        }
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < RN; ++q)
                        if (q < rn) acc[q] = fma(fv, ur[q], acc[q]);
                }
            }
        };
        if (on) {
            if (un_rows > 0) run(sU);
            else run(Un);
        }
        __syncthreads();  // this buffer may be refilled (by the issue two chunks ahead, or the next row's first)
        if (nbuf == 2) buf ^= 1;
        else if (tid == 0 && base + chunk < s1) issue(base + chunk, 0, false);
    }
    const int C = ra * rn;
    if (on)
#pragma unroll
        for (int q = 0; q < RN; ++q)
            if (q < rn) part[g * C + r_a + q * ra] = acc[q];
    __syncthreads();
    for (int cc = tid; cc < C; cc += blockDim.x) {
        T s = T(0);
        for (int q = 0; q < G; ++q) s += part[q * C + cc];
        const int a_ = cc % ra, n_ = cc / ra;
        Y[row + static_cast<long long>(a_ * sa + n_ * sn) * rows] = s;
    }
    __syncthreads();  // the next row's bulk copies overwrite the partials
    }
}

}  // namespace

bool build_segment_groups(Ctx* ctx, ModePlan& P, int b_rows) {
    if (P.b < 0) return false;
    if (P.seg_ptr.get()) return true;
    const long long nslot = P.n_task * 32;
    DBuf<int> key(ctx, nslot + 1), id(ctx, nslot + 1), skey(ctx, nslot + 1), sid(ctx, nslot + 1);
    P.seg_pos.alloc(ctx, nslot + 1);
    P.seg_row.alloc(ctx, nslot + 8);  // +8: bulk copies read 16-byte-aligned supersets
    P.seg_ptr.alloc(ctx, b_rows + 1);
    if (nslot > 0) {
        MB_LAUNCH(ctx, seg_keys_kernel, ceil_div(nslot, 256), 256, 0, P.tasks.get(), P.desc.get(), P.n_task, b_rows,
                  key.get(), id.get());
        std::size_t tmp = 0;
        const int bits = bits_for(b_rows + 1);
        MB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key.get(), skey.get(), id.get(), sid.get(), nslot, 0, bits,
                                                ctx->stream));
        DBuf<unsigned char> t(ctx, tmp);
        MB_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, key.get(), skey.get(), id.get(), sid.get(), nslot, 0, bits,
                                                ctx->stream));
        ctx->launches += 4;
        MB_LAUNCH(ctx, seg_pos_kernel, ceil_div(nslot, 256), 256, 0, sid.get(), nslot, P.tasks.get(), P.seg_pos.get(),
                  P.seg_row.get());
    }
    MB_LAUNCH(ctx, seg_bounds_kernel, ceil_div(b_rows + 1, 256), 256, 0, skey.get(), nslot, b_rows, P.seg_ptr.get());
    int nseg = 0;
    to_host(ctx, &nseg, P.seg_ptr.get() + b_rows, 1);
    sync(ctx);
    P.n_seg = nseg;
    return true;
}

template <typename T>
void y_from_segments(Ctx* ctx, ModePlan& P, const std::vector<int>& dims, const std::vector<int>& ranks, const T* fseg,
                     const T* Un, T* Y) {
    const int n = P.mode, a = P.a, b = P.b;
    const int rows = dims[b];
    build_segment_groups(ctx, P, rows);
    const int ra = ranks[a], rn = ranks[n];
    int sa, sn;  // Y_(b) columns: the two remaining modes, earliest fastest
    if (a < n) { sa = 1; sn = ra; }
    else { sn = 1; sa = rn; }
    const int threads = (512 / ra) * ra;  // whole groups of ra threads
    const int G = threads / ra;
    const int rns = ttm_stride(rn, sizeof(T));
    const std::size_t ubytes = static_cast<std::size_t>(dims[n]) * rns * sizeof(T);
    // U_n rows are staged in shared memory when they fit beside two resident
    // CTAs (C5: 1024 rows x 80 B = 80 KB; gathering them from L2 instead made
    // this kernel latency-bound); large staged copies run on a persistent grid
    // whose CTAs keep the copy across their rows
    static const std::size_t stage_max =
        std::getenv("MACH_S2_STAGE_MAX") ? static_cast<std::size_t>(std::atoll(std::getenv("MACH_S2_STAGE_MAX"))) : 80 * 1024;
    const bool stage = ubytes <= stage_max;
    const int chunk = static_cast<int>(std::min<std::size_t>(2048, (24 * 1024) / (ra * sizeof(T))));
    // shared memory: [U][fibre-sum chunk, later the group partials][i_n chunk]; ~55 KB at C2: four CTAs per SM
    // large staged U: one persistent CTA per SM, so its chunk loads are double-buffered against the compute
    const int nbuf = (stage && ubytes > 32 * 1024) ? 2 : 1;
    const std::size_t fcap = (static_cast<std::size_t>(chunk) * ra * sizeof(T) + 16 + 15) & ~std::size_t(15);
    const std::size_t rcap = (static_cast<std::size_t>(chunk) * sizeof(int) + 16 + 15) & ~std::size_t(15);
    const std::size_t fbytes = std::max(nbuf * fcap, (static_cast<std::size_t>(G) * ra * rn * sizeof(T) + 15) & ~std::size_t(15));
    const std::size_t smem = (stage ? ubytes : 0) + fbytes + nbuf * rcap;
    auto launch = [&](auto y_from_segments_kernel_rn) {  // (the name is the profiler's kernel label)
        auto kern = y_from_segments_kernel_rn;
        MB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        int grid = rows;
        if (stage && ubytes > 32 * 1024) {
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
            grid = std::min<int>(rows, sms * std::max<int>(1, static_cast<int>((227 * 1024) / (smem + 1024))));
        }
        MB_LAUNCH_PDL(ctx, y_from_segments_kernel_rn, grid, threads, smem, P.seg_ptr.get(), P.seg_row.get(), fseg, ra, Un, rns, rn, sa, sn, rows,
                  stage ? dims[n] : 0, chunk, 1, nbuf, Y);
    };
    // RN >= rn register accumulators
    if (rn <= 4) launch(y_from_segments_kernel<T, 4>);
    else if (rn <= 8) launch(y_from_segments_kernel<T, 8>);
    else if (rn <= 12) launch(y_from_segments_kernel<T, 12>);
    else if (rn <= 16) launch(y_from_segments_kernel<T, 16>);
    else if (rn <= 24) launch(y_from_segments_kernel<T, 24>);
    else launch(y_from_segments_kernel<T, 32>);
}

namespace {
__global__ void seg_ib_kernel(const TtmTask* __restrict__ tasks, const int2* __restrict__ desc, long long n_task,
                              int* __restrict__ ib) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= n_task * 32) return;
    const long long t = i >> 5;
    const int lane = static_cast<int>(i & 31);
    ib[i] = lane < tasks[t].nseg ? desc[t * kDesc + lane].x : 0;
}
}  // namespace

template <typename T>
void sparse_mode_stage1(Ctx* ctx, ModePlan& P, const std::vector<int>& dims, const std::vector<int>& ranks,
                        const std::vector<const T*>& Ur, T* F, int ctas, bool overlapped) {
    const int a = P.a;
    auto fill = [&](auto& A) {
        A.vals = reinterpret_cast<const T*>(P.jv.get());
        A.tasks = P.tasks.get();
        A.desc = P.desc.get();
        A.n_task = P.n_task;
        A.Ua = Ur[a]; A.ra = ranks[a];
        A.Ub = Ur[a]; A.rb = 1; A.rbs = 1;  // stage 2 does not run: no U_b
        A.sa = 1; A.sb = 0; A.C = ranks[a]; A.P = nullptr;
        A.ua_rows = dims[a];
        A.ub_elems = 0;
        A.fseg = F;
        A.fpos = nullptr;
        A.stage1 = overlapped ? 1 : 2;
    };
    const int rab = ra_bucket(ranks[a]);
    if (P.ia16) {
        TtmArgs<T, unsigned short> A{};
        A.ia = reinterpret_cast<const unsigned short*>(P.ia.get());
        fill(A);
        dispatch_ttm(ctx, A, rab, ctas);
    } else {
        TtmArgs<T, unsigned int> A{};
        A.ia = reinterpret_cast<const unsigned int*>(P.ia.get());
        fill(A);
        dispatch_ttm(ctx, A, rab, ctas);
    }
}

template <typename T>
void sparse_mode_stage2(Ctx* ctx, ModePlan& P, const std::vector<int>& dims, const std::vector<int>& ranks, const T* F,
                        const T* Ub, T* Y) {
    const int n = P.mode, a = P.a, b = P.b;
    const long long nslot = P.n_task * 32;
    if (!P.seg_ib.get()) {
        P.seg_ib.alloc(ctx, nslot + 8);  // +8: bulk copies read 16-byte-aligned supersets
        if (nslot > 0)
            MB_LAUNCH(ctx, seg_ib_kernel, ceil_div(nslot, 256), 256, 0, P.tasks.get(), P.desc.get(), P.n_task, P.seg_ib.get());
    }
    const int ra = ranks[a], rb = ranks[b];
    int sa, sb;  // Y_(n) columns: the two remaining modes, earliest fastest
    if (a < b) { sa = 1; sb = ra; }
    else { sb = 1; sa = rb; }
    const int rows = dims[n];
    const int threads = (512 / ra) * ra;
    const int G = threads / ra;
    const int rbs = ttm_stride(rb, sizeof(T));
    const std::size_t ubytes = static_cast<std::size_t>(dims[b]) * rbs * sizeof(T);
    // U_n rows are staged in shared memory when they fit beside two resident
    // CTAs (C5: 1024 rows x 80 B = 80 KB; gathering them from L2 instead made
    // this kernel latency-bound); large staged copies run on a persistent grid
    // whose CTAs keep the copy across their rows
    static const std::size_t stage_max =
        std::getenv("MACH_S2_STAGE_MAX") ? static_cast<std::size_t>(std::atoll(std::getenv("MACH_S2_STAGE_MAX"))) : 80 * 1024;
    const bool stage = ubytes <= stage_max;
    const int chunk = static_cast<int>(std::min<std::size_t>(2048, (24 * 1024) / (ra * sizeof(T))));
    const int nbuf = (stage && ubytes > 32 * 1024) ? 2 : 1;  // see y_from_segments
    const std::size_t fcap = (static_cast<std::size_t>(chunk) * ra * sizeof(T) + 16 + 15) & ~std::size_t(15);
    const std::size_t rcap = (static_cast<std::size_t>(chunk) * sizeof(int) + 16 + 15) & ~std::size_t(15);
    const std::size_t fbytes = std::max(nbuf * fcap, (static_cast<std::size_t>(G) * ra * rb * sizeof(T) + 15) & ~std::size_t(15));
    const std::size_t smem = (stage ? ubytes : 0) + fbytes + nbuf * rcap;
    auto launch = [&](auto y_from_segments_kernel_rn) {  // (the name is the profiler's kernel label)
        auto kern = y_from_segments_kernel_rn;
        MB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        static const int rpc = std::getenv("MACH_S2_RPC") ? std::atoi(std::getenv("MACH_S2_RPC")) : 1;  // rows per CTA (1 measured best)
        int grid = (rows + rpc - 1) / rpc;
        if (stage && ubytes > 32 * 1024) {  // persistent: each CTA stages the large U_b once
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
            grid = std::min<int>(grid, sms * std::max<int>(1, static_cast<int>((227 * 1024) / (smem + 1024))));
        }
        MB_LAUNCH_PDL(ctx, y_from_segments_kernel_rn, grid, threads, smem, P.st_base.get(), P.seg_ib.get(), F, ra, Ub, rbs,
                      rb, sa, sb, rows, stage ? dims[b] : 0, chunk, 32, nbuf, Y);
    };
    if (rb <= 4) launch(y_from_segments_kernel<T, 4>);
    else if (rb <= 8) launch(y_from_segments_kernel<T, 8>);
    else if (rb <= 12) launch(y_from_segments_kernel<T, 12>);
    else if (rb <= 16) launch(y_from_segments_kernel<T, 16>);
    else if (rb <= 24) launch(y_from_segments_kernel<T, 24>);
    else launch(y_from_segments_kernel<T, 32>);
}

// ---- order-4 stage 2 ---------------------------------------------------------
// Mode n of a 4-way tensor: stage 1 (the TTM kernel) leaves one fibre sum
// F = sum_{i_a} x U_a[i_a, :] per segment slot; the segment's composite i_b
// packs (i_b2 << bits(b1)) | i_b1.  Per row i_n of Y_(n):
//   Z[i_b2, (r_a, r_b1)] = sum over the row's segments with that i_b2 of
//                          F[r_a] * U_b1[i_b1, r_b1]
//   Y_(n)[i_n, (r_a, r_b1, r_b2)] = sum_{i_b2} Z[i_b2, (r_a, r_b1)] U_b2[i_b2, r_b2]
// (a dimension tree: the per-segment work is r_a r_b1, the r_b2 contraction
// runs once per (row, i_b2) on the dense Z).  One CTA per row; Z lives in
// shared memory; group g of E = r_a r_b1 threads owns the i_b2 range
// [g Ib2 / G, (g+1) Ib2 / G) and walks only the row's tasks overlapping it
// (a row's tasks are in key order, so i_b2 is nondecreasing across them; the
// per-task i_b2 range is precomputed).  Each Z element has one owner thread
// and the segments are taken in a fixed order: deterministic, no atomics.
namespace {
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<std::uint32_t>(__cvta_generic_to_shared(smem))),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<std::uint32_t>(__cvta_generic_to_shared(smem))),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// Per row the pieces (fibre segments) are kept in key order, i.e. sorted by
// (i_b2, i_b1), with the slot their fibre sum went to (pslot) and their
// composite i_b (pib).  The row is cut into R slices of i_b2 (CTAs; pieces
// found by binary search on pib) and every slice's piece range is split
// evenly over the CTA's warps.  A warp walks its pieces in batches of 32:
// lane l gathers piece l's fibre sum row (r_a contiguous values) into its
// strip of shared memory and the 32 composite i_b stay in a register; then,
// per piece (warp-uniform control), lane-owned Z elements e = lane + 32 j
// accumulate F[r_a] U_b1[i_b1, r_b1], and whenever i_b2 changes the Z block
// is folded into the warp's register partial of the Y row:
//   y[e, q] += z[e] U_b2[i_b2, q].
// The warps' partial rows are summed in warp order; with R > 1 the slices go
// through global memory and the last CTA of the row (ticket) sums them in
// slice order.  Fixed summation order throughout: deterministic.
template <typename T, int EPL, int RB2>
__global__ void __launch_bounds__(512) stage2_4way_kernel(const long long* __restrict__ prs, const long long* __restrict__ pre,
                                                          const int* __restrict__ pslot, const int* __restrict__ pib,
                                                          const T* __restrict__ F, int ra, int ras, int rb1, int rb2,
                                                          const T* __restrict__ Ub1, int rb1s, const T* __restrict__ Ub2,
                                                          int rb2s, int Ib1, int Ib2, int bits1, int sa, int sb1, int sb2,
                                                          int rows, int R, T* __restrict__ Ypart,
                                                          unsigned* __restrict__ ticket, T* __restrict__ Y) {
    pdl_enter_strict();
    extern __shared__ __align__(16) unsigned char s4raw[];
    __shared__ bool last;
    const int row = blockIdx.x / R, q = blockIdx.x - (blockIdx.x / R) * R;
    const int E = ra * rb1;
    const int C = E * rb2;
    const int W = blockDim.x >> 5;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int ea[EPL], eb[EPL];
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
        const int e = lane + 32 * j;
        ea[j] = e < E ? e % ra : 0;
        eb[j] = e < E ? e / ra : 0;
    }
    const int mask1 = (1 << bits1) - 1;
    const int c0 = static_cast<int>((static_cast<long long>(Ib2) * q) / R);
    const int c1 = static_cast<int>((static_cast<long long>(Ib2) * (q + 1)) / R);
    T* Us1 = reinterpret_cast<T*>(s4raw);                           // Ib1 x rb1s
    T* Us2 = Us1 + static_cast<std::size_t>(Ib1) * rb1s;            // Ib2 x rb2s
    T* Yw = Us2 + static_cast<std::size_t>(Ib2) * rb2s;             // W x C warp partials
    T* strip = Yw + static_cast<std::size_t>(W) * C + static_cast<std::size_t>(warp) * (2 * 32 * ras + 32 * 4 / sizeof(T));
    for (int i = tid; i < Ib1 * rb1s; i += blockDim.x) Us1[i] = Ub1[i];
    for (int i = tid; i < Ib2 * rb2s; i += blockDim.x) Us2[i] = Ub2[i];
    __syncthreads();
    T y[EPL][RB2];
#pragma unroll
    for (int j = 0; j < EPL; ++j)
#pragma unroll
        for (int k = 0; k < RB2; ++k) y[j][k] = T(0);
    if (row < rows) {
        // this slice's pieces: pib within the row is ascending
        const long long r0 = prs[row], r1 = pre[row];
        long long P0, P1;
        {
            long long lo = r0, hi = r1;
            const int key = c0 << bits1;
            while (lo < hi) { const long long m = (lo + hi) >> 1; if (pib[m] < key) lo = m + 1; else hi = m; }
            P0 = lo;
            hi = r1;
            const int key1 = c1 << bits1;
            while (lo < hi) { const long long m = (lo + hi) >> 1; if (pib[m] < key1) lo = m + 1; else hi = m; }
            P1 = lo;
        }
        const long long L = P1 - P0;
        const long long w0 = P0 + (L * warp) / W, w1 = P0 + (L * (warp + 1)) / W;
        int cur = -1;
        T z[EPL];
#pragma unroll
        for (int j = 0; j < EPL; ++j) z[j] = T(0);
        auto fold = [&]() {
            const T* u2 = Us2 + cur * rb2s;
#pragma unroll
            for (int k = 0; k < RB2; ++k) {
                if (k < rb2) {
                    const T u = u2[k];
#pragma unroll
                    for (int j = 0; j < EPL; ++j) y[j][k] = fma(z[j], u, y[j][k]);
                }
            }
#pragma unroll
            for (int j = 0; j < EPL; ++j) z[j] = T(0);
        };
        // software pipeline over batches of 32 pieces: batch b + 1's fibre-sum
        // rows are in flight (cp.async into the other strip) and batch b + 2's
        // indices in registers while batch b is consumed
        int* su = reinterpret_cast<int*>(strip + 2 * 32 * ras);  // the batch's U_b1 row offsets
        const int vec = (sizeof(T) == 4 && (ra & 3) == 0) ? 4 : 1;  // 16-byte copies when rows are whole units
        auto fetch = [&](long long base, int& ib, int& slot) {
            ib = -1;
            slot = 0;
            if (base < w1 && lane < static_cast<int>(min(32ll, w1 - base))) {
                ib = pib[base + lane];
                slot = pslot[base + lane];
            }
        };
        auto issue = [&](long long base, int ib, int slot, int buf) {
            if (base < w1 && ib >= 0) {
                const T* fr = F + static_cast<long long>(slot) * ra;
                T* dst = strip + buf * 32 * ras + lane * ras;
                if (vec == 4) {
                    for (int a2 = 0; a2 < ra; a2 += 4)
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                                         static_cast<std::uint32_t>(__cvta_generic_to_shared(dst + a2))),
                                     "l"(fr + a2)
                                     : "memory");
                } else {
                    for (int a2 = 0; a2 < ra; ++a2) {
                        if constexpr (sizeof(T) == 4) cp_async4(dst + a2, fr + a2);
                        else cp_async8(dst + a2, fr + a2);
                    }
                }
            }
            cp_async_commit();
        };
        int ib_c, sl_c, ib_n, sl_n;
        fetch(w0, ib_c, sl_c);
        issue(w0, ib_c, sl_c, 0);
        fetch(w0 + 32, ib_n, sl_n);
        for (long long base = w0, buf = 0; base < w1; base += 32, buf ^= 1) {
            const int nb = static_cast<int>(min(32ll, w1 - base));
            const int ibv = ib_c;
            issue(base + 32, ib_n, sl_n, static_cast<int>(buf ^ 1));
            ib_c = ib_n;
            fetch(base + 64, ib_n, sl_n);
            __syncwarp();
            if (lane < nb) su[lane] = (ibv & mask1) * rb1s;
            cp_async_wait1();  // this batch's rows have landed
            // runs of equal i_b2 inside the batch (pib ascending): a fold only between runs
            const int i2v = ibv >> bits1;
            const int prev = __shfl_up_sync(0xffffffffu, i2v, 1);
            unsigned starts = __ballot_sync(0xffffffffu, lane < nb && (lane == 0 || i2v != prev));
            __syncwarp();
            const T* sb = strip + buf * 32 * ras;
            while (starts) {
                const int s0 = __ffs(starts) - 1;
                starts &= starts - 1;
                const int s1 = starts ? __ffs(starts) - 1 : nb;
                const int i2 = __shfl_sync(0xffffffffu, i2v, s0);
                if (i2 != cur) {
                    if (cur >= 0) fold();
                    cur = i2;
                }
                const T* fl = sb + s0 * ras;
                for (int l = s0; l < s1; ++l, fl += ras) {  // branch-free FMA run
                    const T* ur = Us1 + su[l];
#pragma unroll
                    for (int j = 0; j < EPL; ++j) z[j] = fma(fl[ea[j]], ur[eb[j]], z[j]);
                }
            }
        }
        (void)sl_c;
        if (cur >= 0) fold();
    }
    // warp partials -> CTA partial, in warp order
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
        const int e = lane + 32 * j;
        if (e < E)
#pragma unroll
            for (int k = 0; k < RB2; ++k)
                if (k < rb2) Yw[static_cast<std::size_t>(warp) * C + e + k * E] = y[j][k];
    }
    __syncthreads();
    if (row >= rows) return;
    auto out_index = [&](int o) {
        const int ee = o % E, qq = o / E;
        return row + static_cast<long long>((ee % ra) * sa + (ee / ra) * sb1 + qq * sb2) * rows;
    };
    if (R == 1) {
        for (int o = tid; o < C; o += blockDim.x) {
            T sum = T(0);
            for (int w = 0; w < W; ++w) sum += Yw[static_cast<std::size_t>(w) * C + o];
            Y[out_index(o)] = sum;
        }
        return;
    }
    T* mine = Ypart + (static_cast<long long>(row) * R + q) * C;
    for (int o = tid; o < C; o += blockDim.x) {
        T sum = T(0);
        for (int w = 0; w < W; ++w) sum += Yw[static_cast<std::size_t>(w) * C + o];
        mine[o] = sum;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) last = atomicAdd(&ticket[row], 1u) == static_cast<unsigned>(R - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    const T* all = Ypart + static_cast<long long>(row) * R * C;
    for (int o = tid; o < C; o += blockDim.x) {
        T sum = T(0);
        for (int p = 0; p < R; ++p) sum += __ldcg(all + static_cast<long long>(p) * C + o);
        Y[out_index(o)] = sum;
    }
    if (tid == 0) ticket[row] = 0u;  // re-armed for the next launch (graph replays)
}

std::size_t stage2_4way_smem(int Ib1, int Ib2, int ra, int rb1, int rb2, int threads, int esz) {
    const int E = ra * rb1;
    const std::size_t rb1s = ttm_stride(rb1, esz), rb2s = ttm_stride(rb2, esz);
    const int ras = (esz == 4 && (ra & 3) == 0) ? ra : (ra | 1);
    return (static_cast<std::size_t>(Ib1) * rb1s + static_cast<std::size_t>(Ib2) * rb2s +
            static_cast<std::size_t>(threads / 32) * (static_cast<std::size_t>(E) * rb2 + 2 * 32 * ras + 128 / esz)) * esz;
}
}  // namespace

bool stage2_4way_ok(const std::vector<int>& dims, const std::vector<int>& ranks, int n, int a, int b1, int b2) {
    const int E = ranks[a] * ranks[b1];
    const int epl = (E + 31) / 32;
    const int rb2 = ranks[b2];
    const int rbb = rb2 <= 4 ? 4 : rb2 <= 8 ? 8 : rb2 <= 16 ? 16 : 32;
    const int eplb = epl <= 1 ? 1 : epl <= 2 ? 2 : epl <= 4 ? 4 : 8;
    if (eplb * rbb > 64) return false;  // register partial of the Y row
    (void)n;
    return stage2_4way_smem(dims[b1], dims[b2], ranks[a], ranks[b1], rb2, 512, 8) <= 200 * 1024;
}

template <typename T>
void sparse_mode_stage2_4way(Ctx* ctx, ModePlan& P, const std::vector<int>& dims, const std::vector<int>& ranks,
                             const T* F, const std::vector<const T*>& Ur, T* Y) {
    const int n = P.mode, a = P.a, b1 = P.bmodes[0], b2 = P.bmodes[1];
    const int bits1 = bits_for(dims[b1]);
    // Y_(n) columns: the remaining modes in original order, earliest fastest
    int sa = 0, sb1 = 0, sb2 = 0, st = 1;
    for (int m = 0; m < static_cast<int>(dims.size()); ++m) {
        if (m == n) continue;
        if (m == a) sa = st;
        if (m == b1) sb1 = st;
        if (m == b2) sb2 = st;
        st *= ranks[m];
    }
    const int ra = ranks[a], rb1 = ranks[b1], rb2 = ranks[b2];
    const int E = ra * rb1, C = E * rb2;
    const int threads = 512;
    const int rows = dims[n];
    int sms = 148;
    MB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    int R = 1;  // CTAs per row (i_b2 slices): two CTAs per SM
    while (R < 16 && static_cast<long long>(rows) * R < 2ll * sms && R * 2 <= dims[b2]) R *= 2;
    if (R > 1) {
        const std::size_t need = static_cast<std::size_t>(rows) * R * C * sizeof(T);
        if (P.s2part.n < need) P.s2part.alloc(ctx, need);
        if (P.s2tick.n < static_cast<std::size_t>(rows)) {
            P.s2tick.alloc(ctx, rows);
            P.s2tick.zero(ctx);
        }
    }
    const std::size_t smem = stage2_4way_smem(dims[b1], dims[b2], ra, rb1, rb2, threads, sizeof(T));
    const int epl = (E + 31) / 32;
    const int eplb = epl <= 1 ? 1 : epl <= 2 ? 2 : epl <= 4 ? 4 : 8;
    const int rbb = rb2 <= 4 ? 4 : rb2 <= 8 ? 8 : rb2 <= 16 ? 16 : 32;
    auto launch = [&](auto kern) {
        MB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        MB_LAUNCH_PDL(ctx, kern, static_cast<unsigned>(rows) * R, threads, smem, P.piece_rs.get(), P.piece_re.get(),
                      P.pslot.get(), P.pib.get(), F, ra, (sizeof(T) == 4 && (ra & 3) == 0) ? ra : (ra | 1), rb1, rb2, Ur[b1], ttm_stride(rb1, sizeof(T)), Ur[b2],
                      ttm_stride(rb2, sizeof(T)), dims[b1], dims[b2], bits1, sa, sb1, sb2, rows, R,
                      reinterpret_cast<T*>(P.s2part.get()), P.s2tick.get(), Y);
    };
    switch (eplb * 100 + rbb) {
        case 104: launch(stage2_4way_kernel<T, 1, 4>); break;
        case 108: launch(stage2_4way_kernel<T, 1, 8>); break;
        case 116: launch(stage2_4way_kernel<T, 1, 16>); break;
        case 132: launch(stage2_4way_kernel<T, 1, 32>); break;
        case 204: launch(stage2_4way_kernel<T, 2, 4>); break;
        case 208: launch(stage2_4way_kernel<T, 2, 8>); break;
        case 216: launch(stage2_4way_kernel<T, 2, 16>); break;
        case 232: launch(stage2_4way_kernel<T, 2, 32>); break;
        case 404: launch(stage2_4way_kernel<T, 4, 4>); break;
        case 408: launch(stage2_4way_kernel<T, 4, 8>); break;
        case 416: launch(stage2_4way_kernel<T, 4, 16>); break;
        case 804: launch(stage2_4way_kernel<T, 8, 4>); break;
        case 808: launch(stage2_4way_kernel<T, 8, 8>); break;
        default: throw Error(MACH_ERR_INTERNAL, "order-4 stage 2: rank combination not instantiated");
    }
}
template void sparse_mode_stage2_4way<float>(Ctx*, ModePlan&, const std::vector<int>&, const std::vector<int>&, const float*,
                                             const std::vector<const float*>&, float*);
template void sparse_mode_stage2_4way<double>(Ctx*, ModePlan&, const std::vector<int>&, const std::vector<int>&,
                                              const double*, const std::vector<const double*>&, double*);

template void sparse_mode_stage1<float>(Ctx*, ModePlan&, const std::vector<int>&, const std::vector<int>&,
                                        const std::vector<const float*>&, float*, int, bool);
template void sparse_mode_stage1<double>(Ctx*, ModePlan&, const std::vector<int>&, const std::vector<int>&,
                                         const std::vector<const double*>&, double*, int, bool);
template void sparse_mode_stage2<float>(Ctx*, ModePlan&, const std::vector<int>&, const std::vector<int>&, const float*,
                                        const float*, float*);
template void sparse_mode_stage2<double>(Ctx*, ModePlan&, const std::vector<int>&, const std::vector<int>&, const double*,
                                         const double*, double*);

template void y_from_segments<float>(Ctx*, ModePlan&, const std::vector<int>&, const std::vector<int>&, const float*,
                                     const float*, float*);
template void y_from_segments<double>(Ctx*, ModePlan&, const std::vector<int>&, const std::vector<int>&, const double*,
                                      const double*, double*);

// ---- sparse HOSVD Grams ----------------------------------------------------
template <typename T>
void sparse_row_gram(Ctx* ctx, const mach_sparse* X, int n, double normX2, double* G) {
    const int d = static_cast<int>(X->dims.size());
    KeyFields kf{};
    const int bn = bits_for(X->dims[n]);
    kf.mode[kf.nf] = n; kf.shift[kf.nf++] = 0;
    int sh = bn;
    for (int m = 0; m < d; ++m) {
        if (m == n) continue;
        kf.mode[kf.nf] = m; kf.shift[kf.nf++] = sh;
        sh += bits_for(X->dims[m]);
    }
    const bool key64 = sh > 32;
    DBuf<unsigned char> keys, vals;
    build_sorted<T>(ctx, X, kf, sh, key64, keys, vals, !(n == 0));
    const int I = X->dims[n];
    DBuf<unsigned long long> Gi(ctx, static_cast<std::size_t>(I) * I);
    Gi.zero(ctx);
    const double scale = (normX2 > 0) ? std::ldexp(1.0, static_cast<int>(std::floor(61.0 - std::log2(normX2)))) : 1.0;
    const long long nnz = X->nnz;
    if (nnz > 0) {
        if (key64) MB_LAUNCH(ctx, (row_gram_kernel<T, unsigned long long>), ceil_div(nnz, 256), 256, 0,
                             reinterpret_cast<const unsigned long long*>(keys.get()), reinterpret_cast<const T*>(vals.get()),
                             nnz, bn, scale, I, Gi.get());
        else MB_LAUNCH(ctx, (row_gram_kernel<T, unsigned int>), ceil_div(nnz, 256), 256, 0,
                       reinterpret_cast<const unsigned int*>(keys.get()), reinterpret_cast<const T*>(vals.get()), nnz, bn,
                       scale, I, Gi.get());
    }
    MB_LAUNCH(ctx, fixed_to_double_kernel, ceil_div(static_cast<long long>(I) * I, 256), 256, 0, Gi.get(),
              static_cast<long long>(I), 1.0 / scale, G);
}

// X_(n) column stride of every mode (remaining modes in original order,
// earliest fastest; tensor.hpp:119-121)
static std::vector<long long> xn_col_strides(const std::vector<int>& dims, int n) {
    std::vector<long long> st(dims.size(), 0);
    long long s = 1;
    for (std::size_t m = 0; m < dims.size(); ++m) {
        if (static_cast<int>(m) == n) continue;
        st[m] = s;
        s *= dims[m];
    }
    return st;
}

ColDecode plan_col_decode(const std::vector<int>& dims, const ModePlan& P) {
    const auto st = xn_col_strides(dims, P.mode);
    ColDecode D;
    for (int j = 0; j < P.nf; ++j) {
        const int m = P.fmode[j];
        if (m == P.mode) continue;
        D.shift[D.nf] = P.fshift[j];
        D.mask[D.nf] = (1ull << bits_for(dims[m])) - 1ull;
        D.stride[D.nf] = st[m];
        ++D.nf;
    }
    return D;
}

template <typename T>
void sparse_col_gram(Ctx* ctx, const mach_sparse* X, const ModePlan& P, long long cols, double normX2, double* G) {
    const ColDecode D = plan_col_decode(X->dims, P);
    DBuf<unsigned long long> Gi(ctx, static_cast<std::size_t>(cols * cols));
    Gi.zero(ctx);
    const double scale = (normX2 > 0) ? std::ldexp(1.0, static_cast<int>(std::floor(61.0 - std::log2(normX2)))) : 1.0;
    const long long nnz = X->nnz;
    if (nnz > 0) {
        if (P.key64) MB_LAUNCH(ctx, (col_gram_kernel<T, unsigned long long>), ceil_div(nnz, 256), 256, 0,
                               reinterpret_cast<const unsigned long long*>(P.keys.get()), reinterpret_cast<const T*>(P.vals.get()),
                               nnz, P.ba + P.bb, D, scale, cols, Gi.get());
        else MB_LAUNCH(ctx, (col_gram_kernel<T, unsigned int>), ceil_div(nnz, 256), 256, 0,
                       reinterpret_cast<const unsigned int*>(P.keys.get()), reinterpret_cast<const T*>(P.vals.get()), nnz,
                       P.ba + P.bb, D, scale, cols, Gi.get());
    }
    MB_LAUNCH(ctx, fixed_to_double_kernel, ceil_div(cols * cols, 256), 256, 0, Gi.get(), cols, 1.0 / scale, G);
}

template <typename T>
void sparse_times(Ctx* ctx, const mach_sparse* X, const ModePlan& P, const double* V, long long vld, int kc, double* W) {
    const ColDecode D = plan_col_decode(X->dims, P);
    const int rows = P.rows;
#define MB_ST(KT)                                                                                                  \
    MB_LAUNCH(ctx, (sparse_times_kernel<T, KT, 32>), ceil_div(static_cast<long long>(rows) * 32, 256), 256, 0,       \
              reinterpret_cast<const KT*>(P.keys.get()), reinterpret_cast<const T*>(P.vals.get()), P.row_start.get(), \
              P.row_end.get(), rows, D, V, vld, kc, W)
    if (P.key64) MB_ST(unsigned long long);
    else MB_ST(unsigned int);
#undef MB_ST
}

// ---- column-grouped layout of X_(n) (tall-mode basis) ----------------------
namespace {
template <typename K>
__global__ void run_flag_kernel(const K* __restrict__ keys, long long nnz, int sh, unsigned char* __restrict__ flag) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= nnz) return;
    flag[i] = (i == 0 || (static_cast<unsigned long long>(keys[i]) >> sh) != (static_cast<unsigned long long>(keys[i - 1]) >> sh))
                  ? 1 : 0;
}
}  // namespace

template <typename T>
void build_col_layout(Ctx* ctx, const mach_sparse* X, int n, ColLayout& L) {
    const int d = static_cast<int>(X->dims.size());
    const auto st = xn_col_strides(X->dims, n);
    KeyFields kf{};
    L.bn = bits_for(X->dims[n]);
    kf.mode[kf.nf] = n; kf.shift[kf.nf++] = 0;
    int sh = L.bn;
    L.dec = ColDecode{};
    for (int m = 0; m < d; ++m) {
        if (m == n) continue;
        kf.mode[kf.nf] = m; kf.shift[kf.nf++] = sh;
        L.dec.shift[L.dec.nf] = sh;
        L.dec.mask[L.dec.nf] = (1ull << bits_for(X->dims[m])) - 1ull;
        L.dec.stride[L.dec.nf] = st[static_cast<std::size_t>(m)];
        ++L.dec.nf;
        sh += bits_for(X->dims[m]);
    }
    L.key64 = sh > 32;
    build_sorted<T>(ctx, X, kf, sh, L.key64, L.keys, L.vals, !(n == 0));
    const long long nnz = X->nnz;
    L.runs.alloc(ctx, nnz + 1);
    if (nnz == 0) {
        L.nruns = 0;
        const long long z = 0;
        to_device(ctx, L.runs.get(), &z, 1);
        return;
    }
    DBuf<unsigned char> flag(ctx, nnz);
    if (L.key64) MB_LAUNCH(ctx, run_flag_kernel<unsigned long long>, ceil_div(nnz, 256), 256, 0,
                           reinterpret_cast<const unsigned long long*>(L.keys.get()), nnz, L.bn, flag.get());
    else MB_LAUNCH(ctx, run_flag_kernel<unsigned int>, ceil_div(nnz, 256), 256, 0,
                   reinterpret_cast<const unsigned int*>(L.keys.get()), nnz, L.bn, flag.get());
    DBuf<long long> nf_d(ctx, 1);
    thrust::counting_iterator<long long> cnt_it(0);
    std::size_t tmp = 0;
    MB_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, cnt_it, flag.get(), L.runs.get(), nf_d.get(), nnz, ctx->stream));
    DBuf<unsigned char> t(ctx, tmp);
    MB_CUDA(cub::DeviceSelect::Flagged(t.get(), tmp, cnt_it, flag.get(), L.runs.get(), nf_d.get(), nnz, ctx->stream));
    ctx->launches += 1;
    to_host(ctx, &L.nruns, nf_d.get(), 1);
    sync(ctx);
    to_device(ctx, L.runs.get() + L.nruns, &nnz, 1);
    sync(ctx);  // the host value above is a stack temporary
}
template void build_col_layout<float>(Ctx*, const mach_sparse*, int, ColLayout&);
template void build_col_layout<double>(Ctx*, const mach_sparse*, int, ColLayout&);

template std::shared_ptr<ModePlan> get_plan<float>(mach_sparse*, int, const std::vector<int>&, int);
template std::shared_ptr<ModePlan> get_plan<double>(mach_sparse*, int, const std::vector<int>&, int);
template void sparse_mode_ttm<float>(Ctx*, const ModePlan&, const std::vector<int>&, const std::vector<int>&,
                                     const std::vector<const float*>&, const float*, float*, float*, float*,
                                     const int*);
template void sparse_mode_ttm<double>(Ctx*, const ModePlan&, const std::vector<int>&, const std::vector<int>&,
                                      const std::vector<const double*>&, const double*, double*, double*, double*,
                                      const int*);
template void sparse_row_gram<float>(Ctx*, const mach_sparse*, int, double, double*);
template void sparse_row_gram<double>(Ctx*, const mach_sparse*, int, double, double*);
template void sparse_col_gram<float>(Ctx*, const mach_sparse*, const ModePlan&, long long, double, double*);
template void sparse_col_gram<double>(Ctx*, const mach_sparse*, const ModePlan&, long long, double, double*);
template void sparse_times<float>(Ctx*, const mach_sparse*, const ModePlan&, const double*, long long, int, double*);
template void sparse_times<double>(Ctx*, const mach_sparse*, const ModePlan&, const double*, long long, int, double*);

}  // namespace machb

mach_sparse::~mach_sparse() {
    plans.clear();
    if (ctx) {
        if (idx) cudaFreeAsync(idx, ctx->stream);
        if (val) cudaFreeAsync(val, ctx->stream);
    }
}
