// Dense mode-n Gram G = X_(n) X_(n)^T on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, accumulators in TMEM, operands staged by TMA).
//
// Reference: the dense HOSVD's row-side Gram a * a^T (proj/src/linalg.cpp:340,
// reached from hosvd(DenseTensor), proj/src/tucker.cpp:135-150 through
// left_singular_basis, linalg.cpp:319-353).  This is the one tensor-bound
// contraction of the path (2 * I_n * numel flops per mode,
// intensity I_n / 2 flop/B; C5 p = 1: 2.2 TFLOP per mode).
//
// No matricisation copy: the mode-n unfolding of a first-mode-fastest tensor
// is read in place through a TMA tensor map over the 3-D view
// {inner = prod_{j<n} I_j, R = I_n, outer = prod_{j>n} I_j}; column k of
// X_(n) is (ki, ko) with k = ki + inner * ko.  For n > 0 the K index is the
// contiguous one (K-major operands: box {32, 128, 1}, 128-byte swizzle); for
// n = 0 the row index is contiguous (MN-major operands: 2-D map {R, K}, boxes
// {32, 32}).  Out-of-range boxes are zero-filled by TMA, so ragged shapes add
// zeros to the sums.
//
// Work split: G is symmetric, so only 128 x 256 tiles (row block I, column
// block J) that touch the lower triangle are computed (20 of 32 at
// I_n = 1024).  Each tile's K tiles are dealt round-robin to `nsplit`
// CTAs (one CTA per (split, tile)), so all resident CTAs stream the same
// narrow window of columns of X_(n) at about the same time (L2 reuse: X is
// read from HBM about once; few memory pages in flight).  A CTA accumulates its chunk in fp32 TMEM (<= 32768 K terms:
// accumulation error ~ sqrt(K/8) * 2^-24 relative) and writes an fp32 partial
// tile; gram_tc_reduce sums the partials of each entry in fp64 in chunk
// order (deterministic) and mirrors the lower triangle (G exactly symmetric).
//
// Precision: kind::tf32 uses the top 19 bits of each fp32 operand (10-bit
// mantissa).  The truncation error of X is a near-uniform relative shrink
// (mean 2^-11 per operand), which scales G without turning its eigenvectors;
// the fluctuating remainder averages over the K >= 10^5 terms of each entry.
// tests/test_gpu_dense_tc.py measures the entrywise error against an fp64
// Gram and the leading-subspace sine against the fp64 eigenvectors.
//
// CTA roles (192 threads, 1 CTA per SM, 4-stage smem ring of 48 KB):
//   warp 0  TMA producer (one elected lane)
//   warp 1  TMEM allocator + MMA issuer (one elected lane): 4 x
//           tcgen05.mma 128x256x8 per stage, tcgen05.commit frees the stage
//   warps 2-5  epilogue: tcgen05.ld 32x32b (warp w reads TMEM lanes
//           32 (w % 4) ...), coalesced column-major fp32 partial store
#include <cuda.h>

#include <algorithm>

#include "common.cuh"
#include "sparse_ttm.cuh"

namespace machb {

namespace {

constexpr int TBM = 128;   // tile rows (UMMA M)
constexpr int TBN = 256;   // tile columns (UMMA N)
constexpr int TBK = 32;    // K per stage: 128 bytes of fp32 (one 128B-swizzle row)
constexpr int TST = 4;     // pipeline stages
constexpr int kGThreads = 192;
constexpr uint32_t kABytes = TBM * TBK * 4;  // 16 KB
constexpr uint32_t kBBytes = TBN * TBK * 4;  // 32 KB
constexpr uint32_t kStageBytes = kABytes + kBBytes;
constexpr uint32_t kTmemCols = 256;
constexpr std::size_t kGramSmem = static_cast<std::size_t>(TST) * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "GW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra GW_%=;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(tm), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(tm), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

// UMMA shared-memory descriptor, version 1; layout 2 = 128-byte swizzle,
// 1 = 128-byte swizzle on 32-byte atoms (the only MN-major layout for tf32)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout = 2) {
    return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
           (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (static_cast<uint64_t>(layout) << 61);
}

__device__ __forceinline__ void umma_tf32(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// MN-major operand strides (LBO: between 32-element MN chunks; SBO: between
// 8-row K groups), in bytes; __constant__ so the probe can vary them
__constant__ uint32_t g_mn_lbo = 4096, g_mn_sbo = 512;

// lower-triangle tile t -> (I, J): row blocks of TBM, column blocks of TBN,
// tiles with TBN*J <= TBM*I + TBM - 1, enumerated row block by row block
__host__ __device__ inline void tile_of(int t, int& I, int& J) {
    I = 0;
    for (;;) {
        const int nj = (TBM * I + TBM - 1) / TBN + 1;
        if (t < nj) { J = t; return; }
        t -= nj;
        ++I;
    }
}
inline int tile_count(int R) {
    const int nrb = (R + TBM - 1) / TBM, ncb = (R + TBN - 1) / TBN;
    int n = 0;
    for (int I = 0; I < nrb; ++I) n += std::min(ncb, (TBM * I + TBM - 1) / TBN + 1);
    return n;
}

// MN: mode 0 (row index contiguous).  kt tiles of TBK columns; for K-major
// views column tile kt is (ki = (kt % nki) * TBK, ko = kt / nki).
template <bool MN>
__global__ void __launch_bounds__(kGThreads, 1)
    gram_tc_kernel(const __grid_constant__ CUtensorMap tm, int nki, long long nkt, int nsplit, int ntile,
                   float* __restrict__ part, unsigned* __restrict__ dbg) {
    extern __shared__ __align__(1024) unsigned char gsm_raw[];
    unsigned char* gsm = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(gsm_raw) + 1023) & ~std::uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(gsm + TST * kStageBytes);
    uint64_t* empty = full + TST;
    uint64_t* done = empty + TST;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int split = blockIdx.x / ntile, tile = blockIdx.x % ntile;
    int I, J;
    tile_of(tile, I, J);
    // K tiles split, split + nsplit, ...: at any time the resident CTAs read
    // one narrow window of columns (for the last mode every row of X_(n) is
    // its own memory page, so a narrow window keeps the pages in flight few)
    const int nk = static_cast<int>((nkt - split + nsplit - 1) / nsplit);

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < TST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tm) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            for (int i = 0; i < nk; ++i) {
                const int s = i % TST;
                const int u = i / TST;
                if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
                unsigned char* a = gsm + s * kStageBytes;
                unsigned char* b = a + kABytes;
                mbar_expect_tx(&full[s], kStageBytes);
                const long long kt = split + static_cast<long long>(i) * nsplit;
                if constexpr (MN) {
                    const int k = static_cast<int>(kt * TBK);
#pragma unroll
                    for (int m = 0; m < TBM / 32; ++m) tma_load_2d(a + m * 4096, &tm, &full[s], TBM * I + 32 * m, k);
#pragma unroll
                    for (int m = 0; m < TBN / 32; ++m) tma_load_2d(b + m * 4096, &tm, &full[s], TBN * J + 32 * m, k);
                } else {
                    const int ki = static_cast<int>(kt % nki) * TBK, ko = static_cast<int>(kt / nki);
                    tma_load_3d(a, &tm, &full[s], ki, TBM * I, ko);
#pragma unroll
                    for (int m = 0; m < TBN / TBM; ++m) tma_load_3d(b + m * kABytes, &tm, &full[s], ki, TBN * J + TBM * m, ko);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // D = F32, A = B = TF32, K- or MN-major, N = 256, M = 128
            const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (MN ? (1u << 15) | (1u << 16) : 0u) |
                                   (static_cast<uint32_t>(TBN >> 3) << 17) | (static_cast<uint32_t>(TBM >> 4) << 24);
            for (int i = 0; i < nk; ++i) {
                const int s = i % TST;
                mbar_wait(&full[s], (i / TST) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (dbg && blockIdx.x == 0 && i == 0)  // probe: the first stage as the MMA sees it
                    for (uint32_t w = 0; w < kStageBytes / 4; ++w) dbg[w] = reinterpret_cast<const unsigned*>(gsm)[w];
                const uint32_t a = smem_u32(gsm + s * kStageBytes);
                const uint32_t b = a + kABytes;
#pragma unroll
                for (int k = 0; k < TBK / 8; ++k) {
                    uint64_t ad, bd;
                    if constexpr (MN) {  // 8 K rows = 1 KB per step (two 4-row 32B-swizzle atoms, SBO apart); 32-element MN chunks LBO apart
                        ad = umma_desc(a + k * 1024, g_mn_lbo, g_mn_sbo, 1);
                        bd = umma_desc(b + k * 1024, g_mn_lbo, g_mn_sbo, 1);
                    } else {  // 8 K-values = 32 B inside the 128-B swizzle row; 8-row groups 1 KB apart
                        ad = umma_desc(a + k * 32, 16, 1024);
                        bd = umma_desc(b + k * 32, 16, 1024);
                    }
                    umma_tf32(tmem, ad, bd, idesc, (i > 0 || k > 0) ? 1u : 0u);
                }
                umma_commit(&empty[s]);  // the stage is free once these MMAs have read it
            }
            if (nk > 0) umma_commit(done);
        }
    } else {
        // epilogue: warp w owns TMEM lanes 32 (w % 4) .. + 31 = tile rows
        const int q = warp & 3;
        const int row = 32 * q + lane;
        float* out = part + (static_cast<std::size_t>(split) * ntile + tile) * (TBM * TBN);
        if (nk > 0) {
            mbar_wait(done, 0);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
#pragma unroll 1
        for (int c0 = 0; c0 < TBN; c0 += 32) {
            uint32_t v[32];
            if (nk > 0) {
                const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * q) << 16) + static_cast<uint32_t>(c0);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                      "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                      "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                      "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                      "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                    : "r"(taddr)
                    : "memory");
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = 0u;
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) out[static_cast<std::size_t>(c0 + j) * TBM + row] = __uint_as_float(v[j]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
    }
}

// G (R x R, column-major fp64) from the partial tiles: lower triangle summed
// over the chunks in chunk order, mirrored to the upper one.
__global__ void gram_tc_reduce_kernel(const float* __restrict__ part, int R, int nsplit, int ntile,
                                      double* __restrict__ G) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= static_cast<long long>(R) * R) return;
    int r = static_cast<int>(e % R), c = static_cast<int>(e / R);
    if (c > r) { const int t = r; r = c; c = t; }
    const int I = r / TBM, J = c / TBN;
    // tile index of (I, J): tiles of the row blocks before I, then J
    int t = 0;
    for (int i = 0; i < I; ++i) t += (TBM * i + TBM - 1) / TBN + 1;
    t += J;
    const std::size_t off = static_cast<std::size_t>(c - TBN * J) * TBM + (r - TBM * I);
    double s = 0.0;
    for (int sp = 0; sp < nsplit; ++sp) s += static_cast<double>(part[(static_cast<std::size_t>(sp) * ntile + t) * (TBM * TBN) + off]);
    G[e] = s;
}

// x' = x with its last two modes swapped, for first-mode-fastest x with
// dims (A..., I, J): x'[a + A (j + J i)] = x[a + A (i + I j)] — contiguous runs
// of A = prod of the leading dims (A % 4 == 0), copied as float4.
__global__ void swap_last2_kernel(const float4* __restrict__ x, float4* __restrict__ y, long long A4, int I, int J) {
    const long long n = A4 * I * J;
    for (long long o = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; o < n;
         o += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long a = o % A4, r = o / A4;
        const long long j = r % J, i = r / J;  // output run (j, i)
        y[o] = __ldcs(x + a + A4 * (i + static_cast<long long>(I) * j));
    }
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                 const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
    static EncodeTiled fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiled>(p);
    }();
    if (!fn) throw Error(MACH_ERR_CUDA, "cuTensorMapEncodeTiled is not available from the driver");
    return fn;
}

}  // namespace

// Mode view of a first-mode-fastest tensor: inner = prod_{j<n} I_j, R = I_n,
// outer = prod_{j>n} I_j.
static void mode_view(const std::vector<int>& dims, int n, long long& inner, long long& R, long long& outer) {
    inner = 1;
    outer = 1;
    for (int j = 0; j < n; ++j) inner *= dims[static_cast<std::size_t>(j)];
    for (std::size_t j = static_cast<std::size_t>(n) + 1; j < dims.size(); ++j) outer *= dims[j];
    R = dims[static_cast<std::size_t>(n)];
}

bool gram_tc_applies(const std::vector<int>& dims, int n) {
    static const bool off = std::getenv("MACH_NO_GRAM_TC") != nullptr;
    if (off) return false;
    long long inner, R, outer;
    mode_view(dims, n, inner, R, outer);
    const long long K = inner * outer;
    if (R < 64 || K < 4096) return false;  // too small to pay for the pipeline
    if (n == 0) return (R % 4) == 0 && R < (1ll << 31) && K < (1ll << 31);
    return (inner % 4) == 0 && inner < (1ll << 31) && R < (1ll << 31) && outer < (1ll << 31);
}

void gram_tc(Ctx* ctx, const float* x, const std::vector<int>& dims, int n, double* G) {
    long long inner, R, outer;
    mode_view(dims, n, inner, R, outer);
    // The last mode's rows are whole hyper-slices apart (4 MB at 1024^3), so
    // each TMA row of a stage lands on its own memory page and the address
    // translation, not the tensor pipe, sets the pace (measured 6.9 ms vs
    // 2.2 ms for the middle mode at C5).  Swapping the last two modes first
    // (one streaming copy, ~1.4 ms at C5) turns it into a middle mode.
    const int d = static_cast<int>(dims.size());
    static const bool no_swap = std::getenv("MACH_GRAM_NO_SWAP") != nullptr;
    if (!no_swap && d >= 3 && n == d - 1 && inner * 4 >= (1ll << 20)) {
        const long long A = inner / dims[static_cast<std::size_t>(d - 2)];
        std::vector<int> sd = dims;
        std::swap(sd[static_cast<std::size_t>(d - 2)], sd[static_cast<std::size_t>(d - 1)]);
        if (A % 4 == 0 && gram_tc_applies(sd, d - 2)) {
            DBuf<float> xs;
            bool have = true;
            try {
                xs.alloc(ctx, static_cast<std::size_t>(inner) * R);
            } catch (const Error&) {
                cudaGetLastError();
                have = false;  // not enough memory for the copy: read in place
            }
            if (have) {
                int nsm = 148;
                cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device);
                MB_LAUNCH(ctx, swap_last2_kernel, 8 * nsm, 512, 0, reinterpret_cast<const float4*>(x),
                          reinterpret_cast<float4*>(xs.get()), A / 4, dims[static_cast<std::size_t>(d - 2)],
                          dims[static_cast<std::size_t>(d - 1)]);
                gram_tc(ctx, xs.get(), sd, d - 2, G);
                return;
            }
        }
    }
    if (!gram_tc_applies(dims, n)) throw Error(MACH_ERR_INTERNAL, "gram_tc: shape not supported");
    const bool mn = n == 0;
    CUtensorMap tm;
    const EncodeTiled enc = encode_fn();
    CUresult rc;
    long long nkt;
    int nki = 1;
    if (mn) {
        const long long K = outer;  // inner == 1
        const cuuint64_t gdim[2] = {static_cast<cuuint64_t>(R), static_cast<cuuint64_t>(K)};
        const cuuint64_t gstride[1] = {static_cast<cuuint64_t>(R) * 4};
        const cuuint32_t box[2] = {32, 32};
        const cuuint32_t estr[2] = {1, 1};
        rc = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(x), gdim, gstride, box, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        nkt = (K + TBK - 1) / TBK;
    } else {
        const cuuint64_t gdim[3] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(R), static_cast<cuuint64_t>(outer)};
        const cuuint64_t gstride[2] = {static_cast<cuuint64_t>(inner) * 4, static_cast<cuuint64_t>(inner * R) * 4};
        const cuuint32_t box[3] = {32, TBM, 1};
        const cuuint32_t estr[3] = {1, 1, 1};
        rc = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(x), gdim, gstride, box, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        nki = static_cast<int>((inner + TBK - 1) / TBK);
        nkt = static_cast<long long>(nki) * outer;
    }
    if (rc != CUDA_SUCCESS) throw Error(MACH_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(rc)) + ")");
    const int ntile = tile_count(static_cast<int>(R));
    // chunks: <= 1024 K tiles (32768 columns) each for the fp32 accumulation
    // bound, and enough CTAs for several waves over the SMs
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device);
    long long nsplit = std::max<long long>((nkt + 1023) / 1024, (4ll * nsm + ntile - 1) / ntile);
    nsplit = std::min<long long>(nsplit, std::max<long long>(1, nkt));
    nsplit = std::min<long long>(nsplit, (1ll << 31) / std::max(1, ntile) - 1);
    DBuf<float> part(ctx, static_cast<std::size_t>(nsplit) * ntile * TBM * TBN);
    static std::uint64_t attr = 0;  // per-device mask
    if (first_on_device(attr, ctx->device)) {
        MB_CUDA(cudaFuncSetAttribute(gram_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kGramSmem)));
        MB_CUDA(cudaFuncSetAttribute(gram_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kGramSmem)));
    }
    const long long grid = nsplit * ntile;
    if (mn)
        MB_LAUNCH(ctx, gram_tc_kernel<true>, static_cast<unsigned>(grid), kGThreads, kGramSmem, tm, nki, nkt,
                  static_cast<int>(nsplit), ntile, part.get(), nullptr);
    else
        MB_LAUNCH(ctx, gram_tc_kernel<false>, static_cast<unsigned>(grid), kGThreads, kGramSmem, tm, nki, nkt,
                  static_cast<int>(nsplit), ntile, part.get(), nullptr);
    const long long n2 = R * R;
    MB_LAUNCH(ctx, gram_tc_reduce_kernel, ceil_div(n2, 256), 256, 0, part.get(), static_cast<int>(R),
              static_cast<int>(nsplit), ntile, G);
}

}  // namespace machb
