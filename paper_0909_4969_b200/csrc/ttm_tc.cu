// Dense mode product Z = X x_m U^T (U: len x r, r <= 32) on the tcgen05 tensor
// cores with 3xTF32 split precision: the first contraction of the dense
// route's projection chain (reference: mode_product(DenseTensor),
// proj/src/tensor.cpp:224-239, called by project_except, tucker.cpp:109-118),
// the only pass of a dense HOOI sweep that streams the whole tensor.
//
// As a GEMM: rows = every index combination of X except mode m, K = I_m,
// N = r (padded to NB = 16 or 32).
//   m == 0: K is the contiguous index, rows = the flattened outer modes:
//           A = X_(0)^T, K-major, 2-D map {I_0, outer}, box {32, 128};
//           out (r x outer, first-mode-fastest) = thread-per-row, r values.
//   m >  0: rows = (a, c) with a < inner contiguous, c < outer:
//           A MN-major (tf32 MN-major needs the 128B swizzle on 32-byte
//           atoms), 3-D map {inner, I_m, outer}, boxes {32, 32, 1};
//           out (inner x r x outer) coalesced along a.
// B = U^T (K-major, N x K) in two fp32 planes, hi = rn_tf32(U) and lo =
// rn_tf32(U - hi), loaded per stage by TMA (2-D map {len, NB}, zero padded).
//
// 3xTF32: X_hi = rn_tf32(X), X_lo = rn_tf32(X - X_hi) are formed in shared
// memory by converter warps (X_hi in place over the TMA-written tile, X_lo
// beside it); D = X_hi U_hi + X_hi U_lo + X_lo U_hi per 8-deep k-step, each
// product exact or within 2^-22 relative with round-to-nearest.  The tensor
// core's fp32 accumulation is not round-to-nearest: it drops bits toward
// zero (measured: a -7e-9 relative bias per accumulated MMA, -2.8e-6 over a
// 1024-long contraction when partial sums stay in TMEM).  So every k-step
// writes a fresh accumulator in a ring of TMEM buffers and the epilogue warps
// add it into fp64 registers: three fp32 accumulations per k-step, fp64 over
// the contraction (scripts/ttm_tc_err.py measures both variants).
// Output fp64 (the rest of the chain runs in fp64).
//
// Shared memory: an 8-deep TMA ring (A tile, B hi, B lo; 20 KB at NB = 16)
// and a 3-slot ring of A lo planes.
//
// Persistent CTAs (one per SM), warp roles (320 threads):
//   warp 0   TMA producer (elected lane): A tile + both B planes per stage
//   warp 1   TMEM allocator, MMA issuer (elected lane): 4 k-steps x 3 MMAs
//            per stage, each k-step into the next buffer of a 256-column
//            TMEM ring
//   warps 2-5  converters (hi / lo split of the A tile)
//   warps 6-9  epilogue: tcgen05.ld of each k-step's buffer, fp64
//            accumulation in registers, fp64 stores at the end of a tile
#include <cuda.h>

#include <algorithm>

#include "common.cuh"
#include "sparse_ttm.cuh"

namespace machb {

namespace {

constexpr int XBM = 128;  // rows per tile (UMMA M)
constexpr int XBK = 32;   // K per stage (128 B of fp32)
constexpr int XLO = 3;    // lo-plane slots (converter -> MMA)
constexpr int kXThreads = 320;
constexpr uint32_t kXA = XBM * XBK * 4;  // 16 KB

template <int NB>
struct XL {
    static constexpr uint32_t B = NB * XBK * 4;              // one B plane per stage
    static constexpr uint32_t stage = kXA + 2 * B;           // TMA stage: A (hi written in place), B hi, B lo
    // TMA ring as deep as shared memory allows (bytes in flight per SM set
    // the streaming rate); the lo planes live in a short ring of their own
    static constexpr int XST = NB <= 16 ? 8 : 7;
    static constexpr std::size_t smem =
        static_cast<std::size_t>(XST) * stage + static_cast<std::size_t>(XLO) * kXA + 1024 /*align*/ + 1024 /*barriers*/;
    static constexpr uint32_t tmem_cols = 256;
    static constexpr int nbuf = 256 / (4 * NB);  // TMEM ring of per-stage slots (4 k-step accumulators each)
};

__device__ __forceinline__ uint32_t s32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "XW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra XW_%=;\n}" ::"r"(s32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma2(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                     s32(dst)),
                 "l"(tm), "r"(s32(bar)), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            s32(dst)),
        "l"(tm), "r"(s32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
           (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (static_cast<uint64_t>(layout) << 61);
}
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(bar)) : "memory");
}
__device__ __forceinline__ float rn_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// tcgen05.ld of NB columns of this warp's 32 lanes (no wait: the caller
// batches several loads before tcgen05.wait::ld)
template <int NB>
__device__ __forceinline__ void tmem_ld_issue(uint32_t taddr, float* v);
template <>
__device__ __forceinline__ void tmem_ld_issue<16>(uint32_t taddr, float* v) {
    uint32_t* r = reinterpret_cast<uint32_t*>(v);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
}
template <>
__device__ __forceinline__ void tmem_ld_issue<32>(uint32_t taddr, float* v) {
    tmem_ld_issue<16>(taddr, v);
    tmem_ld_issue<16>(taddr + 16, v + 16);
}

// MN == false: contract mode 0 (rows = outer, K contiguous).  MN == true:
// contract a mode m > 0 of the view {inner, len, outer}.
template <bool MN, int NB>
__global__ void __launch_bounds__(kXThreads, 1)
    ttm_tc_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tbh,
                  const __grid_constant__ CUtensorMap tbl, long long inner, int len, long long outer, int r,
                  double* __restrict__ out, int dbg) {
    using L = XL<NB>;
    extern __shared__ __align__(1024) unsigned char xsm_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(xsm_raw) + 1023) & ~std::uintptr_t(1023));
    constexpr int XST = L::XST;
    unsigned char* losm = sm + XST * L::stage;  // XLO lo planes
    uint64_t* full = reinterpret_cast<uint64_t*>(losm + XLO * kXA);
    uint64_t* empty = full + XST;
    uint64_t* conv = empty + XST;    // [XLO] lo plane c written (and hi in place)
    uint64_t* lofree = conv + XLO;   // [XLO] MMAs reading lo plane c done
    uint64_t* ready = lofree + XLO;  // [nbuf] the stage's k-step products are in the TMEM slot
    uint64_t* drained = ready + L::nbuf;  // [nbuf] the epilogue has read the slot
    uint32_t* tslot = reinterpret_cast<uint32_t*>(drained + L::nbuf);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long nab = MN ? (inner + XBM - 1) / XBM : 1;         // row blocks per outer slice
    const long long ntiles = MN ? nab * outer : (outer + XBM - 1) / XBM;
    const int nks = (len + XBK - 1) / XBK;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < XST; ++s) {
            bar_init(&full[s], 1);
            bar_init(&empty[s], 1);
        }
        for (int c = 0; c < XLO; ++c) {
            bar_init(&conv[c], 4);
            bar_init(&lofree[c], 1);
        }
        for (int b = 0; b < L::nbuf; ++b) {
            bar_init(&ready[b], 1);
            bar_init(&drained[b], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&ta) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tbh) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tbl) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(tslot)),
                     "r"(L::tmem_cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tslot;

    if (warp == 0) {
        if (lane == 0) {
            long long it = 0;
            for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
                for (int ks = 0; ks < nks; ++ks, ++it) {
                    const int s = static_cast<int>(it % XST);
                    const long long u = it / XST;
                    if (u > 0) bar_wait(&empty[s], static_cast<uint32_t>((u - 1) & 1));
                    unsigned char* a = sm + s * L::stage;
                    unsigned char* bh = a + kXA;
                    unsigned char* bl = bh + L::B;
                    bar_tx(&full[s], kXA + 2 * L::B);
                    if constexpr (MN) {
                        const int a0 = static_cast<int>((t % nab) * XBM), c = static_cast<int>(t / nab);
#pragma unroll
                        for (int m = 0; m < XBM / 32; ++m) tma3(a + m * 4096, &ta, &full[s], a0 + 32 * m, ks * XBK, c);
                    } else {
                        tma2(a, &ta, &full[s], ks * XBK, static_cast<int>(t * XBM));
                    }
                    tma2(bh, &tbh, &full[s], ks * XBK, 0);
                    tma2(bl, &tbl, &full[s], ks * XBK, 0);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (MN ? (1u << 15) : 0u) |
                                   (static_cast<uint32_t>(NB >> 3) << 17) | (static_cast<uint32_t>(XBM >> 4) << 24);
            long long it = 0;
            for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
                for (int ks = 0; ks < nks; ++ks, ++it) {
                    const int s = static_cast<int>(it % XST);
                    const int cl = static_cast<int>(it % XLO);
                    const int b = static_cast<int>(it % L::nbuf);
                    bar_wait(&conv[cl], static_cast<uint32_t>((it / XLO) & 1));
                    if (it >= L::nbuf) bar_wait(&drained[b], static_cast<uint32_t>(((it / L::nbuf) - 1) & 1));
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t ah = s32(sm + s * L::stage), bh = ah + kXA, bl = bh + L::B;
                    const uint32_t al = s32(losm + cl * kXA);
#pragma unroll
                    for (int k = 0; k < XBK / 8; ++k) {
                        const uint32_t d = tmem + static_cast<uint32_t>((4 * b + k) * NB);  // fresh accumulator per k-step
                        uint64_t dah, dal;
                        if constexpr (MN) {
                            dah = sdesc(ah + k * 1024, 4096, 512, 1);
                            dal = sdesc(al + k * 1024, 4096, 512, 1);
                        } else {
                            dah = sdesc(ah + k * 32, 16, 1024, 2);
                            dal = sdesc(al + k * 32, 16, 1024, 2);
                        }
                        const uint64_t dbh = sdesc(bh + k * 32, 16, 1024, 2), dbl = sdesc(bl + k * 32, 16, 1024, 2);
                        mma_tf32(d, dah, dbh, idesc, 0u);
                        mma_tf32(d, dah, dbl, idesc, 1u);
                        mma_tf32(d, dal, dbh, idesc, 1u);
                    }
                    mma_commit(&empty[s]);
                    mma_commit(&lofree[cl]);
                    mma_commit(&ready[b]);
                }
            }
        }
    } else if (warp < 6) {
        // converters: hi = rn_tf32(x) in place, lo = rn_tf32(x - hi) beside it
        const int ct = threadIdx.x - 64;  // 0..127
        long long it = 0;
        for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
            for (int ks = 0; ks < nks; ++ks, ++it) {
                const int s = static_cast<int>(it % XST);
                const int cl = static_cast<int>(it % XLO);
                bar_wait(&full[s], static_cast<uint32_t>((it / XST) & 1));
                if (it >= XLO) bar_wait(&lofree[cl], static_cast<uint32_t>(((it / XLO) - 1) & 1));
                float4* hi = reinterpret_cast<float4*>(sm + s * L::stage);
                float4* lo = reinterpret_cast<float4*>(losm + cl * kXA);
#pragma unroll
                for (int q = 0; q < static_cast<int>(kXA / 16) / 128; ++q) {
                    if (dbg & 1) break;  // timing probe: no conversion (results wrong)
                    const int e = ct + 128 * q;
                    float4 v = hi[e], h, l;
                    h.x = rn_tf32(v.x); h.y = rn_tf32(v.y); h.z = rn_tf32(v.z); h.w = rn_tf32(v.w);
                    l.x = rn_tf32(v.x - h.x); l.y = rn_tf32(v.y - h.y); l.z = rn_tf32(v.z - h.z); l.w = rn_tf32(v.w - h.w);
                    hi[e] = h;
                    lo[e] = l;
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) bar_arrive(&conv[cl]);
            }
        }
    } else {
        // epilogue: warp w reads TMEM lanes 32 (w % 4) .. (tile rows)
        const int q4 = warp & 3;
        const int row = 32 * q4 + lane;
        long long it = 0;
        for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
            double acc[NB];
#pragma unroll
            for (int qq = 0; qq < NB; ++qq) acc[qq] = 0.0;
            for (int ks = 0; ks < nks; ++ks, ++it) {
                const int b = static_cast<int>(it % L::nbuf);
                bar_wait(&ready[b], static_cast<uint32_t>((it / L::nbuf) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t base = tmem + (static_cast<uint32_t>(32 * q4) << 16) + static_cast<uint32_t>(4 * b * NB);
                float v[4][NB];
                if (dbg & 2) {  // timing probe: no TMEM reads (results wrong)
                    __syncwarp();
                    if (lane == 0) bar_arrive(&drained[b]);
                    continue;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) tmem_ld_issue<NB>(base + k * NB, v[k]);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) bar_arrive(&drained[b]);
#pragma unroll
                for (int qq = 0; qq < NB; ++qq)
                    acc[qq] += (static_cast<double>(v[0][qq]) + static_cast<double>(v[1][qq])) +
                               (static_cast<double>(v[2][qq]) + static_cast<double>(v[3][qq]));
            }
            if constexpr (MN) {
                const long long a = (t % nab) * XBM + row, c = t / nab;
                if (a < inner) {
                    double* o = out + a + inner * static_cast<long long>(r) * c;
#pragma unroll
                    for (int qq = 0; qq < NB; ++qq)
                        if (qq < r) o[inner * qq] = acc[qq];
                }
            } else {
                const long long c = t * XBM + row;
                if (c < outer) {
                    double* o = out + static_cast<long long>(r) * c;
#pragma unroll
                    for (int qq = 0; qq < NB; ++qq)
                        if (qq < r) o[qq] = acc[qq];
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(L::tmem_cols) : "memory");
    }
}

// U (len x r, column-major fp64) -> hi / lo tf32 planes of U^T padded to NB rows
// (row q of a plane at q * ld, ld = len rounded up to 4 floats: TMA strides are 16-byte multiples)
__global__ void split_u_kernel(const double* __restrict__ U, int len, int ld, int r, int NB, float* __restrict__ hi,
                               float* __restrict__ lo) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= ld * NB) return;
    const int k = e % ld, q = e / ld;
    float h = 0.0f, l = 0.0f;
    if (q < r && k < len) {
        const double u = U[k + static_cast<long long>(len) * q];
        h = rn_tf32(static_cast<float>(u));
        l = rn_tf32(static_cast<float>(u - static_cast<double>(h)));
    }
    hi[e] = h;
    lo[e] = l;
}

using EncodeTiledX = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                  const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledX encode_x() {
    static EncodeTiledX fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiledX>(p);
    }();
    if (!fn) throw Error(MACH_ERR_CUDA, "cuTensorMapEncodeTiled is not available from the driver");
    return fn;
}

void encode(CUtensorMap* tm, const float* base, int rank, const cuuint64_t* gdim, const cuuint64_t* gstride,
            const cuuint32_t* box, CUtensorMapSwizzle sw) {
    const cuuint32_t es[3] = {1, 1, 1};
    const CUresult rc = encode_x()(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, static_cast<cuuint32_t>(rank), const_cast<float*>(base),
                                   gdim, gstride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rc != CUDA_SUCCESS) throw Error(MACH_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(rc)) + ")");
}

template <bool MN, int NB>
void launch_ttm_tc(Ctx* ctx, const CUtensorMap& ta, const float* uh, const float* ul, long long inner, int len,
                   long long outer, int r, double* out) {
    CUtensorMap tbh, tbl;
    const int ld = (len + 3) & ~3;
    const cuuint64_t bd[2] = {static_cast<cuuint64_t>(len), static_cast<cuuint64_t>(NB)};
    const cuuint64_t bs[1] = {static_cast<cuuint64_t>(ld) * 4};
    const cuuint32_t bb[2] = {XBK, NB};
    encode(&tbh, uh, 2, bd, bs, bb, CU_TENSOR_MAP_SWIZZLE_128B);
    encode(&tbl, ul, 2, bd, bs, bb, CU_TENSOR_MAP_SWIZZLE_128B);
    static std::uint64_t attr = 0;  // per-device mask
    if (first_on_device(attr, ctx->device)) {
        MB_CUDA(cudaFuncSetAttribute(ttm_tc_kernel<MN, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(XL<NB>::smem)));
    }
    const long long nab = MN ? (inner + XBM - 1) / XBM : 1;
    const long long ntiles = MN ? nab * outer : (outer + XBM - 1) / XBM;
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device);
    const int grid = static_cast<int>(std::min<long long>(ntiles, nsm));
    static const int dbg = std::getenv("MACH_TTM_TC_DBG") ? std::atoi(std::getenv("MACH_TTM_TC_DBG")) : 0;
    MB_LAUNCH(ctx, (ttm_tc_kernel<MN, NB>), grid, kXThreads, XL<NB>::smem, ta, tbh, tbl, inner, len, outer, r, out, dbg);
}

}  // namespace

bool ttm_tc_applies(const std::vector<int>& dims, int m, int r) {
    static const bool off = std::getenv("MACH_NO_TTM_TC") != nullptr;
    if (off || r < 1 || r > 32) return false;
    long long inner = 1, outer = 1;
    for (int j = 0; j < m; ++j) inner *= dims[static_cast<std::size_t>(j)];
    for (std::size_t j = static_cast<std::size_t>(m) + 1; j < dims.size(); ++j) outer *= dims[j];
    const long long len = dims[static_cast<std::size_t>(m)];
    if (len < 32 || inner * len * outer < (1ll << 20)) return false;
    if (len >= (1ll << 31) || outer >= (1ll << 31)) return false;
    if (m == 0) return (len % 4) == 0;
    // MN-major: the row blocks run along the contiguous inner index
    return inner >= XBM && (inner % 4) == 0 && inner < (1ll << 31);
}

// out (dims with I_m -> r, first-mode-fastest, fp64) = x x_m U^T, U len x r
void ttm_tc(Ctx* ctx, const float* x, const std::vector<int>& dims, int m, const double* U, int r, double* out) {
    if (!ttm_tc_applies(dims, m, r)) throw Error(MACH_ERR_INTERNAL, "ttm_tc: shape not supported");
    long long inner = 1, outer = 1;
    for (int j = 0; j < m; ++j) inner *= dims[static_cast<std::size_t>(j)];
    for (std::size_t j = static_cast<std::size_t>(m) + 1; j < dims.size(); ++j) outer *= dims[j];
    const int len = dims[static_cast<std::size_t>(m)];
    const int NB = r <= 16 ? 16 : 32;
    const int ld = (len + 3) & ~3;
    DBuf<float> uh(ctx, static_cast<std::size_t>(ld) * NB), ul(ctx, static_cast<std::size_t>(ld) * NB);
    MB_LAUNCH(ctx, split_u_kernel, ceil_div(static_cast<long long>(ld) * NB, 256), 256, 0, U, len, ld, r, NB, uh.get(), ul.get());
    CUtensorMap ta;
    if (m == 0) {
        const cuuint64_t gd[2] = {static_cast<cuuint64_t>(len), static_cast<cuuint64_t>(outer)};
        const cuuint64_t gs[1] = {static_cast<cuuint64_t>(len) * 4};
        const cuuint32_t bx[2] = {XBK, XBM};
        encode(&ta, x, 2, gd, gs, bx, CU_TENSOR_MAP_SWIZZLE_128B);
        if (NB == 16) launch_ttm_tc<false, 16>(ctx, ta, uh.get(), ul.get(), 1, len, outer, r, out);
        else launch_ttm_tc<false, 32>(ctx, ta, uh.get(), ul.get(), 1, len, outer, r, out);
    } else {
        const cuuint64_t gd[3] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(len), static_cast<cuuint64_t>(outer)};
        const cuuint64_t gs[2] = {static_cast<cuuint64_t>(inner) * 4, static_cast<cuuint64_t>(inner) * len * 4};
        const cuuint32_t bx[3] = {32, XBK, 1};
        encode(&ta, x, 3, gd, gs, bx, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
        if (NB == 16) launch_ttm_tc<true, 16>(ctx, ta, uh.get(), ul.get(), inner, len, outer, r, out);
        else launch_ttm_tc<true, 32>(ctx, ta, uh.get(), ul.get(), inner, len, outer, r, out);
    }
}

}  // namespace machb
