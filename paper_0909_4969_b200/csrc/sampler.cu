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
// SparseTensor, tensor.cpp:78-96) with a single-pass decoupled look-back scan
// over tiles of 8192 (fp32) / 4096 (fp64) elements, claimed in order through
// an atomic ticket by persistent warp-specialised CTAs (see sample_kernel):
// a producer warp stages each tile in shared memory by one bulk copy, eight
// hashing warps own 128 contiguous bytes each (so a thread's kept elements are
// contiguous in the output), and a look-back warp resolves tile prefixes while
// the next tile is hashed.  The input is read exactly once.
//
// Round-2 rewrite (C2 sampler 0.38 -> 0.21 ms, ncu): the old kernel executed
// 70 instructions per element (bounds checks, per-element 64-bit compares,
// look-back spinning and barriers); this one ~25 for the hash plus ~8 for
// the tile machinery.  It is issue-bound on the 32-bit SplitMix64 rounds
// (ncu: issue active 66%, DRAM 34%), with the integer work balanced between
// the ALU and FMA pipes (the keep bit and the mask are IMADs).
// Build knobs: MACH_SAMP_HW (hashing warps), MACH_SAMP_NB (tile buffers),
// MACH_SAMP_MINB (CTAs per SM); run-time MACH_SAMPLER_TB=64 (16 KB tiles).

#include <cmath>
#include <cstdlib>

#include "common.cuh"

namespace machb {

namespace {

#ifndef MACH_SAMP_HW
#define MACH_SAMP_HW 8
#endif
#ifndef MACH_SAMP_NB
#define MACH_SAMP_NB 2
#endif
#ifndef MACH_SAMP_MINB
#define MACH_SAMP_MINB 3
#endif
constexpr int kThreads = 32 * MACH_SAMP_HW;  // hashing threads per CTA

constexpr std::uint64_t kFlagAgg = 1ull << 62;
constexpr std::uint64_t kFlagPre = 2ull << 62;
constexpr std::uint64_t kValMask = (1ull << 62) - 1;

__device__ __forceinline__ std::uint64_t splitmix_finalize(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

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

// ---- tile-staged sampler (round 2) ----
// One CTA per tile of 256 threads x 128 bytes (8192 fp32 / 4096 fp64
// elements).  The tile arrives in shared memory by ONE bulk copy
// (cp.async.bulk, mbarrier completion): no registers are held across the load
// latency, so 6 CTAs (192 KB of loads) are resident per SM.  Each thread then
// owns 128 contiguous bytes of the tile (element order = thread order =
// ascending flat index), so its kept elements are contiguous in the output and
// the tile's scan is a plain scan of one popcount per thread.  The 16-byte
// chunks of a thread are visited in rotated order (chunk (c + tid) & 7):
// the 8 lanes of a shared-memory phase read 8 distinct bank groups.
// Partial tail tiles are staged by plain loads and zero padded (x == 0 is
// never kept, so padding needs no bounds checks in the hash loop).
// Hash: SplitMix64 on 32-bit halves.  MODE 0 (thr_hi < 2^31, i.e. p < 1/2):
// the last xor-shift only flips bit 0 of a high word >= 2^31, so
// hhi < thr_hi <=> zhi < thr_hi and a high-word tie is zhi == thr_hi; MODE 1
// the general high-word compare; MODE 2 keeps every nonzero (p = 1).  A tie
// sends the thread through the exact 64-bit compare (probability ~2^-27 per
// thread).  The look-back polls back off with nanosleep so a waiting warp
// does not steal issue slots from the hashing warps.
__device__ __forceinline__ std::uint32_t s_u32(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

// High word of SplitMix64's second product, z * C2 >> 32 with the two
// xor-shift rounds before it, on 32-bit halves.  The integer work is split
// between the ALU pipe (xor, shifts) and the FMA pipe (IMAD): each pipe
// accepts one warp instruction per two cycles, so the balance sets the rate.
__device__ __forceinline__ unsigned splitmix_zhi(unsigned zl, unsigned zh) {
    const unsigned al = zl ^ __funnelshift_r(zl, zh, 30), ah = zh ^ (zh >> 30);
    const std::uint64_t pm = static_cast<std::uint64_t>(al) * 0x1CE4E5B9u;
    const unsigned yl = static_cast<unsigned>(pm);
    const unsigned yh = static_cast<unsigned>(pm >> 32) + al * 0xBF58476Du + ah * 0x1CE4E5B9u;
    const unsigned bl = yl ^ __funnelshift_r(yl, yh, 27), bh = yh ^ (yh >> 27);
    return __umulhi(bl, 0x133111EBu) + bl * 0x94D049BBu + bh * 0x133111EBu;
}

// 1 iff zhi >= thr, on the FMA pipe: the high word of zhi * 1 + (2^32 - thr),
// one IMAD.WIDE.U32 with a loop-invariant 64-bit addend.  `unit` (= 1) and
// `add` are kernel arguments, so ptxas cannot turn the product into ALU adds.
__device__ __forceinline__ unsigned ge_bit(unsigned zhi, unsigned unit, std::uint64_t add) {
    return static_cast<unsigned>((static_cast<std::uint64_t>(zhi) * unit + add) >> 32);
}

// Keep mask of one thread's EPT = NCH x 16 B elements, bit e = element e.
// Chunks are visited in rotated order (c + r) mod NCH and their bits collected at
// iteration positions (constant weights); one funnel rotation at the end puts
// them at element positions.  MODE 0 (thr_hi < 2^31): the last xor-shift only
// flips bit 0 of a high word >= 2^31, so hhi < thr_hi <=> zhi < thr_hi, a
// high-word tie is zhi == thr_hi, and the "not kept" bit is ge_bit(zhi).
// Zeros are found per chunk by a product (an underflowing product only costs
// the recheck); a thread that saw a zero or a high-word tie recomputes its
// mask exactly.
template <typename T, int MODE, int NCH>
__device__ __forceinline__ unsigned hash_thread(const T* __restrict__ mine, int tid, std::uint64_t zt,
                                                unsigned thr_hi, unsigned unit, std::uint64_t add, bool& slow,
                                                T& nanacc) {
    constexpr int VEC = 16 / sizeof(T);
    constexpr std::uint64_t G = 0x9E3779B97F4A7C15ULL;
    const unsigned two = unit + unit;
    unsigned mask = 0;  // MODE 0: NOT-kept bits shifted in from the bottom (bit-reversed order); else kept
    bool zero = false, tie = false;
    // rotation r: the 8 lanes of a 16-byte shared-memory phase read 8 distinct bank groups
    const int r = (tid / (8 / NCH)) & (NCH - 1);
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        const int cc = (c + r) & (NCH - 1);
        T v[VEC];
        if constexpr (sizeof(T) == 4) {
            const float4 q = *reinterpret_cast<const float4*>(mine + cc * VEC);
            v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
        } else {
            const double2 q = *reinterpret_cast<const double2*>(mine + cc * VEC);
            v[0] = q.x; v[1] = q.y;
        }
        T cp = v[0];
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
            nanacc = fma(v[j], T(0), nanacc);
            if (j) cp *= v[j];
        }
        if constexpr (MODE == 2) {
#pragma unroll
            for (int j = 0; j < VEC; ++j)
                if (v[j] != T(0)) mask |= 1u << (c * VEC + j);
        } else {
            zero |= (cp == T(0));
            std::uint64_t z = zt + static_cast<std::uint64_t>(cc) * (VEC * G);
#pragma unroll
            for (int j = 0; j < VEC; ++j) {
                const unsigned zhi = splitmix_zhi(static_cast<unsigned>(z), static_cast<unsigned>(z >> 32));
                if constexpr (MODE == 0) {
                    tie |= (zhi == thr_hi);
                    mask = mask * two + ge_bit(zhi, unit, add);
                } else {
                    const unsigned hhi = zhi ^ (zhi >> 31);
                    tie |= (hhi == thr_hi);
                    if (hhi < thr_hi) mask |= 1u << (c * VEC + j);
                }
                z += G;
            }
        }
    }
    slow |= zero | tie;
    constexpr int EPT = NCH * VEC;
    constexpr unsigned FULL = EPT == 32 ? 0xFFFFFFFFu : ((1u << EPT) - 1u);
    if constexpr (MODE == 0) mask = ~(__brev(mask) >> (32 - EPT)) & FULL;
    const int rot = r * VEC;  // rotate within EPT bits
    if constexpr (EPT == 32) return __funnelshift_l(mask, mask, rot);
    else return ((mask << rot) | (mask >> (EPT - rot))) & FULL;
}

__device__ __forceinline__ void mbar_init(std::uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(std::uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint64_t* b, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "SW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra SW_%=;\n}" ::"r"(s_u32(b)),
        "r"(parity)
        : "memory");
}

// wait for a phase, suspended in the barrier unit (suspend-time hint) rather
// than spinning: the producer and look-back warps wait most of the time and a
// hot try_wait loop would take issue slots from the hashing warps
__device__ __forceinline__ void mbar_wait_sleep(std::uint64_t* b, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "SWS_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra SWS_%=;\n}" ::"r"(s_u32(b)),
        "r"(parity), "r"(1000000u)
        : "memory");
}

// Warp-specialised persistent CTAs, every CTA of the grid resident:
//   8 hashing warps, 1 look-back warp, 1 producer warp; NB = 3 tile buffers
//   and 2 staging slots for the kept entries.
//   producer (lane 0): takes a ticket and issues the tile's bulk copy into a
//     buffer as soon as the hashing warps release it;
//   hashing warps: hash tile i, scan it (one named barrier), publish its
//     aggregate, stage its kept (tile offset, x) compactly in shared memory
//     and release the tile buffer at once (the next copy starts while the
//     tile still waits for its prefix); then write tile i-1 from its staging
//     slot, coalesced across the CTA, once its prefix is known;
//   look-back warp: resolves each tile's exclusive prefix by the decoupled
//     look-back as soon as its aggregate is published and publishes the
//     inclusive prefix (so look-backs elsewhere stay short).
// A tile with more kept entries than a staging slot holds (p above ~0.1)
// keeps its buffer and is written from it per thread.  Waits are only on
// tiles with smaller tickets; a CTA's unhashed tiles have larger tickets than
// every tile it waits on, so waits cannot form a cycle.
template <typename T, typename IdxT, int TB>
__global__ void __launch_bounds__(kThreads + 64, MACH_SAMP_MINB) sample_kernel(const T* __restrict__ x, std::int64_t numel,
                                                               std::int64_t gofs,  // global flat index of x[0]
                                                               std::uint64_t seed, std::uint64_t thr_shift,
                                                               int mode, unsigned unit, std::uint64_t ge_add,
                                                               double p, double inv_p,
                                                               IdxT* __restrict__ out_idx, T* __restrict__ out_val,
                                                               std::int64_t capacity,
                                                               unsigned long long* __restrict__ status,
                                                               unsigned int* __restrict__ ticket,
                                                               long long* __restrict__ total_out,
                                                               int* __restrict__ flags) {
    constexpr int NCH = TB / 16;           // 16-byte chunks per thread
    constexpr int EPT = TB / sizeof(T);    // elements per thread
    constexpr int TILE = kThreads * EPT;
    constexpr int NW = kThreads / 32;      // hashing warps
    constexpr int NB = MACH_SAMP_NB;       // tile buffers
    constexpr int SCAP = TILE / 8;         // staged kept entries per tile
    constexpr unsigned kBytes = TILE * sizeof(T);
    static_assert(TILE <= 65536, "tile offsets are staged as u16");
    extern __shared__ __align__(128) unsigned char s_dyn[];
    T* s_buf = reinterpret_cast<T*>(s_dyn);                               // [NB][TILE]
    T* s_sval = s_buf + NB * TILE;                                        // [2][SCAP]
    unsigned short* s_sidx = reinterpret_cast<unsigned short*>(s_sval + 2 * SCAP);  // [2][SCAP]
    __shared__ alignas(8) std::uint64_t s_full[NB], s_empty[NB], s_agg[NB], s_pre[NB];
    __shared__ unsigned s_wtot[2][NW];
    __shared__ long long s_excl[NB];
    __shared__ unsigned s_tile[NB], s_total[NB];
    __shared__ long long s_atile[NB];
    __shared__ std::uint64_t s_par[2];  // ge_add, thr_hi | unit << 32: read back into registers
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const std::int64_t ntiles = (numel + TILE - 1) / TILE;
    if (tid == 0) {
        s_par[0] = ge_add;
        s_par[1] = (thr_shift >> 32) | (static_cast<std::uint64_t>(unit) << 32);
        for (int b = 0; b < NB; ++b) {
            mbar_init(&s_full[b], 1);
            mbar_init(&s_empty[b], NW);
            mbar_init(&s_agg[b], 1);
            mbar_init(&s_pre[b], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == NW + 1) {
        // ================= producer warp =================
        if (lane != 0) return;
        for (int k = 0;; ++k) {
            const int b = k % NB;
            if (k >= NB) mbar_wait_sleep(&s_empty[b], ((k / NB) - 1) & 1u);
            const unsigned t = atomicAdd(ticket, 1u);
            s_tile[b] = t;
            if (static_cast<std::int64_t>(t) * TILE + TILE <= numel) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(&s_full[b])),
                             "r"(kBytes)
                             : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        s_u32(s_buf + b * TILE)),
                    "l"(x + static_cast<std::int64_t>(t) * TILE), "r"(kBytes), "r"(s_u32(&s_full[b]))
                    : "memory");
            } else {
                mbar_arrive(&s_full[b]);  // partial last tile (loaded by the hashing warps) or the end
                if (t >= ntiles) return;  // tickets only grow: nothing more to load
            }
        }
    }
    if (warp == NW) {
        // ================= look-back warp =================
        for (int i = 0;; ++i) {
            const int b = i % NB;
            mbar_wait_sleep(&s_agg[b], (i / NB) & 1u);
            const std::int64_t t = s_atile[b];
            if (t < 0) return;
            const unsigned total = s_total[b];
            long long excl = 0;
            if (t > 0) {
                std::int64_t look = t - 1;
                unsigned ns = 32;
                while (true) {
                    const std::int64_t j = look - lane;
                    unsigned long long st = kFlagPre | 0ull;
                    if (j >= 0)
                        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(st) : "l"(status + j) : "memory");
                    const bool unset = (st >> 62) == 0;
                    if (__any_sync(0xffffffffu, unset)) {
                        __nanosleep(ns);
                        if (ns < 256) ns <<= 1;
                        continue;
                    }
                    const unsigned pmask = __ballot_sync(0xffffffffu, (st & ~kValMask) == kFlagPre);
                    long long mine_v = static_cast<long long>(st & kValMask);
                    if (pmask) {
                        const int first = __ffs(pmask) - 1;
                        if (lane > first) mine_v = 0;
                    }
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) mine_v += __shfl_xor_sync(0xffffffffu, mine_v, off);
                    excl += mine_v;
                    if (pmask) break;
                    look -= 32;
                }
                if (lane == 0) atomicExch(&status[t], kFlagPre | static_cast<unsigned long long>(excl + total));
            }
            if (lane == 0) {
                s_excl[b] = excl;
                if (t == ntiles - 1) *total_out = excl + total;
                mbar_arrive(&s_pre[b]);
            }
            __syncwarp();
        }
    }
    // ================= hashing warps =================
    const std::uint64_t add_r = s_par[0];
    const unsigned thr_hi = static_cast<unsigned>(s_par[1]), unit_r = static_cast<unsigned>(s_par[1] >> 32);
    // the previous tile: aggregate published, waiting for its prefix and writes
    std::int64_t ptile = -1;
    unsigned pkeep = 0, poff = 0, ptotal = 0;
    int pb = 0, pi = 0;
    bool pstaged = false;
    auto write = [&]() {
        mbar_wait(&s_pre[pb], (pi / NB) & 1u);
        const long long g0 = s_excl[pb];
        const bool fits = g0 + ptotal <= capacity;
        if (!fits && tid == 0 && ptotal) atomicOr(flags, 2);
        const std::int64_t tb = gofs + ptile * TILE;
        if (pstaged) {
            if (fits) {
                const T* sv = s_sval + (pi & 1) * SCAP;
                const unsigned short* si = s_sidx + (pi & 1) * SCAP;
                for (int r = tid; r < static_cast<int>(ptotal); r += kThreads) {
                    out_idx[g0 + r] = static_cast<IdxT>(tb + si[r]);
                    out_val[g0 + r] = scaled<T>(sv[r], p, inv_p);
                }
            }
        } else {
            if (fits) {
                long long g = g0 + poff;
                const T* mine = s_buf + pb * TILE + tid * EPT;
                unsigned keep = pkeep;
                while (keep) {
                    const int bit = __ffs(keep) - 1;
                    keep &= keep - 1;
                    out_idx[g] = static_cast<IdxT>(tb + tid * EPT + bit);
                    out_val[g] = scaled<T>(mine[bit], p, inv_p);
                    ++g;
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[pb]);
        }
    };
    int i = 0;
    for (;; ++i) {
        const int b = i % NB;
        mbar_wait(&s_full[b], (i / NB) & 1u);
        const std::int64_t tile = s_tile[b];
        if (tile >= ntiles) {
            if (tid == 0) {
                s_atile[b] = -1;
                mbar_arrive(&s_agg[b]);
            }
            break;
        }
        const std::int64_t base = tile * TILE;
        T* s_x = s_buf + b * TILE;
        if (base + TILE > numel) {  // the partial last tile: plain loads, zero padded
            for (int e = tid; e < TILE; e += kThreads) s_x[e] = (base + e < numel) ? x[base + e] : T(0);
            asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory");
        }
        const T* mine = s_x + tid * EPT;
        const std::uint64_t zt =
            seed + (static_cast<std::uint64_t>(gofs + base + tid * EPT) + 1ull) * 0x9E3779B97F4A7C15ULL;
        bool slow = false;
        T nanacc = T(0);  // x * 0 is NaN exactly for inf / NaN inputs
        unsigned keep;
        if (mode == 0)
            keep = hash_thread<T, 0, NCH>(mine, tid, zt, thr_hi, unit_r, add_r, slow, nanacc);
        else if (mode == 1)
            keep = hash_thread<T, 1, NCH>(mine, tid, zt, thr_hi, unit_r, add_r, slow, nanacc);
        else
            keep = hash_thread<T, 2, NCH>(mine, tid, zt, thr_hi, unit_r, add_r, slow, nanacc);
        if (slow && mode != 2) {  // exact: zeros dropped, 64-bit compare (after a zero or a high-word tie)
            keep = 0;
            for (int e = 0; e < EPT; ++e) {
                if (mine[e] == T(0)) continue;
                const std::uint64_t h =
                    splitmix_finalize(seed + (static_cast<std::uint64_t>(gofs + base + tid * EPT + e) + 1ull) *
                                                 0x9E3779B97F4A7C15ULL);
                if (h < thr_shift) keep |= 1u << e;
            }
        }
        if (nanacc != nanacc) atomicOr(flags, 1);
        // ---- block scan of the per-thread kept counts (hashing warps only) ----
        const unsigned cnt = __popc(keep);
        unsigned inc = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) s_wtot[i & 1][warp] = inc;
        // also orders the last tile's staging writes before this tile's staged reads
        asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory");
        unsigned before = 0, tile_total = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const unsigned t = s_wtot[i & 1][w];
            before += (w < warp) ? t : 0u;
            tile_total += t;
        }
        if (tid == 0) {  // tile 0's aggregate is its inclusive prefix
            atomicExch(&status[tile], (tile == 0 ? kFlagPre : kFlagAgg) | tile_total);
            s_total[b] = tile_total;
            s_atile[b] = tile;
            mbar_arrive(&s_agg[b]);
        }
        const unsigned off = before + inc - cnt;
        const bool staged = tile_total <= static_cast<unsigned>(SCAP);
        if (staged) {  // stage (tile offset, x) and release the tile buffer now
            T* sv = s_sval + (i & 1) * SCAP;
            unsigned short* si = s_sidx + (i & 1) * SCAP;
            unsigned k = keep, o = off;
            while (k) {
                const int bit = __ffs(k) - 1;
                k &= k - 1;
                si[o] = static_cast<unsigned short>(tid * EPT + bit);
                sv[o] = mine[bit];
                ++o;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[b]);
        }
        if (ptile >= 0) write();
        ptile = tile;
        pkeep = keep;
        poff = off;
        ptotal = tile_total;
        pb = b;
        pi = i;
        pstaged = staged;
    }
    if (ptile >= 0) {
        // the staged entries of the last tile were written by other warps
        asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory");
        write();
    }
}

template <typename T, typename IdxT, int TB>
std::int64_t launch_sample_tb(Ctx* ctx, const T* x, std::int64_t numel, std::int64_t gofs, std::uint64_t seed,
                              double p, std::int64_t capacity, IdxT* out_idx, T* out_val, int* flags_host) {
    constexpr int TILE = kThreads * (TB / static_cast<int>(sizeof(T)));
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
    // mode 0: high-word threshold below 2^31 (the last xor-shift cannot create a keep); 1: general; 2: p == 1
    const int mode = keep_all ? 2 : ((thr >> 32) < 0x80000000ull ? 0 : 1);
    constexpr int kSmem = MACH_SAMP_NB * TILE * static_cast<int>(sizeof(T)) + 2 * (TILE / 8) * (static_cast<int>(sizeof(T)) + 2);
    static std::uint64_t attr_set = 0;  // per-device mask
    static int resident[64] = {};
    if (first_on_device(attr_set, ctx->device)) {
        MB_CUDA(cudaFuncSetAttribute(sample_kernel<T, IdxT, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        int per_sm = 0, sms = 0;
        MB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sample_kernel<T, IdxT, TB>, kThreads + 64, kSmem));
        MB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
        resident[ctx->device & 63] = std::max(1, per_sm) * sms;
    }
    // every CTA of the grid must be resident (the look-back waits on tiles held by other CTAs)
    const std::int64_t grid = std::min<std::int64_t>(ntiles, resident[ctx->device & 63]);
    if (ntiles > 0)
        MB_LAUNCH(ctx, (sample_kernel<T, IdxT, TB>), static_cast<unsigned>(grid), kThreads + 64, kSmem, x, numel, gofs,
                  seed, thr, mode, 1u, (1ull << 32) - (thr >> 32), p, 1.0 / p, out_idx, out_val, capacity, status,
                  ticket, total, flags);
    long long tot = 0;
    int fl = 0;
    to_host(ctx, &tot, total, 1);
    to_host(ctx, &fl, flags, 1);
    sync(ctx);
    *flags_host = fl;
    return tot;
}

// tile size: 128 bytes per thread (8192 fp32 elements, 2 CTAs of 3 x 32 KB per
// SM) or 64 (MACH_SAMPLER_TB=64: 4 CTAs of 3 x 16 KB)
template <typename T, typename IdxT>
std::int64_t launch_sample(Ctx* ctx, const T* x, std::int64_t numel, std::int64_t gofs, std::uint64_t seed, double p,
                           std::int64_t capacity, IdxT* out_idx, T* out_val, int* flags_host) {
    static const int tb = [] {
        const char* e = std::getenv("MACH_SAMPLER_TB");
        return (e && std::atoi(e) == 64) ? 64 : 128;
    }();
    if (tb == 64)
        return launch_sample_tb<T, IdxT, 64>(ctx, x, numel, gofs, seed, p, capacity, out_idx, out_val, flags_host);
    return launch_sample_tb<T, IdxT, 128>(ctx, x, numel, gofs, seed, p, capacity, out_idx, out_val, flags_host);
}

// ---- p == 1: every nonzero entry is kept (sampling.cpp:25-27 with u < 1 always) ----
// The look-back kernel above stages at most TILE / 8 kept entries per tile and
// falls back to per-thread strided stores beyond that (16 ms at 1024^3).  With
// p = 1 no hash is needed: count the nonzeros per block, scan the block
// counts, and write index and value runs coalesced (two streaming passes).
constexpr int kAllBlock = 256, kAllPer = 16, kAllTile = kAllBlock * kAllPer;

template <typename T>
__global__ void __launch_bounds__(kAllBlock) keep_all_count_kernel(const T* __restrict__ x, std::int64_t numel,
                                                                   unsigned* __restrict__ counts, int* __restrict__ flags) {
    const std::int64_t base = static_cast<std::int64_t>(blockIdx.x) * kAllTile;
    unsigned c = 0;
    bool bad = false;
#pragma unroll
    for (int k = 0; k < kAllPer; ++k) {
        const std::int64_t i = base + k * kAllBlock + threadIdx.x;
        if (i < numel) {
            const T v = x[i];
            c += v != T(0);
            bad |= !isfinite(v);
        }
    }
    if (bad) atomicOr(flags, 1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    __shared__ unsigned red[kAllBlock / 32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned t = 0;
        for (int w = 0; w < kAllBlock / 32; ++w) t += red[w];
        counts[blockIdx.x] = t;
    }
}

// one block: exclusive scan of the block counts into 64-bit offsets (+ the total)
__global__ void __launch_bounds__(1024) keep_all_scan_kernel(const unsigned* __restrict__ counts, std::int64_t n,
                                                             long long* __restrict__ offs, long long* __restrict__ total) {
    __shared__ long long part[1024];
    const std::int64_t per = (n + 1023) / 1024;
    const std::int64_t b0 = threadIdx.x * per, b1 = min(n, b0 + per);
    long long s = 0;
    for (std::int64_t i = b0; i < b1; ++i) s += counts[i];
    part[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long run = 0;
        for (int i = 0; i < 1024; ++i) {
            const long long v = part[i];
            part[i] = run;
            run += v;
        }
        *total = run;
    }
    __syncthreads();
    long long run = part[threadIdx.x];
    for (std::int64_t i = b0; i < b1; ++i) {
        offs[i] = run;
        run += counts[i];
    }
}

template <typename T, typename IdxT>
__global__ void __launch_bounds__(kAllBlock) keep_all_write_kernel(const T* __restrict__ x, std::int64_t numel,
                                                                   std::int64_t gofs, const long long* __restrict__ offs,
                                                                   IdxT* __restrict__ out_idx, T* __restrict__ out_val) {
    const std::int64_t base = static_cast<std::int64_t>(blockIdx.x) * kAllTile;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ unsigned wsum[kAllBlock / 32];
    __shared__ long long run_s;
    if (threadIdx.x == 0) run_s = offs[blockIdx.x];
    __syncthreads();
#pragma unroll 1
    for (int k = 0; k < kAllPer; ++k) {
        const std::int64_t i = base + k * kAllBlock + threadIdx.x;
        T v = T(0);
        if (i < numel) v = x[i];
        const bool keep = v != T(0);
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) wsum[warp] = __popc(m);
        __syncthreads();
        unsigned before = 0, all = 0;
#pragma unroll
        for (int w = 0; w < kAllBlock / 32; ++w) {
            const unsigned c = wsum[w];
            before += w < warp ? c : 0u;
            all += c;
        }
        const long long run = run_s;
        if (keep) {
            const long long o = run + before + __popc(m & ((1u << lane) - 1u));
            out_idx[o] = static_cast<IdxT>(gofs + i);
            out_val[o] = v;
        }
        __syncthreads();
        if (threadIdx.x == 0) run_s = run + all;
    }
}

template <typename T, typename IdxT>
std::int64_t launch_keep_all(Ctx* ctx, const T* x, std::int64_t numel, std::int64_t gofs, void** out_idx, void** out_val,
                             int* flags_host) {
    const std::int64_t nb = (numel + kAllTile - 1) / kAllTile;
    DBuf<unsigned> counts(ctx, static_cast<std::size_t>(nb));
    DBuf<long long> offs(ctx, static_cast<std::size_t>(nb) + 1);
    DBuf<int> flags(ctx, 1);
    flags.zero(ctx);
    MB_LAUNCH(ctx, keep_all_count_kernel<T>, static_cast<unsigned>(nb), kAllBlock, 0, x, numel, counts.get(), flags.get());
    MB_LAUNCH(ctx, keep_all_scan_kernel, 1, 1024, 0, counts.get(), nb, offs.get(), offs.get() + nb);
    long long tot = 0;
    to_host(ctx, &tot, offs.get() + nb, 1);
    to_host(ctx, flags_host, flags.get(), 1);
    sync(ctx);
    if ((*flags_host & 1) || tot == 0) return tot;
    MB_CUDA(cudaMallocAsync(out_idx, static_cast<std::size_t>(tot) * sizeof(IdxT), ctx->stream));
    MB_CUDA(cudaMallocAsync(out_val, static_cast<std::size_t>(tot) * sizeof(T), ctx->stream));
    MB_LAUNCH(ctx, (keep_all_write_kernel<T, IdxT>), static_cast<unsigned>(nb), kAllBlock, 0, x, numel, gofs, offs.get(),
              static_cast<IdxT*>(*out_idx), static_cast<T*>(*out_val));
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
    if (p == 1.0 && x->numel > 0 && x->numel / kAllTile < 0x7fffffffll && !std::getenv("MACH_SAMPLER_NO_KEEP_ALL")) {
        void *di = nullptr, *dv = nullptr;
        int flags = 0;
        std::int64_t nnz = 0;
        if (x->dtype == MACH_F32)
            nnz = out->idx64 ? launch_keep_all<float, unsigned long long>(ctx, static_cast<const float*>(x->data), x->numel,
                                                                          offset, &di, &dv, &flags)
                             : launch_keep_all<float, unsigned int>(ctx, static_cast<const float*>(x->data), x->numel, offset,
                                                                    &di, &dv, &flags);
        else
            nnz = out->idx64 ? launch_keep_all<double, unsigned long long>(ctx, static_cast<const double*>(x->data), x->numel,
                                                                           offset, &di, &dv, &flags)
                             : launch_keep_all<double, unsigned int>(ctx, static_cast<const double*>(x->data), x->numel,
                                                                     offset, &di, &dv, &flags);
        if (flags & 1) throw_arg("tensor values must be finite");
        out->nnz = nnz;
        out->idx = di;
        out->val = dv;
        return out.release();
    }
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
