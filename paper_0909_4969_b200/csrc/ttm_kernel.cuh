// Fused mode-n TTM kernel (included by sparse_ttm.cu).
//
// Persistent warps, one sorted sub-tile (<= 32*seg nonzeros of one output row)
// at a time.  Each warp double-buffers its sub-tiles in shared memory with 1-D
// TMA bulk copies (cp.async.bulk ... mbarrier::complete_tx) so the HBM stream
// is in flight while the previous sub-tile is reduced; lanes then walk `seg`
// consecutive nonzeros each (seg odd => conflict-free shared-memory reads of
// the linear TMA layout).  Factor rows (U_a, U_b) are staged once per CTA in
// shared memory when they fit.
#pragma once

namespace machb {
namespace ttm {

constexpr int kFB = 4;  // fibre queue depth per lane

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(std::uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* bar, std::uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, std::uint32_t bytes, std::uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, std::uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

inline std::size_t al16(std::size_t x) { return (x + 15) & ~static_cast<std::size_t>(15); }

// Per-warp shared-memory carve-up (host and device agree on this).
template <typename T, typename K, int RA>
struct WarpLayout {
    int seg;
    std::size_t kbuf, vbuf, f, eib, ord, total;
    __host__ __device__ explicit WarpLayout(int s) : seg(s) {
        kbuf = ((32ull * s * sizeof(K) + 32 + 15) / 16) * 16;  // +32: alignment slack of the bulk copy
        vbuf = ((32ull * s * sizeof(T) + 32 + 15) / 16) * 16;
        f = ((32ull * kFB * RA * sizeof(T) + 15) / 16) * 16;
        eib = ((32ull * kFB * sizeof(int) + 15) / 16) * 16;
        ord = ((32ull * kFB * sizeof(short) + 15) / 16) * 16;
        total = 16 /*2 mbarriers*/ + 2 * (kbuf + vbuf) + f + eib + ord;
    }
};

template <typename T, typename K, int RA>
__global__ void __launch_bounds__(256) ttm_mode_kernel(TtmArgs<T, K> A) {
    extern __shared__ __align__(128) unsigned char smraw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    const WarpLayout<T, K, RA> L(A.seg);

    // ---- CTA-shared factor rows ----
    unsigned char* fac = smraw;
    const T* Ua = A.Ua;
    const T* Ub = A.Ub;
    if (A.fac_smem) {
        T* ua = reinterpret_cast<T*>(fac);
        T* ub = ua + A.ua_elems;
        for (long long i = threadIdx.x; i < A.ua_elems; i += blockDim.x) ua[i] = A.Ua[i];
        for (long long i = threadIdx.x; i < A.ub_elems; i += blockDim.x) ub[i] = A.Ub[i];
        Ua = ua;
        Ub = ub;
    }
    unsigned char* wbase = smraw + A.fac_bytes + L.total * wib;
    std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(wbase);
    unsigned char* kb[2] = {wbase + 16, wbase + 16 + L.kbuf};
    unsigned char* vb[2] = {wbase + 16 + 2 * L.kbuf, wbase + 16 + 2 * L.kbuf + L.vbuf};
    T* F = reinterpret_cast<T*>(wbase + 16 + 2 * (L.kbuf + L.vbuf));
    int* EIB = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(F) + L.f);
    short* ord = reinterpret_cast<short*>(reinterpret_cast<unsigned char*>(EIB) + L.eib);
    if (lane == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const long long gw = static_cast<long long>(blockIdx.x) * nw + wib;
    const long long stride = static_cast<long long>(gridDim.x) * nw;

    // issue the bulk copies of sub-tile s into buffer b (lane 0 only)
    auto prefetch = [&](long long s, int b) {
        const SubTile st = A.subs[s];
        const unsigned char* kg = reinterpret_cast<const unsigned char*>(A.keys) + st.start * sizeof(K);
        const unsigned char* vg = reinterpret_cast<const unsigned char*>(A.vals) + st.start * sizeof(T);
        const unsigned char* k0 = reinterpret_cast<const unsigned char*>(reinterpret_cast<std::uintptr_t>(kg) & ~std::uintptr_t(15));
        const unsigned char* v0 = reinterpret_cast<const unsigned char*>(reinterpret_cast<std::uintptr_t>(vg) & ~std::uintptr_t(15));
        const std::uint32_t kbytes = static_cast<std::uint32_t>(((kg - k0) + st.len * sizeof(K) + 15) & ~std::size_t(15));
        const std::uint32_t vbytes = static_cast<std::uint32_t>(((vg - v0) + st.len * sizeof(T) + 15) & ~std::size_t(15));
        fence_proxy_async();
        mbar_expect_tx(&bars[b], kbytes + vbytes);
        bulk_g2s(kb[b], k0, kbytes, &bars[b]);
        bulk_g2s(vb[b], v0, vbytes, &bars[b]);
    };

    const int rb = A.rb;
    const int G = 32 / rb;
    const int g = lane / rb, beta = lane - g * rb;
    const bool gactive = g < G;
    const int seg = A.seg;
    const K maska = A.maska, maskb = A.maskb;

    if (gw < A.n_sub && lane == 0) prefetch(gw, 0);
    int it = 0;
    for (long long s = gw; s < A.n_sub; s += stride, ++it) {
        const int b = it & 1;
        if (s + stride < A.n_sub && lane == 0) prefetch(s + stride, b ^ 1);
        const SubTile st = A.subs[s];
        mbar_wait(&bars[b], static_cast<std::uint32_t>((it >> 1) & 1));
        const K* sk = reinterpret_cast<const K*>(kb[b]) + ((st.start * sizeof(K)) & 15) / sizeof(K);
        const T* sv = reinterpret_cast<const T*>(vb[b]) + ((st.start * sizeof(T)) & 15) / sizeof(T);

        T acc1[RA];
        T acc2[RA];
#pragma unroll
        for (int a = 0; a < RA; ++a) { acc1[a] = T(0); acc2[a] = T(0); }
        int nb = 0;
        bool has = false;
        int cur = 0;

        auto push = [&]() {
            T* f = F + (lane * kFB + nb) * RA;
#pragma unroll
            for (int a = 0; a < RA; ++a) { f[a] = acc1[a]; acc1[a] = T(0); }
            EIB[lane * kFB + nb] = cur;
            ++nb;
        };
        auto drain = [&]() {
            int incl = nb;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            const int excl = incl - nb;
            for (int q = 0; q < nb; ++q) ord[excl + q] = static_cast<short>(lane * kFB + q);
            __syncwarp();
            for (int e0 = 0; e0 < total; e0 += G) {
                const int e = e0 + g;
                if (gactive && e < total) {
                    const int slot = ord[e];
                    const T u = Ub[static_cast<long long>(EIB[slot]) * A.rbs + beta];
                    const T* f = F + slot * RA;
#pragma unroll
                    for (int a = 0; a < RA; ++a) acc2[a] = fma(f[a], u, acc2[a]);
                }
            }
            __syncwarp();
            nb = 0;
        };

        const int my0 = lane * seg;
        for (int j = 0; j < seg; ++j) {
            const int e = my0 + j;
            if (e < st.len) {
                const K key = sk[e];
                const T v = sv[e];
                const int ib = static_cast<int>((key >> A.ba) & maskb);
                if (has && ib != cur) push();
                cur = ib;
                has = true;
                const T* u = Ua + static_cast<long long>(key & maska) * RA;
#pragma unroll
                for (int a = 0; a < RA; ++a) acc1[a] = fma(v, u[a], acc1[a]);
            }
            if (__any_sync(0xffffffffu, nb == kFB)) drain();
        }
        if (has) push();
        drain();

        for (int gg = 1; gg < G; ++gg) {
#pragma unroll
            for (int a = 0; a < RA; ++a) {
                const T o = __shfl_sync(0xffffffffu, acc2[a], (lane + gg * rb) & 31);
                if (g == 0) acc2[a] += o;
            }
        }
        if (g == 0) {
            T* out = A.P + s * A.C;
#pragma unroll
            for (int a = 0; a < RA; ++a)
                if (a < A.ra) out[a * A.sa + beta * A.sb] = acc2[a];
        }
        __syncwarp();  // buffer b is refilled two iterations later
    }
}

}  // namespace ttm
}  // namespace machb
