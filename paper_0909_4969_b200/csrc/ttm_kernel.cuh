// Fused mode-n TTM kernel (included by sparse_ttm.cu).
//
// Persistent warps, one sorted sub-tile (<= 32*seg nonzeros of one output row)
// at a time.  Each warp double-buffers its sub-tiles in shared memory with 1-D
// TMA bulk copies (cp.async.bulk ... mbarrier::complete_tx) so the HBM stream
// is in flight while the previous sub-tile is reduced; lanes then walk `seg`
// consecutive nonzeros each (seg odd => conflict-free shared-memory reads of
// the linear TMA layout).  Factor rows (U_a, U_b) are staged once per CTA in
// shared memory when they fit (FS = true) and read with 128-bit loads.
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

template <typename T>
struct Vec4;
template <>
struct Vec4<float> {
    using type = float4;
    static constexpr int n = 4;
};
template <>
struct Vec4<double> {
    using type = double2;
    static constexpr int n = 2;
};

// Per-warp shared-memory carve-up (host and device agree on this).
template <typename T, typename K, int RA>
struct WarpLayout {
    int seg;
    std::size_t kbuf, vbuf, f, eib, ord, total;
    __host__ __device__ explicit WarpLayout(int s) : seg(s) {
        kbuf = ((32ull * s * sizeof(K) + 32 + 15) / 16) * 16;  // +32: alignment slack of the bulk copy
        vbuf = ((32ull * s * sizeof(T) + 32 + 15) / 16) * 16;
        // per-lane fibre queue blocks padded by 16 B so the lanes' 128-bit push
        // stores land in different bank groups
        f = ((32ull * (kFB * RA * sizeof(T) + 16) + 15) / 16) * 16;
        eib = ((32ull * kFB * sizeof(int) + 15) / 16) * 16;
        ord = ((32ull * kFB * sizeof(short) + 15) / 16) * 16;
        total = 16 /*2 mbarriers*/ + 2 * (kbuf + vbuf) + f + eib + ord;
    }
};

template <typename T, typename K, int RA, bool FS>
__global__ void __launch_bounds__(512) ttm_mode_kernel(TtmArgs<T, K> A) {
    using V = typename Vec4<T>::type;
    constexpr int VN = Vec4<T>::n;
    constexpr int LB = kFB * RA + 16 / static_cast<int>(sizeof(T));  // padded per-lane queue block
    extern __shared__ __align__(128) unsigned char smraw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    const WarpLayout<T, K, RA> L(A.seg);

    // ---- CTA-shared factor rows ----
    T* ua_s = reinterpret_cast<T*>(smraw);
    T* ub_s = ua_s + A.ua_elems;
    if (FS) {
        const V* ga = reinterpret_cast<const V*>(A.Ua);
        V* sa = reinterpret_cast<V*>(ua_s);
        for (long long i = threadIdx.x; i < A.ua_elems / VN; i += blockDim.x) sa[i] = ga[i];
        for (long long i = threadIdx.x; i < A.ub_elems; i += blockDim.x) ub_s[i] = A.Ub[i];
    }
    const T* Ua = FS ? ua_s : A.Ua;
    const T* Ub = FS ? ub_s : A.Ub;

    unsigned char* wbase = smraw + A.fac_bytes + L.total * wib;
    std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(wbase);
    unsigned char* kbuf0 = wbase + 16;
    unsigned char* vbuf0 = wbase + 16 + 2 * L.kbuf;
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
        bulk_g2s(kbuf0 + b * L.kbuf, k0, kbytes, &bars[b]);
        bulk_g2s(vbuf0 + b * L.vbuf, v0, vbytes, &bars[b]);
    };

    const int rb = A.rb;
    const int G = 32 / rb;
    const int g = lane / rb, beta = lane - g * rb;
    const bool gactive = g < G;
    const int seg = A.seg;
    const K maska = A.maska, maskb = A.maskb;
    const int ba = A.ba;
    const int rbs = A.rbs;

    if (gw < A.n_sub && lane == 0) prefetch(gw, 0);
    SubTile st = (gw < A.n_sub) ? A.subs[gw] : SubTile{0, 0, 0};
    int it = 0;
    for (long long s = gw; s < A.n_sub; s += stride, ++it) {
        const int b = it & 1;
        SubTile nxt{0, 0, 0};
        if (s + stride < A.n_sub) {
            nxt = A.subs[s + stride];
            if (lane == 0) prefetch(s + stride, b ^ 1);
        }
        mbar_wait(&bars[b], static_cast<std::uint32_t>((it >> 1) & 1));
        const K* sk = reinterpret_cast<const K*>(kbuf0 + b * L.kbuf) + ((st.start * sizeof(K)) & 15) / sizeof(K);
        const T* sv = reinterpret_cast<const T*>(vbuf0 + b * L.vbuf) + ((st.start * sizeof(T)) & 15) / sizeof(T);

        T acc1[RA];
        T acc2[RA];
#pragma unroll
        for (int a = 0; a < RA; ++a) { acc1[a] = T(0); acc2[a] = T(0); }
        int nb = 0;
        int cur = -1;

        auto push = [&]() {
            T* f = F + lane * LB + nb * RA;
#pragma unroll
            for (int a = 0; a < RA; a += VN) {
                V v;
                if constexpr (VN == 4) v = V{acc1[a], acc1[a + 1], acc1[a + 2], acc1[a + 3]};
                else v = V{acc1[a], acc1[a + 1]};
                *reinterpret_cast<V*>(f + a) = v;
            }
#pragma unroll
            for (int a = 0; a < RA; ++a) acc1[a] = T(0);
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
                    const T u = Ub[static_cast<long long>(EIB[slot]) * rbs + beta];
                    const T* f = F + (slot / kFB) * LB + (slot % kFB) * RA;
#pragma unroll
                    for (int a = 0; a < RA; a += VN) {
                        const V fv = *reinterpret_cast<const V*>(f + a);
                        if constexpr (VN == 4) {
                            acc2[a] = fma(fv.x, u, acc2[a]);
                            acc2[a + 1] = fma(fv.y, u, acc2[a + 1]);
                            acc2[a + 2] = fma(fv.z, u, acc2[a + 2]);
                            acc2[a + 3] = fma(fv.w, u, acc2[a + 3]);
                        } else {
                            acc2[a] = fma(fv.x, u, acc2[a]);
                            acc2[a + 1] = fma(fv.y, u, acc2[a + 1]);
                        }
                    }
                }
            }
            __syncwarp();
            nb = 0;
        };

        const int my0 = lane * seg;
        const int cnt = max(0, min(seg, st.len - my0));
        // software pipeline: the next nonzero's key, value and factor row are
        // loaded while the current one is accumulated
        auto load_row = [&](K key, V* dst) {
            const V* u = reinterpret_cast<const V*>(Ua + static_cast<long long>(key & maska) * RA);
#pragma unroll
            for (int a = 0; a < RA / VN; ++a) dst[a] = FS ? u[a] : __ldg(u + a);
        };
        K key_n = K(0);
        T v_n = T(0);
        V un[RA / VN];
        if (cnt > 0) {
            key_n = sk[my0];
            v_n = sv[my0];
            load_row(key_n, un);
        }
        for (int j = 0; j < seg; ++j) {
            const K key = key_n;
            const T v = v_n;
            V u[RA / VN];
#pragma unroll
            for (int a = 0; a < RA / VN; ++a) u[a] = un[a];
            if (j + 1 < cnt) {
                key_n = sk[my0 + j + 1];
                v_n = sv[my0 + j + 1];
                load_row(key_n, un);
            }
            if (j < cnt) {
                const int ib = static_cast<int>((key >> ba) & maskb);
                if (ib != cur) {
                    if (cur >= 0) push();
                    cur = ib;
                }
#pragma unroll
                for (int a = 0; a < RA; a += VN) {
                    const V uv = u[a / VN];
                    if constexpr (VN == 4) {
                        acc1[a] = fma(v, uv.x, acc1[a]);
                        acc1[a + 1] = fma(v, uv.y, acc1[a + 1]);
                        acc1[a + 2] = fma(v, uv.z, acc1[a + 2]);
                        acc1[a + 3] = fma(v, uv.w, acc1[a + 3]);
                    } else {
                        acc1[a] = fma(v, uv.x, acc1[a]);
                        acc1[a + 1] = fma(v, uv.y, acc1[a + 1]);
                    }
                }
            }
            if (__any_sync(0xffffffffu, nb == kFB)) drain();
        }
        if (cur >= 0) push();
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
        st = nxt;
        __syncwarp();  // buffer b is refilled two iterations later
    }
}

}  // namespace ttm
}  // namespace machb
