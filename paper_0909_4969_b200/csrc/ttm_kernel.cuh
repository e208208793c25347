// Fused mode-n TTM kernel (included by sparse_ttm.cu).
//
// Work unit: a task = up to 32 fibre segments (<= kSegMax nonzeros each) of
// one output row, stored in jagged-diagonal order — segments sorted by length
// (descending) and the task's nonzeros interleaved position-major, so at step
// j the lanes whose segment is still running (lanes 0 .. a_j-1) read
// consecutive words: ia[ptr + lane], v[ptr + lane].  One lane owns one
// segment: it accumulates the fibre sum f = sum_j v_j * U_a[ia_j, :] in
// registers without any cross-lane traffic (the product is one __ffma2_rn per
// two ranks).  The warp then forms the task's partial row block
// sum_s f_s (x) U_b[ib_s, :] (lane groups over segments, fixed order) and
// writes it; a second small kernel sums a row's task partials in task order.
//
// Persistent warps double-buffer their tasks in shared memory with 1-D TMA
// bulk copies (cp.async.bulk ... mbarrier::complete_tx): the next task's
// nonzeros stream from HBM while the current one is reduced.  Factor rows
// are staged once per CTA in shared memory when they fit (FS = true).
#pragma once

namespace machb {
namespace ttm {

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
__device__ __forceinline__ void mbar_arrive(std::uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 128-bit shared loads by 32-bit shared address (factor rows are immutable
// once staged, so these need no ordering against other memory operations)
__device__ __forceinline__ float4 lds128f(std::uint32_t a) {
    float4 v;
    asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ double2 lds128d(std::uint32_t a) {
    double2 v;
    asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}

inline std::size_t al16(std::size_t x) { return (x + 15) & ~static_cast<std::size_t>(15); }

// Shared-memory carve-up (host and device agree on this):
//   [factor rows][S full + S empty mbarriers][S task slots][W fibre-sum tiles]
template <typename T, typename IA, int RS>
struct RingLayout {
    static constexpr std::size_t hdr = 32;  // TtmTask copy + task id
    static constexpr std::size_t ibuf = ((kTaskNnz * sizeof(IA) + 32 + 15) / 16) * 16;  // +32: alignment slack
    static constexpr std::size_t vbuf = ((kTaskNnz * sizeof(T) + 32 + 15) / 16) * 16;
    static constexpr std::size_t dbuf = kDesc * sizeof(int2);
    static constexpr std::size_t slot = hdr + ibuf + vbuf + dbuf;
    static constexpr std::size_t fbuf = 32ull * (((RS / (16 / sizeof(T))) & 1) ? RS : RS + 16 / sizeof(T)) * sizeof(T);  // 32 rows, odd-unit stride
    static std::size_t bytes(std::size_t fac, int S, int W) { return fac + 16ull * S + S * slot + W * fbuf; }
};

// Block = W consumer warps + 1 producer warp.  The producer streams the CTA's
// tasks (t = blockIdx.x + i * gridDim.x, i = 0, 1, ...) into a ring of S
// slots with TMA bulk copies; consumer warp w takes i = w, w + W, ...
template <typename T, typename IA, int RA, bool FS>
__global__ void __launch_bounds__(544, 1) ttm_mode_kernel(TtmArgs<T, IA> A) {
    // Stage-1-only launches (fibre sums for a later stage 2) overlap the
    // preceding mode-basis kernel: they read only data that was complete
    // before it started, so they skip the wait here and instead wait at the
    // end, making their completion imply the predecessor's.
    if (A.stage1 == 1) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    else pdl_enter();  // programmatic dependent launch: predecessor complete and visible
    constexpr int VN = 16 / static_cast<int>(sizeof(T));  // elements per 128-bit load
    constexpr int RS = ((RA + VN - 1) / VN) * VN;         // ranks rounded to whole 16-B units
    constexpr int RSS = ((RS / VN) & 1) ? RS : RS + VN;   // factor row stride: odd number of 16-B units
    constexpr int FS_ = RSS;                              // fibre-sum row stride (same reason)
    using L = RingLayout<T, IA, RS>;
    extern __shared__ __align__(128) unsigned char smraw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int W = A.n_cons, S = A.n_slot;
    std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smraw + A.fac_bytes);
    std::uint64_t* empty = full + S;
    unsigned char* slots = smraw + A.fac_bytes + 16ull * S;
    T* ua_s = reinterpret_cast<T*>(smraw);
    T* ub_s = ua_s + A.ua_rows * RSS;
    __shared__ __align__(8) std::uint64_t fbar;
    unsigned long long* ts = A.ts ? A.ts + 8ull * blockIdx.x : nullptr;
    if (ts && threadIdx.x == 0) ts[0] = gtimer();

    if (threadIdx.x == 0) {
        for (int q = 0; q < S; ++q) {
            mbar_init(&full[q], 1);
            mbar_init(&empty[q], 1);
        }
        if (FS) mbar_init(&fbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (ts && threadIdx.x == 0) ts[1] = gtimer();

    if (warp == W) {
        // ---------------- producer ----------------
        if (FS && lane == 0 && A.dbg != 4) {  // factor rows (global rows already use the shared stride RSS)
            const std::uint32_t ua_bytes = static_cast<std::uint32_t>(A.ua_rows * RSS * sizeof(T));
            const std::uint32_t ub_bytes = static_cast<std::uint32_t>(A.ub_elems * sizeof(T));
            fence_proxy_async();
            mbar_expect_tx(&fbar, ua_bytes + ub_bytes);
            bulk_g2s(ua_s, A.Ua, ua_bytes, &fbar);
            if (ub_bytes) bulk_g2s(ub_s, A.Ub, ub_bytes, &fbar);
        }
        // lane k < S owns slot k and feeds it tasks i = r * S + k, r = 0, 1, ...
        // (S <= 32): the slots are refilled in parallel, and each lane's next
        // task record is loaded while it waits for its slot to drain
        if (lane < S) {
            const long long G0 = gridDim.x;
            long long t = blockIdx.x + static_cast<long long>(lane) * G0;
            TtmTask tk{};
            if (t < A.n_task) tk = A.tasks[t];
            unsigned char* sl = slots + lane * L::slot;
            for (int r = 0; t < A.n_task; ++r) {
                const long long tn = t + static_cast<long long>(S) * G0;
                TtmTask nx{};
                if (tn < A.n_task) nx = A.tasks[tn];
                if (r > 0) mbar_wait(&empty[lane], static_cast<std::uint32_t>((r - 1) & 1));
                *reinterpret_cast<TtmTask*>(sl) = tk;
                *reinterpret_cast<long long*>(sl + 24) = t;
                if (A.dbg == 2 || A.dbg == 4) {
                    mbar_arrive(&full[lane]);
                } else {
                    const unsigned char* ig = reinterpret_cast<const unsigned char*>(A.ia) + tk.base * sizeof(IA);
                    const unsigned char* vg = reinterpret_cast<const unsigned char*>(A.vals) + tk.base * sizeof(T);
                    const unsigned char* i0 = reinterpret_cast<const unsigned char*>(reinterpret_cast<std::uintptr_t>(ig) & ~std::uintptr_t(15));
                    const unsigned char* v0 = reinterpret_cast<const unsigned char*>(reinterpret_cast<std::uintptr_t>(vg) & ~std::uintptr_t(15));
                    const std::uint32_t ib = static_cast<std::uint32_t>(((ig - i0) + tk.len * sizeof(IA) + 15) & ~std::size_t(15));
                    const std::uint32_t vb = static_cast<std::uint32_t>(((vg - v0) + tk.len * sizeof(T) + 15) & ~std::size_t(15));
                    // (the empty-barrier wait orders the consumers' reads of this
                    // slot before the bulk writes; no proxy fence is needed for WAR)
                    mbar_expect_tx(&full[lane], ib + vb + static_cast<std::uint32_t>(L::dbuf));
                    bulk_g2s(sl + L::hdr, i0, ib, &full[lane]);
                    bulk_g2s(sl + L::hdr + L::ibuf, v0, vb, &full[lane]);
                    bulk_g2s(sl + L::hdr + L::ibuf + L::vbuf, A.desc + t * kDesc, static_cast<std::uint32_t>(L::dbuf), &full[lane]);
                }
                tk = nx;
                t = tn;
            }
        }
        if (ts && lane == 0) ts[2] = gtimer();
        return;
    }

    // ---------------- consumers ----------------
    if (FS && A.dbg != 4) mbar_wait(&fbar, 0);
    if (ts && threadIdx.x == 0) ts[3] = gtimer();
    const T* Ua = FS ? ua_s : A.Ua;
    const T* Ub = FS ? ub_s : A.Ub;
    T* F = reinterpret_cast<T*>(slots + S * L::slot + warp * L::fbuf);

    const int rb = A.rb;
    const int G = 32 / rb;
    const int g = lane / rb, beta = lane - g * rb;
    const bool gactive = g < G;
    const int rbs = A.rbs;

    // f += v * U_a[ia, :]
    const std::uint32_t ua_addr = smem_u32(ua_s);
    auto gather_fma = [&](T (&f)[RS], long long ia, T v) {
        const T* u = Ua + ia * RSS;
        const std::uint32_t ua = ua_addr + static_cast<std::uint32_t>(ia) * static_cast<std::uint32_t>(RSS * sizeof(T));
        if constexpr (sizeof(T) == 4) {
            const float2 vv = make_float2(v, v);
#pragma unroll
            for (int a = 0; a < RS; a += 4) {
                if (a < RA) {  // a partial last unit reads the row padding
                    const float4 q = FS ? lds128f(ua + a * 4) : __ldg(reinterpret_cast<const float4*>(u + a));
                    const float2 lo = __ffma2_rn(vv, make_float2(q.x, q.y), make_float2(f[a], f[a + 1]));
                    f[a] = lo.x; f[a + 1] = lo.y;
                    if (a + 2 < RA) {
                        const float2 hi = __ffma2_rn(vv, make_float2(q.z, q.w), make_float2(f[a + 2], f[a + 3]));
                        f[a + 2] = hi.x; f[a + 3] = hi.y;
                    }
                }
            }
        } else {
#pragma unroll
            for (int a = 0; a < RA; a += 2) {
                const double2 q = FS ? lds128d(ua + a * 8) : __ldg(reinterpret_cast<const double2*>(u + a));
                f[a] = fma(v, q.x, f[a]);
                f[a + 1] = fma(v, q.y, f[a + 1]);
            }
        }
    };

    int q = warp;  // slot of task i = i mod S (S a multiple of W: one wrap per step at most)
    std::uint32_t par = 0u;
    for (long long i = warp;; i += W) {
        const long long t0 = blockIdx.x + i * static_cast<long long>(gridDim.x);
        if (t0 >= A.n_task) break;
        mbar_wait(&full[q], par);
        const unsigned char* sl = slots + q * L::slot;
        const TtmTask tk = *reinterpret_cast<const TtmTask*>(sl);
        const long long t = *reinterpret_cast<const long long*>(sl + 24);
        const IA* si = reinterpret_cast<const IA*>(sl + L::hdr) + ((tk.base * sizeof(IA)) & 15) / sizeof(IA);
        const T* sv = reinterpret_cast<const T*>(sl + L::hdr + L::ibuf) + ((tk.base * sizeof(T)) & 15) / sizeof(T);
        const int2* sd = reinterpret_cast<const int2*>(sl + L::hdr + L::ibuf + L::vbuf);
        const int2 my = sd[lane];  // {i_b, length}; length 0 past nseg
        // fibre-sum position (fseg): loaded now, used after stage 1 (latency hidden)
        const int fpos = (A.fpos && lane < tk.nseg) ? __ldg(A.fpos + t * 32 + lane) : 0;
        if (A.dbg >= 1) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[q]);
            q += W;
            if (q >= S) {
                q -= S;
                par ^= 1u;
            }
            continue;
        }

        // ---- stage 1: this lane's fibre segment, PU positions per step.
        // Position offsets come precomputed with the task. ----
        const unsigned short* joff = reinterpret_cast<const unsigned short*>(sd + 32);
        T f[RS];
#pragma unroll
        for (int a = 0; a < RS; ++a) f[a] = T(0);
        constexpr int PU = sizeof(T) == 4 ? 8 : 4;  // positions per step (register budget)
        for (int j = 0; j < tk.maxlen; j += PU) {
            int ix[PU];
            T vx[PU];
            bool act[PU];
#pragma unroll
            for (int k = 0; k < PU; ++k) {
                const int off = static_cast<int>(joff[j + k]) + lane;
                act[k] = j + k < my.y;
                ix[k] = act[k] ? static_cast<int>(si[off]) : 0;
                vx[k] = act[k] ? sv[off] : T(0);
            }
#pragma unroll
            for (int k = 0; k < PU; ++k)
                if (act[k]) gather_fma(f, ix[k], vx[k]);
        }

        if (A.stage1) {  // fibre sums only, in task order (segments past nseg write zeros)
            T* o = A.fseg + (t * 32 + lane) * static_cast<long long>(A.ra);
            if (sizeof(T) == 4 && (A.ra & 1) == 0) {
#pragma unroll
                for (int a = 0; a < RA; a += 2)
                    if (a < A.ra) *reinterpret_cast<float2*>(o + a) = make_float2(f[a], f[a + 1]);
            } else {
#pragma unroll
                for (int a = 0; a < RA; ++a)
                    if (a < A.ra) o[a] = f[a];
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[q]);
            q += W;
            if (q >= S) {
                q -= S;
                par ^= 1u;
            }
            continue;
        }
        if (A.fseg && lane < tk.nseg) {  // fibre sums for the next mode (y_from_segments)
            T* o = A.fseg + static_cast<long long>(fpos) * A.ra;
            if (sizeof(T) == 4 && (A.ra & 1) == 0) {  // 8-byte stores (pos * ra even: 8-byte aligned)
#pragma unroll
                for (int a = 0; a < RA; a += 2)
                    if (a < A.ra) *reinterpret_cast<float2*>(o + a) = make_float2(f[a], f[a + 1]);
            } else {
#pragma unroll
                for (int a = 0; a < RA; ++a)
                    if (a < A.ra) o[a] = f[a];
            }
        }

        // ---- stage 2: sum_s f_s (x) U_b[i_b(s), :] over the task's segments ----
        {
            T* fr = F + lane * FS_;
#pragma unroll
            for (int a = 0; a < RS; a += VN) {
                if constexpr (sizeof(T) == 4) *reinterpret_cast<float4*>(fr + a) = make_float4(f[a], f[a + 1], f[a + 2], f[a + 3]);
                else *reinterpret_cast<double2*>(fr + a) = make_double2(f[a], f[a + 1]);
            }
        }
        __syncwarp();
        T acc[RS];
#pragma unroll
        for (int a = 0; a < RS; ++a) acc[a] = T(0);
        if (gactive) {
#pragma unroll 4
            for (int q = g; q < tk.nseg; q += G) {
                const T u = Ub[static_cast<long long>(sd[q].x) * rbs + beta];
                const T* fq = F + q * FS_;
#pragma unroll
                for (int a = 0; a < RS; a += VN) {
                    if constexpr (sizeof(T) == 4) {
                        const float4 fv = *reinterpret_cast<const float4*>(fq + a);
                        const float2 uu = make_float2(u, u);
                        float2 lo = __ffma2_rn(uu, make_float2(fv.x, fv.y), make_float2(acc[a], acc[a + 1]));
                        float2 hi = __ffma2_rn(uu, make_float2(fv.z, fv.w), make_float2(acc[a + 2], acc[a + 3]));
                        acc[a] = lo.x; acc[a + 1] = lo.y; acc[a + 2] = hi.x; acc[a + 3] = hi.y;
                    } else {
                        const double2 fv = *reinterpret_cast<const double2*>(fq + a);
                        acc[a] = fma(fv.x, u, acc[a]);
                        acc[a + 1] = fma(fv.y, u, acc[a + 1]);
                    }
                }
            }
        }
        for (int gg = 1; gg < G; ++gg) {
#pragma unroll
            for (int a = 0; a < RA; ++a) {
                const T o = __shfl_sync(0xffffffffu, acc[a], (lane + gg * rb) & 31);
                if (g == 0) acc[a] += o;
            }
        }
        if (g == 0) {
            T* out = A.P + t * A.C;
#pragma unroll
            for (int a = 0; a < RA; ++a)
                if (a < A.ra) out[a * A.sa + beta * A.sb] = acc[a];
        }
        __syncwarp();  // all lanes are done with the slot and with F
        if (lane == 0) mbar_arrive(&empty[q]);
        q += W;
        if (q >= S) {
            q -= S;
            par ^= 1u;
        }
    }
    if (ts && lane == 0) atomicMax(&ts[4], gtimer());
    if (A.stage1 == 1) asm volatile("griddepcontrol.wait;" ::: "memory");  // complete only after the predecessor
}

}  // namespace ttm
}  // namespace machb
