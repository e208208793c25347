// Internal plumbing for libmach_b200: error type, context, stream-ordered
// device buffers, launch accounting.  sm_100a only.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "mach_b200.h"

namespace machb {

struct Error : std::runtime_error {
    int code;
    int index;
    Error(int c, const std::string& m, int idx = 0) : std::runtime_error(m), code(c), index(idx) {}
};

[[noreturn]] inline void throw_arg(const std::string& m) { throw Error(MACH_ERR_ARGUMENT, m); }
[[noreturn]] inline void throw_shape(const std::string& m) { throw Error(MACH_ERR_SHAPE, m); }

#define MB_CUDA(x)                                                                                   \
    do {                                                                                             \
        cudaError_t e_ = (x);                                                                        \
        if (e_ != cudaSuccess)                                                                       \
            throw ::machb::Error(e_ == cudaErrorMemoryAllocation ? MACH_ERR_OOM : MACH_ERR_CUDA,     \
                                 std::string(#x) + ": " + cudaGetErrorString(e_));                   \
    } while (0)

struct KStat {
    std::int64_t launches = 0;
    double ms = 0.0;
};

struct PendingEvent {
    const char* name;
    cudaEvent_t a, b;
};

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    // launched right after the next fused mode-basis kernel, ahead of its
    // fallback kernels (consumed once): the overlapped sweep's next stage 1
    std::function<void()> after_basis;
    // NCCL communicator of the time-slab shards (comm.cpp), or null
    void* comm = nullptr;
    int comm_world = 1, comm_rank = 0;
    std::int64_t launches = 0;
    bool profile = false;                      // per-kernel CUDA-event timing (bench roofline)
    std::map<std::string, KStat> stats;
    std::vector<PendingEvent> pending;
    void resolve() {
        for (auto& p : pending) {
            cudaEventSynchronize(p.b);
            float ms = 0;
            cudaEventElapsedTime(&ms, p.a, p.b);
            auto& st = stats[p.name];
            st.launches += 1;
            st.ms += ms;
            cudaEventDestroy(p.a);
            cudaEventDestroy(p.b);
        }
        pending.clear();
    }
};

// Every kernel launch in the library goes through this so the bench can
// report how many of our kernels ran (gpu_launches) and, when profiling is on,
// each kernel's device time from CUDA events on the launching stream.
inline bool max_carveout(const void* f) {
    return cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100) == cudaSuccess;
}

// Every kernel prefers the maximum shared-memory carve-out: the big kernels
// need it and a uniform carve-out avoids SM reconfiguration between launches.
#define MB_LAUNCH(ctx, kernel, grid, block, smem, ...)                                               \
    do {                                                                                             \
        static const bool carve_ = ::machb::max_carveout(reinterpret_cast<const void*>(kernel));     \
        (void)carve_;                                                                                \
        ::machb::PendingEvent pe_{#kernel, nullptr, nullptr};                                        \
        if ((ctx)->profile) {                                                                        \
            MB_CUDA(cudaEventCreate(&pe_.a));                                                        \
            MB_CUDA(cudaEventCreate(&pe_.b));                                                        \
            MB_CUDA(cudaEventRecord(pe_.a, (ctx)->stream));                                          \
        }                                                                                            \
        kernel<<<(grid), (block), (smem), (ctx)->stream>>>(__VA_ARGS__);                              \
        {                                                                                            \
            cudaError_t le_ = cudaGetLastError();                                                    \
            if (le_ != cudaSuccess)                                                                  \
                throw ::machb::Error(MACH_ERR_CUDA, std::string("launch of " #kernel ": ") +         \
                                                        cudaGetErrorString(le_));                    \
        }                                                                                            \
        ++(ctx)->launches;                                                                           \
        if ((ctx)->profile) {                                                                        \
            MB_CUDA(cudaEventRecord(pe_.b, (ctx)->stream));                                          \
            (ctx)->pending.push_back(pe_);                                                           \
        }                                                                                            \
    } while (0)

// Same for an extended launch (clusters): cfgp is a cudaLaunchConfig_t*.
#define MB_LAUNCH_EX(ctx, name, cfgp, kernel, ...)                                                 \
    do {                                                                                             \
        static const bool carve_ = ::machb::max_carveout(reinterpret_cast<const void*>(kernel));     \
        (void)carve_;                                                                                \
        ::machb::PendingEvent pe_{name, nullptr, nullptr};                                           \
        if ((ctx)->profile) {                                                                        \
            MB_CUDA(cudaEventCreate(&pe_.a));                                                        \
            MB_CUDA(cudaEventCreate(&pe_.b));                                                        \
            MB_CUDA(cudaEventRecord(pe_.a, (ctx)->stream));                                          \
        }                                                                                            \
        {                                                                                            \
            cudaError_t le_ = cudaLaunchKernelEx((cfgp), kernel, __VA_ARGS__);                       \
            if (le_ != cudaSuccess)                                                                  \
                throw ::machb::Error(le_ == cudaErrorMemoryAllocation ? MACH_ERR_OOM : MACH_ERR_CUDA, \
                                     std::string("launch of ") + (name) + ": " + cudaGetErrorString(le_)); \
        }                                                                                            \
        ++(ctx)->launches;                                                                           \
        if ((ctx)->profile) {                                                                        \
            MB_CUDA(cudaEventRecord(pe_.b, (ctx)->stream));                                          \
            (ctx)->pending.push_back(pe_);                                                           \
        }                                                                                            \
    } while (0)

// Programmatic dependent launch for the sweep's kernel chain: the launch of
// kernel N+1 (and its CTAs' prologue) overlaps kernel N; every kernel launched
// this way starts with pdl_enter(), whose griddepcontrol.wait blocks until the
// predecessor grid has completed and its writes are visible (a no-op when the
// kernel was launched without the attribute).  MACH_NO_PDL=1 disables it.
#ifndef MACH_PDL_TRIGGER_FIRST
#define MACH_PDL_TRIGGER_FIRST 1
#endif
__device__ __forceinline__ constexpr bool pdl_trigger_first() { return MACH_PDL_TRIGGER_FIRST != 0; }
__device__ __forceinline__ void pdl_enter() {
    // trigger first: the dependent grid may launch (and queue its CTAs) as
    // soon as all of this grid's CTAs have started; it still waits for this
    // grid's completion in its own griddepcontrol.wait
    if (pdl_trigger_first()) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (!pdl_trigger_first()) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// Wait first, then trigger: the dependent grid launches only after this
// grid's predecessor has completed.  Used by the kernels that bound a
// consumer of data a later, non-waiting (overlapped) launch overwrites.
__device__ __forceinline__ void pdl_enter_strict() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
inline bool pdl_on() {
    static const bool off = std::getenv("MACH_NO_PDL") != nullptr;
    return !off;
}
#define MB_LAUNCH_PDL(ctx, kernel, grid, block, smem, ...)                                           \
    do {                                                                                             \
        if (!::machb::pdl_on()) {                                                                    \
            MB_LAUNCH(ctx, kernel, grid, block, smem, __VA_ARGS__);                                  \
            break;                                                                                   \
        }                                                                                            \
        cudaLaunchConfig_t cfg_{};                                                                   \
        cfg_.gridDim = dim3(grid);                                                                   \
        cfg_.blockDim = dim3(block);                                                                 \
        cfg_.dynamicSmemBytes = (smem);                                                              \
        cfg_.stream = (ctx)->stream;                                                                 \
        cudaLaunchAttribute at_[1];                                                                  \
        at_[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                              \
        at_[0].val.programmaticStreamSerializationAllowed = 1;                                       \
        cfg_.attrs = at_;                                                                            \
        cfg_.numAttrs = 1;                                                                           \
        MB_LAUNCH_EX(ctx, #kernel, &cfg_, kernel, __VA_ARGS__);                                      \
    } while (0)

// Stream-ordered device allocation owned by RAII.
template <typename T>
struct DBuf {
    T* p = nullptr;
    std::size_t n = 0;
    cudaStream_t s = nullptr;
    DBuf() = default;
    DBuf(Ctx* ctx, std::size_t count) { alloc(ctx, count); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p; n = o.n; s = o.s;
            o.p = nullptr; o.n = 0;
        }
        return *this;
    }
    ~DBuf() { release(); }
    void alloc(Ctx* ctx, std::size_t count) {
        release();
        s = ctx->stream;
        n = count;
        if (count) MB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), s));
    }
    void zero(Ctx* ctx) {
        if (n) MB_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), ctx->stream));
    }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
    }
    T* get() const { return p; }
};

template <typename T>
inline void to_host(Ctx* ctx, T* dst, const T* src, std::size_t count) {
    if (count) MB_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
}
template <typename T>
inline void to_device(Ctx* ctx, T* dst, const T* src, std::size_t count) {
    if (count) MB_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
}
inline void sync(Ctx* ctx) { MB_CUDA(cudaStreamSynchronize(ctx->stream)); }

inline int dtype_size(int dtype) { return dtype == MACH_F64 ? 8 : 4; }

// ---- tensor layout helpers (first mode fastest; reference tensor.cpp:15-45) ----
std::int64_t checked_size(const std::vector<int>& dims);
struct Split {
    std::int64_t inner = 1, outer = 1;
    int len = 0;
};
Split split_at(const std::vector<int>& dims, int mode);

// ---- NCCL (comm.cpp), bound at run time ----
void comm_unique_id(unsigned char* out);
void comm_init(Ctx* ctx, int world, int rank, const unsigned char* id);
void comm_destroy(Ctx* ctx);
void comm_allreduce_sum(Ctx* ctx, void* buf, std::size_t count, bool f64);

// One-time per-device setup (kernel attributes are per device): true the
// first time `dev` is seen for this mask.
inline bool first_on_device(std::uint64_t& mask, int dev) {
    const std::uint64_t bit = 1ull << (static_cast<unsigned>(dev) & 63u);
    if (mask & bit) return false;
    mask |= bit;
    return true;
}

inline int ceil_div(std::int64_t a, std::int64_t b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace machb

// ---- opaque handle types of the C ABI ----
struct mach_ctx {
    machb::Ctx c;
};

struct mach_dense {
    machb::Ctx* ctx = nullptr;
    int dtype = MACH_F64;
    std::vector<int> dims;
    std::int64_t numel = 0;
    void* data = nullptr;
    bool owns = true;
};

namespace machb {
struct ModePlan;  // per-mode sorted layout (layout.cu)
}

struct mach_sparse {
    machb::Ctx* ctx = nullptr;
    int dtype = MACH_F64;
    std::vector<int> dims;
    std::int64_t numel = 0;
    std::int64_t nnz = 0;
    bool idx64 = false;        // flat index stored as u64 (numel > 2^32) else u32
    void* idx = nullptr;       // ascending flat index
    void* val = nullptr;       // dtype values
    double norm2 = -1.0;       // cached |X|^2 (fp64), -1 = unknown
    std::vector<std::shared_ptr<machb::ModePlan>> plans;  // lazily built per mode
    ~mach_sparse();
};

struct mach_model {
    int order = 0;
    std::vector<int> dims, ranks;
    std::vector<double> core;                  // prod(ranks), first mode fastest
    std::vector<std::vector<double>> factors;  // I_n x r_n column-major
    int iterations = 0;
    double fit = 0.0;
    std::vector<double> sweep_fits;
    std::vector<std::string> warnings;
    double sample_ms = 0, setup_ms = 0, hosvd_ms = 0;
    std::vector<double> sweep_ms;
};
