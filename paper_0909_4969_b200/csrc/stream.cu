// Streaming sample-on-arrival ingest and binary tensor files
// (SURVEY §8f.4).
//
// Stream: the paper's Remark 2 flips the keep coin per
// arriving measurement; the reference gets the same effect offline because the
// RNG counter is the global flat index (proj/src/sampling.cpp:27).  With the
// first-mode-fastest layout (tensor.hpp:10-12) a time slab is a contiguous
// flat range, so sampling each arriving slab with its global offset and
// appending the kept entries keeps the sampled tensor in canonical ascending
// order and identical, bit for bit, to mach_sparsify of everything seen so
// far.  Host slabs go through two device staging buffers: the H2D copy of slab
// k (copy stream) overlaps the sampling of slab k-1 (library stream).
//
// Records: proj/src/ingest.cpp:90-134 restated for one time slab of
// pre-indexed records (the name -> index maps stay on the host): radix sort
// by value then stably by cell = (cell, value) order, one thread per cell run
// sums its records in that order and divides by the count (bit-identical to
// the reference's order-independent mean), carry-forward keeps the last seen
// value per (machine, metric) across slabs.
#include <cub/cub.cuh>

#include <cstdio>
#include <cstring>

#include "sparse_ttm.cuh"

namespace machb {
mach_sparse* sample_slab(const mach_dense* x, const std::vector<int>& gdims, std::int64_t offset, double p,
                         std::uint64_t seed);
}

struct mach_stream {
    machb::Ctx* ctx = nullptr;
    int dtype = MACH_F32;
    std::vector<int> cap_dims;      // leading dims + capacity ticks
    std::int64_t slab = 1;          // elements per tick
    std::int64_t ticks = 0, nnz = 0, cap = 0;
    bool idx64 = false;
    double p = 1.0;
    std::uint64_t seed = 0;
    void* idx = nullptr;
    void* val = nullptr;
    // host-slab pipeline
    cudaStream_t copy = nullptr;
    cudaEvent_t ready[2] = {nullptr, nullptr}, freed[2] = {nullptr, nullptr};
    void* stage[2] = {nullptr, nullptr};
    std::size_t stage_bytes[2] = {0, 0};
    int pending = -1;               // staging buffer holding an unsampled slab
    int pending_ticks = 0;
    int next = 0;
    // last dense slab (records / host appends)
    void* last = nullptr;
    int last_ticks = 0;
    // carry-forward state per (machine, metric)
    double* cf_last = nullptr;
    unsigned char* cf_seen = nullptr;
};

namespace machb {

namespace {

__global__ void narrow_idx_kernel(const unsigned long long* __restrict__ in, long long n, unsigned int* __restrict__ out) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i < n) out[i] = static_cast<unsigned int>(in[i]);
}

__device__ __forceinline__ unsigned long long order_bits(double v) {  // total order matching operator< on finite doubles
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ double from_order_bits(unsigned long long k) {
    return __longlong_as_double(static_cast<long long>((k >> 63) ? (k ^ 0x8000000000000000ull) : ~k));
}

__global__ void record_keys_kernel(const int* __restrict__ machine, const int* __restrict__ metric,
                                   const int* __restrict__ tick, const double* __restrict__ value, long long n, int M,
                                   int J, int ticks, unsigned long long* __restrict__ vkey, long long* __restrict__ cell,
                                   int* __restrict__ bad) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const int m = machine[i], j = metric[i], t = tick[i];
    const double v = value[i];
    if (m < 0 || m >= M || j < 0 || j >= J || t < 0 || t >= ticks) atomicOr(bad, 1);
    if (!isfinite(v)) atomicOr(bad, 2);
    vkey[i] = order_bits(v);
    cell[i] = m + static_cast<long long>(M) * (j + static_cast<long long>(J) * t);
}

// one thread per record; the head of a run of equal cells sums the run in order
template <typename T>
__global__ void cell_mean_kernel(const long long* __restrict__ cell, const unsigned long long* __restrict__ vbits, long long n,
                                 T* __restrict__ slab, unsigned char* __restrict__ filled) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const long long c = cell[i];
    if (i > 0 && cell[i - 1] == c) return;
    double sum = 0.0;
    long long cnt = 0;
    for (long long k = i; k < n && cell[k] == c; ++k) {
        sum += from_order_bits(vbits[k]);
        ++cnt;
    }
    slab[c] = static_cast<T>(sum / static_cast<double>(cnt));
    filled[c] = 1;
}

template <typename T>
__global__ void carry_forward_kernel(T* __restrict__ slab, const unsigned char* __restrict__ filled, long long MJ,
                                     int ticks, double* __restrict__ last, unsigned char* __restrict__ seen) {
    const long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (c >= MJ) return;
    double l = last[c];
    bool s = seen[c] != 0;
    for (int t = 0; t < ticks; ++t) {
        const long long cellx = c + MJ * t;
        if (filled[cellx]) {
            l = static_cast<double>(slab[cellx]);
            s = true;
        } else if (s) {
            slab[cellx] = static_cast<T>(l);
        }
    }
    last[c] = l;
    seen[c] = s ? 1 : 0;
}

void ensure_capacity(mach_stream* s, std::int64_t need) {
    if (need <= s->cap) return;
    Ctx* ctx = s->ctx;
    std::int64_t cap = std::max<std::int64_t>(need, s->cap + s->cap / 2 + 4096);
    const int isz = s->idx64 ? 8 : 4, vsz = dtype_size(s->dtype);
    void *ni = nullptr, *nv = nullptr;
    MB_CUDA(cudaMallocAsync(&ni, static_cast<std::size_t>(cap) * isz, ctx->stream));
    MB_CUDA(cudaMallocAsync(&nv, static_cast<std::size_t>(cap) * vsz, ctx->stream));
    if (s->nnz > 0) {
        MB_CUDA(cudaMemcpyAsync(ni, s->idx, static_cast<std::size_t>(s->nnz) * isz, cudaMemcpyDeviceToDevice, ctx->stream));
        MB_CUDA(cudaMemcpyAsync(nv, s->val, static_cast<std::size_t>(s->nnz) * vsz, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    if (s->idx) cudaFreeAsync(s->idx, ctx->stream);
    if (s->val) cudaFreeAsync(s->val, ctx->stream);
    s->idx = ni;
    s->val = nv;
    s->cap = cap;
}

// sample `ticks` ticks resident at `data` and append the kept entries
void append_device(mach_stream* s, void* data, int ticks) {
    if (ticks < 0) throw_arg("ticks must be >= 0");
    if (ticks == 0) return;
    if (s->ticks + ticks > s->cap_dims.back()) throw_shape("stream capacity (dims[order-1] ticks) exceeded");
    mach_dense view;
    view.ctx = s->ctx;
    view.dtype = s->dtype;
    view.dims = s->cap_dims;
    view.dims.back() = ticks;
    view.numel = s->slab * ticks;
    view.data = data;
    view.owns = false;
    std::unique_ptr<mach_sparse> kept(sample_slab(&view, s->cap_dims, s->ticks * s->slab, s->p, s->seed));
    if (kept->nnz > 0) {
        ensure_capacity(s, s->nnz + kept->nnz);
        const int isz = s->idx64 ? 8 : 4, vsz = dtype_size(s->dtype);
        MB_CUDA(cudaMemcpyAsync(static_cast<char*>(s->idx) + static_cast<std::size_t>(s->nnz) * isz, kept->idx,
                                static_cast<std::size_t>(kept->nnz) * isz, cudaMemcpyDeviceToDevice, s->ctx->stream));
        MB_CUDA(cudaMemcpyAsync(static_cast<char*>(s->val) + static_cast<std::size_t>(s->nnz) * vsz, kept->val,
                                static_cast<std::size_t>(kept->nnz) * vsz, cudaMemcpyDeviceToDevice, s->ctx->stream));
        s->nnz += kept->nnz;
    }
    s->ticks += ticks;
}

void flush_pending(mach_stream* s) {
    if (s->pending < 0) return;
    const int b = s->pending;
    s->pending = -1;
    MB_CUDA(cudaStreamWaitEvent(s->ctx->stream, s->ready[b], 0));
    append_device(s, s->stage[b], s->pending_ticks);
    MB_CUDA(cudaEventRecord(s->freed[b], s->ctx->stream));
    s->last = s->stage[b];
    s->last_ticks = s->pending_ticks;
}

}  // namespace

mach_stream* stream_begin(Ctx* ctx, int dtype, const std::vector<int>& dims, double p, std::uint64_t seed) {
    if (dims.size() < 2) throw_arg("a stream needs at least two modes (the last one is time)");
    for (int d : dims)
        if (d < 1) throw_arg("every dimension must be >= 1");
    if (!(p > 0.0 && p <= 1.0)) throw_arg("p must be in (0, 1]");
    auto s = std::make_unique<mach_stream>();
    s->ctx = ctx;
    s->dtype = dtype;
    s->cap_dims = dims;
    const std::int64_t numel = checked_size(dims);
    s->slab = numel / dims.back();
    s->idx64 = numel > 0xFFFFFFFFll;
    s->p = p;
    s->seed = seed;
    MB_CUDA(cudaStreamCreateWithFlags(&s->copy, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
        MB_CUDA(cudaEventCreateWithFlags(&s->ready[b], cudaEventDisableTiming));
        MB_CUDA(cudaEventCreateWithFlags(&s->freed[b], cudaEventDisableTiming));
    }
    return s.release();
}

void stream_append(mach_stream* s, const mach_dense* slab) {
    flush_pending(s);
    if (slab->dtype != s->dtype) throw_arg("slab value type differs from the stream's");
    if (slab->dims.size() != s->cap_dims.size()) throw_shape("slab order differs from the stream's");
    for (std::size_t m = 0; m + 1 < s->cap_dims.size(); ++m)
        if (slab->dims[m] != s->cap_dims[m]) throw_shape("slab leading dims differ from the stream's");
    append_device(s, slab->data, slab->dims.back());
    s->last = nullptr;
}

void stream_append_host(mach_stream* s, const void* host, int ticks) {
    if (ticks < 0) throw_arg("ticks must be >= 0");
    if (ticks == 0) return;
    if (!host) throw_arg("host slab is null");
    if (s->ticks + (s->pending >= 0 ? s->pending_ticks : 0) + ticks > s->cap_dims.back())
        throw_shape("stream capacity (dims[order-1] ticks) exceeded");
    const int b = s->next;
    s->next ^= 1;
    const std::size_t bytes = static_cast<std::size_t>(s->slab) * ticks * dtype_size(s->dtype);
    // buffer b's previous slab (two appends ago) was sampled on the library stream
    MB_CUDA(cudaStreamWaitEvent(s->copy, s->freed[b], 0));
    if (s->stage_bytes[b] < bytes) {
        if (s->stage[b]) {
            MB_CUDA(cudaStreamSynchronize(s->ctx->stream));  // (rare: slab size grew) its last reader is done
            MB_CUDA(cudaFree(s->stage[b]));
        }
        MB_CUDA(cudaMalloc(&s->stage[b], bytes));
        s->stage_bytes[b] = bytes;
    }
    MB_CUDA(cudaMemcpyAsync(s->stage[b], host, bytes, cudaMemcpyHostToDevice, s->copy));
    MB_CUDA(cudaEventRecord(s->ready[b], s->copy));
    // sample the previous slab while this one is in flight
    try {
        flush_pending(s);
    } catch (...) {  // (e.g. a non-finite value in the previous slab) this slab is dropped with it
        cudaStreamSynchronize(s->copy);  // the host buffer must not be read after we return
        throw;
    }
    s->pending = b;
    s->pending_ticks = ticks;
    MB_CUDA(cudaStreamSynchronize(s->copy));  // the host buffer may be reused on return
}

void stream_append_records(mach_stream* s, std::int64_t n, const std::int32_t* machine, const std::int32_t* metric,
                           const std::int32_t* tick, const double* value, int ticks, bool carry) {
    if (s->cap_dims.size() != 3) throw_arg("record ingest needs a machines x metrics x time stream");
    if (ticks < 0 || n < 0) throw_arg("ticks and n must be >= 0");
    flush_pending(s);
    if (ticks == 0) {
        if (n > 0) throw_arg("records for an empty slab");
        return;
    }
    Ctx* ctx = s->ctx;
    const int M = s->cap_dims[0], J = s->cap_dims[1];
    const long long MJ = static_cast<long long>(M) * J;
    const std::size_t cells = static_cast<std::size_t>(MJ) * ticks;
    const std::size_t bytes = cells * dtype_size(s->dtype);
    const int b = s->next;
    s->next ^= 1;
    MB_CUDA(cudaStreamSynchronize(s->copy));
    if (s->stage_bytes[b] < bytes) {
        MB_CUDA(cudaStreamSynchronize(ctx->stream));
        if (s->stage[b]) MB_CUDA(cudaFree(s->stage[b]));
        MB_CUDA(cudaMalloc(&s->stage[b], bytes));
        s->stage_bytes[b] = bytes;
    }
    MB_CUDA(cudaMemsetAsync(s->stage[b], 0, bytes, ctx->stream));
    DBuf<unsigned char> filled(ctx, cells);
    filled.zero(ctx);
    if (n > 0) {
        if (!machine || !metric || !tick || !value) throw_arg("record arrays are null");
        const std::size_t N = static_cast<std::size_t>(n);
        DBuf<int> dm(ctx, N), dj(ctx, N), dt(ctx, N);
        DBuf<double> dv(ctx, N);
        DBuf<unsigned long long> vk(ctx, N), vk2(ctx, N);
        DBuf<long long> ck(ctx, N), ck2(ctx, N);
        DBuf<int> bad(ctx, 1);
        bad.zero(ctx);
        to_device(ctx, dm.get(), machine, N);
        to_device(ctx, dj.get(), metric, N);
        to_device(ctx, dt.get(), tick, N);
        to_device(ctx, dv.get(), value, N);
        MB_LAUNCH(ctx, record_keys_kernel, ceil_div(n, 256), 256, 0, dm.get(), dj.get(), dt.get(), dv.get(),
                  static_cast<long long>(n), M, J, ticks, vk.get(), ck.get(), bad.get());
        int hb = 0;
        to_host(ctx, &hb, bad.get(), 1);
        sync(ctx);
        if (hb & 2) throw_arg("record value is not finite");
        if (hb & 1) throw_arg("record names a machine, metric or tick outside the slab");
        // (cell, value) order: radix sort by the value's order-preserving bits (cells as payload), then
        // stably by cell (value bits as payload)
        const int ni = static_cast<int>(n);
        std::size_t tb1 = 0, tb2 = 0;
        MB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb1, vk.get(), vk2.get(), ck.get(), ck2.get(), ni, 0, 64, ctx->stream));
        MB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb2, ck2.get(), ck.get(), vk2.get(), vk.get(), ni, 0, 64, ctx->stream));
        DBuf<unsigned char> tmp(ctx, std::max(tb1, tb2));
        MB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb1, vk.get(), vk2.get(), ck.get(), ck2.get(), ni, 0, 64, ctx->stream));
        MB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb2, ck2.get(), ck.get(), vk2.get(), vk.get(), ni, 0, 64, ctx->stream));
        ctx->launches += 2;
        if (s->dtype == MACH_F32)
            MB_LAUNCH(ctx, cell_mean_kernel<float>, ceil_div(n, 256), 256, 0, ck.get(), vk.get(), static_cast<long long>(n),
                      static_cast<float*>(s->stage[b]), filled.get());
        else
            MB_LAUNCH(ctx, cell_mean_kernel<double>, ceil_div(n, 256), 256, 0, ck.get(), vk.get(), static_cast<long long>(n),
                      static_cast<double*>(s->stage[b]), filled.get());
    }
    if (carry) {
        if (!s->cf_last) {
            MB_CUDA(cudaMalloc(&s->cf_last, static_cast<std::size_t>(MJ) * sizeof(double)));
            MB_CUDA(cudaMalloc(&s->cf_seen, static_cast<std::size_t>(MJ)));
            MB_CUDA(cudaMemsetAsync(s->cf_last, 0, static_cast<std::size_t>(MJ) * sizeof(double), ctx->stream));
            MB_CUDA(cudaMemsetAsync(s->cf_seen, 0, static_cast<std::size_t>(MJ), ctx->stream));
        }
        if (s->dtype == MACH_F32)
            MB_LAUNCH(ctx, carry_forward_kernel<float>, ceil_div(MJ, 128), 128, 0, static_cast<float*>(s->stage[b]),
                      filled.get(), MJ, ticks, s->cf_last, s->cf_seen);
        else
            MB_LAUNCH(ctx, carry_forward_kernel<double>, ceil_div(MJ, 128), 128, 0, static_cast<double*>(s->stage[b]),
                      filled.get(), MJ, ticks, s->cf_last, s->cf_seen);
    }
    append_device(s, s->stage[b], ticks);
    MB_CUDA(cudaEventRecord(s->freed[b], ctx->stream));
    s->last = s->stage[b];
    s->last_ticks = ticks;
}

void stream_state(mach_stream* s, std::int64_t* ticks, std::int64_t* nnz) {
    flush_pending(s);
    if (ticks) *ticks = s->ticks;
    if (nnz) *nnz = s->nnz;
}

mach_sparse* stream_tensor(mach_stream* s) {
    flush_pending(s);
    Ctx* ctx = s->ctx;
    auto t = std::make_unique<mach_sparse>();
    t->ctx = ctx;
    t->dtype = s->dtype;
    t->dims = s->cap_dims;
    t->dims.back() = static_cast<int>(s->ticks);
    if (s->ticks < 1) throw_shape("the stream holds no time ticks yet");
    t->numel = checked_size(t->dims);
    t->idx64 = t->numel > 0xFFFFFFFFll;
    t->nnz = s->nnz;
    if (s->nnz > 0) {
        const std::size_t N = static_cast<std::size_t>(s->nnz);
        const int vsz = dtype_size(s->dtype);
        MB_CUDA(cudaMallocAsync(&t->idx, N * (t->idx64 ? 8 : 4), ctx->stream));
        MB_CUDA(cudaMallocAsync(&t->val, N * vsz, ctx->stream));
        if (s->idx64 && !t->idx64)
            MB_LAUNCH(ctx, narrow_idx_kernel, ceil_div(s->nnz, 256), 256, 0, static_cast<const unsigned long long*>(s->idx),
                      static_cast<long long>(s->nnz), static_cast<unsigned int*>(t->idx));
        else
            MB_CUDA(cudaMemcpyAsync(t->idx, s->idx, N * (t->idx64 ? 8 : 4), cudaMemcpyDeviceToDevice, ctx->stream));
        MB_CUDA(cudaMemcpyAsync(t->val, s->val, N * vsz, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    return t.release();
}

mach_dense* stream_last_slab(mach_stream* s) {
    flush_pending(s);
    if (!s->last) throw_arg("no host or record slab has been appended");
    Ctx* ctx = s->ctx;
    auto t = std::make_unique<mach_dense>();
    t->ctx = ctx;
    t->dtype = s->dtype;
    t->dims = s->cap_dims;
    t->dims.back() = s->last_ticks;
    t->numel = s->slab * s->last_ticks;
    const std::size_t bytes = static_cast<std::size_t>(t->numel) * dtype_size(s->dtype);
    MB_CUDA(cudaMallocAsync(&t->data, bytes, ctx->stream));
    MB_CUDA(cudaMemcpyAsync(t->data, s->last, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
    t->owns = true;
    return t.release();
}

void stream_free(mach_stream* s) {
    if (!s) return;
    cudaStreamSynchronize(s->copy);
    cudaStreamSynchronize(s->ctx->stream);
    if (s->idx) cudaFreeAsync(s->idx, s->ctx->stream);
    if (s->val) cudaFreeAsync(s->val, s->ctx->stream);
    for (int b = 0; b < 2; ++b) {
        if (s->stage[b]) cudaFree(s->stage[b]);
        cudaEventDestroy(s->ready[b]);
        cudaEventDestroy(s->freed[b]);
    }
    if (s->cf_last) cudaFree(s->cf_last);
    if (s->cf_seen) cudaFree(s->cf_seen);
    cudaStreamDestroy(s->copy);
    delete s;
}

// ---- binary tensor files ------------------------------------------------------
namespace {

struct FileHeader {
    char magic[8];
    std::uint32_t version, kind, dtype, order;
    std::int32_t dims[8];
    std::int64_t count;       // numel (dense) or nnz (sparse)
    std::uint32_t idx_bytes, reserved;
};
static_assert(sizeof(FileHeader) == 72, "file header layout");
const char kMagic[8] = {'M', 'A', 'C', 'H', 'B', '2', 0, 0};

struct File {
    std::FILE* f = nullptr;
    std::string path;
    File(const char* p, const char* mode) : path(p ? p : "") {
        if (!p) throw_arg("path is null");
        f = std::fopen(p, mode);
        if (!f) throw Error(MACH_ERR_IO, std::string("cannot open '") + p + "' for " + (mode[0] == 'r' ? "reading" : "writing"));
    }
    ~File() {
        if (f) std::fclose(f);
    }
    void write(const void* p, std::size_t n) {
        if (n && std::fwrite(p, 1, n, f) != n) throw Error(MACH_ERR_IO, "write to '" + path + "' failed");
    }
    void read(void* p, std::size_t n) {
        if (n && std::fread(p, 1, n, f) != n) throw Error(MACH_ERR_PARSE, "'" + path + "': truncated tensor file");
    }
    void close() {
        const int rc = std::fclose(f);
        f = nullptr;
        if (rc != 0) throw Error(MACH_ERR_IO, "write to '" + path + "' failed");
    }
};

constexpr std::size_t kChunk = 64u << 20;  // pinned staging, bytes

struct Pinned {
    void* p = nullptr;
    Pinned() { MB_CUDA(cudaMallocHost(&p, kChunk)); }
    ~Pinned() {
        if (p) cudaFreeHost(p);
    }
};

void device_to_file(Ctx* ctx, File& f, const void* dev, std::size_t bytes, Pinned& pin) {
    for (std::size_t o = 0; o < bytes; o += kChunk) {
        const std::size_t n = std::min(kChunk, bytes - o);
        MB_CUDA(cudaMemcpyAsync(pin.p, static_cast<const char*>(dev) + o, n, cudaMemcpyDeviceToHost, ctx->stream));
        sync(ctx);
        f.write(pin.p, n);
    }
}

void file_to_device(Ctx* ctx, File& f, void* dev, std::size_t bytes, Pinned& pin) {
    for (std::size_t o = 0; o < bytes; o += kChunk) {
        const std::size_t n = std::min(kChunk, bytes - o);
        f.read(pin.p, n);
        MB_CUDA(cudaMemcpyAsync(static_cast<char*>(dev) + o, pin.p, n, cudaMemcpyHostToDevice, ctx->stream));
        sync(ctx);
    }
}

FileHeader read_header(File& f) {
    FileHeader h{};
    f.read(&h, sizeof h);
    if (std::memcmp(h.magic, kMagic, 8) != 0) throw Error(MACH_ERR_PARSE, "'" + f.path + "': not a MACHB2 tensor file");
    if (h.version != 1) throw Error(MACH_ERR_PARSE, "'" + f.path + "': unsupported file version");
    if (h.kind > 1 || h.dtype > 1 || h.order < 1 || h.order > 8) throw Error(MACH_ERR_PARSE, "'" + f.path + "': malformed header");
    for (std::uint32_t m = 0; m < h.order; ++m)
        if (h.dims[m] < 1) throw Error(MACH_ERR_PARSE, "'" + f.path + "': malformed dims");
    if (h.count < 0) throw Error(MACH_ERR_PARSE, "'" + f.path + "': malformed count");
    return h;
}

FileHeader make_header(int kind, int dtype, const std::vector<int>& dims, std::int64_t count, int idx_bytes) {
    if (dims.size() > 8) throw_shape("tensor files hold at most 8 modes");
    FileHeader h{};
    std::memcpy(h.magic, kMagic, 8);
    h.version = 1;
    h.kind = static_cast<std::uint32_t>(kind);
    h.dtype = static_cast<std::uint32_t>(dtype);
    h.order = static_cast<std::uint32_t>(dims.size());
    for (std::size_t m = 0; m < dims.size(); ++m) h.dims[m] = dims[m];
    h.count = count;
    h.idx_bytes = static_cast<std::uint32_t>(idx_bytes);
    return h;
}

__global__ void ascending_check_kernel(const void* __restrict__ idx, int idx64, long long n, long long numel,
                                       int* __restrict__ bad) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const unsigned long long a = idx64 ? static_cast<const unsigned long long*>(idx)[i] : static_cast<const unsigned int*>(idx)[i];
    if (a >= static_cast<unsigned long long>(numel)) atomicOr(bad, 1);
    if (i > 0) {
        const unsigned long long b =
            idx64 ? static_cast<const unsigned long long*>(idx)[i - 1] : static_cast<const unsigned int*>(idx)[i - 1];
        if (b >= a) atomicOr(bad, 2);
    }
}

}  // namespace

void dense_save(const mach_dense* t, const char* path) {
    File f(path, "wb");
    const FileHeader h = make_header(0, t->dtype, t->dims, t->numel, 0);
    f.write(&h, sizeof h);
    Pinned pin;
    device_to_file(t->ctx, f, t->data, static_cast<std::size_t>(t->numel) * dtype_size(t->dtype), pin);
    f.close();
}

mach_dense* dense_load(Ctx* ctx, const char* path) {
    File f(path, "rb");
    const FileHeader h = read_header(f);
    if (h.kind != 0) throw Error(MACH_ERR_PARSE, "'" + f.path + "': holds a sparse tensor, a dense one was expected");
    auto t = std::make_unique<mach_dense>();
    t->ctx = ctx;
    t->dtype = static_cast<int>(h.dtype);
    t->dims.assign(h.dims, h.dims + h.order);
    t->numel = checked_size(t->dims);
    if (t->numel != h.count) throw Error(MACH_ERR_PARSE, "'" + f.path + "': element count does not match dims");
    const std::size_t bytes = static_cast<std::size_t>(t->numel) * dtype_size(t->dtype);
    MB_CUDA(cudaMallocAsync(&t->data, bytes, ctx->stream));
    t->owns = true;
    Pinned pin;
    file_to_device(ctx, f, t->data, bytes, pin);
    return t.release();
}

void sparse_save(const mach_sparse* t, const char* path) {
    File f(path, "wb");
    const FileHeader h = make_header(1, t->dtype, t->dims, t->nnz, t->idx64 ? 8 : 4);
    f.write(&h, sizeof h);
    Pinned pin;
    device_to_file(t->ctx, f, t->idx, static_cast<std::size_t>(t->nnz) * (t->idx64 ? 8 : 4), pin);
    device_to_file(t->ctx, f, t->val, static_cast<std::size_t>(t->nnz) * dtype_size(t->dtype), pin);
    f.close();
}

mach_sparse* sparse_load(Ctx* ctx, const char* path) {
    File f(path, "rb");
    const FileHeader h = read_header(f);
    if (h.kind != 1) throw Error(MACH_ERR_PARSE, "'" + f.path + "': holds a dense tensor, a sparse one was expected");
    auto t = std::make_unique<mach_sparse>();
    t->ctx = ctx;
    t->dtype = static_cast<int>(h.dtype);
    t->dims.assign(h.dims, h.dims + h.order);
    t->numel = checked_size(t->dims);
    t->idx64 = t->numel > 0xFFFFFFFFll;
    if (h.idx_bytes != (t->idx64 ? 8u : 4u)) throw Error(MACH_ERR_PARSE, "'" + f.path + "': index width does not match dims");
    if (h.count > t->numel) throw Error(MACH_ERR_PARSE, "'" + f.path + "': more entries than elements");
    t->nnz = h.count;
    if (t->nnz > 0) {
        const std::size_t N = static_cast<std::size_t>(t->nnz);
        MB_CUDA(cudaMallocAsync(&t->idx, N * h.idx_bytes, ctx->stream));
        MB_CUDA(cudaMallocAsync(&t->val, N * dtype_size(t->dtype), ctx->stream));
        Pinned pin;
        file_to_device(ctx, f, t->idx, N * h.idx_bytes, pin);
        file_to_device(ctx, f, t->val, N * dtype_size(t->dtype), pin);
        DBuf<int> bad(ctx, 1);
        bad.zero(ctx);
        MB_LAUNCH(ctx, ascending_check_kernel, ceil_div(t->nnz, 256), 256, 0, static_cast<const void*>(t->idx),
                  t->idx64 ? 1 : 0, static_cast<long long>(t->nnz), static_cast<long long>(t->numel), bad.get());
        int hb = 0;
        to_host(ctx, &hb, bad.get(), 1);
        sync(ctx);
        if (hb) throw Error(MACH_ERR_PARSE, "'" + f.path + "': indices are not ascending, distinct and in range");
    }
    return t.release();
}

void tensor_file_kind(const char* path, int* kind, int* dtype, int* order, int* dims, std::int64_t* count) {
    File f(path, "rb");
    const FileHeader h = read_header(f);
    if (kind) *kind = static_cast<int>(h.kind);
    if (dtype) *dtype = static_cast<int>(h.dtype);
    if (order) *order = static_cast<int>(h.order);
    if (dims)
        for (std::uint32_t m = 0; m < h.order; ++m) dims[m] = h.dims[m];
    if (count) *count = h.count;
}

}  // namespace machb

namespace machb {
int stream_device(const mach_stream* s) { return s->ctx->device; }
}  // namespace machb
