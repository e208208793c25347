/*
 * mach_b200.h — C ABI of the B200-native MACH sampler + Tucker (HOSVD/HOOI)
 * hot path.  Plain pointers, sizes and opaque handles; no C++ or torch types.
 *
 * The reference exposes this path as C++ value-semantics functions in
 * /root/reference/proj/include/mach/{tensor,sampling,tucker,linalg}.hpp.
 * Each entry point below names the reference interface it replaces.  The C++
 * mirror of that interface (include/mach/*.hpp, same names and exceptions) is
 * implemented on top of this ABI inside libmach_b200.so.
 *
 * Conventions
 *  - Dense tensors are first-mode-fastest (tensor.hpp:10-12); matrices are
 *    column-major (tensor.hpp:77-105); sparse entries are flat indices.
 *  - Every function returns a mach_status; on failure mach_last_error()
 *    returns a thread-local message and, for MACH_ERR_CONVERGENCE,
 *    mach_last_error_index() the 1-based singular index
 *    (errors.hpp:37-45).  No exception crosses this boundary.
 *  - Handles are device-resident (HBM) and bound to the context's device and
 *    stream.  Host buffers are caller-owned.
 */
#ifndef MACH_B200_H
#define MACH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MACH_OK = 0,
    MACH_ERR_ARGUMENT = 1,    /* mach::ArgumentError (errors.hpp:9-13)    */
    MACH_ERR_SHAPE = 2,       /* mach::ShapeError (errors.hpp:15-19)      */
    MACH_ERR_CONVERGENCE = 3, /* mach::ConvergenceError (errors.hpp:37-45)*/
    MACH_ERR_CUDA = 4,
    MACH_ERR_OOM = 5,
    MACH_ERR_NCCL = 6,
    MACH_ERR_INTERNAL = 7,
    MACH_ERR_IO = 8,          /* mach::IoError (errors.hpp:21-25)         */
    MACH_ERR_PARSE = 9        /* mach::ParseError (errors.hpp:27-35)      */
} mach_status;

typedef enum { MACH_F32 = 0, MACH_F64 = 1 } mach_dtype;

typedef struct mach_ctx mach_ctx;       /* device + stream                   */
typedef struct mach_dense mach_dense;   /* DenseTensor in HBM                */
typedef struct mach_sparse mach_sparse; /* canonical SparseTensor in HBM     */
typedef struct mach_model mach_model;   /* TuckerModel in HBM (+host scalars) */

/* ---- errors / context --------------------------------------------------- */
const char* mach_last_error(void);
int mach_last_error_index(void);
const char* mach_version(void);

mach_status mach_ctx_create(int device, mach_ctx** out);
mach_status mach_ctx_destroy(mach_ctx* ctx);
/* Run all work of this context on an external cudaStream_t (NULL = own). */
mach_status mach_ctx_set_stream(mach_ctx* ctx, void* cuda_stream);
mach_status mach_ctx_synchronize(mach_ctx* ctx);
/* Number of kernels this library launched on the context (bench evidence). */
mach_status mach_ctx_launch_count(mach_ctx* ctx, int64_t* out);

/* ---- dense tensors: DenseTensor (tensor.hpp:13-39) ----------------------- */
/* Copy a host tensor into HBM; values must be finite (tensor.cpp:60-65).    */
mach_status mach_dense_upload(mach_ctx* ctx, mach_dtype dtype, int order, const int* dims,
                              const void* host, mach_dense** out);
/* Wrap caller-owned device memory (no copy, not freed by mach_dense_free).   */
mach_status mach_dense_wrap(mach_ctx* ctx, mach_dtype dtype, int order, const int* dims,
                            void* device_ptr, mach_dense** out);
mach_status mach_dense_download(const mach_dense* t, void* host);
mach_status mach_dense_free(mach_dense* t);

/* ---- sampler: sparsify (sampling.hpp:22, sampling.cpp:21-31) ------------- */
/* Keep x_i != 0 iff counter_uniform01(seed, i) < p; value x_i / p (fp64
 * division, rounded to the tensor dtype).  Output ascending flat index.     */
mach_status mach_sparsify(mach_ctx* ctx, const mach_dense* x, double p, uint64_t seed,
                          mach_sparse** out);
/* Same, with host input and host output (the reference call end to end).   */
mach_status mach_sparsify_host(mach_ctx* ctx, mach_dtype dtype, int order, const int* dims,
                               const void* host_x, double p, uint64_t seed, int64_t* nnz_out,
                               int64_t** idx_out, double** val_out);
void mach_free_host(void* p);
/* Sample the flat range [offset, offset + numel(slab)) of a tensor of dims
   global_dims whose values are `slab` (a time slab under first-mode-fastest
   layout).  The RNG counter and the stored indices are global, so the kept set
   equals the full tensor's restricted to the slab (sampling.cpp:21-31). */
mach_status mach_sparsify_slab(mach_ctx* ctx, const mach_dense* slab, int order, const int* global_dims,
                               int64_t offset, double p, uint64_t seed, mach_sparse** out);

/* ---- sparse tensors: SparseTensor (tensor.hpp:48-75) --------------------- */
/* From host flat-index entries; canonicalised (sorted, merged, zeros
 * dropped) like tensor.cpp:78-96.                                           */
mach_status mach_sparse_upload(mach_ctx* ctx, mach_dtype dtype, int order, const int* dims,
                               int64_t nnz, const int64_t* idx, const double* vals,
                               mach_sparse** out);
mach_status mach_sparse_nnz(const mach_sparse* s, int64_t* nnz);
mach_status mach_sparse_download(const mach_sparse* s, int64_t* idx, double* vals);
/* tensor_norm(SparseTensor) (tensor.hpp:114, tensor.cpp:166-171).           */
mach_status mach_sparse_norm(const mach_sparse* s, double* out);
mach_status mach_sparse_free(mach_sparse* s);
/* device pointers of the (ascending flat index, value) arrays; idx_bytes 4|8 */
mach_status mach_sparse_device_view(const mach_sparse* s, void** idx, void** vals, int* idx_bytes);
/* new tensor from device arrays already in canonical form (ascending unique
   flat indices, u32 when numel < 2^32 else u64; values of dtype), copied */
mach_status mach_sparse_from_device(mach_ctx* ctx, mach_dtype dtype, int order, const int* dims, int64_t nnz,
                                    const void* idx, const void* vals, mach_sparse** out);

/* ---- decompositions (tucker.hpp:34-44, sampling.hpp:32-36) -------------- */
mach_status mach_hosvd_sparse(mach_ctx* ctx, const mach_sparse* t, const int* ranks,
                              mach_model** out);
mach_status mach_hosvd_dense(mach_ctx* ctx, const mach_dense* t, const int* ranks,
                             mach_model** out);
mach_status mach_hooi_sparse(mach_ctx* ctx, const mach_sparse* t, const int* ranks,
                             int max_iterations, double fit_tolerance, mach_model** out);
mach_status mach_hooi_dense(mach_ctx* ctx, const mach_dense* t, const int* ranks,
                            int max_iterations, double fit_tolerance, mach_model** out);
/* mach_hooi (sampling.cpp:41-47): sparsify then hooi; *sampled optional.    */
mach_status mach_mach_hooi(mach_ctx* ctx, const mach_dense* t, const int* ranks, double p,
                           uint64_t seed, int max_iterations, double fit_tolerance,
                           mach_model** out, mach_sparse** sampled);
mach_status mach_mach_hosvd(mach_ctx* ctx, const mach_dense* t, const int* ranks, double p,
                            uint64_t seed, mach_model** out, mach_sparse** sampled);

/* ---- incremental HOOI: hooi_loop (tucker.cpp:80-106) split into begin /
 *      step so sweeps can be driven (and timed) one at a time -------------- */
typedef struct mach_session mach_session;
/* setup (per-mode layouts) + HOSVD initialisation (tucker.cpp:152-169).     */
mach_status mach_hooi_begin(mach_ctx* ctx, const mach_sparse* t, const int* ranks, mach_session** out);
mach_status mach_hooi_begin_dense(mach_ctx* ctx, const mach_dense* t, const int* ranks,
                                  mach_session** out);
/* Up to n sweeps with the reference stop rule (fit - prev < tol ends the
 * iteration, tucker.cpp:102); *done = sweeps run, *stopped = rule fired.
 * fit_tolerance < 0 runs exactly n sweeps (extension for fixed-length runs). */
mach_status mach_hooi_step(mach_session* s, int n, double fit_tolerance, int* done, int* stopped);
mach_status mach_hooi_state(mach_session* s, double* fit, int* iterations);
mach_status mach_hooi_model(mach_session* s, mach_model** out);
/* Algorithmic bytes one mode-`mode` TTM launch moves on the sparse route
   (inner indices + values, task records, partial rows written); -1 when the
   session is on the dense route.  Used for the roofline report. */
mach_status mach_hooi_ttm_bytes(mach_session* s, int mode, long long* bytes);

/* ---- split sweeps (time-slab sharding) ----------------------
   A rank holds the nonzeros of its time slab in a tensor of the GLOBAL dims
   (mach_sparsify_slab).  Each sweep, per mode: mach_hooi_mode_y runs the TTM
   of the local nonzeros and returns the device buffer Y_(mode) (rows x cols,
   column-major, the tensor dtype); the caller sums it over the ranks in place
   (e.g. ncclAllReduce); mach_hooi_mode_update then updates the factor from
   the summed Y.  mach_hooi_sweep_end computes core and fit from the last
   mode's Y (tucker.cpp:80-106 bookkeeping and stop rule). */
mach_status mach_hooi_begin_from(mach_ctx* ctx, const mach_sparse* t, const int* ranks, const mach_model* init,
                                 mach_session** out);  /* start from init's factors (e.g. a replicated HOSVD) */
mach_status mach_hooi_set_norm2(mach_session* s, double norm2);
/* Time-slab sharding over NCCL inside the library.  Rank 0 gets
 * a unique id, the caller broadcasts it, every rank binds its context; then
 * mach_hooi_shard marks a session (built on the rank's slab, e.g. by
 * mach_hooi_begin_from) as one shard: |X|^2 is all-reduced and every sweep
 * of mach_hooi_step all-reduces each mode's partial Y_(n) on the library
 * stream (graph-captured with the rest of the sweep).                      */
#define MACH_COMM_ID_BYTES 128
mach_status mach_comm_unique_id(unsigned char* out);
mach_status mach_ctx_comm_init(mach_ctx* ctx, int world, int rank, const unsigned char* id);
mach_status mach_hooi_shard(mach_session* s);  /* global |X|^2 for the fit */
mach_status mach_hooi_mode_y(mach_session* s, int mode, void** y, int* rows, int* cols);
mach_status mach_hooi_mode_update(mach_session* s, int mode);
mach_status mach_hooi_sweep_end(mach_session* s, double fit_tolerance, int* stopped);
/* Shard HOSVD from partial Grams: with time-slab shards the row
 * Gram of every mode but the last is the sum of the shards' Grams
 * (mach_sparse_row_gram of the local tensor, all-reduced by the caller; the
 * last mode's Gram has cross-slab blocks and comes from the gathered
 * nonzeros).  mach_hosvd_from_grams turns the d full Grams (host, I_n x I_n
 * column-major) into the HOSVD factors (model core / fit left zero);
 * mach_hooi_begin_from starts the shard session from them, and after the
 * caller has reduced mach_hooi_mode_y(order-1), mach_hooi_refresh_fit sets
 * the starting fit (sweep_fits[0]).                                          */
mach_status mach_sparse_row_gram(mach_ctx* ctx, const mach_sparse* t, int mode, double* host);
mach_status mach_hosvd_from_grams(mach_ctx* ctx, int order, const int* dims, const int* ranks,
                                  const double* const* grams, mach_model** out);
mach_status mach_hooi_refresh_fit(mach_session* s);
mach_status mach_session_free(mach_session* s);

/* ---- per-kernel device timing (CUDA events on the context stream) -------- */
mach_status mach_ctx_profile(mach_ctx* ctx, int enable);
/* i-th kernel name with its launch count and summed device milliseconds;
 * returns MACH_ERR_ARGUMENT past the end.  Resets with enable=1.           */
mach_status mach_ctx_kernel_stat(mach_ctx* ctx, int i, char* name, size_t len, int64_t* launches,
                                 double* total_ms);

/* ---- model access (TuckerModel, tucker.hpp:14-22) ------------------------ */
mach_status mach_model_info(const mach_model* m, int* order, int* iterations, double* fit,
                            int* n_sweep_fits, int* n_warnings);
mach_status mach_model_dims(const mach_model* m, int* dims, int* ranks);
mach_status mach_model_core(const mach_model* m, double* host);          /* prod(ranks) */
mach_status mach_model_factor(const mach_model* m, int mode, double* host); /* I x r    */
mach_status mach_model_sweep_fits(const mach_model* m, double* host);
mach_status mach_model_warning(const mach_model* m, int i, char* buf, size_t len);
/* Per-phase device times of the last run (ms): sample, setup, hosvd, sweeps. */
mach_status mach_model_times(const mach_model* m, double* sample_ms, double* setup_ms,
                             double* hosvd_ms, double* sweep_ms, int max_sweeps);
mach_status mach_model_free(mach_model* m);

/* ---- model evaluation (tucker.hpp:47-55) --------------------------------- */
/* accuracy(t, model) = 1 - |t - reconstruct(model)| / |t|                   */
mach_status mach_accuracy(mach_ctx* ctx, const mach_dense* t, const mach_model* m, double* out);
/* accuracy(t, model) from host model arrays (core prod(ranks), factors[m]
 * I_m x r_m column-major): one fused device pass, no reconstruction
 * (tucker.cpp:211-217; compare, metrics.cpp:155-156)                        */
mach_status mach_model_accuracy(mach_ctx* ctx, const mach_dense* t, const int* ranks,
                                const double* core, const double* const* factors, double* out);
/* subspace_sin (metrics.cpp:59-66): largest principal-angle sine between the
 * spans of the leading r columns of host n x r column-major a and b          */
mach_status mach_subspace_sin(mach_ctx* ctx, int n, int r, const double* a, const double* b,
                              double* out);
/* reconstruct(model) into a new dense fp64 tensor                           */
mach_status mach_reconstruct(mach_ctx* ctx, const mach_model* m, mach_dense** out);

/* ---- linear algebra building blocks (linalg.hpp:42, tensor.hpp:121-132) -- */
/* left_singular_basis of a host column-major rows x cols fp64 matrix, on
 * device; basis rows x k, sv k; numerical_rank / completed as in the ref.  */
mach_status mach_left_singular_basis(mach_ctx* ctx, int rows, int cols, const double* a, int k,
                                     double* basis, double* sv, int* numerical_rank,
                                     int* completed);
/* truncated_svd (linalg.hpp:23): top-k singular triplets of a host
 * column-major rows x cols fp64 matrix, 1 <= k <= min(rows, cols); left
 * rows x k, sv k, right cols x k (caller-allocated), reference sign rule.   */
mach_status mach_truncated_svd(mach_ctx* ctx, int rows, int cols, const double* a, int k,
                               double* left, double* sv, double* right);
/* low_rank_approx (linalg.hpp:29): left diag(sv) right^T, rows x cols       */
mach_status mach_low_rank_approx(mach_ctx* ctx, int rows, int cols, const double* a, int k,
                                 double* out);
/* mode_product(DenseTensor / SparseTensor, Matrix, mode) -> new dense fp64   */
mach_status mach_mode_product_dense(mach_ctx* ctx, const mach_dense* t, int rows, int cols,
                                    const double* m, int mode, mach_dense** out);
mach_status mach_mode_product_sparse(mach_ctx* ctx, const mach_sparse* t, int rows, int cols,
                                     const double* m, int mode, mach_dense** out);
/* Mode-n Gram X_(n) X_(n)^T of a dense tensor (the dense HOSVD's row-side
 * Gram, linalg.cpp:340 via tucker.cpp:135-150), I_n x I_n column-major fp64
 * into host.  fp32 tensors of supported shape use the tcgen05 TF32 kernel
 * (*tensor_cores = 1); otherwise the fp64 CUDA-core Gram (*tensor_cores = 0). */
mach_status mach_dense_mode_gram(mach_ctx* ctx, const mach_dense* t, int mode, double* host,
                                 int* tensor_cores);

/* ---- Theorem-1 bound (bounds.hpp:10-66) ---------------------- */
typedef struct mach_bound_mode {   /* BoundModeReport (bounds.hpp:24-30)       */
    int rank;
    double x_residual;             /* |X_(i) - X_(i),r_i|, original tensor      */
    double xhat_residual;          /* same residual on the sampled tensor       */
    double x_lowrank_norm;         /* |X_(i),r_i|                               */
    double t_i;
} mach_bound_mode;
typedef struct mach_bound_report { /* BoundReport (bounds.hpp:35-46)            */
    double b, p, p_min, t, success_probability;
    int dims_large_enough, dims_balanced, p_above_min, conditions_met;
} mach_bound_report;
/* achlioptas_bounds (bounds.hpp:17): (4 b sqrt(n/p), 4 b sqrt(n k/p))         */
mach_status mach_achlioptas_bounds(double b, int64_t n, int64_t k, double p, double* two_norm,
                                   double* frobenius);
/* min_sampling_probability (bounds.hpp:22)                                    */
mach_status mach_min_sampling_probability(int order, const int* dims, double* out);
/* theorem1_conditions (bounds.hpp:51): shape-only part of the report          */
mach_status mach_theorem1_conditions(int order, const int* dims, double p, mach_bound_report* rep);
/* theorem1_bound (bounds.hpp:62): full mode spectra of x and xhat from the
 * device Gram kernels and the on-device eigensolver; per_mode holds one entry
 * per mode (caller-allocated).  The shorter side of every mode unfolding must
 * be <= 1700 (one-CTA spectrum solver).                                        */
mach_status mach_theorem1_bound(mach_ctx* ctx, const mach_dense* x, const mach_sparse* xhat,
                                const int* ranks, double p, mach_bound_report* rep,
                                mach_bound_mode* per_mode);

/* ---- streaming sample-on-arrival ingest (PAPER Remark 2,
 * ingest.hpp:44) ------------------------------------------------------------
 * A stream is a tensor growing along its last (time) mode.  dims gives the
 * leading modes and, in dims[order-1], the CAPACITY in time ticks.  Every
 * arriving time slab is sampled on the device with the global flat index as
 * the RNG counter (sampling.cpp:27) and appended to the sampled tensor in HBM,
 * so at any time the kept set equals mach_sparsify of the tensor seen so far,
 * bit for bit.                                                                */
typedef struct mach_stream mach_stream;
mach_status mach_stream_begin(mach_ctx* ctx, mach_dtype dtype, int order, const int* dims, double p,
                              uint64_t seed, mach_stream** out);
/* append a device-resident slab (leading dims x ticks, first mode fastest)    */
mach_status mach_stream_append(mach_stream* s, const mach_dense* slab);
/* append a host slab of `ticks` time ticks (dtype values): the host->device
 * copy of this slab overlaps the sampling of the previous one (two staging
 * buffers); the host buffer may be reused on return                           */
mach_status mach_stream_append_host(mach_stream* s, const void* host, int ticks);
/* ingest (ingest.cpp:90-134) of one time slab of pre-indexed measurement
 * records on the device: the cell (machine, metric, tick) means are formed in
 * (cell, value) order (independent of record order), empty cells are zero or,
 * with carry_forward, the cell's latest earlier value (state kept across
 * slabs); the slab is then sampled and appended.  order must be 3.            */
mach_status mach_stream_append_records(mach_stream* s, int64_t n, const int32_t* machine,
                                       const int32_t* metric, const int32_t* tick,
                                       const double* value, int ticks, int carry_forward);
mach_status mach_stream_state(mach_stream* s, int64_t* ticks, int64_t* nnz);
/* the sampled tensor seen so far (dims: leading modes x ticks), a copy        */
mach_status mach_stream_tensor(mach_stream* s, mach_sparse** out);
/* the last appended dense slab (records / host appends), for inspection       */
mach_status mach_stream_last_slab(mach_stream* s, mach_dense** out);
mach_status mach_stream_free(mach_stream* s);

/* ---- binary tensor files (replaces the text formats of
 * tensor_io.hpp:24-26 at scale) ----------------------------------------------
 * Little-endian: "MACHB2\0\0", u32 version (1), u32 kind (0 dense, 1 sparse),
 * u32 dtype (mach_dtype), u32 order, i32 dims[order], i64 nnz (numel for
 * dense), u32 index bytes (0 dense, 4|8 sparse), u32 reserved; then the raw
 * arrays (sparse: ascending flat indices, then values).                       */
mach_status mach_dense_save(const mach_dense* t, const char* path);
mach_status mach_dense_load(mach_ctx* ctx, const char* path, mach_dense** out);
mach_status mach_sparse_save(const mach_sparse* t, const char* path);
mach_status mach_sparse_load(mach_ctx* ctx, const char* path, mach_sparse** out);
/* kind of a tensor file without loading it: 0 dense, 1 sparse                 */
mach_status mach_tensor_file_kind(const char* path, int* kind, mach_dtype* dtype, int* order,
                                  int* dims /* >= 8 */, int64_t* nnz);

#ifdef __cplusplus
}
#endif
#endif /* MACH_B200_H */
