// Shared declarations of the sparse route (sparse_ttm.cu) and the device
// linear-algebra helpers (linalg.cu, eig.cu, dense.cu) used by the drivers.
#pragma once

#include "common.cuh"

namespace machb {

// TTM work unit: <= 32 fibre segments of one output row, <= kSegMax nonzeros
// each, stored in jagged-diagonal order at [base, base + len).
constexpr int kSegMax = 32;
constexpr int kTaskNnz = 32 * kSegMax;
// task descriptor: 32 int2 {i_b, length} (lengths descending) followed by the
// 32 u16 jagged-diagonal offsets of positions 0..31 (8 int2)
constexpr int kDesc = 40;

struct TtmTask {
    long long base;
    int len;
    int row;
    int nseg;
    int maxlen;
};

template <typename T, typename IA>
struct TtmArgs {
    const IA* ia;          // inner-mode index per nonzero (task JDS order)
    const T* vals;         // values, same order
    const TtmTask* tasks;
    const int2* desc;      // kDesc int2 per task (see kDesc)
    long long n_task;
    const T* Ua;
    int ra;
    const T* Ub;
    int rb, rbs;
    int sa, sb, C;
    T* P;
    long long ua_rows, ub_elems;   // U_a rows; U_b elements (row-major, padded stride)
    std::size_t fac_bytes;         // shared-memory bytes of the staged factors
    int fac_smem;                  // 1: factors staged in shared memory
    int n_cons, n_slot;            // consumer warps, task slots of the TMA ring
    int dbg;                       // experiments: 1 = stream only (no arithmetic)
    unsigned long long* ts;        // experiments: per-CTA %globaltimer stamps (8 per CTA) or null
    T* fseg;                       // optional: every segment's fibre sum (ra values at fpos[t * 32 + lane] * ra)
    const int* fpos;               // position of each segment in the i_b-grouped order (with fseg)
    int stage1;                    // 1: fibre sums only, to fseg in task order, overlapping the preceding
                                   //    kernel (no wait at entry; see ttm_mode_kernel); 2: same, waiting
};

// Per-mode sorted layout of a sampled tensor (built once, reused by HOSVD and
// every sweep).
struct ModePlan {
    int mode = 0, a = 0, b = -1;
    int ba = 0, bb = 0;
    bool key64 = false;
    int rows = 0;
    DBuf<unsigned char> keys, vals;  // sorted (key, value) pairs (HOSVD Grams)
    DBuf<long long> row_start, row_end;
    // TTM layout
    bool ia16 = false;             // inner index stored as u16
    long long n_task = 0;
    DBuf<unsigned char> ia, jv;    // inner index / value per nonzero, task JDS order
    DBuf<TtmTask> tasks;
    DBuf<int2> desc;
    DBuf<int> st_base;             // tasks of row r: [st_base[r], st_base[r+1])
    // segments grouped by their i_b (built on first use): the fibre sums of
    // this mode's TTM give mode b's Y_(b) without another pass over X
    DBuf<int> seg_pos, seg_ptr;    // segment t * 32 + lane -> position in i_b order; row i_b: [seg_ptr[i], seg_ptr[i+1])
    DBuf<int> seg_row;             // i_n (this mode's row) of the segment at each position
    long long n_seg = -1;          // segments (valid positions), known once grouped
    DBuf<int> seg_ib;              // i_b of every segment slot t * 32 + lane, task order (0 past nseg)
    // order 4 (stage2_4way_kernel): pieces in key order with their slot and
    // composite i_b, each row's piece range, slice partials and row tickets
    bool keep_pieces = false;
    long long n_piece = 0;
    DBuf<int> pslot, pib;
    DBuf<long long> piece_rs, piece_re;
    DBuf<unsigned char> s2part;
    DBuf<unsigned> s2tick;
    // packed-key fields (least significant first): mode and bit offset
    int nf = 0;
    int fmode[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int fshift[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    std::vector<int> bmodes;       // modes folded into the composite i_b (outer first is last)
};

// X_(n) column of a packed key: sum over the fields of ((key >> shift) &
// mask) * stride (the column order of matricize, tensor.hpp:119-121).
struct ColDecode {
    int nf = 0;
    int shift[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    unsigned long long mask[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long stride[8] = {0, 0, 0, 0, 0, 0, 0, 0};
};
ColDecode plan_col_decode(const std::vector<int>& dims, const ModePlan& P);

// Nonzeros of X_(n) grouped by column (mode n in the low key bits, the other
// modes above it in increasing order), with the start of every nonempty
// column run; built on demand for the tall-mode basis.
struct ColLayout {
    bool key64 = false;
    int bn = 0;
    long long nruns = 0;
    DBuf<unsigned char> keys, vals;
    DBuf<long long> runs;  // nruns + 1 (sentinel nnz)
    ColDecode dec;
};
template <typename T>
void build_col_layout(Ctx* ctx, const mach_sparse* X, int n, ColLayout& L);
// group P's segments by i_b (once); false when P has no b mode
bool build_segment_groups(Ctx* ctx, ModePlan& P, int b_rows);

// ---- sparse route ----
bool sparse_fast_path_ok(const std::vector<int>& dims, const std::vector<int>& ranks);
int ttm_ra_bucket(int r);
int ttm_stride(int r, int elem_bytes);  // factor row stride of the TTM kernel copies
template <typename T>
std::shared_ptr<ModePlan> get_plan(mach_sparse* X, int n, const std::vector<int>& ranks, int force_a = -1);
template <typename T>
void sparse_mode_ttm(Ctx* ctx, const ModePlan& P, const std::vector<int>& dims, const std::vector<int>& ranks,
                     const std::vector<const T*>& Ur, const T* one, T* Pbuf, T* Y, T* fseg = nullptr,
                     const int* fpos = nullptr);
// Y_(b) (b = P.b) from the fibre sums F (= X x_a U_a, one ra-vector per
// segment of P's TTM, written by sparse_mode_ttm with fseg) and U_n (row-major
// kernel copy of mode P.mode's factor): Y_(b)[i_b, :] = sum over the segments
// s with i_b(s) = i_b of F_s (x) U_n[i_n(s), :], segments in a fixed order.
template <typename T>
void y_from_segments(Ctx* ctx, ModePlan& P, const std::vector<int>& dims, const std::vector<int>& ranks, const T* fseg,
                     const T* Un, T* Y);
// Split TTM for overlapped sweeps: stage 1 = the fibre sums F (X x_a U_a, one
// ra-vector per segment slot, task order) on `ctas` CTAs, launched so that it
// may overlap the preceding kernel (see ttm_mode_kernel); stage 2 = Y_(n) =
// sum over each row's segments of F (x) U_b[i_b, :] (fixed order).
template <typename T>
void sparse_mode_stage1(Ctx* ctx, ModePlan& P, const std::vector<int>& dims, const std::vector<int>& ranks,
                        const std::vector<const T*>& Ur, T* F, int ctas, bool overlapped = true);
template <typename T>
void sparse_mode_stage2(Ctx* ctx, ModePlan& P, const std::vector<int>& dims, const std::vector<int>& ranks, const T* F,
                        const T* Ub, T* Y);
// order 4: Y_(n) from stage 1's fibre sums through a per-row dense block
// over the outer composite mode (see stage2_4way_kernel)
template <typename T>
void sparse_mode_stage2_4way(Ctx* ctx, ModePlan& P, const std::vector<int>& dims, const std::vector<int>& ranks,
                             const T* F, const std::vector<const T*>& Ur, T* Y);
bool stage2_4way_ok(const std::vector<int>& dims, const std::vector<int>& ranks, int n, int a, int b1, int b2);
template <typename T>
void sparse_row_gram(Ctx* ctx, const mach_sparse* X, int n, double normX2, double* G);
template <typename T>
void sparse_col_gram(Ctx* ctx, const mach_sparse* X, const ModePlan& P, long long cols, double normX2, double* G);
template <typename T>
void sparse_times(Ctx* ctx, const mach_sparse* X, const ModePlan& P, const double* V, long long vld, int kc, double* W);
// Leading-k left singular basis of X_(n) when the column side is too wide for
// a Gram (tall time modes): implicit subspace iteration on
// X_(n) X_(n)^T (tall_basis.cu).  U (I_n x k), sv (k), st (3) as basis_from_side.
template <typename T>
void sparse_tall_basis(Ctx* ctx, const mach_sparse* X, const ModePlan& P, int k, double* U, double* sv, int* st);
// Same for a dense column-major Y (rows x cols) whose column side is too wide.
template <typename T>
void dense_tall_basis(Ctx* ctx, const T* Y, int rows, long long cols, int k, double* U, double* sv, int* st);
// columns of X_(n) above which the tall-mode basis replaces the column Gram
long long tall_min_cols();

// ---- eigen step (eig.cu, linalg.cu) ----
void eig_topk(Ctx* ctx, const double* G, int n, int k, double* work, double* V, double* sig, int* status,
              const int* skip = nullptr);
bool eig_subspace(Ctx* ctx, const double* G, int n, int k, const double* X0, int x0_cols, double* Xkeep, int b,
                  double* V, double* sig, int* status);
// Warm blocks (Xkeep) hold n*b vectors followed by their b Ritz values.
inline std::size_t warm_doubles(int n, int b) { return static_cast<std::size_t>(n) * b + b; }
// top-k eigenpairs of G: warm-started subspace solver when it applies, with the
// exact selected-eigenpair solver as the in-stream fallback.  status[1]==1
// flags an exactly zero G.
bool eig_select(Ctx* ctx, const double* G, int n, int k, const double* X0, int x0_cols, double* Xkeep, int b,
                double* V, double* sig, int* status);
int eig_block(int n, int k);
// whether eig_select uses the warm-startable subspace solver for this shape
bool subspace_applies(int n, int k);
struct EigJob {
    const double* G;
    int n, k;
    const double* X0;
    int x0_cols;
    double* Xkeep;
    double* V;
    double* sig;
    int* status;
    double* Gw;  // workspaces (set by the launcher)
    double* Bw;
    const double* th0 = nullptr;  // Ritz values of X0 (warm start with them: filter first)
};
void eig_select_batched(Ctx* ctx, std::vector<EigJob> jobs);
// multi-kernel subspace solver for G too large for one CTA's shared memory
bool eig_large_batched(Ctx* ctx, const std::vector<EigJob>& jobs, int b);
std::size_t eig_work_doubles(int n, int k);
template <typename T>
void gram(Ctx* ctx, const T* a, long long sk, long long sn, int K, int N, double* G);
template <typename T>
void matmul_yv(Ctx* ctx, const T* Y, int rows, int C, const double* V, int kc, double* W);
void basis_from_side(Ctx* ctx, const double* V, const double* sig, int n, int k, const int* eig_status, double* U,
                     double* sv, int* st);
void basis_from_products(Ctx* ctx, const double* W, int n, int wc, int k, const double* sig, const int* eig_status,
                         double* U, double* sv, int* st);
void identity_basis(Ctx* ctx, double* U, int n, int k, double* sv, int* st);
template <typename T>
void core_from_last(Ctx* ctx, const T* Y, int rows, int C, const double* U, int r, double* core);
// core_from_last + |core|^2 into *out in one launch (part: >= blocks doubles; ticket: zeroed once, re-armed)
template <typename T>
void core_sumsq(Ctx* ctx, const T* Y, int rows, int C, const double* U, int r, double* core, double* part,
                unsigned* ticket, double* out);
template <typename T>
void sumsq(Ctx* ctx, const T* x, long long n, double* scratch, double* out);
int sumsq_scratch();
template <typename T>
void factor_rowmajor(Ctx* ctx, const double* U, int n, int r, int rs, T* out);
// flag-gated variants (run only when need[0] != 0; the fused mode basis queues them as fallbacks)
template <typename T>
void matmul_yv_gated(Ctx* ctx, const T* Y, int rows, int C, const double* V, int kc, double* W, const int* need);
void basis_from_products_gated(Ctx* ctx, const double* W, int n, int wc, int k, const double* sig,
                               const int* eig_status, double* U, double* sv, int* st, const int* need);
template <typename T>
void factor_rowmajor_gated(Ctx* ctx, const double* U, int n, int r, int rs, T* out, const int* need);
// the fused mode basis's fallback chain (W = Y V, basis, row-major copy) in one flag-gated launch
template <typename T>
void mb_fallback(Ctx* ctx, const T* Y, int rows, int C, const double* V, int k, double* W, const double* sig, double* U,
                 double* sv, int* st, T* Ur, int rs, const int* flags);
// the whole fallback chain (exact eigensolver + mb_fallback) in one flag-gated launch (eig.cu)
template <typename T>
void mb_fallback_all(Ctx* ctx, const double* Gout, int n, int k, double* work, double* V, double* sig, int* est,
                     const T* Y, int rows, double* W, double* U, double* sv, int* st, T* Ur, int rs, const int* flags);
// fused column-side mode basis (mode_basis.cu); false = not applicable
template <typename T>
bool mode_basis_fused(Ctx* ctx, const T* Y, int rows, int n, int k, const double* X0, int x0_cols, double* Xkeep, int b,
                      double* U, double* sv, int* st, T* Ur, int rs);

// ---- dense route (dense.cu) ----
// out[a + inner*(q + J*c)] = sum_r in[a + inner*(r + len*c)] * M(q, r) where
// M(q, r) = U[r + len*q] when transpose (U is len x J: projection by U^T) or
// U[q + J*r] otherwise (U is J x len: expansion by U).
template <typename Tin>
void dense_mode_product(Ctx* ctx, const Tin* in, const std::vector<int>& dims, int mode, const double* U, int J,
                        bool transpose, double* out);
// mode_product(SparseTensor, Matrix, mode) from the nonzeros, reference
// summation order (sparse_mode_product.cu); M: J x len column-major
void sparse_mode_product(Ctx* ctx, const mach_sparse* s, int mode, const double* M, int J, double* y);
// |x - reconstruct(core, U)|^2 in one fused pass (metrics.cu)
template <typename T>
double residual2_fused(Ctx* ctx, const T* x, const std::vector<int>& dims, const std::vector<int>& ranks,
                       const double* core, const std::vector<const double*>& U);
double subspace_sin_dev(Ctx* ctx, const double* A, const double* B, int n, int r);
// truncated_svd family on the device (tsvd.cu); A rows x cols column-major
void truncated_svd_dev(Ctx* ctx, const double* A, int rows, int cols, int k, double* left, double* sv, double* right);
void low_rank_dev(Ctx* ctx, const double* L, const double* sv, const double* R, int rows, int cols, int k, double* out);
// work model of mode n's sparse TTM with inner mode a (sparse_ttm.cu)
double inner_cost(const mach_sparse* X, int n, const std::vector<int>& ranks, int a);
// dense mode-n Gram X_(n) X_(n)^T on tcgen05 (gram_tc.cu), read in place
bool gram_tc_applies(const std::vector<int>& dims, int n);
void gram_tc(Ctx* ctx, const float* x, const std::vector<int>& dims, int n, double* G);
// dense mode product out = x x_m U^T (U: I_m x r fp64, r <= 32) on tcgen05, 3xTF32 (ttm_tc.cu)
bool ttm_tc_applies(const std::vector<int>& dims, int m, int r);
void ttm_tc(Ctx* ctx, const float* x, const std::vector<int>& dims, int m, const double* U, int r, double* out);
template <typename Tin, typename Tout>
void dense_matricize(Ctx* ctx, const Tin* in, const std::vector<int>& dims, int mode, Tout* out);
template <typename T>
void densify(Ctx* ctx, const mach_sparse* X, T* out);
// fp32 sampled tensor into a zeroed dense buffer, values rounded to TF32 (for the tensor-core Gram)
void densify_tf32(Ctx* ctx, const mach_sparse* X, float* out);
template <typename T>
void sumsq_diff(Ctx* ctx, const T* x, const double* y, long long n, double* scratch, double* out);
template <typename T>
void scatter_sub(Ctx* ctx, const mach_sparse* X, double* dense);

}  // namespace machb
