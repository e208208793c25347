// TEST INFRASTRUCTURE ONLY — flat C ABI over the CPU oracle for ctypes
// (tests/, smoke() and bench.py's CPU arms).  Not part of the product.

#include "oracle.hpp"

#include <cstring>
#include <string>

using namespace orc;

namespace {
thread_local std::string g_err;
thread_local int g_kind = 0;
thread_local int g_index = 0;

template <typename F>
int guard(F&& f) {
    try {
        f();
        g_kind = 0;
        return 0;
    } catch (const Error& e) {
        g_err = e.what();
        g_kind = static_cast<int>(e.kind);
        g_index = e.singular_index;
        return g_kind;
    } catch (const std::exception& e) {
        g_err = e.what();
        g_kind = 99;
        return 99;
    }
}

std::vector<int> to_dims(int order, const int* dims) { return std::vector<int>(dims, dims + order); }
}  // namespace

extern "C" {

int orc_last_error(char* buf, int len) {
    if (buf && len > 0) {
        std::strncpy(buf, g_err.c_str(), static_cast<std::size_t>(len - 1));
        buf[len - 1] = 0;
    }
    return g_kind;
}
int orc_last_error_index() { return g_index; }

unsigned long long orc_counter_hash64(unsigned long long seed, unsigned long long c) { return counter_hash64(seed, c); }
double orc_counter_uniform01(unsigned long long seed, unsigned long long c) { return counter_uniform01(seed, c); }

// ---- dense / sparse handles ----
int orc_dense_new(int order, const int* dims, const double* v, void** out) {
    return guard([&] {
        std::vector<int> d = to_dims(order, dims);
        const std::int64_t n = checked_size(d);
        *out = new Dense(make_dense(d, std::vector<double>(v, v + n)));
    });
}
void orc_dense_free(void* h) { delete static_cast<Dense*>(h); }
long long orc_dense_size(void* h) { return static_cast<Dense*>(h)->size(); }
void orc_dense_get(void* h, double* out) {
    auto* t = static_cast<Dense*>(h);
    std::memcpy(out, t->v.data(), t->v.size() * sizeof(double));
}

int orc_sparse_new(int order, const int* dims, long long nnz, const long long* idx, const double* vals, void** out) {
    return guard([&] {
        std::vector<Entry> en(static_cast<std::size_t>(nnz));
        for (long long i = 0; i < nnz; ++i) en[static_cast<std::size_t>(i)] = {idx[i], vals[i]};
        *out = new Sparse(make_sparse(to_dims(order, dims), std::move(en)));
    });
}
void orc_sparse_free(void* h) { delete static_cast<Sparse*>(h); }
long long orc_sparse_nnz(void* h) { return static_cast<Sparse*>(h)->nnz(); }
void orc_sparse_get(void* h, long long* idx, double* vals) {
    auto* s = static_cast<Sparse*>(h);
    for (std::size_t i = 0; i < s->e.size(); ++i) {
        idx[i] = s->e[i].index;
        vals[i] = s->e[i].value;
    }
}
int orc_densify(void* sparse, double* out) {
    return guard([&] {
        Dense d = densify(*static_cast<Sparse*>(sparse));
        std::memcpy(out, d.v.data(), d.v.size() * sizeof(double));
    });
}

int orc_sparsify(void* dense, double p, unsigned long long seed, void** out) {
    return guard([&] { *out = new Sparse(sparsify(*static_cast<Dense*>(dense), p, seed)); });
}

double orc_tensor_norm_dense(void* h) { return tensor_norm(*static_cast<Dense*>(h)); }
double orc_tensor_norm_sparse(void* h) { return tensor_norm(*static_cast<Sparse*>(h)); }

// ---- tensor ops ----
int orc_matricize(void* dense, int mode, double* out) {
    return guard([&] {
        Mat m = matricize(*static_cast<Dense*>(dense), mode);
        std::memcpy(out, m.v.data(), m.v.size() * sizeof(double));
    });
}
static Mat mk_mat(int rows, int cols, const double* v) {
    Mat m(rows, cols);
    std::memcpy(m.v.data(), v, m.v.size() * sizeof(double));
    return m;
}
int orc_mode_product_dense(void* dense, int rows, int cols, const double* m, int mode, double* out) {
    return guard([&] {
        Dense y = mode_product(*static_cast<Dense*>(dense), mk_mat(rows, cols, m), mode);
        std::memcpy(out, y.v.data(), y.v.size() * sizeof(double));
    });
}
int orc_mode_product_sparse(void* sparse, int rows, int cols, const double* m, int mode, double* out) {
    return guard([&] {
        Dense y = mode_product(*static_cast<Sparse*>(sparse), mk_mat(rows, cols, m), mode);
        std::memcpy(out, y.v.data(), y.v.size() * sizeof(double));
    });
}
int orc_sparse_row_gram(void* sparse, int mode, double* out) {
    return guard([&] {
        Mat g = sparse_row_gram(*static_cast<Sparse*>(sparse), mode);
        std::memcpy(out, g.v.data(), g.v.size() * sizeof(double));
    });
}

// ---- linalg ----
int orc_sym_eig(int n, const double* a, double* evals, double* evecs) {
    return guard([&] {
        std::vector<double> ev;
        Mat vec;
        sym_eig(mk_mat(n, n, a), ev, vec);
        std::memcpy(evals, ev.data(), ev.size() * sizeof(double));
        std::memcpy(evecs, vec.v.data(), vec.v.size() * sizeof(double));
    });
}
int orc_jacobi_eig(int n, const double* a, double* evals_desc, double* evecs) {
    return guard([&] {
        std::vector<double> ev;
        Mat vec;
        jacobi_eig(mk_mat(n, n, a), ev, vec);
        std::memcpy(evals_desc, ev.data(), ev.size() * sizeof(double));
        std::memcpy(evecs, vec.v.data(), vec.v.size() * sizeof(double));
    });
}
int orc_left_singular_basis(int rows, int cols, const double* a, int k, double* basis, double* sv, int* nr,
                            int* completed) {
    return guard([&] {
        Basis b = left_singular_basis(mk_mat(rows, cols, a), k);
        std::memcpy(basis, b.basis.v.data(), b.basis.v.size() * sizeof(double));
        std::memcpy(sv, b.sv.data(), b.sv.size() * sizeof(double));
        *nr = b.numerical_rank;
        *completed = b.completed ? 1 : 0;
    });
}
int orc_truncated_svd(int rows, int cols, const double* a, int k, double* left, double* sv, double* right) {
    return guard([&] {
        Svd r = truncated_svd(mk_mat(rows, cols, a), k);
        std::memcpy(left, r.left.v.data(), r.left.v.size() * sizeof(double));
        std::memcpy(sv, r.sv.data(), r.sv.size() * sizeof(double));
        std::memcpy(right, r.right.v.data(), r.right.v.size() * sizeof(double));
    });
}
int orc_low_rank_approx(int rows, int cols, const double* a, int k, double* out) {
    return guard([&] {
        Mat r = low_rank_approx(mk_mat(rows, cols, a), k);
        std::memcpy(out, r.v.data(), r.v.size() * sizeof(double));
    });
}
double orc_subspace_gap(int n, int k, const double* a, const double* b) {
    return subspace_gap(mk_mat(n, k, a), mk_mat(n, k, b));
}

// ---- Tucker ----
int orc_hosvd_dense(void* dense, const int* ranks, void** out) {
    return guard([&] {
        auto* t = static_cast<Dense*>(dense);
        *out = new Model(hosvd(*t, std::vector<int>(ranks, ranks + t->order())));
    });
}
int orc_hosvd_sparse(void* sparse, const int* ranks, void** out) {
    return guard([&] {
        auto* t = static_cast<Sparse*>(sparse);
        *out = new Model(hosvd(*t, std::vector<int>(ranks, ranks + t->order())));
    });
}
int orc_hooi_dense(void* dense, const int* ranks, int max_it, double tol, void** out) {
    return guard([&] {
        auto* t = static_cast<Dense*>(dense);
        *out = new Model(hooi(*t, std::vector<int>(ranks, ranks + t->order()), max_it, tol));
    });
}
int orc_hooi_sparse(void* sparse, const int* ranks, int max_it, double tol, void** out) {
    return guard([&] {
        auto* t = static_cast<Sparse*>(sparse);
        *out = new Model(hooi(*t, std::vector<int>(ranks, ranks + t->order()), max_it, tol));
    });
}
int orc_mach_hooi(void* dense, const int* ranks, double p, unsigned long long seed, int max_it, double tol,
                  void** model_out, void** sparse_out) {
    return guard([&] {
        auto* t = static_cast<Dense*>(dense);
        MachResult r = mach_hooi(*t, std::vector<int>(ranks, ranks + t->order()), p, seed, max_it, tol);
        *model_out = new Model(std::move(r.model));
        *sparse_out = new Sparse(std::move(r.sparsified));
    });
}
int orc_mach_hosvd(void* dense, const int* ranks, double p, unsigned long long seed, void** model_out,
                   void** sparse_out) {
    return guard([&] {
        auto* t = static_cast<Dense*>(dense);
        MachResult r = mach_hosvd(*t, std::vector<int>(ranks, ranks + t->order()), p, seed);
        *model_out = new Model(std::move(r.model));
        *sparse_out = new Sparse(std::move(r.sparsified));
    });
}
int orc_pearson(int n, const double* x, const double* y, double* out) {
    return guard([&] { *out = pearson(std::vector<double>(x, x + n), std::vector<double>(y, y + n)); });
}
int orc_pc_correlation(void* a, void* b, int mode, int component, double* out, int* flipped) {
    return guard([&] {
        bool f = false;
        *out = pc_correlation(*static_cast<Model*>(a), *static_cast<Model*>(b), mode, component, &f);
        *flipped = f ? 1 : 0;
    });
}
int orc_compare(void* a, void* b, void* ref, double* rho, int* flipped, int* tied, double* tie_sin, double* acc2,
                double* core2) {
    return guard([&] {
        Report r = compare(*static_cast<Model*>(a), *static_cast<Model*>(b), *static_cast<Dense*>(ref));
        for (std::size_t m = 0; m < r.rho.size(); ++m) {
            rho[m] = r.rho[m];
            flipped[m] = r.flipped[m] ? 1 : 0;
            tied[m] = r.tied[m] ? 1 : 0;
            tie_sin[m] = r.tie_sin[m];
        }
        acc2[0] = r.accuracy_exact;
        acc2[1] = r.accuracy_mach;
        core2[0] = r.core_exact;
        core2[1] = r.core_mach;
    });
}
int orc_accuracy(void* dense, void* model, double* out) {
    return guard([&] { *out = accuracy(*static_cast<Dense*>(dense), *static_cast<Model*>(model)); });
}
int orc_reconstruct(void* model, double* out) {
    return guard([&] {
        Dense r = reconstruct(*static_cast<Model*>(model));
        std::memcpy(out, r.v.data(), r.v.size() * sizeof(double));
    });
}
int orc_core_tensor(void* dense, int nf, const int* rows, const int* cols, const double* const* fac, double* out) {
    return guard([&] {
        std::vector<Mat> f;
        for (int i = 0; i < nf; ++i) f.push_back(mk_mat(rows[i], cols[i], fac[i]));
        Dense c = core_tensor(*static_cast<Dense*>(dense), f);
        std::memcpy(out, c.v.data(), c.v.size() * sizeof(double));
    });
}

void orc_model_free(void* h) { delete static_cast<Model*>(h); }
int orc_model_order(void* h) { return static_cast<Model*>(h)->core.order(); }
int orc_model_rank(void* h, int m) { return static_cast<Model*>(h)->core.dims[static_cast<std::size_t>(m)]; }
int orc_model_dim(void* h, int m) { return static_cast<Model*>(h)->factors[static_cast<std::size_t>(m)].rows; }
int orc_model_iterations(void* h) { return static_cast<Model*>(h)->iterations; }
double orc_model_fit(void* h) { return static_cast<Model*>(h)->fit; }
int orc_model_n_sweep_fits(void* h) { return static_cast<int>(static_cast<Model*>(h)->sweep_fits.size()); }
void orc_model_sweep_fits(void* h, double* out) {
    auto& s = static_cast<Model*>(h)->sweep_fits;
    std::memcpy(out, s.data(), s.size() * sizeof(double));
}
void orc_model_core(void* h, double* out) {
    auto& c = static_cast<Model*>(h)->core.v;
    std::memcpy(out, c.data(), c.size() * sizeof(double));
}
void orc_model_factor(void* h, int m, double* out) {
    auto& f = static_cast<Model*>(h)->factors[static_cast<std::size_t>(m)].v;
    std::memcpy(out, f.data(), f.size() * sizeof(double));
}
int orc_model_n_warnings(void* h) { return static_cast<int>(static_cast<Model*>(h)->warnings.size()); }
void orc_model_warning(void* h, int i, char* buf, int len) {
    const auto& w = static_cast<Model*>(h)->warnings[static_cast<std::size_t>(i)];
    std::strncpy(buf, w.c_str(), static_cast<std::size_t>(len - 1));
    buf[len - 1] = 0;
}

// ---- fixtures ----
void orc_random_tensor(int order, const int* dims, unsigned long long seed, double* out) {
    Dense t = random_tensor(to_dims(order, dims), seed);
    std::memcpy(out, t.v.data(), t.v.size() * sizeof(double));
}
void orc_random_matrix(int rows, int cols, unsigned long long seed, double* out) {
    Mat m = random_matrix(rows, cols, seed);
    std::memcpy(out, m.v.data(), m.v.size() * sizeof(double));
}
void orc_random_orthogonal(int n, unsigned long long seed, double* out) {
    Mat m = random_orthogonal(n, seed);
    std::memcpy(out, m.v.data(), m.v.size() * sizeof(double));
}

void orc_phase_times(double* sample, double* hosvd, double* sweeps, int max_sweeps, int* n_sweeps) {
    auto& p = last_phase_times();
    *sample = p.sample;
    *hosvd = p.hosvd;
    const int n = static_cast<int>(p.sweeps.size());
    *n_sweeps = n;
    for (int i = 0; i < n && i < max_sweeps; ++i) sweeps[i] = p.sweeps[static_cast<std::size_t>(i)];
}

}  // extern "C"
