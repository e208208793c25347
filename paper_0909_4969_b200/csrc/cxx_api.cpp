// C++ drop-in for the reference API (include/mach/*.hpp mirrors
// /root/reference/proj/include/mach/*.hpp).  Value types stay on the host;
// every computation goes through the C ABI onto the B200 (thread-local
// context on device MACH_DEVICE, default 0).  C ABI status codes are rethrown
// as the reference's exception types.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>

#include "mach/errors.hpp"
#include "mach/linalg.hpp"
#include "mach/metrics.hpp"
#include "mach/sampling.hpp"
#include "mach/tensor.hpp"
#include "mach/tucker.hpp"
#include "mach_b200.h"

namespace mach {

namespace {

void rethrow(mach_status st) {
    if (st == MACH_OK) return;
    std::string msg = mach_last_error();
    switch (st) {
        case MACH_ERR_ARGUMENT: throw ArgumentError(msg);
        case MACH_ERR_SHAPE: throw ShapeError(msg);
        case MACH_ERR_CONVERGENCE: {
            const auto p = msg.rfind(" (singular index ");
            if (p != std::string::npos) msg = msg.substr(0, p);
            throw ConvergenceError(msg, mach_last_error_index());
        }
        case MACH_ERR_IO: throw IoError(msg);
        case MACH_ERR_PARSE: throw ParseError(msg, 1);
        default: throw std::runtime_error("mach-b200: " + msg);
    }
}

struct CtxHolder {
    mach_ctx* ctx = nullptr;
    CtxHolder() {
        const char* dev = std::getenv("MACH_DEVICE");
        rethrow(mach_ctx_create(dev ? std::atoi(dev) : 0, &ctx));
    }
    ~CtxHolder() { mach_ctx_destroy(ctx); }
};

mach_ctx* ctx() {
    thread_local CtxHolder h;
    return h.ctx;
}

}  // namespace

namespace b200 {  // shared with cxx_api_ext.cpp
mach_ctx* context() { return ctx(); }
void check(mach_status st) { rethrow(st); }
}  // namespace b200

namespace {

std::int64_t checked_size(const std::vector<int>& dims) {
    if (dims.empty()) throw ArgumentError("tensor must have at least one mode");
    std::int64_t n = 1;
    for (int d : dims) {
        if (d < 1) throw ArgumentError("every dimension must be >= 1");
        if (n > std::numeric_limits<std::int64_t>::max() / d) throw ArgumentError("shape product overflows");
        n *= d;
    }
    return n;
}

struct DenseH {
    mach_dense* h = nullptr;
    explicit DenseH(const DenseTensor& t) {
        rethrow(mach_dense_upload(ctx(), MACH_F64, t.order(), t.dims().data(), t.data(), &h));
    }
    ~DenseH() { mach_dense_free(h); }
};

struct SparseH {
    mach_sparse* h = nullptr;
    explicit SparseH(const SparseTensor& t) {
        std::vector<std::int64_t> idx(static_cast<std::size_t>(t.nnz()));
        std::vector<double> val(static_cast<std::size_t>(t.nnz()));
        for (std::size_t i = 0; i < idx.size(); ++i) {
            idx[i] = t.entries()[i].index;
            val[i] = t.entries()[i].value;
        }
        rethrow(mach_sparse_upload(ctx(), MACH_F64, t.order(), t.dims().data(), t.nnz(), idx.data(), val.data(), &h));
    }
    explicit SparseH(mach_sparse* p) : h(p) {}
    ~SparseH() { mach_sparse_free(h); }
};

DenseTensor from_device(mach_dense* d, const std::vector<int>& dims) {
    std::vector<double> v(static_cast<std::size_t>(checked_size(dims)));
    const mach_status st = mach_dense_download(d, v.data());
    mach_dense_free(d);
    rethrow(st);
    return DenseTensor(dims, std::move(v));
}

SparseTensor sparse_to_value(mach_sparse* s, const std::vector<int>& dims) {
    std::int64_t nnz = 0;
    rethrow(mach_sparse_nnz(s, &nnz));
    std::vector<std::int64_t> idx(static_cast<std::size_t>(nnz));
    std::vector<double> val(static_cast<std::size_t>(nnz));
    rethrow(mach_sparse_download(s, idx.data(), val.data()));
    std::vector<SparseEntry> e(static_cast<std::size_t>(nnz));
    for (std::size_t i = 0; i < e.size(); ++i) e[i] = {idx[i], val[i]};
    return SparseTensor::from_canonical(dims, std::move(e));
}

TuckerModel model_to_value(mach_model* m) {
    int order = 0, iters = 0, nfits = 0, nwarn = 0;
    double fit = 0;
    rethrow(mach_model_info(m, &order, &iters, &fit, &nfits, &nwarn));
    std::vector<int> dims(static_cast<std::size_t>(order)), ranks(static_cast<std::size_t>(order));
    rethrow(mach_model_dims(m, dims.data(), ranks.data()));
    TuckerModel out;
    std::vector<double> core(static_cast<std::size_t>(checked_size(ranks)));
    rethrow(mach_model_core(m, core.data()));
    out.core = DenseTensor(ranks, std::move(core));
    for (int q = 0; q < order; ++q) {
        Matrix f(dims[static_cast<std::size_t>(q)], ranks[static_cast<std::size_t>(q)]);
        rethrow(mach_model_factor(m, q, f.data()));
        out.factors.push_back(std::move(f));
    }
    out.ranks = ranks;
    out.iterations = iters;
    out.fit = fit;
    out.sweep_fits.resize(static_cast<std::size_t>(nfits));
    rethrow(mach_model_sweep_fits(m, out.sweep_fits.data()));
    for (int i = 0; i < nwarn; ++i) {
        char buf[512];
        rethrow(mach_model_warning(m, i, buf, sizeof buf));
        out.warnings.emplace_back(buf);
    }
    mach_model_free(m);
    return out;
}

}  // namespace

// ---- DenseTensor / SparseTensor / Matrix (tensor.cpp:47-147 contracts) ----
DenseTensor::DenseTensor(std::vector<int> dims)
    : dims_(std::move(dims)), values_(static_cast<std::size_t>(checked_size(dims_)), 0.0) {}

DenseTensor::DenseTensor(std::vector<int> dims, std::vector<double> values) : dims_(std::move(dims)), values_(std::move(values)) {
    if (static_cast<std::int64_t>(values_.size()) != checked_size(dims_))
        throw ShapeError("value count does not match shape product");
    for (double x : values_)
        if (!std::isfinite(x)) throw ArgumentError("tensor values must be finite");
}

std::int64_t DenseTensor::flat_index(std::span<const int> index) const {
    if (index.size() != dims_.size()) throw ArgumentError("multi-index order mismatch");
    std::int64_t f = 0, stride = 1;
    for (std::size_t m = 0; m < dims_.size(); ++m) {
        if (index[m] < 0 || index[m] >= dims_[m]) throw ArgumentError("multi-index out of bounds");
        f += index[m] * stride;
        stride *= dims_[m];
    }
    return f;
}

SparseTensor::SparseTensor(std::vector<int> dims, std::vector<SparseEntry> entries) : dims_(std::move(dims)) {
    // canonicalise on the device (sort, merge, drop zeros)
    std::vector<std::int64_t> idx(entries.size());
    std::vector<double> val(entries.size());
    for (std::size_t i = 0; i < entries.size(); ++i) {
        idx[i] = entries[i].index;
        val[i] = entries[i].value;
    }
    mach_sparse* s = nullptr;
    rethrow(mach_sparse_upload(ctx(), MACH_F64, static_cast<int>(dims_.size()), dims_.data(),
                               static_cast<std::int64_t>(idx.size()), idx.data(), val.data(), &s));
    SparseH guard(s);
    *this = sparse_to_value(s, dims_);
    guard.h = s;
}

SparseTensor::SparseTensor(std::vector<int> dims, const std::vector<std::pair<std::vector<int>, double>>& entries)
    : SparseTensor(dims, [&] {
          std::vector<SparseEntry> flat;
          flat.reserve(entries.size());
          for (const auto& [idx, v] : entries) {
              if (idx.size() != dims.size()) throw ArgumentError("multi-index order mismatch");
              std::int64_t f = 0, stride = 1;
              for (std::size_t m = 0; m < idx.size(); ++m) {
                  if (idx[m] < 0 || idx[m] >= dims[m]) throw ArgumentError("multi-index out of bounds");
                  f += idx[m] * stride;
                  stride *= dims[m];
              }
              flat.push_back({f, v});
          }
          return flat;
      }()) {}

SparseTensor SparseTensor::from_canonical(std::vector<int> dims, std::vector<SparseEntry> entries) {
    SparseTensor t;
    t.dims_ = std::move(dims);
    t.entries_ = std::move(entries);
    return t;
}

std::int64_t SparseTensor::size() const noexcept {
    std::int64_t n = 1;
    for (int d : dims_) n *= d;
    return n;
}

std::vector<int> SparseTensor::multi_index(std::int64_t flat) const {
    std::vector<int> idx(dims_.size());
    for (std::size_t m = 0; m < dims_.size(); ++m) {
        idx[m] = static_cast<int>(flat % dims_[m]);
        flat /= dims_[m];
    }
    return idx;
}

Matrix::Matrix(int rows, int cols) : rows_(rows), cols_(cols) {
    if (rows < 0 || cols < 0) throw ArgumentError("matrix dimensions must be nonnegative");
    values_.assign(static_cast<std::size_t>(rows) * static_cast<std::size_t>(cols), 0.0);
}

Matrix::Matrix(int rows, int cols, std::vector<double> values) : rows_(rows), cols_(cols), values_(std::move(values)) {
    if (rows < 0 || cols < 0) throw ArgumentError("matrix dimensions must be nonnegative");
    if (values_.size() != static_cast<std::size_t>(rows) * static_cast<std::size_t>(cols))
        throw ShapeError("value count does not match rows*cols");
}

Matrix Matrix::identity(int n) {
    Matrix m(n, n);
    for (int i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
}

Matrix transpose(const Matrix& m) {
    Matrix t(m.cols(), m.rows());
    for (int c = 0; c < m.cols(); ++c)
        for (int r = 0; r < m.rows(); ++r) t(c, r) = m(r, c);
    return t;
}

// Pairwise (cascade) summation of f(lo..hi-1) in the reference's order
// (internal.hpp:36-46): blocks of <= 64 summed left to right, halves added,
// so host-side norms agree with the reference bit for bit.
template <typename F>
double pairwise_sum(std::int64_t lo, std::int64_t hi, F&& f) {
    const std::int64_t n = hi - lo;
    if (n <= 64) {
        double s = 0.0;
        for (std::int64_t i = lo; i < hi; ++i) s += f(i);
        return s;
    }
    const std::int64_t mid = lo + n / 2;
    return pairwise_sum(lo, mid, f) + pairwise_sum(mid, hi, f);
}

double frobenius_norm(const Matrix& m) {
    const double* v = m.data();
    return std::sqrt(pairwise_sum(0, static_cast<std::int64_t>(m.values().size()), [&](std::int64_t i) { return v[i] * v[i]; }));
}

double tensor_norm(const DenseTensor& t) {
    const double* v = t.data();
    return std::sqrt(pairwise_sum(0, t.size(), [&](std::int64_t i) { return v[i] * v[i]; }));
}

double tensor_norm(const SparseTensor& t) {
    SparseH h(t);
    double n = 0.0;
    rethrow(mach_sparse_norm(h.h, &n));
    return n;
}

double inner_product(const DenseTensor& x, const DenseTensor& y) {
    if (x.dims() != y.dims()) throw ShapeError("inner_product requires identical shapes");
    return pairwise_sum(0, x.size(), [&](std::int64_t i) { return x.data()[i] * y.data()[i]; });
}

Matrix matricize(const DenseTensor& t, int mode) {
    if (mode < 0 || mode >= t.order()) throw ArgumentError("mode out of range");
    std::int64_t inner = 1, outer = 1;
    for (int m = 0; m < mode; ++m) inner *= t.dim(m);
    for (int m = mode + 1; m < t.order(); ++m) outer *= t.dim(m);
    const int len = t.dim(mode);
    Matrix out(len, static_cast<int>(inner * outer));
    for (std::int64_t c = 0; c < outer; ++c)
        for (int r = 0; r < len; ++r)
            for (std::int64_t a = 0; a < inner; ++a)
                out(r, static_cast<int>(a + inner * c)) = t.data()[a + inner * (r + static_cast<std::int64_t>(len) * c)];
    return out;
}

DenseTensor refold(const Matrix& m, int mode, const std::vector<int>& dims) {
    if (mode < 0 || mode >= static_cast<int>(dims.size())) throw ArgumentError("mode out of range");
    std::int64_t inner = 1, outer = 1;
    for (int q = 0; q < mode; ++q) inner *= dims[static_cast<std::size_t>(q)];
    for (int q = mode + 1; q < static_cast<int>(dims.size()); ++q) outer *= dims[static_cast<std::size_t>(q)];
    const int len = dims[static_cast<std::size_t>(mode)];
    if (m.rows() != len || static_cast<std::int64_t>(m.cols()) != inner * outer)
        throw ShapeError("matrix shape does not match refold target dims");
    DenseTensor t(dims);
    for (std::int64_t c = 0; c < outer; ++c)
        for (int r = 0; r < len; ++r)
            for (std::int64_t a = 0; a < inner; ++a)
                t.data()[a + inner * (r + static_cast<std::int64_t>(len) * c)] = m(r, static_cast<int>(a + inner * c));
    return t;
}

DenseTensor mode_product(const DenseTensor& t, const Matrix& m, int mode) {
    DenseH h(t);
    mach_dense* out = nullptr;
    rethrow(mach_mode_product_dense(ctx(), h.h, m.rows(), m.cols(), m.data(), mode, &out));
    std::vector<int> od = t.dims();
    od[static_cast<std::size_t>(mode)] = m.rows();
    return from_device(out, od);
}

DenseTensor mode_product(const SparseTensor& t, const Matrix& m, int mode) {
    SparseH h(t);
    mach_dense* out = nullptr;
    rethrow(mach_mode_product_sparse(ctx(), h.h, m.rows(), m.cols(), m.data(), mode, &out));
    std::vector<int> od = t.dims();
    od[static_cast<std::size_t>(mode)] = m.rows();
    return from_device(out, od);
}

DenseTensor densify(const SparseTensor& s) {
    DenseTensor t(s.dims());
    for (const auto& e : s.entries()) t.data()[e.index] = e.value;
    return t;
}

SparseTensor sparsify_exact(const DenseTensor& t) {
    std::vector<SparseEntry> e;
    for (std::int64_t i = 0; i < t.size(); ++i)
        if (t.data()[i] != 0.0) e.push_back({i, t.data()[i]});
    return SparseTensor::from_canonical(t.dims(), std::move(e));
}

// ---- sampling.hpp ----
SparseTensor sparsify(const DenseTensor& t, const SparsifyConfig& cfg) {
    DenseH h(t);
    mach_sparse* s = nullptr;
    rethrow(mach_sparsify(ctx(), h.h, cfg.p, cfg.seed, &s));
    SparseH g(s);
    return sparse_to_value(s, t.dims());
}

MachResult mach_hosvd(const DenseTensor& t, const std::vector<int>& ranks, const SparsifyConfig& cfg) {
    DenseH h(t);
    mach_model* m = nullptr;
    mach_sparse* s = nullptr;
    if (ranks.size() != t.dims().size()) throw ArgumentError("ranks must name one rank per mode");
    rethrow(mach_mach_hosvd(ctx(), h.h, ranks.data(), cfg.p, cfg.seed, &m, &s));
    SparseH g(s);
    MachResult r;
    r.sparsified = sparse_to_value(s, t.dims());
    r.model = model_to_value(m);
    return r;
}

MachResult mach_hooi(const DenseTensor& t, const std::vector<int>& ranks, const SparsifyConfig& scfg, const HooiConfig& hcfg) {
    DenseH h(t);
    mach_model* m = nullptr;
    mach_sparse* s = nullptr;
    if (ranks.size() != t.dims().size()) throw ArgumentError("ranks must name one rank per mode");
    rethrow(mach_mach_hooi(ctx(), h.h, ranks.data(), scfg.p, scfg.seed, hcfg.max_iterations, hcfg.fit_tolerance, &m, &s));
    SparseH g(s);
    MachResult r;
    r.sparsified = sparse_to_value(s, t.dims());
    r.model = model_to_value(m);
    return r;
}

// ---- tucker.hpp ----
TuckerModel hosvd(const DenseTensor& t, const std::vector<int>& ranks) {
    if (ranks.size() != t.dims().size()) throw ArgumentError("ranks must name one rank per mode");
    DenseH h(t);
    mach_model* m = nullptr;
    rethrow(mach_hosvd_dense(ctx(), h.h, ranks.data(), &m));
    return model_to_value(m);
}

TuckerModel hosvd(const SparseTensor& t, const std::vector<int>& ranks) {
    if (ranks.size() != t.dims().size()) throw ArgumentError("ranks must name one rank per mode");
    SparseH h(t);
    mach_model* m = nullptr;
    rethrow(mach_hosvd_sparse(ctx(), h.h, ranks.data(), &m));
    return model_to_value(m);
}

TuckerModel hooi(const DenseTensor& t, const std::vector<int>& ranks, const HooiConfig& cfg) {
    if (ranks.size() != t.dims().size()) throw ArgumentError("ranks must name one rank per mode");
    DenseH h(t);
    mach_model* m = nullptr;
    rethrow(mach_hooi_dense(ctx(), h.h, ranks.data(), cfg.max_iterations, cfg.fit_tolerance, &m));
    return model_to_value(m);
}

TuckerModel hooi(const SparseTensor& t, const std::vector<int>& ranks, const HooiConfig& cfg) {
    if (ranks.size() != t.dims().size()) throw ArgumentError("ranks must name one rank per mode");
    SparseH h(t);
    mach_model* m = nullptr;
    rethrow(mach_hooi_sparse(ctx(), h.h, ranks.data(), cfg.max_iterations, cfg.fit_tolerance, &m));
    return model_to_value(m);
}

DenseTensor core_tensor(const DenseTensor& t, const std::vector<Matrix>& factors) {
    if (static_cast<int>(factors.size()) != t.order()) throw ArgumentError("one factor per mode required");
    DenseTensor y = t;
    for (int m = 0; m < t.order(); ++m) y = mode_product(y, transpose(factors[static_cast<std::size_t>(m)]), m);
    return y;
}

DenseTensor reconstruct(const TuckerModel& model) {
    DenseTensor y = model.core;
    for (int m = 0; m < model.core.order(); ++m) y = mode_product(y, model.factors[static_cast<std::size_t>(m)], m);
    return y;
}

// accuracy (tucker.cpp:211-217): one fused device pass over t, the
// reconstruction is never materialised (metrics.cu)
double accuracy(const DenseTensor& t, const TuckerModel& model) {
    if (static_cast<int>(model.factors.size()) != t.order()) throw ShapeError("model reconstructs to a different shape");
    for (int m = 0; m < t.order(); ++m)
        if (model.factors[static_cast<std::size_t>(m)].rows() != t.dim(m))
            throw ShapeError("model reconstructs to a different shape");
    DenseH h(t);
    std::vector<const double*> f;
    for (const Matrix& u : model.factors) f.push_back(u.data());
    double out = 0.0;
    rethrow(mach_model_accuracy(ctx(), h.h, model.ranks.data(), model.core.data(), f.data(), &out));
    return out;
}

// ---- metrics.hpp (metrics.cpp:15-159) ----
namespace {
constexpr double kTieGap = 1e-6;  // metrics.cpp:19

void check_same_shape(const TuckerModel& a, const TuckerModel& b) {
    if (a.factors.size() != b.factors.size())
        throw ShapeError("models have orders " + std::to_string(a.factors.size()) + " and " + std::to_string(b.factors.size()));
    for (std::size_t m = 0; m < a.factors.size(); ++m)
        if (a.factors[m].rows() != b.factors[m].rows())
            throw ShapeError("mode " + std::to_string(m + 1) + " has " + std::to_string(a.factors[m].rows()) +
                             " rows in one model and " + std::to_string(b.factors[m].rows()) + " in the other");
}

std::vector<double> core_slice_norms(const DenseTensor& core, int mode) {
    std::int64_t stride = 1;
    for (int m = 0; m < mode; ++m) stride *= core.dim(m);
    const std::int64_t len = core.dim(mode);
    std::vector<double> sq(static_cast<std::size_t>(len), 0.0);
    for (std::int64_t i = 0; i < core.size(); ++i) sq[static_cast<std::size_t>((i / stride) % len)] += core.data()[i] * core.data()[i];
    for (double& v : sq) v = std::sqrt(v);
    return sq;
}

bool top_two_tied(std::vector<double> n) {
    if (n.size() < 2) return false;
    std::sort(n.begin(), n.end(), std::greater<>());
    return n[0] - n[1] <= kTieGap * n[0];
}
}  // namespace

double pearson(std::span<const double> x, std::span<const double> y) {
    if (x.size() != y.size())
        throw ShapeError("correlation inputs have lengths " + std::to_string(x.size()) + " and " + std::to_string(y.size()));
    const std::int64_t n = static_cast<std::int64_t>(x.size());
    if (n < 2) throw ArgumentError("correlation needs at least 2 samples");
    const bool xc = std::all_of(x.begin(), x.end(), [&](double v) { return v == x[0]; });
    const bool yc = std::all_of(y.begin(), y.end(), [&](double v) { return v == y[0]; });
    if (xc || yc) throw ArgumentError("correlation is undefined for a zero-variance input");
    const double mx = pairwise_sum(0, n, [&](std::int64_t i) { return x[static_cast<std::size_t>(i)]; }) / static_cast<double>(n);
    const double my = pairwise_sum(0, n, [&](std::int64_t i) { return y[static_cast<std::size_t>(i)]; }) / static_cast<double>(n);
    const double sxx = pairwise_sum(0, n, [&](std::int64_t i) {
        const double d = x[static_cast<std::size_t>(i)] - mx;
        return d * d;
    });
    const double syy = pairwise_sum(0, n, [&](std::int64_t i) {
        const double d = y[static_cast<std::size_t>(i)] - my;
        return d * d;
    });
    const double sxy = pairwise_sum(0, n, [&](std::int64_t i) {
        return (x[static_cast<std::size_t>(i)] - mx) * (y[static_cast<std::size_t>(i)] - my);
    });
    if (sxx == 0.0 || syy == 0.0) throw ArgumentError("correlation is undefined for a zero-variance input");
    return sxy / std::sqrt(sxx * syy);
}

double pc_correlation(const TuckerModel& exact, const TuckerModel& approx, int mode, int component, bool* flipped) {
    check_same_shape(exact, approx);
    const int d = static_cast<int>(exact.factors.size());
    if (mode < 0 || mode >= d)
        throw ArgumentError("mode " + std::to_string(mode + 1) + " out of range for order " + std::to_string(d));
    const int limit = std::min(exact.ranks[static_cast<std::size_t>(mode)], approx.ranks[static_cast<std::size_t>(mode)]);
    if (component < 1 || component > limit)
        throw ArgumentError("component " + std::to_string(component) + " out of range; mode " + std::to_string(mode + 1) +
                            " has at most " + std::to_string(limit) + " shared components");
    const Matrix& fa = exact.factors[static_cast<std::size_t>(mode)];
    const Matrix& fb = approx.factors[static_cast<std::size_t>(mode)];
    const std::span<const double> a(fa.data() + static_cast<std::size_t>(component - 1) * fa.rows(), static_cast<std::size_t>(fa.rows()));
    const std::span<const double> b(fb.data() + static_cast<std::size_t>(component - 1) * fb.rows(), static_cast<std::size_t>(fb.rows()));
    const double dot = pairwise_sum(0, static_cast<std::int64_t>(a.size()),
                                    [&](std::int64_t i) { return a[static_cast<std::size_t>(i)] * b[static_cast<std::size_t>(i)]; });
    const bool flip = dot < 0.0;
    if (flipped) *flipped = flip;
    if (!flip) return pearson(a, b);
    std::vector<double> aligned(b.begin(), b.end());
    for (double& v : aligned) v = -v;
    return pearson(a, aligned);
}

ComparisonReport compare(const TuckerModel& exact, const TuckerModel& approx, const DenseTensor& reference) {
    check_same_shape(exact, approx);
    if (reference.order() != static_cast<int>(exact.factors.size()))
        throw ShapeError("reference has order " + std::to_string(reference.order()) + ", models have order " +
                         std::to_string(exact.factors.size()));
    for (int m = 0; m < reference.order(); ++m)
        if (reference.dim(m) != exact.factors[static_cast<std::size_t>(m)].rows())
            throw ShapeError("mode " + std::to_string(m + 1) + " has " + std::to_string(reference.dim(m)) +
                             " entries in the reference and " +
                             std::to_string(exact.factors[static_cast<std::size_t>(m)].rows()) + " in the models");
    const int d = reference.order();
    ComparisonReport rep;
    rep.per_mode_rho.resize(static_cast<std::size_t>(d));
    rep.flipped.assign(static_cast<std::size_t>(d), false);
    rep.tied.assign(static_cast<std::size_t>(d), false);
    rep.tie_subspace_sin.assign(static_cast<std::size_t>(d), 0.0);
    for (int m = 0; m < d; ++m) {
        bool flip = false;
        rep.per_mode_rho[static_cast<std::size_t>(m)] = pc_correlation(exact, approx, m, 1, &flip);
        rep.flipped[static_cast<std::size_t>(m)] = flip;
        if (top_two_tied(core_slice_norms(exact.core, m)) || top_two_tied(core_slice_norms(approx.core, m))) {
            rep.tied[static_cast<std::size_t>(m)] = true;
            const int r = std::min(exact.ranks[static_cast<std::size_t>(m)], approx.ranks[static_cast<std::size_t>(m)]);
            double s = 0.0;
            rethrow(mach_subspace_sin(ctx(), exact.factors[static_cast<std::size_t>(m)].rows(), r,
                                      exact.factors[static_cast<std::size_t>(m)].data(),
                                      approx.factors[static_cast<std::size_t>(m)].data(), &s));
            rep.tie_subspace_sin[static_cast<std::size_t>(m)] = s;
        }
    }
    rep.accuracy_exact = accuracy(reference, exact);
    rep.accuracy_mach = accuracy(reference, approx);
    rep.core_interaction = {exact.core.data()[0], approx.core.data()[0]};
    return rep;
}

// ---- linalg.hpp ----
LeftSingularBasis left_singular_basis(const Matrix& m, int k) {
    if (m.rows() < 1 || m.cols() < 1) throw ArgumentError("matrix must be nonempty");
    if (k < 1 || k > m.rows()) throw ArgumentError("k must satisfy 1 <= k <= rows");
    LeftSingularBasis out;
    out.basis = Matrix(m.rows(), k);
    out.singular_values.assign(static_cast<std::size_t>(k), 0.0);
    int nr = 0, comp = 0;
    rethrow(mach_left_singular_basis(ctx(), m.rows(), m.cols(), m.data(), k, out.basis.data(), out.singular_values.data(),
                                     &nr, &comp));
    out.numerical_rank = nr;
    out.completed = comp != 0;
    return out;
}

TruncatedSvd truncated_svd(const Matrix& m, int k) {
    if (m.rows() < 1 || m.cols() < 1) throw ArgumentError("matrix must be nonempty");
    if (k < 1 || k > std::min(m.rows(), m.cols())) throw ArgumentError("k must satisfy 1 <= k <= min(rows, cols)");
    TruncatedSvd out;
    out.left = Matrix(m.rows(), k);
    out.right = Matrix(m.cols(), k);
    out.singular_values.assign(static_cast<std::size_t>(k), 0.0);
    rethrow(mach_truncated_svd(ctx(), m.rows(), m.cols(), m.data(), k, out.left.data(), out.singular_values.data(),
                               out.right.data()));
    return out;
}

Matrix leading_left_singular_vectors(const Matrix& m, int k) { return truncated_svd(m, k).left; }

Matrix low_rank_approx(const Matrix& m, int k) {
    if (m.rows() < 1 || m.cols() < 1) throw ArgumentError("matrix must be nonempty");
    if (k < 1 || k > std::min(m.rows(), m.cols())) throw ArgumentError("k must satisfy 1 <= k <= min(rows, cols)");
    Matrix out(m.rows(), m.cols());
    rethrow(mach_low_rank_approx(ctx(), m.rows(), m.cols(), m.data(), k, out.data()));
    return out;
}

void set_thread_count(int) {}

}  // namespace mach
