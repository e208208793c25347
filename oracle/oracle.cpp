// TEST INFRASTRUCTURE ONLY — see oracle.hpp for the scope and pinning notes.
// Restates /root/reference/proj/src/{internal.hpp,tensor.cpp,sampling.cpp,
// sparse_kernels.cpp,linalg.cpp,tucker.cpp} without Eigen.  Citations are
// relative to /root/reference/proj.

#include "oracle.hpp"

#include <algorithm>
#include <cstdlib>
#include <thread>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <random>

namespace orc {

namespace {

// src/internal.hpp:36-46 — cascade summation, base case 64.
template <typename F>
double pairwise_seq(std::int64_t lo, std::int64_t hi, F&& f) {
    const std::int64_t n = hi - lo;
    if (n <= 64) {
        double s = 0.0;
        for (std::int64_t i = lo; i < hi; ++i) s += f(i);
        return s;
    }
    const std::int64_t mid = lo + n / 2;
    return pairwise_seq(lo, mid, f) + pairwise_seq(mid, hi, f);
}

#ifdef ORC_THREADS
// The all-cores build (liboracle_omp.so, the CPU baseline's second line):
// std::thread workers (this image's g++ has no OpenMP runtime) over
// independent outputs; every output is computed by one thread in the serial
// order, so results are bit-identical to the one-thread build.
template <typename Fn>
void parallel_for(std::int64_t n, Fn&& fn) {
    static const int nt = [] {
        const char* e = std::getenv("ORC_THREADS");
        const int v = e ? std::atoi(e) : static_cast<int>(std::thread::hardware_concurrency());
        return v > 0 ? v : 1;
    }();
    const int t = static_cast<int>(std::min<std::int64_t>(nt, n));
    if (t <= 1) {
        for (std::int64_t i = 0; i < n; ++i) fn(i);
        return;
    }
    std::vector<std::thread> th;
    th.reserve(static_cast<std::size_t>(t));
    for (int w = 0; w < t; ++w)
        th.emplace_back([&, w] {
            for (std::int64_t i = w; i < n; i += t) fn(i);  // cyclic: balanced for any work shape
        });
    for (auto& x : th) x.join();
}
// the 2^kParDepth subtrees of the cascade's top levels summed in parallel and
// combined in the reference's order (bit-identical to pairwise_seq)
constexpr int kParDepth = 7;
inline double pairwise_combine(std::int64_t lo, std::int64_t hi, int depth, const std::vector<double>& leaf, std::size_t& k) {
    if (depth == kParDepth || hi - lo <= 64) return leaf[k++];
    const std::int64_t mid = lo + (hi - lo) / 2;
    const double a = pairwise_combine(lo, mid, depth + 1, leaf, k);
    const double b = pairwise_combine(mid, hi, depth + 1, leaf, k);
    return a + b;
}
inline void pairwise_leaves(std::int64_t lo, std::int64_t hi, int depth, std::vector<std::pair<std::int64_t, std::int64_t>>& out) {
    if (depth == kParDepth || hi - lo <= 64) {
        out.emplace_back(lo, hi);
        return;
    }
    const std::int64_t mid = lo + (hi - lo) / 2;
    pairwise_leaves(lo, mid, depth + 1, out);
    pairwise_leaves(mid, hi, depth + 1, out);
}
template <typename F>
double pairwise_sum(std::int64_t lo, std::int64_t hi, F&& f) {
    if (hi - lo < (1 << 16)) return pairwise_seq(lo, hi, f);
    std::vector<std::pair<std::int64_t, std::int64_t>> rg;
    pairwise_leaves(lo, hi, 0, rg);
    std::vector<double> leaf(rg.size());
    parallel_for(static_cast<std::int64_t>(rg.size()), [&](std::int64_t i) { leaf[static_cast<std::size_t>(i)] = pairwise_seq(rg[static_cast<std::size_t>(i)].first, rg[static_cast<std::size_t>(i)].second, f); });
    std::size_t k = 0;
    return pairwise_combine(lo, hi, 0, leaf, k);
}
#else
template <typename Fn>
void parallel_for(std::int64_t n, Fn&& fn) {
    for (std::int64_t i = 0; i < n; ++i) fn(i);
}
template <typename F>
double pairwise_sum(std::int64_t lo, std::int64_t hi, F&& f) {
    return pairwise_seq(lo, hi, f);
}
#endif

[[noreturn]] void arg_error(const std::string& m) { throw Error(ErrKind::Argument, m); }
[[noreturn]] void shape_error(const std::string& m) { throw Error(ErrKind::Shape, m); }
[[noreturn]] void conv_error(const std::string& m, int idx) {
    throw Error(ErrKind::Convergence, m + " (singular index " + std::to_string(idx) + ")", idx);
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

PhaseTimes g_phase;

// ---- tiny dense helpers (stand-ins for the Eigen expressions) --------------
// c = a^T b  (a: n x p, b: n x q)
Mat mul_tn(const Mat& a, const Mat& b) {
    Mat c(a.cols, b.cols);
    for (int j = 0; j < b.cols; ++j)
        for (int i = 0; i < a.cols; ++i) {
            const double* x = a.col(i);
            const double* y = b.col(j);
            double s = 0.0;
            for (int r = 0; r < a.rows; ++r) s += x[r] * y[r];
            c(i, j) = s;
        }
    return c;
}

// c = a b  (a: n x p, b: p x q)
Mat mul_nn(const Mat& a, const Mat& b) {
    Mat c(a.rows, b.cols);
    for (int j = 0; j < b.cols; ++j) {
        double* out = c.col(j);
        for (int k = 0; k < a.cols; ++k) {
            const double f = b(k, j);
            const double* x = a.col(k);
            for (int r = 0; r < a.rows; ++r) out[r] += x[r] * f;
        }
    }
    return c;
}

// c = a a^T
Mat mul_aat(const Mat& a) {
    Mat c(a.rows, a.rows);
    for (int k = 0; k < a.cols; ++k) {
        const double* x = a.col(k);
        for (int j = 0; j < a.rows; ++j) {
            const double f = x[j];
            if (f == 0.0) continue;
            double* out = c.col(j);
            for (int r = 0; r < a.rows; ++r) out[r] += x[r] * f;
        }
    }
    return c;
}

double vnorm(const double* x, int n) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += x[i] * x[i];
    return std::sqrt(s);
}

// v -= B[:, :count] (B[:, :count]^T v)
void project_out(const Mat& b, int count, std::vector<double>& v) {
    if (count <= 0) return;
    std::vector<double> t(static_cast<std::size_t>(count));
    for (int c = 0; c < count; ++c) {
        const double* x = b.col(c);
        double s = 0.0;
        for (int r = 0; r < b.rows; ++r) s += x[r] * v[static_cast<std::size_t>(r)];
        t[static_cast<std::size_t>(c)] = s;
    }
    for (int c = 0; c < count; ++c) {
        const double* x = b.col(c);
        const double f = t[static_cast<std::size_t>(c)];
        for (int r = 0; r < b.rows; ++r) v[static_cast<std::size_t>(r)] -= x[r] * f;
    }
}

// Thin Q (rows x cols) of a Householder QR, Eigen's reflector convention
// (HouseholderQR::householderQ() * Identity(rows, cols), linalg.cpp:144-145).
Mat householder_thin_q(Mat a) {
    const int m = a.rows, n = a.cols;
    const int kmax = std::min(m, n);
    std::vector<double> tau(static_cast<std::size_t>(kmax), 0.0);
    for (int k = 0; k < kmax; ++k) {
        double* x = a.col(k) + k;
        const int len = m - k;
        double tail = 0.0;
        for (int i = 1; i < len; ++i) tail += x[i] * x[i];
        const double c0 = x[0];
        double beta, t;
        if (tail == 0.0) {
            t = 0.0;
            beta = c0;
            for (int i = 1; i < len; ++i) x[i] = 0.0;
        } else {
            beta = std::sqrt(c0 * c0 + tail);
            if (c0 >= 0.0) beta = -beta;
            for (int i = 1; i < len; ++i) x[i] /= (c0 - beta);
            t = (beta - c0) / beta;
        }
        x[0] = beta;
        tau[static_cast<std::size_t>(k)] = t;
        // apply H_k = I - t v v^T (v = [1; x[1:]]) to the trailing columns
        for (int j = k + 1; j < n; ++j) {
            double* y = a.col(j) + k;
            double s = y[0];
            for (int i = 1; i < len; ++i) s += x[i] * y[i];
            s *= t;
            y[0] -= s;
            for (int i = 1; i < len; ++i) y[i] -= s * x[i];
        }
    }
    // Q[:, :n] = H_0 ... H_{kmax-1} I[:, :n]
    Mat q(m, n);
    for (int j = 0; j < n && j < m; ++j) q(j, j) = 1.0;
    for (int k = kmax - 1; k >= 0; --k) {
        const double* x = a.col(k) + k;
        const double t = tau[static_cast<std::size_t>(k)];
        const int len = m - k;
        for (int j = 0; j < n; ++j) {
            double* y = q.col(j) + k;
            double s = y[0];
            for (int i = 1; i < len; ++i) s += x[i] * y[i];
            s *= t;
            y[0] -= s;
            for (int i = 1; i < len; ++i) y[i] -= s * x[i];
        }
    }
    return q;
}

}  // namespace

// ============================================================================
// RNG — src/internal.hpp:68-77 (SplitMix64 output function on a counter).
// ============================================================================
std::uint64_t counter_hash64(std::uint64_t seed, std::uint64_t counter) {
    std::uint64_t z = seed + (counter + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

double counter_uniform01(std::uint64_t seed, std::uint64_t counter) {
    return static_cast<double>(counter_hash64(seed, counter) >> 11) * 0x1.0p-53;
}

// ============================================================================
// Layout — src/tensor.cpp:15-45.
// ============================================================================
std::int64_t checked_size(const std::vector<int>& dims) {
    if (dims.empty()) arg_error("tensor must have at least one mode");
    std::int64_t n = 1;
    for (int d : dims) {
        if (d < 1) arg_error("every dimension must be >= 1");
        if (n > std::numeric_limits<std::int64_t>::max() / d) arg_error("shape product overflows");
        n *= d;
    }
    return n;
}

Split split_at(const std::vector<int>& dims, int mode) {
    if (mode < 0 || mode >= static_cast<int>(dims.size())) arg_error("mode out of range");
    Split s;
    for (int m = 0; m < mode; ++m) s.inner *= dims[static_cast<std::size_t>(m)];
    for (int m = mode + 1; m < static_cast<int>(dims.size()); ++m) s.outer *= dims[static_cast<std::size_t>(m)];
    s.len = dims[static_cast<std::size_t>(mode)];
    return s;
}

std::int64_t Sparse::size() const {
    std::int64_t n = 1;
    for (int d : dims) n *= d;
    return n;
}

// tensor.cpp:60-65
Dense make_dense(std::vector<int> dims, std::vector<double> v) {
    if (static_cast<std::int64_t>(v.size()) != checked_size(dims))
        shape_error("value count does not match shape product");
    for (double x : v)
        if (!std::isfinite(x)) arg_error("tensor values must be finite");
    return Dense{std::move(dims), std::move(v)};
}

// tensor.cpp:78-96 — validate, sort by flat index, merge duplicates by
// summation, drop exact zeros.
Sparse make_sparse(std::vector<int> dims, std::vector<Entry> entries) {
    const std::int64_t total = checked_size(dims);
    for (const auto& e : entries) {
        if (e.index < 0 || e.index >= total) arg_error("sparse entry index out of bounds");
        if (!std::isfinite(e.value)) arg_error("tensor values must be finite");
    }
    std::stable_sort(entries.begin(), entries.end(),
                     [](const Entry& a, const Entry& b) { return a.index < b.index; });
    std::size_t out = 0;
    for (std::size_t i = 0; i < entries.size();) {
        const std::int64_t idx = entries[i].index;
        double sum = 0.0;
        while (i < entries.size() && entries[i].index == idx) sum += entries[i++].value;
        if (sum != 0.0) entries[out++] = {idx, sum};
    }
    entries.resize(out);
    return Sparse{std::move(dims), std::move(entries)};
}

// ============================================================================
// Tensor ops — src/tensor.cpp:149-276.
// ============================================================================
Mat transpose(const Mat& m) {                                   // :149-154
    Mat t(m.cols, m.rows);
    for (int c = 0; c < m.cols; ++c)
        for (int r = 0; r < m.rows; ++r) t(c, r) = m(r, c);
    return t;
}

double frobenius_norm(const Mat& m) {                            // :156-159
    const double* v = m.v.data();
    return std::sqrt(pairwise_sum(0, static_cast<std::int64_t>(m.v.size()),
                                  [v](std::int64_t i) { return v[i] * v[i]; }));
}

double tensor_norm(const Dense& t) {                             // :161-164
    const double* v = t.v.data();
    return std::sqrt(pairwise_sum(0, t.size(), [v](std::int64_t i) { return v[i] * v[i]; }));
}

double tensor_norm(const Sparse& t) {                            // :166-171
    const Entry* e = t.e.data();
    return std::sqrt(pairwise_sum(0, t.nnz(), [e](std::int64_t i) { return e[i].value * e[i].value; }));
}

Mat matricize(const Dense& t, int mode) {                        // :180-200
    const Split s = split_at(t.dims, mode);
    const std::int64_t cols = s.inner * s.outer;
    Mat m(s.len, static_cast<int>(cols));
    if (s.inner == 1) {
        std::memcpy(m.v.data(), t.v.data(), t.v.size() * sizeof(double));
        return m;
    }
    for (std::int64_t c = 0; c < s.outer; ++c) {
        const double* slab = t.v.data() + c * s.inner * s.len;
        for (int r = 0; r < s.len; ++r) {
            const double* row = slab + static_cast<std::int64_t>(r) * s.inner;
            double* out = m.v.data() + r + (c * s.inner) * s.len;
            for (std::int64_t a = 0; a < s.inner; ++a) out[a * s.len] = row[a];
        }
    }
    return m;
}

Dense refold(const Mat& m, int mode, const std::vector<int>& dims) {  // :202-222
    const Split s = split_at(dims, mode);
    if (m.rows != s.len || static_cast<std::int64_t>(m.cols) != s.inner * s.outer)
        shape_error("matrix shape does not match refold target dims");
    Dense t{dims, std::vector<double>(static_cast<std::size_t>(checked_size(dims)), 0.0)};
    if (s.inner == 1) {
        std::memcpy(t.v.data(), m.v.data(), t.v.size() * sizeof(double));
        return t;
    }
    for (std::int64_t c = 0; c < s.outer; ++c) {
        double* slab = t.v.data() + c * s.inner * s.len;
        for (int r = 0; r < s.len; ++r) {
            double* row = slab + static_cast<std::int64_t>(r) * s.inner;
            const double* in = m.v.data() + r + (c * s.inner) * s.len;
            for (std::int64_t a = 0; a < s.inner; ++a) row[a] = in[a * s.len];
        }
    }
    return t;
}

// :224-239 — per outer slab c: dst(inner x J) = slab(inner x len) * m^T.
Dense mode_product(const Dense& t, const Mat& m, int mode) {
    const Split s = split_at(t.dims, mode);
    if (m.cols != s.len) shape_error("mode_product inner dimensions disagree");
    std::vector<int> od = t.dims;
    od[static_cast<std::size_t>(mode)] = m.rows;
    Dense out{od, std::vector<double>(static_cast<std::size_t>(checked_size(od)), 0.0)};
    const int j = m.rows;
    // (c, q) output columns are independent; each is summed in the same order
    // by one thread, so the all-cores build is bit-identical
    parallel_for(s.outer * j, [&](std::int64_t cq) {
        const std::int64_t c = cq / j;
        const int q = static_cast<int>(cq % j);
        const double* slab = t.v.data() + c * s.inner * s.len;
        double* dcol = out.v.data() + c * s.inner * j + static_cast<std::int64_t>(q) * s.inner;
        for (int r = 0; r < s.len; ++r) {
            const double f = m(q, r);
            const double* scol = slab + static_cast<std::int64_t>(r) * s.inner;
            for (std::int64_t a = 0; a < s.inner; ++a) dcol[a] += scol[a] * f;
        }
    });
    return out;
}

// :241-259 — scatter each nonzero into the dense result.
Dense mode_product(const Sparse& t, const Mat& m, int mode) {
    const Split s = split_at(t.dims, mode);
    if (m.cols != s.len) shape_error("mode_product inner dimensions disagree");
    std::vector<int> od = t.dims;
    od[static_cast<std::size_t>(mode)] = m.rows;
    Dense out{od, std::vector<double>(static_cast<std::size_t>(checked_size(od)), 0.0)};
    const int j = m.rows;
    double* o = out.v.data();
    for (const auto& e : t.e) {
        const std::int64_t a = e.index % s.inner;
        const std::int64_t r = (e.index / s.inner) % s.len;
        const std::int64_t c = e.index / (s.inner * s.len);
        const double* mcol = m.v.data() + r * j;
        double* base = o + a + c * s.inner * j;
        for (int q = 0; q < j; ++q) base[q * s.inner] += mcol[q] * e.value;
    }
    return out;
}

Dense densify(const Sparse& s) {                                 // :261-266
    Dense t{s.dims, std::vector<double>(static_cast<std::size_t>(checked_size(s.dims)), 0.0)};
    for (const auto& e : s.e) t.v[static_cast<std::size_t>(e.index)] = e.value;
    return t;
}

Sparse sparsify_exact(const Dense& t) {                          // :268-274
    std::vector<Entry> en;
    for (std::int64_t i = 0; i < t.size(); ++i)
        if (t.v[static_cast<std::size_t>(i)] != 0.0) en.push_back({i, t.v[static_cast<std::size_t>(i)]});
    return make_sparse(t.dims, std::move(en));
}

// ============================================================================
// Sampler — src/sampling.cpp:15-31.
// ============================================================================
Sparse sparsify(const Dense& t, double p, std::uint64_t seed) {
    if (!(p > 0.0 && p <= 1.0)) arg_error("p must be in (0, 1]");
    std::vector<Entry> kept;
    const double* v = t.v.data();
    for (std::int64_t i = 0; i < t.size(); ++i) {
        if (v[i] == 0.0) continue;
        if (counter_uniform01(seed, static_cast<std::uint64_t>(i)) < p) kept.push_back({i, v[i] / p});
    }
    return make_sparse(t.dims, std::move(kept));
}

// ============================================================================
// Symmetric eigendecomposition (stand-in for Eigen::SelfAdjointEigenSolver,
// used at src/linalg.cpp:108): Householder tridiagonalisation followed by the
// implicit QL iteration with eigenvector accumulation (EISPACK tred2/tql2
// algorithm class).  Eigenvalues ascending, eigenvectors in columns.
// ============================================================================
void sym_eig(const Mat& a, std::vector<double>& evals, Mat& evecs) {
    const int n = a.rows;
    if (a.cols != n) shape_error("sym_eig needs a square matrix");
    // V row-major scratch: V[i][j] = w[i*n + j]
    std::vector<double> w(static_cast<std::size_t>(n) * n);
    auto V = [&](int i, int j) -> double& { return w[static_cast<std::size_t>(i) * n + j]; };
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) V(i, j) = a(i, j);
    std::vector<double> d(static_cast<std::size_t>(n)), e(static_cast<std::size_t>(n));
    if (n == 1) {
        evals.assign(1, a(0, 0));
        evecs = Mat(1, 1);
        evecs(0, 0) = 1.0;
        return;
    }
    // --- tridiagonalise (lower triangle used) ---
    for (int j = 0; j < n; ++j) d[j] = V(n - 1, j);
    for (int i = n - 1; i > 0; --i) {
        double scale = 0.0, h = 0.0;
        for (int k = 0; k < i; ++k) scale += std::abs(d[k]);
        if (scale == 0.0) {
            e[i] = d[i - 1];
            for (int j = 0; j < i; ++j) {
                d[j] = V(i - 1, j);
                V(i, j) = 0.0;
                V(j, i) = 0.0;
            }
        } else {
            for (int k = 0; k < i; ++k) {
                d[k] /= scale;
                h += d[k] * d[k];
            }
            double f = d[i - 1];
            double g = std::sqrt(h);
            if (f > 0) g = -g;
            e[i] = scale * g;
            h -= f * g;
            d[i - 1] = f - g;
            for (int j = 0; j < i; ++j) e[j] = 0.0;
            for (int j = 0; j < i; ++j) {
                f = d[j];
                V(j, i) = f;
                g = e[j] + V(j, j) * f;
                for (int k = j + 1; k <= i - 1; ++k) {
                    g += V(k, j) * d[k];
                    e[k] += V(k, j) * f;
                }
                e[j] = g;
            }
            f = 0.0;
            for (int j = 0; j < i; ++j) {
                e[j] /= h;
                f += e[j] * d[j];
            }
            const double hh = f / (h + h);
            for (int j = 0; j < i; ++j) e[j] -= hh * d[j];
            for (int j = 0; j < i; ++j) {
                f = d[j];
                g = e[j];
                for (int k = j; k <= i - 1; ++k) V(k, j) -= (f * e[k] + g * d[k]);
                d[j] = V(i - 1, j);
                V(i, j) = 0.0;
            }
        }
        d[i] = h;
    }
    // accumulate the transformations
    for (int i = 0; i < n - 1; ++i) {
        V(n - 1, i) = V(i, i);
        V(i, i) = 1.0;
        const double h = d[i + 1];
        if (h != 0.0) {
            for (int k = 0; k <= i; ++k) d[k] = V(k, i + 1) / h;
            for (int j = 0; j <= i; ++j) {
                double g = 0.0;
                for (int k = 0; k <= i; ++k) g += V(k, i + 1) * V(k, j);
                for (int k = 0; k <= i; ++k) V(k, j) -= g * d[k];
            }
        }
        for (int k = 0; k <= i; ++k) V(k, i + 1) = 0.0;
    }
    for (int j = 0; j < n; ++j) {
        d[j] = V(n - 1, j);
        V(n - 1, j) = 0.0;
    }
    V(n - 1, n - 1) = 1.0;
    e[0] = 0.0;

    // --- implicit QL on the tridiagonal ---
    for (int i = 1; i < n; ++i) e[i - 1] = e[i];
    e[n - 1] = 0.0;
    double f = 0.0, tst1 = 0.0;
    const double eps = std::ldexp(1.0, -52);
    for (int l = 0; l < n; ++l) {
        tst1 = std::max(tst1, std::abs(d[l]) + std::abs(e[l]));
        int m = l;
        while (m < n) {
            if (std::abs(e[m]) <= eps * tst1) break;
            ++m;
        }
        if (m == n) m = n - 1;
        if (m > l) {
            int iter = 0;
            do {
                if (++iter > 60) conv_error("symmetric eigendecomposition failed", 1);
                double g = d[l];
                double p = (d[l + 1] - g) / (2.0 * e[l]);
                double r = std::hypot(p, 1.0);
                if (p < 0) r = -r;
                d[l] = e[l] / (p + r);
                d[l + 1] = e[l] * (p + r);
                const double dl1 = d[l + 1];
                double h = g - d[l];
                for (int i = l + 2; i < n; ++i) d[i] -= h;
                f += h;
                p = d[m];
                double c = 1.0, c2 = c, c3 = c;
                const double el1 = e[l + 1];
                double s = 0.0, s2 = 0.0;
                for (int i = m - 1; i >= l; --i) {
                    c3 = c2;
                    c2 = c;
                    s2 = s;
                    g = c * e[i];
                    h = c * p;
                    r = std::hypot(p, e[i]);
                    e[i + 1] = s * r;
                    s = e[i] / r;
                    c = p / r;
                    p = c * d[i] - s * g;
                    d[i + 1] = h + s * (c * g + s * d[i]);
                    for (int k = 0; k < n; ++k) {
                        h = V(k, i + 1);
                        V(k, i + 1) = s * V(k, i) + c * h;
                        V(k, i) = c * V(k, i) - s * h;
                    }
                }
                p = -s * s2 * c3 * el1 * e[l] / dl1;
                e[l] = s * p;
                d[l] = c * p;
            } while (std::abs(e[l]) > eps * tst1);
        }
        d[l] += f;
        e[l] = 0.0;
    }
    // sort ascending
    std::vector<int> ord(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) ord[i] = i;
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return d[x] < d[y]; });
    evals.resize(static_cast<std::size_t>(n));
    evecs = Mat(n, n);
    for (int j = 0; j < n; ++j) {
        evals[static_cast<std::size_t>(j)] = d[ord[j]];
        for (int i = 0; i < n; ++i) evecs(i, j) = V(i, ord[j]);
    }
}

// ============================================================================
// Eigen step — src/linalg.cpp:18-357, constants src/linalg_internal.hpp:13-23.
// ============================================================================
namespace {

constexpr int kGramPathLimit = 512;
constexpr int kOversample = 8;
constexpr int kMaxSubspaceIters = 300;
constexpr double kSubspaceTol = 1e-10;
constexpr double kDeficiencyFloor = 1e-10;
constexpr double kRankFloor = 1e-6;
constexpr std::uint64_t kSubspaceSeed = 0x4D414348u;
constexpr double kCollapseFloor = 1e-3;

// linalg.cpp:18-32
double canonical_sign(double* u, int n) {
    int pivot = 0;
    double best = std::abs(u[0]);
    for (int i = 1; i < n; ++i)
        if (std::abs(u[i]) > best) {
            best = std::abs(u[i]);
            pivot = i;
        }
    if (u[pivot] < 0.0) {
        for (int i = 0; i < n; ++i) u[i] = -u[i];
        return -1.0;
    }
    return 1.0;
}

// linalg.cpp:41-51
std::vector<double> completion_column(const Mat& basis, int count) {
    const int n = basis.rows;
    for (int e = 0; e < n; ++e) {
        std::vector<double> v(static_cast<std::size_t>(n), 0.0);
        v[static_cast<std::size_t>(e)] = 1.0;
        for (int pass = 0; pass < 2; ++pass) project_out(basis, count, v);
        const double nv = vnorm(v.data(), n);
        if (nv > 0.5) {
            for (double& x : v) x /= nv;
            return v;
        }
    }
    conv_error("orthonormal completion found no free direction", count + 1);
}

struct Ortho {
    Mat basis;
    std::vector<double> flips;
    std::vector<bool> backed;
    int numerical_rank = 0;
    bool completed = false;
};

// linalg.cpp:66-100
Ortho orthonormal_columns(const Mat& w, int k, double sigma1, bool canonicalize) {
    Ortho out;
    out.basis = Mat(w.rows, k);
    out.flips.assign(static_cast<std::size_t>(k), 1.0);
    out.backed.assign(static_cast<std::size_t>(k), false);
    const double floor = sigma1 * kRankFloor;
    for (int i = 0; i < k; ++i) {
        bool data_backed = false;
        if (i < w.cols) {
            std::vector<double> v(w.col(i), w.col(i) + w.rows);
            const double nv = vnorm(v.data(), w.rows);
            if (nv > floor) {
                for (int pass = 0; pass < 2; ++pass)
                    if (i > 0) project_out(out.basis, i, v);
                const double res = vnorm(v.data(), w.rows);
                if (res > kCollapseFloor * nv) {
                    for (int r = 0; r < w.rows; ++r) out.basis(r, i) = v[static_cast<std::size_t>(r)] / res;
                    data_backed = true;
                }
            }
        }
        if (!data_backed) {
            const auto c = completion_column(out.basis, i);
            std::copy(c.begin(), c.end(), out.basis.col(i));
            out.completed = true;
        } else {
            out.backed[static_cast<std::size_t>(i)] = true;
            ++out.numerical_rank;
        }
        if (canonicalize) out.flips[static_cast<std::size_t>(i)] = canonical_sign(out.basis.col(i), w.rows);
    }
    return out;
}

struct Side {
    Mat vectors;
    std::vector<double> sigma;
};

// linalg.cpp:106-120
Side gram_side_basis(const Mat& gram, int k) {
    const int n = gram.rows;
    Mat sym(n, n);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) sym(i, j) = 0.5 * (gram(i, j) + gram(j, i));
    std::vector<double> ev;
    Mat vec;
    sym_eig(sym, ev, vec);
    Side out;
    out.vectors = Mat(n, k);
    out.sigma.resize(static_cast<std::size_t>(k));
    for (int i = 0; i < k; ++i) {
        std::copy(vec.col(n - 1 - i), vec.col(n - 1 - i) + n, out.vectors.col(i));
        out.sigma[static_cast<std::size_t>(i)] = std::sqrt(std::max(0.0, ev[static_cast<std::size_t>(n - 1 - i)]));
    }
    return out;
}

// linalg.cpp:128-193
Side subspace_side_basis(const Mat& a, bool side_is_rows, int k) {
    const int side = side_is_rows ? a.rows : a.cols;
    const int block = std::min(k + kOversample, side);
    const Mat at = transpose(a);
    auto apply = [&](const Mat& q) {
        if (side_is_rows) return mul_nn(a, mul_nn(at, q));
        return mul_nn(at, mul_nn(a, q));
    };
    Mat q(side, block);
    for (int c = 0; c < block; ++c)
        for (int r = 0; r < side; ++r)
            q(r, c) = 2.0 * counter_uniform01(kSubspaceSeed, static_cast<std::uint64_t>(c) * side +
                                                                  static_cast<std::uint64_t>(r)) - 1.0;
    q = householder_thin_q(q);
    Mat prev;
    for (int iter = 0; iter < kMaxSubspaceIters; ++iter) {
        Mat z = apply(q);
        Mat t = mul_tn(q, z);
        Mat ts(block, block);
        for (int j = 0; j < block; ++j)
            for (int i = 0; i < block; ++i) ts(i, j) = 0.5 * (t(i, j) + t(j, i));
        std::vector<double> ev;
        Mat vec;
        sym_eig(ts, ev, vec);
        Mat sel(block, k);
        std::vector<double> theta(static_cast<std::size_t>(k));
        for (int i = 0; i < k; ++i) {
            std::copy(vec.col(block - 1 - i), vec.col(block - 1 - i) + block, sel.col(i));
            theta[static_cast<std::size_t>(i)] = ev[static_cast<std::size_t>(block - 1 - i)];
        }
        Mat ritz = mul_nn(q, sel);
        const double theta_floor = theta[0] * kDeficiencyFloor * kDeficiencyFloor;
        if (!prev.v.empty()) {
            bool converged = true;
            for (int i = 0; i < k && converged; ++i) {
                if (theta[static_cast<std::size_t>(i)] <= theta_floor) continue;
                std::vector<double> r(prev.col(i), prev.col(i) + side);
                project_out(ritz, k, r);
                if (vnorm(r.data(), side) > kSubspaceTol) converged = false;
            }
            if (converged) {
                Side out;
                out.vectors = std::move(ritz);
                out.sigma.resize(static_cast<std::size_t>(k));
                for (int i = 0; i < k; ++i)
                    out.sigma[static_cast<std::size_t>(i)] = std::sqrt(std::max(0.0, theta[static_cast<std::size_t>(i)]));
                return out;
            }
        }
        prev = std::move(ritz);
        if (iter + 1 < kMaxSubspaceIters) q = householder_thin_q(z);
    }
    for (int i = 0; i < k; ++i) {
        std::vector<double> r(prev.col(i), prev.col(i) + side);
        project_out(q, q.cols, r);
        if (vnorm(r.data(), side) > kSubspaceTol) conv_error("subspace iteration did not converge", i + 1);
    }
    conv_error("subspace iteration did not converge", k);
}

// linalg.cpp:261-276
Basis basis_from_side(Side side, int k) {
    Basis out;
    const double sigma1 = side.sigma.empty() ? 0.0 : side.sigma[0];
    out.sv.assign(static_cast<std::size_t>(k), 0.0);
    while (out.numerical_rank < k && side.sigma[static_cast<std::size_t>(out.numerical_rank)] > sigma1 * kRankFloor)
        ++out.numerical_rank;
    for (int i = 0; i < out.numerical_rank; ++i) {
        canonical_sign(side.vectors.col(i), side.vectors.rows);
        out.sv[static_cast<std::size_t>(i)] = side.sigma[static_cast<std::size_t>(i)];
    }
    for (int i = out.numerical_rank; i < k; ++i) {
        const auto c = completion_column(side.vectors, i);
        std::copy(c.begin(), c.end(), side.vectors.col(i));
    }
    out.completed = out.numerical_rank < k;
    out.basis = std::move(side.vectors);
    return out;
}

// linalg.cpp:278-281
Basis basis_from_row_gram(const Mat& gram, int k) {
    if (k < 1 || k > gram.rows) arg_error("k must satisfy 1 <= k <= rows");
    return basis_from_side(gram_side_basis(gram, k), k);
}

// linalg.cpp:283-296
Basis basis_from_products(const Mat& w, const std::vector<double>& sigma, int k, double sigma1) {
    if (k < 1 || k > w.rows) arg_error("k must satisfy 1 <= k <= rows");
    Ortho cols = orthonormal_columns(w, k, sigma1, true);
    Basis out;
    out.basis = std::move(cols.basis);
    out.sv.assign(static_cast<std::size_t>(k), 0.0);
    for (int i = 0; i < k && i < static_cast<int>(sigma.size()); ++i)
        if (cols.backed[static_cast<std::size_t>(i)]) out.sv[static_cast<std::size_t>(i)] = sigma[static_cast<std::size_t>(i)];
    out.numerical_rank = cols.numerical_rank;
    out.completed = cols.completed;
    return out;
}

// linalg.cpp:196-214
void check_svd_args(const Mat& m, int k) {
    if (m.rows < 1 || m.cols < 1) arg_error("matrix must be nonempty");
    if (k < 1 || k > std::min(m.rows, m.cols)) arg_error("k must satisfy 1 <= k <= min(rows, cols)");
}

Svd zero_matrix_svd(int rows, int cols, int k) {
    Svd out;
    out.left = Mat(rows, k);
    out.right = Mat(cols, k);
    for (int i = 0; i < k; ++i) {
        out.left(i, i) = 1.0;
        out.right(i, i) = 1.0;
    }
    out.sv.assign(static_cast<std::size_t>(k), 0.0);
    return out;
}

// linalg.cpp:218-241
Svd assemble_svd(const Mat& a, bool side_is_rows, Side side, int k) {
    const double sigma1 = side.sigma.empty() ? 0.0 : side.sigma[0];
    Svd out;
    out.sv.assign(side.sigma.begin(), side.sigma.begin() + k);
    if (side_is_rows) {
        for (int i = 0; i < k; ++i) canonical_sign(side.vectors.col(i), side.vectors.rows);
        Mat w = mul_tn(a, side.vectors);
        Ortho right = orthonormal_columns(w, k, sigma1, false);
        out.left = std::move(side.vectors);
        out.right = std::move(right.basis);
    } else {
        Mat w = mul_nn(a, side.vectors);
        Ortho left = orthonormal_columns(w, k, sigma1, true);
        for (int i = 0; i < k; ++i)
            if (left.flips[static_cast<std::size_t>(i)] < 0)
                for (int r = 0; r < side.vectors.rows; ++r) side.vectors(r, i) = -side.vectors(r, i);
        out.left = std::move(left.basis);
        out.right = std::move(side.vectors);
    }
    return out;
}

Svd truncated_svd_gram(const Mat& m, int k) {                    // :245-253
    check_svd_args(m, k);
    if (frobenius_norm(m) == 0.0) return zero_matrix_svd(m.rows, m.cols, k);
    const bool rows_side = m.rows <= m.cols;
    Mat gram = rows_side ? mul_aat(m) : mul_tn(m, m);
    return assemble_svd(m, rows_side, gram_side_basis(gram, k), k);
}

Svd truncated_svd_subspace(const Mat& m, int k) {                // :255-263
    check_svd_args(m, k);
    if (frobenius_norm(m) == 0.0) return zero_matrix_svd(m.rows, m.cols, k);
    const bool rows_side = m.rows <= m.cols;
    const int side = std::min(m.rows, m.cols);
    if (k + kOversample >= side) return truncated_svd_gram(m, k);
    return assemble_svd(m, rows_side, subspace_side_basis(m, rows_side, k), k);
}

}  // namespace

Svd truncated_svd(const Mat& m, int k) {                         // linalg.cpp:301-305
    check_svd_args(m, k);
    if (std::min(m.rows, m.cols) <= kGramPathLimit) return truncated_svd_gram(m, k);
    return truncated_svd_subspace(m, k);
}

Mat low_rank_approx(const Mat& m, int k) {                       // linalg.cpp:311-317
    Svd s = truncated_svd(m, k);
    Mat out(m.rows, m.cols);
    for (int i = 0; i < k; ++i)
        for (int c = 0; c < m.cols; ++c) {
            const double f = s.sv[static_cast<std::size_t>(i)] * s.right(c, i);
            for (int r = 0; r < m.rows; ++r) out(r, c) += s.left(r, i) * f;
        }
    return out;
}

// linalg.cpp:319-353
Basis left_singular_basis(const Mat& m, int k) {
    if (m.rows < 1 || m.cols < 1) arg_error("matrix must be nonempty");
    if (k < 1 || k > m.rows) arg_error("k must satisfy 1 <= k <= rows");
    if (frobenius_norm(m) == 0.0) {
        Basis out;
        out.basis = Mat(m.rows, k);
        for (int i = 0; i < k; ++i) out.basis(i, i) = 1.0;
        out.sv.assign(static_cast<std::size_t>(k), 0.0);
        out.numerical_rank = 0;
        out.completed = true;
        return out;
    }
    if (m.rows <= m.cols && k <= m.cols) {
        if (m.rows <= kGramPathLimit || k + kOversample >= m.rows) return basis_from_row_gram(mul_aat(m), k);
        return basis_from_side(subspace_side_basis(m, true, k), k);
    }
    const int kc = std::min(k, m.cols);
    Side side;
    if (m.cols <= kGramPathLimit || kc + kOversample >= m.cols)
        side = gram_side_basis(mul_tn(m, m), kc);
    else
        side = subspace_side_basis(m, false, kc);
    Mat w = mul_nn(m, side.vectors);
    return basis_from_products(w, side.sigma, k, side.sigma[0]);
}

// ============================================================================
// Sparse kernels — src/sparse_kernels.cpp:15-101.
// ============================================================================
namespace {

struct Triple {
    std::int64_t major, minor;
    double value;
};

// :21-39
std::vector<Triple> matricization_triples(const Sparse& t, int mode, bool by_column) {
    const Split s = split_at(t.dims, mode);
    std::vector<Triple> tr;
    tr.reserve(t.e.size());
    for (const auto& e : t.e) {
        const std::int64_t a = e.index % s.inner;
        const std::int64_t rest = e.index / s.inner;
        const std::int64_t row = rest % s.len;
        const std::int64_t col = a + (rest / s.len) * s.inner;
        if (by_column) tr.push_back({col, row, e.value});
        else tr.push_back({row, col, e.value});
    }
    std::sort(tr.begin(), tr.end(), [](const Triple& x, const Triple& y) {
        return x.major != y.major ? x.major < y.major : x.minor < y.minor;
    });
    return tr;
}

// :43-56
Mat bucket_gram(const std::vector<Triple>& tr, std::int64_t n) {
    Mat g(static_cast<int>(n), static_cast<int>(n));
    std::size_t i = 0;
    while (i < tr.size()) {
        std::size_t j = i;
        while (j < tr.size() && tr[j].major == tr[i].major) ++j;
        for (std::size_t x = i; x < j; ++x)
            for (std::size_t y = i; y <= x; ++y)
                g(static_cast<int>(tr[y].minor), static_cast<int>(tr[x].minor)) += tr[y].value * tr[x].value;
        i = j;
    }
    for (int c = 0; c < g.cols; ++c)
        for (int r = c + 1; r < g.rows; ++r) g(r, c) = g(c, r);
    return g;
}

// :69-80
Mat sparse_matricization_times(const Sparse& t, int mode, const Mat& v) {
    const Split s = split_at(t.dims, mode);
    Mat w(s.len, v.cols);
    for (const auto& e : t.e) {
        const std::int64_t a = e.index % s.inner;
        const std::int64_t rest = e.index / s.inner;
        const std::int64_t col = a + (rest / s.len) * s.inner;
        const int row = static_cast<int>(rest % s.len);
        for (int c = 0; c < v.cols; ++c) w(row, c) += e.value * v(static_cast<int>(col), c);
    }
    return w;
}

}  // namespace

Mat sparse_row_gram(const Sparse& t, int mode) {
    const Split s = split_at(t.dims, mode);
    return bucket_gram(matricization_triples(t, mode, true), s.len);
}

Mat sparse_col_gram(const Sparse& t, int mode, std::int64_t cols) {
    return bucket_gram(matricization_triples(t, mode, false), cols);
}

Basis sparse_mode_basis(const Sparse& t, int mode, int k) {
    const Split s = split_at(t.dims, mode);
    const std::int64_t cols = s.inner * s.outer;
    if (s.len <= cols) return basis_from_row_gram(sparse_row_gram(t, mode), k);
    const int kc = static_cast<int>(std::min<std::int64_t>(k, cols));
    Side side = gram_side_basis(sparse_col_gram(t, mode, cols), kc);
    Mat w = sparse_matricization_times(t, mode, side.vectors);
    return basis_from_products(w, side.sigma, k, side.sigma[0]);
}

// ============================================================================
// Tucker — src/tucker.cpp:18-217.
// ============================================================================
namespace {

void check_ranks(const std::vector<int>& dims, const std::vector<int>& ranks) {   // :20-27
    if (ranks.size() != dims.size()) arg_error("ranks must name one rank per mode");
    for (std::size_t m = 0; m < dims.size(); ++m)
        if (ranks[m] < 1 || ranks[m] > dims[m])
            arg_error("rank for mode " + std::to_string(m + 1) + " must be in [1, " +
                      std::to_string(dims[m]) + "]");
}

void check_hooi_config(int max_iterations, double tol) {                            // :29-32
    if (max_iterations < 1) arg_error("max_iterations must be >= 1");
    if (!(tol >= 0.0)) arg_error("fit_tolerance must be >= 0");
}

std::string completion_warning(int mode, int nr, int requested) {                  // :34-38
    return "mode " + std::to_string(mode + 1) + " matricization has numerical rank " +
           std::to_string(nr) + " below requested rank " + std::to_string(requested) +
           "; remaining directions were basis-completed";
}

double residual_norm(const Dense& t, const Dense& rec) {                           // :40-45
    const double* a = t.v.data();
    const double* b = rec.v.data();
    return std::sqrt(pairwise_sum(0, t.size(), [a, b](std::int64_t i) { return (a[i] - b[i]) * (a[i] - b[i]); }));
}

double model_fit(const Dense& t, double norm_t, const Model& model) {              // :51-54
    if (norm_t == 0.0) return 1.0;
    return 1.0 - residual_norm(t, reconstruct(model)) / norm_t;
}

double model_fit(const Sparse& t, double norm_t, const Model& model) {             // :56-64
    if (norm_t == 0.0) return 1.0;
    Dense diff = reconstruct(model);
    double* b = diff.v.data();
    for (const auto& e : t.e) b[e.index] -= e.value;
    const double err = std::sqrt(pairwise_sum(0, diff.size(), [b](std::int64_t i) { return b[i] * b[i]; }));
    return 1.0 - err / norm_t;
}

constexpr double kDensifyThreshold = 0.25;                                          // :69

Dense sparse_core(const Sparse& t, const std::vector<Mat>& f) {                    // :71-75
    Dense y = mode_product(t, transpose(f[0]), 0);
    for (int m = 1; m < t.order(); ++m) y = mode_product(y, transpose(f[static_cast<std::size_t>(m)]), m);
    return y;
}

Dense project_except(const Dense& t, const std::vector<Mat>& f, int skip) {        // :109-118
    Dense y;
    bool first = true;
    for (int m = 0; m < t.order(); ++m) {
        if (m == skip) continue;
        y = mode_product(first ? t : y, transpose(f[static_cast<std::size_t>(m)]), m);
        first = false;
    }
    return first ? t : y;
}

Dense project_except(const Sparse& t, const std::vector<Mat>& f, int skip) {       // :120-131
    const int d = t.order();
    const int first_mode = skip == 0 ? 1 : 0;
    if (d == 1) return densify(t);
    Dense y = mode_product(t, transpose(f[static_cast<std::size_t>(first_mode)]), first_mode);
    for (int m = first_mode + 1; m < d; ++m) {
        if (m == skip) continue;
        y = mode_product(y, transpose(f[static_cast<std::size_t>(m)]), m);
    }
    return y;
}

// :80-106
template <typename T, typename P, typename C>
Model hooi_loop(const T& t, const std::vector<int>& ranks, int max_it, double tol, Model init,
                P&& project, C&& core_of) {
    const double norm_t = tensor_norm(t);
    Model model = std::move(init);
    model.sweep_fits.assign(1, model.fit);
    model.iterations = 0;
    double prev_fit = model.fit;
    g_phase.sweeps.clear();
    for (int sweep = 1; sweep <= max_it; ++sweep) {
        const double t0 = now_s();
        std::vector<std::string> warnings;
        for (int i = 0; i < t.order(); ++i) {
            Dense y = project(model.factors, i);
            Basis b = left_singular_basis(matricize(y, i), ranks[static_cast<std::size_t>(i)]);
            if (b.completed) warnings.push_back(completion_warning(i, b.numerical_rank, ranks[static_cast<std::size_t>(i)]));
            model.factors[static_cast<std::size_t>(i)] = std::move(b.basis);
        }
        model.core = core_of(model.factors);
        model.fit = model_fit(t, norm_t, model);
        model.sweep_fits.push_back(model.fit);
        model.iterations = sweep;
        model.warnings = std::move(warnings);
        g_phase.sweeps.push_back(now_s() - t0);
        if (model.fit - prev_fit < tol) break;
        prev_fit = model.fit;
    }
    return model;
}

}  // namespace

Model hosvd(const Dense& t, const std::vector<int>& ranks) {                        // :135-150
    check_ranks(t.dims, ranks);
    Model model;
    model.ranks = ranks;
    for (int m = 0; m < t.order(); ++m) {
        Basis b = left_singular_basis(matricize(t, m), ranks[static_cast<std::size_t>(m)]);
        if (b.completed) model.warnings.push_back(completion_warning(m, b.numerical_rank, ranks[static_cast<std::size_t>(m)]));
        model.factors.push_back(std::move(b.basis));
    }
    model.core = core_tensor(t, model.factors);
    model.fit = model_fit(t, tensor_norm(t), model);
    model.sweep_fits.assign(1, model.fit);
    return model;
}

Model hosvd(const Sparse& t, const std::vector<int>& ranks) {                       // :152-169
    check_ranks(t.dims, ranks);
    if (static_cast<double>(t.nnz()) >= kDensifyThreshold * static_cast<double>(t.size()))
        return hosvd(densify(t), ranks);
    Model model;
    model.ranks = ranks;
    for (int m = 0; m < t.order(); ++m) {
        Basis b = sparse_mode_basis(t, m, ranks[static_cast<std::size_t>(m)]);
        if (b.completed) model.warnings.push_back(completion_warning(m, b.numerical_rank, ranks[static_cast<std::size_t>(m)]));
        model.factors.push_back(std::move(b.basis));
    }
    model.core = sparse_core(t, model.factors);
    model.fit = model_fit(t, tensor_norm(t), model);
    model.sweep_fits.assign(1, model.fit);
    return model;
}

Model hooi(const Dense& t, const std::vector<int>& ranks, int max_it, double tol) {  // :171-180
    check_ranks(t.dims, ranks);
    check_hooi_config(max_it, tol);
    const double t0 = now_s();
    Model init = hosvd(t, ranks);
    g_phase.hosvd = now_s() - t0;
    return hooi_loop(
        t, ranks, max_it, tol, std::move(init),
        [&](const std::vector<Mat>& f, int skip) { return project_except(t, f, skip); },
        [&](const std::vector<Mat>& f) { return core_tensor(t, f); });
}

Model hooi(const Sparse& t, const std::vector<int>& ranks, int max_it, double tol) { // :182-193
    check_ranks(t.dims, ranks);
    check_hooi_config(max_it, tol);
    if (static_cast<double>(t.nnz()) >= kDensifyThreshold * static_cast<double>(t.size()))
        return hooi(densify(t), ranks, max_it, tol);
    const double t0 = now_s();
    Model init = hosvd(t, ranks);
    g_phase.hosvd = now_s() - t0;
    return hooi_loop(
        t, ranks, max_it, tol, std::move(init),
        [&](const std::vector<Mat>& f, int skip) { return project_except(t, f, skip); },
        [&](const std::vector<Mat>& f) { return sparse_core(t, f); });
}

Dense core_tensor(const Dense& t, const std::vector<Mat>& factors) {               // :195-202
    if (static_cast<int>(factors.size()) != t.order()) arg_error("one factor per mode required");
    Dense y = t;
    for (int m = 0; m < t.order(); ++m) y = mode_product(y, transpose(factors[static_cast<std::size_t>(m)]), m);
    return y;
}

Dense reconstruct(const Model& model) {                                             // :204-209
    Dense y = model.core;
    for (int m = 0; m < model.core.order(); ++m) y = mode_product(y, model.factors[static_cast<std::size_t>(m)], m);
    return y;
}

double accuracy(const Dense& t, const Model& model) {                               // :211-217
    const double norm_t = tensor_norm(t);
    if (norm_t == 0.0) arg_error("accuracy needs a reference tensor with nonzero norm");
    Dense rec = reconstruct(model);
    if (rec.dims != t.dims) shape_error("model reconstructs to a different shape");
    return 1.0 - residual_norm(t, rec) / norm_t;
}

// src/sampling.cpp:33-47
MachResult mach_hosvd(const Dense& t, const std::vector<int>& ranks, double p, std::uint64_t seed) {
    MachResult r;
    r.sparsified = sparsify(t, p, seed);
    r.model = hosvd(r.sparsified, ranks);
    return r;
}

MachResult mach_hooi(const Dense& t, const std::vector<int>& ranks, double p, std::uint64_t seed,
                     int max_it, double tol) {
    MachResult r;
    const double t0 = now_s();
    r.sparsified = sparsify(t, p, seed);
    const double ts = now_s() - t0;
    r.model = hooi(r.sparsified, ranks, max_it, tol);
    g_phase.sample = ts;
    return r;
}

PhaseTimes& last_phase_times() { return g_phase; }

// ============================================================================
// Fixtures — proj/tests/oracles.hpp:111-262 (libstdc++ random streams).
// ============================================================================
Dense random_tensor(const std::vector<int>& dims, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> dist(0.0, 1.0);
    std::int64_t n = 1;
    for (int d : dims) n *= d;
    std::vector<double> v(static_cast<std::size_t>(n));
    for (auto& x : v) x = dist(rng);
    return make_dense(dims, std::move(v));
}

Mat random_matrix(int rows, int cols, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> dist(0.0, 1.0);
    Mat m(rows, cols);
    for (auto& x : m.v) x = dist(rng);
    return m;
}

Mat random_orthogonal(int n, std::uint64_t seed) {
    Mat m = random_matrix(n, n, seed);
    for (int c = 0; c < n; ++c) {
        for (int prev = 0; prev < c; ++prev) {
            double dot = 0.0;
            for (int r = 0; r < n; ++r) dot += m(r, c) * m(r, prev);
            for (int r = 0; r < n; ++r) m(r, c) -= dot * m(r, prev);
        }
        double nrm = 0.0;
        for (int r = 0; r < n; ++r) nrm += m(r, c) * m(r, c);
        nrm = std::sqrt(nrm);
        for (int r = 0; r < n; ++r) m(r, c) /= nrm;
    }
    return m;
}

void jacobi_eig(const Mat& in, std::vector<double>& evals, Mat& evecs) {
    const int n = in.rows;
    std::vector<std::vector<double>> a(static_cast<std::size_t>(n), std::vector<double>(static_cast<std::size_t>(n)));
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) a[i][j] = in(i, j);
    std::vector<std::vector<double>> v(static_cast<std::size_t>(n), std::vector<double>(static_cast<std::size_t>(n), 0.0));
    for (int i = 0; i < n; ++i) v[i][i] = 1.0;
    for (int sweep = 0; sweep < 200; ++sweep) {
        double off = 0.0;
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) off += a[p][q] * a[p][q];
        if (std::sqrt(off) < 1e-14 * (1.0 + std::abs(a[0][0]))) break;
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) {
                if (a[p][q] == 0.0) continue;
                const double theta = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
                const double t = (theta >= 0.0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0);
                const double s = t * c;
                for (int k = 0; k < n; ++k) {
                    const double akp = a[k][p], akq = a[k][q];
                    a[k][p] = c * akp - s * akq;
                    a[k][q] = s * akp + c * akq;
                }
                for (int k = 0; k < n; ++k) {
                    const double apk = a[p][k], aqk = a[q][k];
                    a[p][k] = c * apk - s * aqk;
                    a[q][k] = s * apk + c * aqk;
                }
                for (int k = 0; k < n; ++k) {
                    const double vkp = v[k][p], vkq = v[k][q];
                    v[k][p] = c * vkp - s * vkq;
                    v[k][q] = s * vkp + c * vkq;
                }
            }
    }
    std::vector<int> order(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](int x, int y) { return a[x][x] > a[y][y]; });
    evals.resize(static_cast<std::size_t>(n));
    evecs = Mat(n, n);
    for (int k = 0; k < n; ++k) {
        evals[static_cast<std::size_t>(k)] = a[order[k]][order[k]];
        for (int i = 0; i < n; ++i) evecs(i, k) = v[i][order[k]];
    }
}

double subspace_gap(const Mat& a, const Mat& b) {
    const int n = a.rows, k = a.cols;
    Mat c = mul_tn(b, a);
    Mat res = a;
    for (int j = 0; j < k; ++j)
        for (int l = 0; l < k; ++l) {
            const double f = c(l, j);
            for (int r = 0; r < n; ++r) res(r, j) -= b(r, l) * f;
        }
    Mat g = mul_tn(res, res);
    std::vector<double> ev;
    Mat vec;
    jacobi_eig(g, ev, vec);
    return std::sqrt(std::max(0.0, ev.front()));
}

// ============================================================================
// Metrics — src/metrics.cpp:15-159.
// ============================================================================
namespace {
constexpr double kTieGap = 1e-6;  // metrics.cpp:19

void check_models(const Model& a, const Model& b) {  // :21-31
    if (a.factors.size() != b.factors.size())
        shape_error("models have orders " + std::to_string(a.factors.size()) + " and " + std::to_string(b.factors.size()));
    for (std::size_t m = 0; m < a.factors.size(); ++m)
        if (a.factors[m].rows != b.factors[m].rows)
            shape_error("mode " + std::to_string(m + 1) + " has " + std::to_string(a.factors[m].rows) +
                        " rows in one model and " + std::to_string(b.factors[m].rows) + " in the other");
}

std::vector<double> core_slice_norms(const Dense& core, int mode) {  // :40-50
    std::int64_t stride = 1;
    for (int m = 0; m < mode; ++m) stride *= core.dims[static_cast<std::size_t>(m)];
    const std::int64_t len = core.dims[static_cast<std::size_t>(mode)];
    std::vector<double> sq(static_cast<std::size_t>(len), 0.0);
    for (std::int64_t i = 0; i < core.size(); ++i) sq[static_cast<std::size_t>((i / stride) % len)] += core.v[static_cast<std::size_t>(i)] * core.v[static_cast<std::size_t>(i)];
    for (double& v : sq) v = std::sqrt(v);
    return sq;
}

bool top_two_tied(std::vector<double> n) {  // :52-56
    if (n.size() < 2) return false;
    std::sort(n.begin(), n.end(), std::greater<>());
    return n[0] - n[1] <= kTieGap * n[0];
}

Mat left_cols(const Mat& a, int r) {
    Mat out(a.rows, r);
    for (int c = 0; c < r; ++c)
        for (int i = 0; i < a.rows; ++i) out(i, c) = a(i, c);
    return out;
}
}  // namespace

double pearson(const std::vector<double>& x, const std::vector<double>& y) {
    if (x.size() != y.size())
        shape_error("correlation inputs have lengths " + std::to_string(x.size()) + " and " + std::to_string(y.size()));
    const std::int64_t n = static_cast<std::int64_t>(x.size());
    if (n < 2) arg_error("correlation needs at least 2 samples");
    const bool xc = std::all_of(x.begin(), x.end(), [&](double v) { return v == x[0]; });
    const bool yc = std::all_of(y.begin(), y.end(), [&](double v) { return v == y[0]; });
    if (xc || yc) arg_error("correlation is undefined for a zero-variance input");
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
    if (sxx == 0.0 || syy == 0.0) arg_error("correlation is undefined for a zero-variance input");
    return sxy / std::sqrt(sxx * syy);
}

double pc_correlation(const Model& exact, const Model& approx, int mode, int component, bool* flipped) {
    check_models(exact, approx);
    const int d = static_cast<int>(exact.factors.size());
    if (mode < 0 || mode >= d) arg_error("mode " + std::to_string(mode + 1) + " out of range for order " + std::to_string(d));
    const int limit = std::min(exact.ranks[static_cast<std::size_t>(mode)], approx.ranks[static_cast<std::size_t>(mode)]);
    if (component < 1 || component > limit)
        arg_error("component " + std::to_string(component) + " out of range; mode " + std::to_string(mode + 1) +
                  " has at most " + std::to_string(limit) + " shared components");
    const Mat& fa = exact.factors[static_cast<std::size_t>(mode)];
    const Mat& fb = approx.factors[static_cast<std::size_t>(mode)];
    std::vector<double> a(fa.col(component - 1), fa.col(component - 1) + fa.rows);
    std::vector<double> b(fb.col(component - 1), fb.col(component - 1) + fb.rows);
    const double dot = pairwise_sum(0, static_cast<std::int64_t>(a.size()),
                                    [&](std::int64_t i) { return a[static_cast<std::size_t>(i)] * b[static_cast<std::size_t>(i)]; });
    const bool flip = dot < 0.0;
    if (flipped) *flipped = flip;
    if (flip)
        for (double& v : b) v = -v;
    return pearson(a, b);
}

Report compare(const Model& exact, const Model& approx, const Dense& reference) {
    check_models(exact, approx);
    const int d = static_cast<int>(exact.factors.size());
    if (reference.order() != d)
        shape_error("reference has order " + std::to_string(reference.order()) + ", models have order " + std::to_string(d));
    for (int m = 0; m < d; ++m)
        if (reference.dims[static_cast<std::size_t>(m)] != exact.factors[static_cast<std::size_t>(m)].rows)
            shape_error("mode " + std::to_string(m + 1) + " has " + std::to_string(reference.dims[static_cast<std::size_t>(m)]) +
                        " entries in the reference and " + std::to_string(exact.factors[static_cast<std::size_t>(m)].rows) +
                        " in the models");
    Report r;
    r.rho.resize(static_cast<std::size_t>(d));
    r.flipped.assign(static_cast<std::size_t>(d), false);
    r.tied.assign(static_cast<std::size_t>(d), false);
    r.tie_sin.assign(static_cast<std::size_t>(d), 0.0);
    for (int m = 0; m < d; ++m) {
        bool flip = false;
        r.rho[static_cast<std::size_t>(m)] = pc_correlation(exact, approx, m, 1, &flip);
        r.flipped[static_cast<std::size_t>(m)] = flip;
        if (top_two_tied(core_slice_norms(exact.core, m)) || top_two_tied(core_slice_norms(approx.core, m))) {
            r.tied[static_cast<std::size_t>(m)] = true;
            const int rk = std::min(exact.ranks[static_cast<std::size_t>(m)], approx.ranks[static_cast<std::size_t>(m)]);
            r.tie_sin[static_cast<std::size_t>(m)] = subspace_gap(left_cols(exact.factors[static_cast<std::size_t>(m)], rk),
                                                                  left_cols(approx.factors[static_cast<std::size_t>(m)], rk));
        }
    }
    r.accuracy_exact = accuracy(reference, exact);
    r.accuracy_mach = accuracy(reference, approx);
    r.core_exact = exact.core.v[0];
    r.core_mach = approx.core.v[0];
    return r;
}

}  // namespace orc
