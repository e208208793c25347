// ============================================================================
//  TEST INFRASTRUCTURE ONLY — CPU oracle: the Theorem-1
//  bound (proj/src/bounds.cpp) and the measurement ingest (proj/src/ingest.cpp),
//  restated on top of oracle.cpp's public functions.  Same rules as
//  oracle.hpp: only tests/, smoke() and bench.py's CPU arms may load it.
// ============================================================================
#include "oracle.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <set>
#include <utility>

namespace orc {

namespace {

[[noreturn]] void arg_err(const std::string& m) { throw Error(ErrKind::Argument, m); }

// bounds.cpp:20-35
double min_probability_core(const std::vector<int>& dims) {
    double worst = 0.0;
    for (std::size_t j = 0; j < dims.size(); ++j) {
        double log_sum = 0.0, prod = 1.0;
        for (std::size_t k = 0; k < dims.size(); ++k) {
            if (k == j) continue;
            log_sum += std::log(static_cast<double>(dims[k]));
            prod *= static_cast<double>(dims[k]);
        }
        const double base = 8.0 * log_sum;
        worst = std::max(worst, base * base * base * base / prod);
    }
    return worst;
}

// descending clamped eigenvalues of the symmetrised Gram (bounds.cpp:46-55)
std::vector<double> spectrum_desc(const Mat& gram) {
    const int n = gram.rows;
    Mat sym(n, n);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) sym(i, j) = 0.5 * (gram(i, j) + gram(j, i));
    std::vector<double> ev;
    Mat vec;
    sym_eig(sym, ev, vec);
    std::vector<double> out(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) out[static_cast<std::size_t>(i)] = std::max(0.0, ev[static_cast<std::size_t>(n - 1 - i)]);
    return out;
}

// bounds.cpp:41-56: Gram of the shorter side of the mode unfolding
std::vector<double> dense_mode_spectrum(const Dense& x, int mode) {
    const Mat m = matricize(x, mode);
    const bool rows_side = m.rows <= m.cols;
    const int n = rows_side ? m.rows : m.cols;
    Mat g(n, n);
    if (rows_side) {
        for (int c = 0; c < m.cols; ++c)
            for (int j = 0; j < n; ++j) {
                const double f = m(j, c);
                if (f == 0.0) continue;
                for (int i = 0; i < n; ++i) g(i, j) += m(i, c) * f;
            }
    } else {
        for (int j = 0; j < n; ++j)
            for (int i = 0; i <= j; ++i) {
                double s = 0.0;
                for (int r = 0; r < m.rows; ++r) s += m(r, i) * m(r, j);
                g(i, j) = s;
                g(j, i) = s;
            }
    }
    return spectrum_desc(g);
}

// bounds.cpp:58-66 -> sparse_kernels.cpp:92-101 (sigma = sqrt(max(0, lambda)), squared again)
std::vector<double> sparse_mode_spectrum(const Sparse& t, int mode) {
    const Split s = split_at(t.dims, mode);
    const std::int64_t cols = s.inner * s.outer;
    Mat gram = s.len <= cols ? sparse_row_gram(t, mode) : sparse_col_gram(t, mode, cols);
    std::vector<double> sig2 = spectrum_desc(gram);
    for (double& v : sig2) {
        const double sg = std::sqrt(v);
        v = sg * sg;
    }
    return sig2;
}

struct SplitNorms {
    double lowrank = 0.0, residual = 0.0;
};

// bounds.cpp:75-88: both sums run smallest-first
SplitNorms split_spectrum(const std::vector<double>& sigma2, int r) {
    const int n = static_cast<int>(sigma2.size());
    const int head = std::min(r, n);
    SplitNorms out;
    double acc = 0.0;
    for (int l = n - 1; l >= head; --l) acc += sigma2[static_cast<std::size_t>(l)];
    out.residual = std::sqrt(acc);
    acc = 0.0;
    for (int l = head - 1; l >= 0; --l) acc += sigma2[static_cast<std::size_t>(l)];
    out.lowrank = std::sqrt(acc);
    return out;
}

}  // namespace

struct BoundMode {
    int rank = 0;
    double x_residual = 0, xhat_residual = 0, x_lowrank_norm = 0, t_i = 0;
};
struct Bound {
    double b = 0, p = 0, p_min = 0, t = 0, success_probability = 0;
    bool dims_large_enough = false, dims_balanced = false, p_above_min = false, conditions_met = false;
    std::vector<BoundMode> per_mode;
};

// bounds.cpp:91-116
Bound conditions_core(const std::vector<int>& dims, double p) {
    Bound rep;
    rep.p = p;
    rep.p_min = min_probability_core(dims);
    rep.success_probability = 1.0;
    const int d = static_cast<int>(dims.size());
    for (int i = 0; i < d; ++i) {
        double log_sum = 0.0;
        for (int k = 0; k < d; ++k)
            if (k != i) log_sum += std::log(static_cast<double>(dims[static_cast<std::size_t>(k)]));
        rep.success_probability *= 1.0 - std::exp(-19.0 * log_sum);
    }
    double total = 1.0;
    for (int n : dims) total *= static_cast<double>(n);
    rep.dims_large_enough = true;
    rep.dims_balanced = true;
    for (int n : dims) {
        if (n < 76) rep.dims_large_enough = false;
        if (static_cast<double>(n) * static_cast<double>(n) > total) rep.dims_balanced = false;
    }
    rep.p_above_min = p >= rep.p_min;
    rep.conditions_met = rep.dims_large_enough && rep.dims_balanced && rep.p_above_min;
    return rep;
}

// bounds.cpp:145-150
double min_sampling_probability(const std::vector<int>& dims) {
    if (dims.size() < 2) arg_err("at least two modes required");
    for (int d : dims)
        if (d < 2) arg_err("every dimension must be >= 2");
    return min_probability_core(dims);
}

// bounds.cpp:152-184
Bound theorem1_bound(const Dense& x, const Sparse& xhat, const std::vector<int>& ranks, double p) {
    if (x.dims != xhat.dims) throw Error(ErrKind::Shape, "x and xhat must share dims");
    if (ranks.size() != x.dims.size()) arg_err("ranks must name one rank per mode");
    for (std::size_t m = 0; m < ranks.size(); ++m)
        if (ranks[m] < 1 || ranks[m] > x.dims[m])
            arg_err("rank for mode " + std::to_string(m + 1) + " must be in [1, " + std::to_string(x.dims[m]) + "]");
    if (!(p > 0.0 && p <= 1.0)) arg_err("p must be in (0, 1]");
    const int d = x.order();
    Bound rep = conditions_core(x.dims, p);
    for (double v : x.v) rep.b = std::max(rep.b, std::abs(v));
    rep.per_mode.resize(static_cast<std::size_t>(d));
    for (int i = 0; i < d; ++i) {
        BoundMode& mode = rep.per_mode[static_cast<std::size_t>(i)];
        mode.rank = ranks[static_cast<std::size_t>(i)];
        const SplitNorms xs = split_spectrum(dense_mode_spectrum(x, i), mode.rank);
        mode.x_residual = xs.residual;
        mode.x_lowrank_norm = xs.lowrank;
        mode.xhat_residual = split_spectrum(sparse_mode_spectrum(xhat, i), mode.rank).residual;
    }
    for (int i = 0; i < d; ++i) {
        BoundMode& mode = rep.per_mode[static_cast<std::size_t>(i)];
        double others = 1.0, cross = 0.0;
        for (int j = 0; j < d; ++j) {
            if (j == i) continue;
            others *= static_cast<double>(x.dims[static_cast<std::size_t>(j)]);
            cross += rep.per_mode[static_cast<std::size_t>(j)].xhat_residual;
        }
        const double ratio = static_cast<double>(mode.rank) / p * others;
        mode.t_i = mode.x_residual + 4.0 * rep.b * std::sqrt(ratio) +
                   4.0 * std::sqrt(mode.x_lowrank_norm * rep.b) * std::pow(ratio, 0.25) + cross;
        rep.t = i == 0 ? mode.t_i : std::min(rep.t, mode.t_i);
    }
    return rep;
}

// ---- ingest (proj/src/ingest.cpp:51-135), on pre-indexed records ------------
// The name -> axis-index maps (ingest.cpp:62-67) are string handling and stay
// with the caller; this restates the numeric part: bucket alignment
// (:69-78), order-independent cell means (:90-117: records sorted by (cell,
// value), summed in that order, divided by the count) and the carry-forward
// fill (:119-134).  policy 0 = zero, 1 = carry_forward.
std::int64_t floor_div(std::int64_t a, std::int64_t b) {
    std::int64_t q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
    return q;
}

Dense ingest_indexed(const std::vector<int>& machine, const std::vector<int>& metric, const std::vector<std::int64_t>& ts,
                     const std::vector<double>& value, int n_machines, int n_metrics, std::int64_t bucket_seconds,
                     int policy, std::int64_t* first_bucket_out) {
    if (ts.empty()) arg_err("no records to ingest");
    if (bucket_seconds <= 0) arg_err("time_bucket_seconds must be positive");
    for (double v : value)
        if (!std::isfinite(v)) arg_err("record value is not finite");
    std::int64_t min_ts = ts.front(), max_ts = ts.front();
    for (std::int64_t t : ts) {
        min_ts = std::min(min_ts, t);
        max_ts = std::max(max_ts, t);
    }
    const std::int64_t first_bucket = floor_div(min_ts, bucket_seconds) * bucket_seconds;
    const std::int64_t buckets = floor_div(max_ts - first_bucket, bucket_seconds) + 1;
    if (first_bucket_out) *first_bucket_out = first_bucket;
    Dense out;
    out.dims = {n_machines, n_metrics, static_cast<int>(buckets)};
    out.v.assign(static_cast<std::size_t>(n_machines) * n_metrics * buckets, 0.0);
    std::vector<std::pair<std::int64_t, double>> cells;
    cells.reserve(ts.size());
    for (std::size_t i = 0; i < ts.size(); ++i) {
        const std::int64_t t = floor_div(ts[i] - first_bucket, bucket_seconds);
        cells.emplace_back(machine[i] + static_cast<std::int64_t>(n_machines) * (metric[i] + static_cast<std::int64_t>(n_metrics) * t),
                           value[i]);
    }
    std::sort(cells.begin(), cells.end());
    std::vector<char> filled(out.v.size(), 0);
    for (std::size_t i = 0; i < cells.size();) {
        const std::int64_t cell = cells[i].first;
        double sum = 0.0;
        std::int64_t count = 0;
        while (i < cells.size() && cells[i].first == cell) {
            sum += cells[i++].second;
            ++count;
        }
        out.v[static_cast<std::size_t>(cell)] = sum / static_cast<double>(count);
        filled[static_cast<std::size_t>(cell)] = 1;
    }
    if (policy == 1) {
        for (std::int64_t m = 0; m < n_machines; ++m)
            for (std::int64_t j = 0; j < n_metrics; ++j) {
                double last = 0.0;
                bool seen = false;
                for (std::int64_t t = 0; t < buckets; ++t) {
                    const std::size_t cell = static_cast<std::size_t>(m + n_machines * (j + n_metrics * t));
                    if (filled[cell]) {
                        last = out.v[cell];
                        seen = true;
                    } else if (seen) {
                        out.v[cell] = last;
                    }
                }
            }
    }
    return out;
}

}  // namespace orc

// ---- C entry points (ctypes) -------------------------------------------------
namespace {
thread_local std::string g_err;
thread_local int g_kind = 0;
template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const orc::Error& e) {
        g_err = e.what();
        g_kind = static_cast<int>(e.kind);
        return g_kind;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 99;
    }
}
}  // namespace

extern "C" {

const char* orc_ext_last_error() { return g_err.c_str(); }

// scal[5] = {b, p, p_min, t, success_probability}; flags[4]; per_mode: order x {rank, x_res, xhat_res, x_lowrank, t_i}
int orc_theorem1_bound(void* dense, void* sparse, const int* ranks, double p, double* scal, int* flags, double* per_mode) {
    return guard([&] {
        auto* x = static_cast<orc::Dense*>(dense);
        auto* xh = static_cast<orc::Sparse*>(sparse);
        const orc::Bound r = orc::theorem1_bound(*x, *xh, std::vector<int>(ranks, ranks + x->order()), p);
        scal[0] = r.b; scal[1] = r.p; scal[2] = r.p_min; scal[3] = r.t; scal[4] = r.success_probability;
        flags[0] = r.dims_large_enough; flags[1] = r.dims_balanced; flags[2] = r.p_above_min; flags[3] = r.conditions_met;
        for (std::size_t i = 0; i < r.per_mode.size(); ++i) {
            per_mode[5 * i + 0] = r.per_mode[i].rank;
            per_mode[5 * i + 1] = r.per_mode[i].x_residual;
            per_mode[5 * i + 2] = r.per_mode[i].xhat_residual;
            per_mode[5 * i + 3] = r.per_mode[i].x_lowrank_norm;
            per_mode[5 * i + 4] = r.per_mode[i].t_i;
        }
    });
}

int orc_theorem1_conditions(int order, const int* dims, double p, double* scal, int* flags) {
    return guard([&] {
        const std::vector<int> d(dims, dims + order);
        if (d.size() < 2) throw orc::Error(orc::ErrKind::Argument, "at least two modes required");
        for (int v : d)
            if (v < 2) throw orc::Error(orc::ErrKind::Argument, "every dimension must be >= 2");
        if (!(p > 0.0 && p <= 1.0)) throw orc::Error(orc::ErrKind::Argument, "p must be in (0, 1]");
        const orc::Bound r = orc::conditions_core(d, p);
        scal[0] = r.b; scal[1] = r.p; scal[2] = r.p_min; scal[3] = r.t; scal[4] = r.success_probability;
        flags[0] = r.dims_large_enough; flags[1] = r.dims_balanced; flags[2] = r.p_above_min; flags[3] = r.conditions_met;
    });
}

int orc_min_sampling_probability(int order, const int* dims, double* out) {
    return guard([&] { *out = orc::min_sampling_probability(std::vector<int>(dims, dims + order)); });
}

// out: n_machines * n_metrics * buckets doubles (caller sizes it from orc_ingest_buckets)
long long orc_ingest_buckets(long long n, const long long* ts, long long bucket_seconds, long long* first_bucket) {
    if (n < 1 || bucket_seconds <= 0) return 1;  // orc_ingest_indexed reports the error
    long long mn = ts[0], mx = ts[0];
    for (long long i = 0; i < n; ++i) {
        mn = std::min(mn, ts[i]);
        mx = std::max(mx, ts[i]);
    }
    const long long fb = orc::floor_div(mn, bucket_seconds) * bucket_seconds;
    if (first_bucket) *first_bucket = fb;
    return orc::floor_div(mx - fb, bucket_seconds) + 1;
}

int orc_ingest_indexed(long long n, const int* machine, const int* metric, const long long* ts, const double* value,
                       int n_machines, int n_metrics, long long bucket_seconds, int policy, double* out) {
    return guard([&] {
        std::vector<std::int64_t> t64(ts, ts + n);
        const orc::Dense d = orc::ingest_indexed(std::vector<int>(machine, machine + n), std::vector<int>(metric, metric + n), t64,
                                                 std::vector<double>(value, value + n), n_machines, n_metrics, bucket_seconds,
                                                 policy, nullptr);
        std::memcpy(out, d.v.data(), d.v.size() * sizeof(double));
    });
}

}  // extern "C"
