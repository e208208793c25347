// C++ drop-in: bounds.hpp, ingest.hpp (+ StreamingIngest)
// and tensor_io.hpp mirrors over the C ABI.  Text parsing / rendering and the
// name -> axis maps are host work; the spectra, the cell means, the sampling
// and the decompositions run on the B200.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <map>
#include <set>
#include <sstream>
#include <string_view>

#include "mach/bounds.hpp"
#include "mach/errors.hpp"
#include "mach/ingest.hpp"
#include "mach/tensor_io.hpp"
#include "mach_b200.h"

namespace mach {

namespace b200 {
mach_ctx* context();
void check(mach_status st);
}  // namespace b200

namespace {

using b200::check;
using b200::context;

struct DenseDev {
    mach_dense* h = nullptr;
    explicit DenseDev(const DenseTensor& t) {
        check(mach_dense_upload(context(), MACH_F64, t.order(), t.dims().data(), t.data(), &h));
    }
    ~DenseDev() { mach_dense_free(h); }
};

struct SparseDev {
    mach_sparse* h = nullptr;
    explicit SparseDev(const SparseTensor& t) {
        const std::size_t n = static_cast<std::size_t>(t.nnz());
        std::vector<std::int64_t> idx(n);
        std::vector<double> val(n);
        for (std::size_t i = 0; i < n; ++i) {
            idx[i] = t.entries()[i].index;
            val[i] = t.entries()[i].value;
        }
        check(mach_sparse_upload(context(), MACH_F64, t.order(), t.dims().data(), t.nnz(), idx.data(), val.data(), &h));
    }
    explicit SparseDev(mach_sparse* p) : h(p) {}
    ~SparseDev() { mach_sparse_free(h); }
};

SparseTensor sparse_value(const mach_sparse* s, std::vector<int> dims) {
    std::int64_t nnz = 0;
    check(mach_sparse_nnz(s, &nnz));
    std::vector<std::int64_t> idx(static_cast<std::size_t>(nnz));
    std::vector<double> val(static_cast<std::size_t>(nnz));
    check(mach_sparse_download(s, idx.data(), val.data()));
    std::vector<SparseEntry> e(idx.size());
    for (std::size_t i = 0; i < e.size(); ++i) e[i] = {idx[i], val[i]};
    return SparseTensor::from_canonical(std::move(dims), std::move(e));
}

TuckerModel model_value(mach_model* m) {
    int order = 0, iters = 0, nfits = 0, nwarn = 0;
    double fit = 0;
    check(mach_model_info(m, &order, &iters, &fit, &nfits, &nwarn));
    std::vector<int> dims(static_cast<std::size_t>(order)), ranks(static_cast<std::size_t>(order));
    check(mach_model_dims(m, dims.data(), ranks.data()));
    TuckerModel out;
    std::size_t cn = 1;
    for (int r : ranks) cn *= static_cast<std::size_t>(r);
    std::vector<double> core(cn);
    check(mach_model_core(m, core.data()));
    out.core = DenseTensor(ranks, std::move(core));
    for (int q = 0; q < order; ++q) {
        Matrix f(dims[static_cast<std::size_t>(q)], ranks[static_cast<std::size_t>(q)]);
        check(mach_model_factor(m, q, f.data()));
        out.factors.push_back(std::move(f));
    }
    out.ranks = ranks;
    out.iterations = iters;
    out.fit = fit;
    out.sweep_fits.resize(static_cast<std::size_t>(nfits));
    check(mach_model_sweep_fits(m, out.sweep_fits.data()));
    for (int i = 0; i < nwarn; ++i) {
        char buf[512];
        check(mach_model_warning(m, i, buf, sizeof buf));
        out.warnings.emplace_back(buf);
    }
    mach_model_free(m);
    return out;
}

BoundReport report_value(const mach_bound_report& r) {
    BoundReport out;
    out.b = r.b;
    out.p = r.p;
    out.p_min = r.p_min;
    out.t = r.t;
    out.success_probability = r.success_probability;
    out.dims_large_enough = r.dims_large_enough != 0;
    out.dims_balanced = r.dims_balanced != 0;
    out.p_above_min = r.p_above_min != 0;
    out.conditions_met = r.conditions_met != 0;
    return out;
}

}  // namespace

namespace b200 {  // shared with cli.cpp
TuckerModel model_from_handle(mach_model* m) { return model_value(m); }
SparseTensor sparse_from_handle(const mach_sparse* s, std::vector<int> dims) { return sparse_value(s, std::move(dims)); }
}  // namespace b200

// ---- bounds.hpp -------------------------------------------------------------
AchlioptasBounds achlioptas_bounds(double b, std::int64_t n, std::int64_t k, double p) {
    AchlioptasBounds out;
    check(mach_achlioptas_bounds(b, n, k, p, &out.two_norm, &out.frobenius));
    return out;
}

double min_sampling_probability(const std::vector<int>& dims) {
    double out = 0.0;
    check(mach_min_sampling_probability(static_cast<int>(dims.size()), dims.data(), &out));
    return out;
}

BoundReport theorem1_conditions(const std::vector<int>& dims, double p) {
    mach_bound_report r{};
    check(mach_theorem1_conditions(static_cast<int>(dims.size()), dims.data(), p, &r));
    return report_value(r);
}

BoundReport theorem1_bound(const DenseTensor& x, const SparseTensor& xhat, const std::vector<int>& ranks, double p) {
    if (x.dims() != xhat.dims()) throw ShapeError("x and xhat must share dims");
    if (ranks.size() != x.dims().size()) throw ArgumentError("ranks must name one rank per mode");
    DenseDev xd(x);
    SparseDev sd(xhat);
    mach_bound_report r{};
    std::vector<mach_bound_mode> modes(x.dims().size());
    check(mach_theorem1_bound(context(), xd.h, sd.h, ranks.data(), p, &r, modes.data()));
    BoundReport out = report_value(r);
    for (const mach_bound_mode& m : modes) out.per_mode.push_back({m.rank, m.x_residual, m.xhat_residual, m.x_lowrank_norm, m.t_i});
    return out;
}

// ---- ingest.hpp -------------------------------------------------------------
namespace {

std::int64_t floor_quot(std::int64_t a, std::int64_t b) {
    const std::int64_t q = a / b, r = a % b;
    return (r != 0 && ((r < 0) != (b < 0))) ? q - 1 : q;
}

std::map<std::string, int> axis_map(const std::vector<std::string>& names, const char* what) {
    std::map<std::string, int> out;
    for (std::size_t i = 0; i < names.size(); ++i)
        if (!out.emplace(names[i], static_cast<int>(i)).second)
            throw ArgumentError(std::string(what) + " ordering repeats '" + names[i] + "'");
    return out;
}

void valid_name(const std::string& name, const char* what) {
    if (name.empty()) throw ArgumentError(std::string(what) + " must be nonempty");
    if (name.find_first_of(",\n\r") != std::string::npos)
        throw ArgumentError(std::string(what) + " '" + name + "' may not contain commas or line breaks");
}

struct Indexed {
    std::vector<std::int32_t> machine, metric, tick;
    std::vector<double> value;
};

// records -> axis indices and bucket numbers relative to `origin`; every bucket must land in [0, buckets)
Indexed index_records(const std::vector<MeasurementRecord>& records, const std::map<std::string, int>& mi,
                      const std::map<std::string, int>& ji, std::int64_t origin, std::int64_t width, std::int64_t buckets) {
    Indexed out;
    out.machine.reserve(records.size());
    out.metric.reserve(records.size());
    out.tick.reserve(records.size());
    out.value.reserve(records.size());
    for (const MeasurementRecord& r : records) {
        if (!std::isfinite(r.value))
            throw ArgumentError("record value for machine '" + r.machine_id + "' metric '" + r.metric + "' is not finite");
        const auto m = mi.find(r.machine_id);
        if (m == mi.end()) throw ArgumentError("unknown machine '" + r.machine_id + "'");
        const auto j = ji.find(r.metric);
        if (j == ji.end()) throw ArgumentError("unknown metric '" + r.metric + "'");
        const std::int64_t t = floor_quot(r.timestamp - origin, width);
        if (t < 0 || t >= buckets) throw ArgumentError("record timestamp " + std::to_string(r.timestamp) + " falls outside the window");
        out.machine.push_back(m->second);
        out.metric.push_back(j->second);
        out.tick.push_back(static_cast<std::int32_t>(t));
        out.value.push_back(r.value);
    }
    return out;
}

std::vector<std::string> names_seen(const std::vector<MeasurementRecord>& records, std::string MeasurementRecord::*field) {
    std::set<std::string> s;
    for (const MeasurementRecord& r : records) s.insert(r.*field);
    return {s.begin(), s.end()};
}

struct StreamDev {
    mach_stream* h = nullptr;
    StreamDev(const std::vector<int>& dims, double p, std::uint64_t seed) {
        check(mach_stream_begin(context(), MACH_F64, static_cast<int>(dims.size()), dims.data(), p, seed, &h));
    }
    ~StreamDev() { mach_stream_free(h); }
};

}  // namespace

IngestResult ingest(const std::vector<MeasurementRecord>& records, const TensorBuildSpec& spec) {
    if (records.empty()) throw ArgumentError("no records to ingest");
    if (spec.time_bucket_seconds <= 0) throw ArgumentError("time_bucket_seconds must be positive");
    IngestResult out;
    out.machines = spec.machine_order.empty() ? names_seen(records, &MeasurementRecord::machine_id) : spec.machine_order;
    out.metrics = spec.metric_order.empty() ? names_seen(records, &MeasurementRecord::metric) : spec.metric_order;
    const auto mi = axis_map(out.machines, "machine");
    const auto ji = axis_map(out.metrics, "metric");
    std::int64_t lo = records.front().timestamp, hi = lo;
    for (const MeasurementRecord& r : records) {
        lo = std::min(lo, r.timestamp);
        hi = std::max(hi, r.timestamp);
    }
    const std::int64_t w = spec.time_bucket_seconds;
    const std::int64_t origin = floor_quot(lo, w) * w;
    const std::int64_t buckets = floor_quot(hi - origin, w) + 1;
    if (buckets > 0x7fffffffll) throw ArgumentError("time range spans too many buckets");
    const Indexed ix = index_records(records, mi, ji, origin, w, buckets);
    const std::vector<int> dims{static_cast<int>(out.machines.size()), static_cast<int>(out.metrics.size()),
                                static_cast<int>(buckets)};
    // one window holding every bucket: the device forms the cell means and the fill
    StreamDev st(dims, 1.0, 0);
    check(mach_stream_append_records(st.h, static_cast<std::int64_t>(ix.value.size()), ix.machine.data(), ix.metric.data(),
                                     ix.tick.data(), ix.value.data(), dims[2],
                                     spec.missing_policy == MissingPolicy::carry_forward ? 1 : 0));
    mach_dense* slab = nullptr;
    check(mach_stream_last_slab(st.h, &slab));
    std::vector<double> v(static_cast<std::size_t>(dims[0]) * dims[1] * dims[2]);
    const mach_status rc = mach_dense_download(slab, v.data());
    mach_dense_free(slab);
    check(rc);
    out.tensor = DenseTensor(dims, std::move(v));
    out.bucket_starts.resize(static_cast<std::size_t>(buckets));
    for (std::int64_t t = 0; t < buckets; ++t) out.bucket_starts[static_cast<std::size_t>(t)] = origin + t * w;
    return out;
}

struct StreamingIngest::Impl {
    std::vector<std::string> machines, metrics;
    std::map<std::string, int> mi, ji;
    std::int64_t origin = 0, width = 300;
    MissingPolicy policy = MissingPolicy::zero;
    std::vector<int> dims;
    std::unique_ptr<StreamDev> dev;
};

StreamingIngest::StreamingIngest(std::vector<std::string> machines, std::vector<std::string> metrics,
                                 std::int64_t first_bucket_start, std::int64_t time_bucket_seconds, int capacity_buckets,
                                 MissingPolicy policy, const SparsifyConfig& cfg)
    : impl_(std::make_unique<Impl>()) {
    if (machines.empty() || metrics.empty()) throw ArgumentError("machine and metric orderings must be nonempty");
    if (time_bucket_seconds <= 0) throw ArgumentError("time_bucket_seconds must be positive");
    if (capacity_buckets < 1) throw ArgumentError("capacity_buckets must be >= 1");
    impl_->mi = axis_map(machines, "machine");
    impl_->ji = axis_map(metrics, "metric");
    impl_->machines = std::move(machines);
    impl_->metrics = std::move(metrics);
    impl_->origin = first_bucket_start;
    impl_->width = time_bucket_seconds;
    impl_->policy = policy;
    impl_->dims = {static_cast<int>(impl_->machines.size()), static_cast<int>(impl_->metrics.size()), capacity_buckets};
    impl_->dev = std::make_unique<StreamDev>(impl_->dims, cfg.p, cfg.seed);
}

StreamingIngest::~StreamingIngest() = default;

void StreamingIngest::append_window(const std::vector<MeasurementRecord>& records, int buckets) {
    if (buckets < 0) throw ArgumentError("buckets must be >= 0");
    const std::int64_t seen = this->buckets();
    const Indexed ix = index_records(records, impl_->mi, impl_->ji, impl_->origin + seen * impl_->width, impl_->width, buckets);
    check(mach_stream_append_records(impl_->dev->h, static_cast<std::int64_t>(ix.value.size()), ix.machine.data(),
                                     ix.metric.data(), ix.tick.data(), ix.value.data(), buckets,
                                     impl_->policy == MissingPolicy::carry_forward ? 1 : 0));
}

std::int64_t StreamingIngest::buckets() const {
    std::int64_t t = 0;
    check(mach_stream_state(impl_->dev->h, &t, nullptr));
    return t;
}

std::int64_t StreamingIngest::nnz() const {
    std::int64_t z = 0;
    check(mach_stream_state(impl_->dev->h, nullptr, &z));
    return z;
}

SparseTensor StreamingIngest::sampled() const {
    mach_sparse* s = nullptr;
    check(mach_stream_tensor(impl_->dev->h, &s));
    SparseDev own(s);
    std::vector<int> dims = impl_->dims;
    dims[2] = static_cast<int>(buckets());
    return sparse_value(s, dims);
}

TuckerModel StreamingIngest::hooi(const std::vector<int>& ranks, const HooiConfig& cfg) const {
    if (ranks.size() != 3) throw ArgumentError("ranks must name one rank per mode");
    mach_sparse* s = nullptr;
    check(mach_stream_tensor(impl_->dev->h, &s));
    SparseDev own(s);
    mach_model* m = nullptr;
    check(mach_hooi_sparse(context(), s, ranks.data(), cfg.max_iterations, cfg.fit_tolerance, &m));
    return model_value(m);
}

// ---- text formats (tensor_io.hpp; ingest.hpp's CSV) ---------------------------
namespace {

// line-oriented reader that keeps the 1-based line number for ParseError
class Lines {
public:
    explicit Lines(const std::string& path) : in_(path) {
        if (!in_) throw IoError("cannot open '" + path + "' for reading");
    }
    bool next(std::string& line) {
        if (!std::getline(in_, line)) return false;
        ++no_;
        if (!line.empty() && line.back() == '\r') line.pop_back();
        return true;
    }
    long no() const { return no_; }

private:
    std::ifstream in_;
    long no_ = 0;
};

template <typename F>
void each_token(std::string_view line, F&& f) {
    std::size_t i = 0;
    while (i < line.size()) {
        while (i < line.size() && (line[i] == ' ' || line[i] == '\t')) ++i;
        const std::size_t b = i;
        while (i < line.size() && line[i] != ' ' && line[i] != '\t') ++i;
        if (i > b) f(line.substr(b, i - b));
    }
}

std::vector<std::string_view> split_ws(std::string_view line) {
    std::vector<std::string_view> out;
    each_token(line, [&](std::string_view t) { out.push_back(t); });
    return out;
}

std::int64_t to_int(std::string_view tok, long line) {
    std::int64_t v = 0;
    const auto r = std::from_chars(tok.data(), tok.data() + tok.size(), v);
    if (r.ec != std::errc{} || r.ptr != tok.data() + tok.size()) throw ParseError("bad integer '" + std::string(tok) + "'", line);
    return v;
}

double to_value(std::string_view tok, long line) {
    double v = 0.0;
    const auto r = std::from_chars(tok.data(), tok.data() + tok.size(), v);
    if (r.ec != std::errc{} || r.ptr != tok.data() + tok.size()) throw ParseError("bad value '" + std::string(tok) + "'", line);
    if (!std::isfinite(v)) throw ParseError("value '" + std::string(tok) + "' is not finite", line);
    return v;
}

std::vector<int> header_dims(std::string_view rest, long line) {
    std::vector<int> dims;
    std::int64_t total = 1;
    each_token(rest, [&](std::string_view t) {
        const std::int64_t v = to_int(t, line);
        if (v < 1) throw ParseError("dimensions must be positive", line);
        if (v > std::numeric_limits<int>::max() || total > std::numeric_limits<std::int64_t>::max() / v)
            throw ParseError("dimensions overflow", line);
        total *= v;
        dims.push_back(static_cast<int>(v));
    });
    if (dims.empty()) throw ParseError("header lists no dimensions", line);
    return dims;
}

struct Out {
    std::ofstream f;
    std::string path;
    explicit Out(const std::string& p) : f(p), path(p) {
        if (!f) throw IoError("cannot open '" + p + "' for writing");
    }
    void done() {
        f.flush();
        if (!f) throw IoError("failed writing '" + path + "'");
    }
};

void dense_text(Out& o, const std::vector<int>& dims, const double* v, std::int64_t n) {
    o.f << "dims:";
    for (int d : dims) o.f << ' ' << d;
    o.f << '\n';
    const std::int64_t fibre = dims[0];
    for (std::int64_t i = 0; i < n; ++i) {
        o.f << format_double(v[i]) << (((i + 1) % fibre == 0) ? '\n' : ' ');
    }
}

bool is_binary_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open '" + path + "' for reading");
    char magic[8] = {};
    in.read(magic, 8);
    static const char want[8] = {'M', 'A', 'C', 'H', 'B', '2', 0, 0};
    return in.gcount() == 8 && std::memcmp(magic, want, 8) == 0;
}

bool binary_suffix(const std::string& path) { return path.size() >= 6 && path.compare(path.size() - 6, 6, ".machb") == 0; }

AnyTensor read_binary(const std::string& path) {
    int kind = 0, order = 0, dims8[8] = {};
    mach_dtype dt = MACH_F64;
    std::int64_t count = 0;
    check(mach_tensor_file_kind(path.c_str(), &kind, &dt, &order, dims8, &count));
    std::vector<int> dims(dims8, dims8 + order);
    if (kind == 1) {
        mach_sparse* s = nullptr;
        check(mach_sparse_load(context(), path.c_str(), &s));
        SparseDev own(s);
        return sparse_value(s, dims);
    }
    mach_dense* d = nullptr;
    check(mach_dense_load(context(), path.c_str(), &d));
    std::vector<double> v(static_cast<std::size_t>(count));
    mach_status rc = MACH_OK;
    if (dt == MACH_F64) {
        rc = mach_dense_download(d, v.data());
    } else {
        std::vector<float> f(static_cast<std::size_t>(count));
        rc = mach_dense_download(d, f.data());
        std::copy(f.begin(), f.end(), v.begin());
    }
    mach_dense_free(d);
    check(rc);
    return DenseTensor(dims, std::move(v));
}

}  // namespace

std::string format_double(double v) {
    char buf[40];
    const auto r = std::to_chars(buf, buf + sizeof buf, v);
    return std::string(buf, r.ptr);
}

AnyTensor read_tensor(const std::string& path) {
    if (is_binary_file(path)) return read_binary(path);
    Lines in(path);
    std::string line;
    if (!in.next(line)) throw ParseError("missing header", 1);
    std::string_view head(line);
    const bool sparse = head.starts_with("sparse dims:");
    if (sparse) head.remove_prefix(12);
    else if (head.starts_with("dims:")) head.remove_prefix(5);
    else throw ParseError("expected 'dims:' or 'sparse dims:' header", 1);
    const std::vector<int> dims = header_dims(head, 1);
    std::int64_t total = 1;
    for (int d : dims) total *= d;
    if (sparse) {
        std::vector<std::pair<std::vector<int>, double>> entries;
        while (in.next(line)) {
            const auto toks = split_ws(line);
            if (toks.empty()) continue;
            if (toks.size() != dims.size() + 1)
                throw ParseError("expected " + std::to_string(dims.size()) + " indices and a value, got " +
                                     std::to_string(toks.size()) + " tokens", in.no());
            std::vector<int> idx(dims.size());
            for (std::size_t m = 0; m < dims.size(); ++m) {
                const std::int64_t v = to_int(toks[m], in.no());
                if (v < 1 || v > dims[m])
                    throw ParseError("index " + std::to_string(v) + " outside [1, " + std::to_string(dims[m]) + "]", in.no());
                idx[m] = static_cast<int>(v - 1);
            }
            entries.emplace_back(std::move(idx), to_value(toks.back(), in.no()));
        }
        return SparseTensor(dims, entries);
    }
    std::vector<double> values;
    values.reserve(static_cast<std::size_t>(total));
    while (in.next(line))
        each_token(line, [&](std::string_view t) {
            if (static_cast<std::int64_t>(values.size()) == total)
                throw ParseError("more than " + std::to_string(total) + " values", in.no());
            values.push_back(to_value(t, in.no()));
        });
    if (static_cast<std::int64_t>(values.size()) != total)
        throw ParseError("expected " + std::to_string(total) + " values, found " + std::to_string(values.size()),
                         in.no() == 0 ? 1 : in.no());
    return DenseTensor(dims, std::move(values));
}

void write_tensor(const DenseTensor& t, const std::string& path) {
    if (t.order() < 1) throw ArgumentError("cannot serialize an order-0 tensor");
    if (binary_suffix(path)) {
        DenseDev d(t);
        check(mach_dense_save(d.h, path.c_str()));
        return;
    }
    Out o(path);
    dense_text(o, t.dims(), t.data(), t.size());
    o.done();
}

void write_tensor(const SparseTensor& t, const std::string& path) {
    if (t.order() < 1) throw ArgumentError("cannot serialize an order-0 tensor");
    if (binary_suffix(path)) {
        SparseDev s(t);
        check(mach_sparse_save(s.h, path.c_str()));
        return;
    }
    Out o(path);
    o.f << "sparse dims:";
    for (int d : t.dims()) o.f << ' ' << d;
    o.f << '\n';
    for (const SparseEntry& e : t.entries()) {
        for (int i : t.multi_index(e.index)) o.f << i + 1 << ' ';
        o.f << format_double(e.value) << '\n';
    }
    o.done();
}

Matrix read_matrix(const std::string& path) {
    AnyTensor t = read_tensor(path);
    const DenseTensor* d = std::get_if<DenseTensor>(&t);
    if (!d || d->order() != 2) throw ParseError("expected an order-2 dense tensor file at '" + path + "'", 1);
    return Matrix(d->dim(0), d->dim(1), d->values());
}

void write_matrix(const Matrix& m, const std::string& path) {
    Out o(path);
    dense_text(o, {m.rows(), m.cols()}, m.data(), m.size());
    o.done();
}

void save_model(const TuckerModel& model, const std::string& dir) {
    std::error_code ec;
    std::filesystem::create_directories(dir, ec);
    if (ec) throw IoError("cannot create directory '" + dir + "': " + ec.message());
    write_tensor(model.core, dir + "/core");
    for (std::size_t m = 0; m < model.factors.size(); ++m) write_matrix(model.factors[m], dir + "/factor_" + std::to_string(m + 1));
    Out o(dir + "/metadata");
    o.f << "ranks:";
    for (int r : model.ranks) o.f << ' ' << r;
    o.f << "\niterations: " << model.iterations << "\nfit: " << format_double(model.fit) << "\nsweep_fits:";
    for (double f : model.sweep_fits) o.f << ' ' << format_double(f);
    o.f << '\n';
    for (const std::string& w : model.warnings) o.f << "warning: " << w << '\n';
    o.done();
}

TuckerModel load_model(const std::string& dir) {
    const std::string meta = dir + "/metadata";
    Lines in(meta);
    std::string line;
    TuckerModel model;
    auto field = [&](const char* key) -> std::vector<std::string_view> {
        if (!in.next(line)) throw ParseError(std::string("missing '") + key + "' line", in.no() + 1);
        std::string_view v(line);
        if (!v.starts_with(key)) throw ParseError(std::string("expected '") + key + "' line", in.no());
        v.remove_prefix(std::strlen(key));
        return split_ws(v);
    };
    auto one = [&](const char* key) -> std::string_view {
        const auto toks = field(key);
        if (toks.size() != 1) throw ParseError(std::string("expected one value after '") + key + "'", in.no());
        return toks[0];
    };
    for (std::string_view t : field("ranks:")) {
        const std::int64_t r = to_int(t, in.no());
        if (r < 1) throw ParseError("ranks must be positive", in.no());
        model.ranks.push_back(static_cast<int>(r));
    }
    if (model.ranks.empty()) throw ParseError("ranks line lists no ranks", in.no());
    model.iterations = static_cast<int>(to_int(one("iterations:"), in.no()));
    model.fit = to_value(one("fit:"), in.no());
    for (std::string_view t : field("sweep_fits:")) model.sweep_fits.push_back(to_value(t, in.no()));
    while (in.next(line)) {
        if (line.empty()) continue;
        if (line.rfind("warning: ", 0) != 0) throw ParseError("expected 'warning: ' line", in.no());
        model.warnings.push_back(line.substr(9));
    }
    AnyTensor core = read_tensor(dir + "/core");
    DenseTensor* dense = std::get_if<DenseTensor>(&core);
    bool ok = dense && dense->order() == static_cast<int>(model.ranks.size());
    for (std::size_t m = 0; ok && m < model.ranks.size(); ++m) ok = dense->dim(static_cast<int>(m)) == model.ranks[m];
    if (!ok) throw ParseError("core does not match the ranks line of '" + meta + "'", 1);
    model.core = std::move(*dense);
    for (std::size_t m = 0; m < model.ranks.size(); ++m) {
        const std::string fp = dir + "/factor_" + std::to_string(m + 1);
        model.factors.push_back(read_matrix(fp));
        if (model.factors.back().cols() != model.ranks[m]) throw ParseError("factor does not match the ranks line at '" + fp + "'", 1);
    }
    return model;
}

namespace {
void put(std::string& s, const std::string& key, const std::string& value) { s += key + " = " + value + "\n"; }
const char* tf(bool b) { return b ? "true" : "false"; }
}  // namespace

std::string render_bound_report(const BoundReport& rep) {
    const bool full = !rep.per_mode.empty();  // a shape-only report omits b, t and the modes
    std::string s;
    if (full) put(s, "b", format_double(rep.b));
    put(s, "p", format_double(rep.p));
    put(s, "p_min", format_double(rep.p_min));
    if (full) put(s, "t", format_double(rep.t));
    put(s, "success_probability", format_double(rep.success_probability));
    put(s, "dims_large_enough", tf(rep.dims_large_enough));
    put(s, "dims_balanced", tf(rep.dims_balanced));
    put(s, "p_above_min", tf(rep.p_above_min));
    put(s, "conditions_met", tf(rep.conditions_met));
    for (std::size_t i = 0; i < rep.per_mode.size(); ++i) {
        const std::string k = "mode_" + std::to_string(i + 1) + ".";
        const BoundModeReport& m = rep.per_mode[i];
        put(s, k + "rank", std::to_string(m.rank));
        put(s, k + "x_residual", format_double(m.x_residual));
        put(s, k + "xhat_residual", format_double(m.xhat_residual));
        put(s, k + "x_lowrank_norm", format_double(m.x_lowrank_norm));
        put(s, k + "t_i", format_double(m.t_i));
    }
    return s;
}

std::string render_comparison_report(const ComparisonReport& rep) {
    std::string s;
    put(s, "accuracy_exact", format_double(rep.accuracy_exact));
    put(s, "accuracy_mach", format_double(rep.accuracy_mach));
    put(s, "core_exact", format_double(rep.core_interaction.first));
    put(s, "core_mach", format_double(rep.core_interaction.second));
    for (std::size_t i = 0; i < rep.per_mode_rho.size(); ++i) {
        const std::string k = "mode_" + std::to_string(i + 1) + ".";
        put(s, k + "rho", format_double(rep.per_mode_rho[i]));
        put(s, k + "flipped", tf(rep.flipped[i]));
        put(s, k + "tied", tf(rep.tied[i]));
        put(s, k + "tie_subspace_sin", format_double(rep.tie_subspace_sin[i]));
    }
    return s;
}

void write_bound_report(const BoundReport& rep, const std::string& path) {
    Out o(path);
    o.f << render_bound_report(rep);
    o.done();
}

void write_comparison_report(const ComparisonReport& rep, const std::string& path) {
    Out o(path);
    o.f << render_comparison_report(rep);
    o.done();
}

std::vector<MeasurementRecord> read_measurements_csv(const std::string& path) {
    Lines in(path);
    std::string line;
    if (!in.next(line)) throw ParseError("empty measurement file", 1);
    if (line != "machine_id,metric,timestamp,value") throw ParseError("expected header machine_id,metric,timestamp,value", in.no());
    std::vector<MeasurementRecord> out;
    while (in.next(line)) {
        if (line.empty()) continue;
        std::vector<std::string_view> f;
        std::string_view rest(line);
        for (std::size_t c; (c = rest.find(',')) != std::string_view::npos; rest.remove_prefix(c + 1)) f.push_back(rest.substr(0, c));
        f.push_back(rest);
        if (f.size() != 4) throw ParseError("expected 4 comma-separated fields, got " + std::to_string(f.size()), in.no());
        if (f[0].empty() || f[1].empty()) throw ParseError("machine_id and metric must be nonempty", in.no());
        MeasurementRecord r;
        r.machine_id = std::string(f[0]);
        r.metric = std::string(f[1]);
        const auto a = std::from_chars(f[2].data(), f[2].data() + f[2].size(), r.timestamp);
        if (a.ec != std::errc{} || a.ptr != f[2].data() + f[2].size()) throw ParseError("bad timestamp '" + std::string(f[2]) + "'", in.no());
        const auto b = std::from_chars(f[3].data(), f[3].data() + f[3].size(), r.value);
        if (b.ec != std::errc{} || b.ptr != f[3].data() + f[3].size() || !std::isfinite(r.value))
            throw ParseError("bad value '" + std::string(f[3]) + "'", in.no());
        out.push_back(std::move(r));
    }
    return out;
}

void write_measurements_csv(const std::vector<MeasurementRecord>& records, const std::string& path) {
    for (const MeasurementRecord& r : records) {
        valid_name(r.machine_id, "machine_id");
        valid_name(r.metric, "metric");
        if (!std::isfinite(r.value)) throw ArgumentError("record values must be finite");
    }
    Out o(path);
    o.f << "machine_id,metric,timestamp,value\n";
    for (const MeasurementRecord& r : records)
        o.f << r.machine_id << ',' << r.metric << ',' << r.timestamp << ',' << format_double(r.value) << '\n';
    o.done();
}

}  // namespace mach
