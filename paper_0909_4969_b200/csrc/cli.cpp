// Command-line tool wired to the B200 backend (mirrors the
// reference's subcommands and exit codes, proj/src/cli.cpp:200-211, :347-450,
// cli.hpp:9-14): ingest, sparsify, hosvd, hooi, mach-hosvd, mach-hooi,
// compare, bound, bench — plus `convert` between the reference's text tensor
// files and the binary MACHB2 format.  Binary inputs are loaded straight into
// HBM and decomposed in their stored precision without a host round trip; text
// inputs go through the C++ mirror.  (`synth` is not provided: the reference's
// generators are outside the hot path.)
#include <algorithm>
#include <array>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstring>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <set>

#include "mach/bounds.hpp"
#include "mach/cli.hpp"
#include "mach/errors.hpp"
#include "mach/ingest.hpp"
#include "mach/metrics.hpp"
#include "mach/sampling.hpp"
#include "mach/tensor_io.hpp"
#include "mach/tucker.hpp"
#include "mach_b200.h"

namespace mach {

namespace b200 {
mach_ctx* context();
void check(mach_status st);
TuckerModel model_from_handle(mach_model* m);
SparseTensor sparse_from_handle(const mach_sparse* s, std::vector<int> dims);
}  // namespace b200

namespace {

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// "--name value" options of one subcommand; flags listed in `flags` take no value
class Options {
public:
    Options(const std::vector<std::string>& args, std::size_t from, std::set<std::string> allowed, std::set<std::string> flags = {}) {
        for (std::size_t i = from; i < args.size(); ++i) {
            const std::string& a = args[i];
            if (a.rfind("--", 0) != 0) throw UsageError("unexpected argument '" + a + "'");
            std::string key = a.substr(2), val;
            const std::size_t eq = key.find('=');
            const bool inline_val = eq != std::string::npos;
            if (inline_val) {
                val = key.substr(eq + 1);
                key = key.substr(0, eq);
            }
            if (!allowed.count(key) && !flags.count(key)) throw UsageError("unknown option '--" + key + "'");
            if (flags.count(key)) {
                kv_[key] = "1";
                continue;
            }
            if (!inline_val) {
                if (i + 1 >= args.size()) throw UsageError("option '--" + key + "' needs a value");
                val = args[++i];
            }
            kv_[key] = val;
        }
    }
    bool has(const std::string& k) const { return kv_.count(k) != 0; }
    std::string str(const std::string& k, const std::string& dflt = "") const {
        const auto it = kv_.find(k);
        return it == kv_.end() ? dflt : it->second;
    }
    std::string need(const std::string& k) const {
        if (!has(k)) throw UsageError("option '--" + k + "' is required");
        return kv_.at(k);
    }
    double real(const std::string& k, double dflt) const {
        if (!has(k)) return dflt;
        const std::string& s = kv_.at(k);
        double v = 0;
        const auto r = std::from_chars(s.data(), s.data() + s.size(), v);
        if (r.ec != std::errc{} || r.ptr != s.data() + s.size()) throw UsageError("option '--" + k + "': bad number '" + s + "'");
        return v;
    }
    std::int64_t integer(const std::string& k, std::int64_t dflt) const {
        if (!has(k)) return dflt;
        const std::string& s = kv_.at(k);
        std::int64_t v = 0;
        const auto r = std::from_chars(s.data(), s.data() + s.size(), v);
        if (r.ec != std::errc{} || r.ptr != s.data() + s.size()) throw UsageError("option '--" + k + "': bad integer '" + s + "'");
        return v;
    }
    std::vector<int> ints(const std::string& k) const {
        std::vector<int> out;
        if (!has(k)) return out;
        std::string_view rest(kv_.at(k));
        while (!rest.empty()) {
            const std::size_t c = rest.find(',');
            const std::string_view tok = rest.substr(0, c);
            int v = 0;
            const auto r = std::from_chars(tok.data(), tok.data() + tok.size(), v);
            if (r.ec != std::errc{} || r.ptr != tok.data() + tok.size())
                throw UsageError("option '--" + k + "': bad integer '" + std::string(tok) + "'");
            out.push_back(v);
            if (c == std::string_view::npos) break;
            rest.remove_prefix(c + 1);
        }
        return out;
    }

private:
    std::map<std::string, std::string> kv_;
};

bool binary_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open '" + path + "' for reading");
    char m[8] = {};
    in.read(m, 8);
    static const char want[8] = {'M', 'A', 'C', 'H', 'B', '2', 0, 0};
    return in.gcount() == 8 && std::memcmp(m, want, 8) == 0;
}

struct FileInfo {
    int kind = 0, order = 0;
    mach_dtype dtype = MACH_F64;
    std::vector<int> dims;
    std::int64_t count = 0;
};

FileInfo file_info(const std::string& path) {
    FileInfo f;
    int d8[8] = {};
    b200::check(mach_tensor_file_kind(path.c_str(), &f.kind, &f.dtype, &f.order, d8, &f.count));
    f.dims.assign(d8, d8 + f.order);
    return f;
}

const DenseTensor& as_dense(const AnyTensor& t, const std::string& path) {
    const DenseTensor* d = std::get_if<DenseTensor>(&t);
    if (!d) throw ShapeError("'" + path + "' holds a sparse tensor; a dense one is required");
    return *d;
}

void report_model(const TuckerModel& model, const std::string& out) {
    save_model(model, out);
    std::cout << "wrote " << out << '\n' << "fit = " << format_double(model.fit) << '\n';
    for (const std::string& w : model.warnings) std::cout << "warning: " << w << '\n';
}

// hosvd / hooi / mach-hosvd / mach-hooi (cli.cpp:188-247)
void cmd_decompose(const std::vector<std::string>& a, bool iterate, bool sample) {
    std::set<std::string> allowed{"input", "ranks", "output"};
    if (sample) allowed.insert({"p", "seed", "sparsified"});
    if (iterate) allowed.insert({"max-iters", "fit-tol"});
    const Options o(a, 1, allowed);
    const std::string input = o.need("input"), output = o.need("output");
    const std::vector<int> ranks = o.ints("ranks");
    if (ranks.empty()) throw UsageError("option '--ranks' is required");
    SparsifyConfig scfg;
    HooiConfig hcfg;
    if (sample) {
        if (!o.has("p")) throw UsageError("option '--p' is required");
        scfg.p = o.real("p", 1.0);
        scfg.seed = static_cast<std::uint64_t>(o.integer("seed", 0));
    }
    hcfg.max_iterations = static_cast<int>(o.integer("max-iters", hcfg.max_iterations));
    hcfg.fit_tolerance = o.real("fit-tol", hcfg.fit_tolerance);
    const std::string sparsified = o.str("sparsified");

    if (binary_file(input)) {  // device path: file -> HBM -> model, stored precision
        const FileInfo fi = file_info(input);
        if (static_cast<int>(ranks.size()) != fi.order) throw ArgumentError("ranks must name one rank per mode");
        mach_model* m = nullptr;
        if (fi.kind == 0) {
            mach_dense* x = nullptr;
            b200::check(mach_dense_load(b200::context(), input.c_str(), &x));
            mach_sparse* sp = nullptr;
            mach_status rc;
            if (sample)
                rc = iterate ? mach_mach_hooi(b200::context(), x, ranks.data(), scfg.p, scfg.seed, hcfg.max_iterations,
                                              hcfg.fit_tolerance, &m, sparsified.empty() ? nullptr : &sp)
                             : mach_mach_hosvd(b200::context(), x, ranks.data(), scfg.p, scfg.seed, &m,
                                               sparsified.empty() ? nullptr : &sp);
            else
                rc = iterate ? mach_hooi_dense(b200::context(), x, ranks.data(), hcfg.max_iterations, hcfg.fit_tolerance, &m)
                             : mach_hosvd_dense(b200::context(), x, ranks.data(), &m);
            mach_dense_free(x);
            if (rc == MACH_OK && sp) {
                if (sparsified.size() >= 6 && sparsified.compare(sparsified.size() - 6, 6, ".machb") == 0)
                    rc = mach_sparse_save(sp, sparsified.c_str());
                else
                    write_tensor(b200::sparse_from_handle(sp, fi.dims), sparsified);
                if (rc == MACH_OK) std::cout << "wrote " << sparsified << '\n';
            }
            if (sp) mach_sparse_free(sp);
            b200::check(rc);
        } else {
            if (sample) throw ShapeError("'" + input + "' holds a sparse tensor; a dense one is required");
            mach_sparse* s = nullptr;
            b200::check(mach_sparse_load(b200::context(), input.c_str(), &s));
            const mach_status rc = iterate ? mach_hooi_sparse(b200::context(), s, ranks.data(), hcfg.max_iterations,
                                                              hcfg.fit_tolerance, &m)
                                           : mach_hosvd_sparse(b200::context(), s, ranks.data(), &m);
            mach_sparse_free(s);
            b200::check(rc);
        }
        report_model(b200::model_from_handle(m), output);
        return;
    }
    const AnyTensor t = read_tensor(input);
    if (sample) {
        const DenseTensor& x = as_dense(t, input);
        const MachResult r = iterate ? mach_hooi(x, ranks, scfg, hcfg) : mach_hosvd(x, ranks, scfg);
        if (!sparsified.empty()) {
            write_tensor(r.sparsified, sparsified);
            std::cout << "wrote " << sparsified << '\n';
        }
        report_model(r.model, output);
        return;
    }
    const TuckerModel model = iterate ? std::visit([&](const auto& x) { return hooi(x, ranks, hcfg); }, t)
                                      : std::visit([&](const auto& x) { return hosvd(x, ranks); }, t);
    report_model(model, output);
}

void cmd_sparsify(const std::vector<std::string>& a) {  // cli.cpp:162-186
    const Options o(a, 1, {"input", "p", "seed", "output"});
    const std::string input = o.need("input"), output = o.need("output");
    if (!o.has("p")) throw UsageError("option '--p' is required");
    const SparsifyConfig cfg{o.real("p", 1.0), static_cast<std::uint64_t>(o.integer("seed", 0))};
    std::int64_t nnz = 0;
    if (binary_file(input)) {
        const FileInfo fi = file_info(input);
        if (fi.kind != 0) throw ShapeError("'" + input + "' holds a sparse tensor; a dense one is required");
        mach_dense* x = nullptr;
        b200::check(mach_dense_load(b200::context(), input.c_str(), &x));
        mach_sparse* s = nullptr;
        mach_status rc = mach_sparsify(b200::context(), x, cfg.p, cfg.seed, &s);
        mach_dense_free(x);
        b200::check(rc);
        mach_sparse_nnz(s, &nnz);
        if (output.size() >= 6 && output.compare(output.size() - 6, 6, ".machb") == 0) rc = mach_sparse_save(s, output.c_str());
        else write_tensor(b200::sparse_from_handle(s, fi.dims), output);
        mach_sparse_free(s);
        b200::check(rc);
    } else {
        const AnyTensor t = read_tensor(input);
        const SparseTensor s = sparsify(as_dense(t, input), cfg);
        nnz = s.nnz();
        write_tensor(s, output);
    }
    std::cout << "wrote " << output << " (" << nnz << " nonzeros)\n";
}

void cmd_ingest(const std::vector<std::string>& a) {  // cli.cpp:117-160
    const Options o(a, 1, {"input", "output", "bucket-seconds", "missing", "labels"});
    TensorBuildSpec spec;
    spec.time_bucket_seconds = o.integer("bucket-seconds", 300);
    const std::string missing = o.str("missing", "zero");
    if (missing != "zero" && missing != "carry_forward") throw UsageError("--missing must be zero or carry_forward");
    spec.missing_policy = missing == "zero" ? MissingPolicy::zero : MissingPolicy::carry_forward;
    const IngestResult r = ingest(read_measurements_csv(o.need("input")), spec);
    write_tensor(r.tensor, o.need("output"));
    if (o.has("labels")) {
        std::ofstream out(o.str("labels"));
        if (!out) throw IoError("cannot open '" + o.str("labels") + "' for writing");
        for (const std::string& m : r.machines) out << "machine: " << m << '\n';
        for (const std::string& m : r.metrics) out << "metric: " << m << '\n';
        for (std::int64_t b : r.bucket_starts) out << "bucket_start: " << b << '\n';
        out.flush();
        if (!out) throw IoError("failed writing '" + o.str("labels") + "'");
    }
    std::cout << "wrote " << o.str("output") << " (" << r.machines.size() << " x " << r.metrics.size() << " x "
              << r.bucket_starts.size() << ")\n";
}

void cmd_compare(const std::vector<std::string>& a) {  // cli.cpp:249-277
    const Options o(a, 1, {"exact", "approx", "reference", "output"});
    const TuckerModel exact = load_model(o.need("exact")), approx = load_model(o.need("approx"));
    const AnyTensor ref = read_tensor(o.need("reference"));
    const ComparisonReport rep = compare(exact, approx, as_dense(ref, o.str("reference")));
    write_comparison_report(rep, o.need("output"));
    std::cout << render_comparison_report(rep) << "wrote " << o.str("output") << '\n';
}

void cmd_bound(const std::vector<std::string>& a) {  // cli.cpp:279-322
    const Options o(a, 1, {"dims", "input", "sparsified", "ranks", "p", "output"});
    if (!o.has("p")) throw UsageError("option '--p' is required");
    const double p = o.real("p", 1.0);
    BoundReport rep;
    if (o.has("dims")) {
        if (o.has("input") || o.has("sparsified") || o.has("ranks")) throw UsageError("--dims excludes --input, --sparsified and --ranks");
        rep = theorem1_conditions(o.ints("dims"), p);
    } else {
        const std::string input = o.need("input"), sparsified = o.need("sparsified");
        const std::vector<int> ranks = o.ints("ranks");
        if (ranks.empty()) throw UsageError("option '--ranks' is required");
        const AnyTensor x = read_tensor(input), xh = read_tensor(sparsified);
        const SparseTensor* s = std::get_if<SparseTensor>(&xh);
        if (!s) throw ShapeError("'" + sparsified + "' holds a dense tensor; a sparse one is required");
        rep = theorem1_bound(as_dense(x, input), *s, ranks, p);
    }
    write_bound_report(rep, o.need("output"));
    std::cout << render_bound_report(rep) << "wrote " << o.str("output") << '\n';
}

template <typename F>
double median_of_three(F&& body) {
    std::array<double, 3> runs{};
    for (double& r : runs) {
        const auto t0 = std::chrono::steady_clock::now();
        body();
        r = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    std::sort(runs.begin(), runs.end());
    return runs[1];
}

void cmd_bench(const std::vector<std::string>& a) {  // cli.cpp:324-407
    const Options o(a, 1, {"input", "ranks", "p", "seed", "max-iters", "fit-tol", "output", "timing"});
    const std::vector<int> ranks = o.ints("ranks");
    if (ranks.empty()) throw UsageError("option '--ranks' is required");
    if (!o.has("p")) throw UsageError("option '--p' is required");
    const SparsifyConfig scfg{o.real("p", 1.0), static_cast<std::uint64_t>(o.integer("seed", 0))};
    HooiConfig hcfg;
    hcfg.max_iterations = static_cast<int>(o.integer("max-iters", hcfg.max_iterations));
    hcfg.fit_tolerance = o.real("fit-tol", hcfg.fit_tolerance);
    const std::string output = o.need("output"), timing = o.need("timing");
    const AnyTensor t = read_tensor(o.need("input"));
    const DenseTensor& x = as_dense(t, o.str("input"));
    TuckerModel exact;
    const double exact_s = median_of_three([&] { exact = hooi(x, ranks, hcfg); });
    MachResult sampled;
    const double mach_s = median_of_three([&] { sampled = mach_hooi(x, ranks, scfg, hcfg); });
    const ComparisonReport rep = compare(exact, sampled.model, x);
    {
        std::ofstream out(output);
        if (!out) throw IoError("cannot open '" + output + "' for writing");
        out << "p,accuracy_exact,accuracy_mach,core_exact,core_mach";
        for (std::size_t m = 0; m < rep.per_mode_rho.size(); ++m) out << ",rho_" << m + 1;
        out << '\n'
            << format_double(scfg.p) << ',' << format_double(rep.accuracy_exact) << ',' << format_double(rep.accuracy_mach) << ','
            << format_double(rep.core_interaction.first) << ',' << format_double(rep.core_interaction.second);
        for (double rho : rep.per_mode_rho) out << ',' << format_double(rho);
        out << '\n';
        out.flush();
        if (!out) throw IoError("failed writing '" + output + "'");
    }
    {
        std::ofstream tim(timing);
        if (!tim) throw IoError("cannot open '" + timing + "' for writing");
        tim << "exact_seconds,mach_seconds,speedup\n"
            << format_double(exact_s) << ',' << format_double(mach_s) << ',' << format_double(exact_s / mach_s) << '\n';
        tim.flush();
        if (!tim) throw IoError("failed writing '" + timing + "'");
    }
    std::cout << "exact_seconds = " << format_double(exact_s) << '\n'
              << "mach_seconds = " << format_double(mach_s) << '\n'
              << "speedup = " << format_double(exact_s / mach_s) << '\n'
              << "accuracy_exact = " << format_double(rep.accuracy_exact) << '\n'
              << "accuracy_mach = " << format_double(rep.accuracy_mach) << '\n'
              << "wrote " << output << '\n'
              << "wrote " << timing << '\n';
}

// text <-> binary (the suffix ".machb" selects the binary format on write)
void cmd_convert(const std::vector<std::string>& a) {
    const Options o(a, 1, {"input", "output"});
    const AnyTensor t = read_tensor(o.need("input"));
    std::visit([&](const auto& x) { write_tensor(x, o.need("output")); }, t);
    std::cout << "wrote " << o.str("output") << '\n';
}

int fail(int code, const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return code;
}

const char* kUsage =
    "usage: mach_b200 <command> [options]\n"
    "commands: ingest sparsify hosvd hooi mach-hosvd mach-hooi compare bound bench convert\n";

}  // namespace

int run_cli(const std::vector<std::string>& args) {
    try {
        if (args.empty()) throw UsageError("a command is required");
        const std::string& c = args[0];
        if (c == "--help" || c == "-h" || c == "help") {
            std::cout << kUsage;
            return 0;
        }
        if (c == "ingest") cmd_ingest(args);
        else if (c == "sparsify") cmd_sparsify(args);
        else if (c == "hosvd") cmd_decompose(args, false, false);
        else if (c == "hooi") cmd_decompose(args, true, false);
        else if (c == "mach-hosvd") cmd_decompose(args, false, true);
        else if (c == "mach-hooi") cmd_decompose(args, true, true);
        else if (c == "compare") cmd_compare(args);
        else if (c == "bound") cmd_bound(args);
        else if (c == "bench") cmd_bench(args);
        else if (c == "convert") cmd_convert(args);
        else throw UsageError("unknown command '" + c + "'");
    } catch (const UsageError& e) {
        std::cerr << "error: " << e.what() << '\n' << kUsage;
        return 2;
    } catch (const ArgumentError& e) {
        return fail(2, e);
    } catch (const ShapeError& e) {
        return fail(3, e);
    } catch (const ParseError& e) {
        return fail(3, e);
    } catch (const IoError& e) {
        return fail(3, e);
    } catch (const ConvergenceError& e) {
        return fail(4, e);
    } catch (const std::exception& e) {
        return fail(1, e);
    }
    return 0;
}

}  // namespace mach
