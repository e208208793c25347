// Reference-style caller of the §8(f) mirrors (include/mach/bounds.hpp,
// ingest.hpp, tensor_io.hpp, cli.hpp), the code shape of
// proj/tests/test_bounds.cpp / test_io.cpp / test_cli.cpp, linked against
// libmach_b200.so.  argv[1] = scratch directory.  Exit code = failures.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "mach/bounds.hpp"
#include "mach/cli.hpp"
#include "mach/errors.hpp"
#include "mach/ingest.hpp"
#include "mach/sampling.hpp"
#include "mach/tensor.hpp"
#include "mach/tensor_io.hpp"
#include "mach/tucker.hpp"

static int failures = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        if (!(c)) {                                                           \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);           \
            ++failures;                                                       \
        }                                                                     \
    } while (0)
#define CHECK_THROWS(expr, Type)                                              \
    do {                                                                      \
        bool t_ = false;                                                      \
        try {                                                                 \
            (void)(expr);                                                     \
        } catch (const Type&) {                                               \
            t_ = true;                                                        \
        } catch (...) {                                                       \
        }                                                                     \
        if (!t_) {                                                            \
            std::printf("FAIL %s:%d %s did not throw %s\n", __FILE__, __LINE__, #expr, #Type); \
            ++failures;                                                       \
        }                                                                     \
    } while (0)

using namespace mach;

static DenseTensor wave(std::vector<int> dims, double f) {
    std::int64_t n = 1;
    for (int d : dims) n *= d;
    std::vector<double> v(static_cast<std::size_t>(n));
    for (std::size_t i = 0; i < v.size(); ++i) v[i] = std::sin(f * static_cast<double>(i + 1)) + 0.25 * std::cos(0.11 * static_cast<double>(i));
    return DenseTensor(std::move(dims), std::move(v));
}

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : "/tmp";

    // ---- bounds (test_bounds.cpp) ----
    {
        const AchlioptasBounds z = achlioptas_bounds(0.0, 10, 3, 0.5);
        CHECK(z.two_norm == 0.0 && z.frobenius == 0.0);
        const AchlioptasBounds b = achlioptas_bounds(1.0, 1000, 4, 1.0);
        CHECK(std::abs(b.two_norm - 4.0 * std::sqrt(1000.0)) < 1e-9 && std::abs(b.frobenius - 4.0 * std::sqrt(4000.0)) < 1e-9);
        CHECK_THROWS(achlioptas_bounds(-1.0, 10, 1, 0.5), ArgumentError);
        CHECK_THROWS(min_sampling_probability({5}), ArgumentError);
        CHECK_THROWS(theorem1_conditions({5, 5}, 1.5), ArgumentError);
        const DenseTensor x = wave({10, 12, 9}, 0.37);
        const SparseTensor all = sparsify(x, SparsifyConfig{1.0, 1});
        const BoundReport rep = theorem1_bound(x, all, {10, 12, 9}, 1.0);
        CHECK(rep.per_mode.size() == 3);
        for (const BoundModeReport& m : rep.per_mode) CHECK(m.x_residual == 0.0 && m.xhat_residual == 0.0 && m.t_i > 0.0);
        CHECK(rep.t == std::min({rep.per_mode[0].t_i, rep.per_mode[1].t_i, rep.per_mode[2].t_i}));
        CHECK(!rep.dims_large_enough && !rep.conditions_met);
        const SparseTensor xh = sparsify(x, SparsifyConfig{0.4, 3});
        const BoundReport full = theorem1_bound(x, xh, {2, 2, 2}, 0.4), half = theorem1_bound(x, xh, {2, 2, 2}, 0.2);
        for (std::size_t i = 0; i < 3; ++i) {  // halving p: test_bounds.cpp:185-203
            const BoundModeReport& m = full.per_mode[i];
            const double others = 10.0 * 12.0 * 9.0 / x.dim(static_cast<int>(i));
            const double ratio = m.rank / 0.4 * others;
            const double pred = (std::sqrt(2.0) - 1.0) * 4.0 * full.b * std::sqrt(ratio) +
                                (std::pow(2.0, 0.25) - 1.0) * 4.0 * std::sqrt(m.x_lowrank_norm * full.b) * std::pow(ratio, 0.25);
            CHECK(std::abs((half.per_mode[i].t_i - m.t_i) - pred) <= 1e-10 * pred);
            CHECK(half.per_mode[i].x_residual == m.x_residual && half.per_mode[i].xhat_residual == m.xhat_residual);
        }
        const BoundReport shape = theorem1_conditions(x.dims(), 0.4);
        CHECK(shape.p_min == full.p_min && shape.per_mode.empty() && shape.b == 0.0 && shape.t == 0.0);
        CHECK_THROWS(theorem1_bound(x, xh, {2, 2}, 0.4), ArgumentError);
        CHECK_THROWS(theorem1_bound(x, sparsify(wave({10, 12, 8}, 0.3), SparsifyConfig{0.5, 1}), {2, 2, 2}, 0.4), ShapeError);
        const std::string text = render_bound_report(full);
        CHECK(text.find("mode_3.t_i = ") != std::string::npos && text.rfind("b = ", 0) == 0);
        CHECK(render_bound_report(shape).find("b = ") == std::string::npos);
    }

    // ---- ingest (test_io.cpp:187-345) ----
    {
        TensorBuildSpec spec;
        spec.time_bucket_seconds = 60;
        const IngestResult r = ingest({{"host", "cpu", 1000, 1.0}, {"host", "cpu", 1060, 2.0}, {"host", "cpu", 1120, 3.0}}, spec);
        CHECK((r.tensor.dims() == std::vector<int>{1, 1, 3}));
        CHECK(r.tensor.data()[0] == 1.0 && r.tensor.data()[1] == 2.0 && r.tensor.data()[2] == 3.0);
        CHECK((r.bucket_starts == std::vector<std::int64_t>{960, 1020, 1080}));
        spec.time_bucket_seconds = 100;
        CHECK(ingest({{"h", "m", 10, 4.0}, {"h", "m", 20, 6.0}}, spec).tensor.data()[0] == 5.0);
        std::vector<MeasurementRecord> rec{{"a", "x", 5, 1e16},  {"a", "x", 15, 1.0},  {"a", "x", 25, -1e16}, {"a", "x", 35, 2.0},
                                           {"a", "x", 45, 0.125}, {"b", "x", 12, -7.5}, {"a", "y", 22, 3.25},  {"b", "y", 91, 2.5},
                                           {"b", "y", 33, 2.5}};
        const IngestResult base = ingest(rec, spec);
        for (int trial = 0; trial < 5; ++trial) {
            std::rotate(rec.begin(), rec.begin() + 2, rec.end());
            std::swap(rec[trial], rec[8 - trial]);
            CHECK(ingest(rec, spec).tensor.values() == base.tensor.values());
        }
        std::vector<MeasurementRecord> gap{{"h", "x", 0, 2.0}, {"h", "x", 200, 8.0}, {"h", "y", 100, 5.0}};
        const IngestResult zero = ingest(gap, spec);
        CHECK(zero.tensor.at(std::vector<int>{0, 0, 1}) == 0.0 && zero.tensor.at(std::vector<int>{0, 1, 2}) == 0.0);
        spec.missing_policy = MissingPolicy::carry_forward;
        const IngestResult cf = ingest(gap, spec);
        CHECK(cf.tensor.at(std::vector<int>{0, 0, 1}) == 2.0 && cf.tensor.at(std::vector<int>{0, 0, 2}) == 8.0);
        CHECK(cf.tensor.at(std::vector<int>{0, 1, 0}) == 0.0 && cf.tensor.at(std::vector<int>{0, 1, 2}) == 5.0);
        CHECK_THROWS(ingest({}, TensorBuildSpec{}), ArgumentError);
        CHECK_THROWS(ingest({{"h", "m", 0, std::nan("")}}, TensorBuildSpec{}), ArgumentError);
        TensorBuildSpec bad;
        bad.time_bucket_seconds = 0;
        CHECK_THROWS(ingest({{"h", "m", 0, 1.0}}, bad), ArgumentError);
        bad = TensorBuildSpec{};
        bad.machine_order = {"a", "a"};
        CHECK_THROWS(ingest({{"a", "m", 0, 1.0}}, bad), ArgumentError);
        bad.machine_order = {"z"};
        CHECK_THROWS(ingest({{"a", "m", 0, 1.0}}, bad), ArgumentError);
        spec = TensorBuildSpec{};
        spec.time_bucket_seconds = 60;
        const IngestResult neg = ingest({{"h", "m", -10, 1.0}, {"h", "m", 10, 2.0}}, spec);
        CHECK((neg.bucket_starts == std::vector<std::int64_t>{-60, 0}) && neg.tensor.data()[0] == 1.0 && neg.tensor.data()[1] == 2.0);

        // sample on arrival == sparsify(ingest(everything))
        std::vector<MeasurementRecord> all;
        for (int t = 0; t < 40; ++t)
            for (int m = 0; m < 5; ++m)
                for (int j = 0; j < 3; ++j)
                    if ((t * 7 + m * 3 + j) % 4 != 0)
                        all.push_back({"m" + std::to_string(m), "k" + std::to_string(j), 6000 + 60 * t + (m * 11 + j) % 60,
                                       std::sin(0.3 * t + m) * (j + 1) + 2.0});
        TensorBuildSpec whole;
        whole.time_bucket_seconds = 60;
        whole.missing_policy = MissingPolicy::carry_forward;
        const IngestResult off = ingest(all, whole);
        const SparsifyConfig scfg{0.5, 9};
        const SparseTensor ref = sparsify(off.tensor, scfg);
        StreamingIngest live(off.machines, off.metrics, off.bucket_starts.front(), 60, 64, MissingPolicy::carry_forward, scfg);
        const int cuts[] = {0, 7, 8, 25, 40};
        for (int w = 0; w + 1 < 5; ++w) {
            std::vector<MeasurementRecord> win;
            for (const MeasurementRecord& r2 : all) {
                const std::int64_t b = (r2.timestamp - off.bucket_starts.front()) / 60;
                if (b >= cuts[w] && b < cuts[w + 1]) win.push_back(r2);
            }
            std::reverse(win.begin(), win.end());
            live.append_window(win, cuts[w + 1] - cuts[w]);
        }
        CHECK(live.buckets() == 40 && live.nnz() == ref.nnz());
        const SparseTensor got = live.sampled();
        CHECK(got.dims() == ref.dims() && got.nnz() == ref.nnz());
        bool same = got.nnz() == ref.nnz();
        for (std::int64_t i = 0; same && i < ref.nnz(); ++i)
            same = got.entries()[static_cast<std::size_t>(i)].index == ref.entries()[static_cast<std::size_t>(i)].index &&
                   got.entries()[static_cast<std::size_t>(i)].value == ref.entries()[static_cast<std::size_t>(i)].value;
        CHECK(same);
        const TuckerModel a = live.hooi({2, 2, 3}, HooiConfig{3, 0.0}), b = hooi(ref, {2, 2, 3}, HooiConfig{3, 0.0});
        CHECK(std::abs(a.fit - b.fit) < 1e-12 && a.iterations == b.iterations);
        CHECK_THROWS(live.append_window({{"nobody", "k0", 6000 + 60 * 40, 1.0}}, 1), ArgumentError);

        const std::string csv = dir + "/m.csv";
        write_measurements_csv(all, csv);
        const std::vector<MeasurementRecord> back = read_measurements_csv(csv);
        bool eq = back.size() == all.size();
        for (std::size_t i = 0; eq && i < all.size(); ++i)
            eq = back[i].machine_id == all[i].machine_id && back[i].metric == all[i].metric && back[i].timestamp == all[i].timestamp &&
                 back[i].value == all[i].value;
        CHECK(eq);
        CHECK_THROWS(write_measurements_csv({{"a,b", "m", 0, 1.0}}, csv), ArgumentError);
        CHECK_THROWS(read_measurements_csv(dir + "/none.csv"), IoError);
    }

    // ---- tensor files: text (reference grammar) and binary, model directory ----
    {
        const DenseTensor x = wave({5, 4, 3}, 0.77);
        const SparseTensor s = sparsify(x, SparsifyConfig{0.5, 2});
        for (const char* suffix : {".txt", ".machb"}) {
            const std::string pd = dir + "/x" + suffix, ps = dir + "/s" + suffix;
            write_tensor(x, pd);
            write_tensor(s, ps);
            const AnyTensor rd = read_tensor(pd), rs = read_tensor(ps);
            const DenseTensor* xd = std::get_if<DenseTensor>(&rd);
            const SparseTensor* xs = std::get_if<SparseTensor>(&rs);
            CHECK(xd && xd->dims() == x.dims() && xd->values() == x.values());
            CHECK(xs && xs->dims() == s.dims() && xs->nnz() == s.nnz());
            for (std::int64_t i = 0; xs && i < s.nnz(); ++i)
                CHECK(xs->entries()[static_cast<std::size_t>(i)].index == s.entries()[static_cast<std::size_t>(i)].index &&
                      xs->entries()[static_cast<std::size_t>(i)].value == s.entries()[static_cast<std::size_t>(i)].value);
        }
        {
            std::ofstream f(dir + "/hand.txt");
            f << "sparse dims: 2 3\n1 1 1.5\n2 3 -2\n1 1 0.5\n";  // duplicate lines sum
        }
        const AnyTensor hand = read_tensor(dir + "/hand.txt");
        const SparseTensor* hs = std::get_if<SparseTensor>(&hand);
        CHECK(hs && hs->nnz() == 2 && hs->entries()[0].value == 2.0 && hs->entries()[1].index == 5);
        {
            std::ofstream f(dir + "/bad.txt");
            f << "dims: 2 2\n1 2 3\n";
        }
        CHECK_THROWS(read_tensor(dir + "/bad.txt"), ParseError);
        CHECK_THROWS(read_tensor(dir + "/nope.txt"), IoError);
        CHECK(format_double(0.1) == "0.1" && format_double(1e300) == "1e+300");
        const TuckerModel m = hooi(x, {2, 2, 2}, HooiConfig{4, 0.0});
        save_model(m, dir + "/model");
        const TuckerModel l = load_model(dir + "/model");
        CHECK(l.ranks == m.ranks && l.iterations == m.iterations && l.fit == m.fit && l.sweep_fits == m.sweep_fits);
        CHECK(l.core.values() == m.core.values() && l.factors[2].values() == m.factors[2].values());
    }

    // ---- CLI (test_cli.cpp shape): exit codes and an end-to-end sampled run ----
    {
        const DenseTensor x = wave({12, 10, 14}, 0.21);
        write_tensor(x, dir + "/cx.txt");
        CHECK(run_cli({"convert", "--input", dir + "/cx.txt", "--output", dir + "/cx.machb"}) == 0);
        CHECK(run_cli({"mach-hooi", "--input", dir + "/cx.machb", "--ranks", "2,2,3", "--p", "0.5", "--seed", "4", "--max-iters", "3",
                       "--fit-tol", "0", "--output", dir + "/cm_bin", "--sparsified", dir + "/cs.machb"}) == 0);
        CHECK(run_cli({"mach-hooi", "--input", dir + "/cx.txt", "--ranks", "2,2,3", "--p", "0.5", "--seed", "4", "--max-iters", "3",
                       "--fit-tol", "0", "--output", dir + "/cm_txt", "--sparsified", dir + "/cs.txt"}) == 0);
        const TuckerModel mb = load_model(dir + "/cm_bin"), mt = load_model(dir + "/cm_txt");
        const MachResult direct = mach_hooi(x, {2, 2, 3}, SparsifyConfig{0.5, 4}, HooiConfig{3, 0.0});
        CHECK(mt.fit == direct.model.fit && std::abs(mb.fit - direct.model.fit) < 1e-12);
        const AnyTensor cs = read_tensor(dir + "/cs.machb");
        CHECK(std::get_if<SparseTensor>(&cs) && std::get_if<SparseTensor>(&cs)->nnz() == direct.sparsified.nnz());
        CHECK(run_cli({"hosvd", "--input", dir + "/cs.machb", "--ranks", "2,2,3", "--output", dir + "/ch"}) == 0);
        CHECK(run_cli({"hooi", "--input", dir + "/cx.txt", "--ranks", "2,2,3", "--output", dir + "/ce"}) == 0);
        CHECK(run_cli({"compare", "--exact", dir + "/ce", "--approx", dir + "/cm_txt", "--reference", dir + "/cx.txt", "--output",
                       dir + "/cmp.txt"}) == 0);
        CHECK(run_cli({"bound", "--input", dir + "/cx.txt", "--sparsified", dir + "/cs.txt", "--ranks", "2,2,3", "--p", "0.5",
                       "--output", dir + "/bound.txt"}) == 0);
        CHECK(run_cli({"bound", "--dims", "200,200,200", "--p", "0.5", "--output", dir + "/cond.txt"}) == 0);
        CHECK(run_cli({"sparsify", "--input", dir + "/cx.machb", "--p", "0.25", "--output", dir + "/s25.machb"}) == 0);
        CHECK(run_cli({"bench", "--input", dir + "/cx.txt", "--ranks", "2,2,3", "--p", "0.5", "--max-iters", "3", "--output",
                       dir + "/bench.csv", "--timing", dir + "/timing.csv"}) == 0);
        CHECK(run_cli({}) == 2);
        CHECK(run_cli({"frobnicate"}) == 2);
        CHECK(run_cli({"hooi", "--input", dir + "/cx.txt", "--output", dir + "/o"}) == 2);                  // no ranks
        CHECK(run_cli({"sparsify", "--input", dir + "/cx.txt", "--p", "1.5", "--output", dir + "/o"}) == 2);  // ArgumentError
        CHECK(run_cli({"hooi", "--input", dir + "/missing.txt", "--ranks", "2,2,3", "--output", dir + "/o"}) == 3);
        CHECK(run_cli({"mach-hooi", "--input", dir + "/cs.txt", "--ranks", "2,2,3", "--p", "0.5", "--output", dir + "/o"}) == 3);
    }

    std::printf("ext_smoke: %d failures\n", failures);
    return failures;
}
