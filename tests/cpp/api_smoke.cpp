// Reference-style caller of the C++ mirror (include/mach/*.hpp): the same
// code shape as proj/tests/test_sampling.cpp / test_tucker.cpp, linked
// against libmach_b200.so.  Prints one line per check; exit code = failures.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

#include "mach/errors.hpp"
#include "mach/linalg.hpp"
#include "mach/metrics.hpp"
#include "mach/sampling.hpp"
#include "mach/tensor.hpp"
#include "mach/tucker.hpp"

static int failures = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        if (!(c)) {                                                           \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);           \
            ++failures;                                                       \
        }                                                                     \
    } while (0)

int main() {
    using namespace mach;
    std::vector<double> v(6 * 7 * 8);
    for (std::size_t i = 0; i < v.size(); ++i) v[i] = std::sin(0.37 * static_cast<double>(i)) + 0.01 * static_cast<double>(i % 5);
    const DenseTensor t({6, 7, 8}, v);

    const SparseTensor keep = sparsify(t, SparsifyConfig{1.0, 3});
    std::int64_t nonzero = 0;  // sparsify skips exact zeros (sampling.cpp:25); v[0] = sin(0) = 0
    for (double x : v) nonzero += x != 0.0;
    CHECK(keep.nnz() == nonzero);
    const SparseTensor half = sparsify(t, SparsifyConfig{0.5, 7});
    CHECK(half.nnz() > 0 && half.nnz() < t.size());
    for (const SparseEntry& e : half.entries()) CHECK(e.value * 0.5 == t.values()[static_cast<std::size_t>(e.index)]);

    const TuckerModel m = hooi(t, {2, 2, 2}, HooiConfig{});
    CHECK(m.iterations >= 1 && m.sweep_fits.size() == static_cast<std::size_t>(m.iterations) + 1);
    CHECK(std::abs(m.fit - accuracy(t, m)) < 1e-10);

    const MachResult r = mach_hooi(t, {2, 2, 2}, SparsifyConfig{0.3, 11}, HooiConfig{5, 0.0});
    CHECK(r.sparsified.nnz() > 0);

    bool threw = false;
    try {
        sparsify(t, SparsifyConfig{0.0, 1});
    } catch (const ArgumentError&) {
        threw = true;
    }
    CHECK(threw);

    const LeftSingularBasis b = left_singular_basis(matricize(t, 1), 3);
    CHECK(b.numerical_rank == 3 && !b.completed);

    // truncated SVD family (linalg.hpp:11-30): orthonormal factors, sorted
    // values, the left factor shared with leading_left_singular_vectors,
    // low_rank_approx = left diag(s) right^T, k checked like the reference
    const Matrix a = matricize(t, 2);  // 8 x 42
    const TruncatedSvd svd = truncated_svd(a, 4);
    CHECK(svd.left.rows() == 8 && svd.left.cols() == 4 && svd.right.rows() == 42 && svd.right.cols() == 4);
    for (int i = 1; i < 4; ++i) CHECK(svd.singular_values[i] <= svd.singular_values[i - 1]);
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
            double l = 0.0, r = 0.0;
            for (int x = 0; x < 8; ++x) l += svd.left(x, i) * svd.left(x, j);
            for (int x = 0; x < 42; ++x) r += svd.right(x, i) * svd.right(x, j);
            CHECK(std::abs(l - (i == j ? 1.0 : 0.0)) < 1e-10 && std::abs(r - (i == j ? 1.0 : 0.0)) < 1e-10);
        }
    const Matrix lead = leading_left_singular_vectors(a, 4);
    CHECK(lead.values() == svd.left.values());
    const Matrix lr = low_rank_approx(a, 4);
    double err = 0.0;
    for (int r = 0; r < 8; ++r)
        for (int c = 0; c < 42; ++c) {
            double v = 0.0;
            for (int i = 0; i < 4; ++i) v += svd.left(r, i) * svd.singular_values[i] * svd.right(c, i);
            err = std::max(err, std::abs(v - lr(r, c)));
        }
    CHECK(err < 1e-12);
    threw = false;
    try {
        truncated_svd(a, 9);
    } catch (const ArgumentError&) {
        threw = true;
    }
    CHECK(threw);
    // metrics.hpp: the reference model against the MACH one
    const ComparisonReport rep = compare(m, r.model, t);
    CHECK(rep.per_mode_rho.size() == 3 && rep.flipped.size() == 3 && rep.tied.size() == 3);
    for (double rho : rep.per_mode_rho) CHECK(rho >= -1.0 && rho <= 1.0);
    CHECK(std::abs(rep.accuracy_exact - accuracy(t, m)) < 1e-14);
    CHECK(rep.core_interaction.first == m.core.data()[0]);
    const std::vector<double> px{1.0, 2.0, 3.0}, py{2.0, 4.0, 6.0};
    CHECK(pearson(px, py) == 1.0);
    std::printf("api_smoke: %d failures\n", failures);
    return failures;
}
