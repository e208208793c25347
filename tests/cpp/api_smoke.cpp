// Reference-style caller of the C++ mirror (include/mach/*.hpp): the same
// code shape as proj/tests/test_sampling.cpp / test_tucker.cpp, linked
// against libmach_b200.so.  Prints one line per check; exit code = failures.
#include <cmath>
#include <cstdio>
#include <vector>

#include "mach/errors.hpp"
#include "mach/linalg.hpp"
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
    CHECK(keep.nnz() == t.size());
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
    std::printf("api_smoke: %d failures\n", failures);
    return failures;
}
