// ============================================================================
//  TEST INFRASTRUCTURE ONLY — CPU oracle for the MACH sampler + Tucker path.
//
//  This is an Eigen-free restatement, in plain C++20, of the reference's hot
//  path (reference = /root/reference/proj, which cannot be compiled here:
//  proj/CMakeLists.txt:10 requires Eigen3, which is absent from the image).
//  Every function below names the reference file:line it restates.
//
//  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / the
//  `--impl reference` arm may load it.  The product library
//  (paper_0909_4969_b200/) never links or calls it.
//
//  Pinning: see tests/test_oracle_*.py — SplitMix64 published known answers,
//  the reference test suites' known answers restated (test_sampling.cpp,
//  test_tucker.cpp, test_tensor.cpp, test_linalg.cpp, acceptance.cpp) and a
//  numpy.linalg.eigh cross-check of the eigensolver.
// ============================================================================
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

// ---- errors (proj/include/mach/errors.hpp:9-47) ---------------------------
enum class ErrKind { Argument = 1, Shape = 2, Convergence = 3 };

struct Error : std::runtime_error {
    ErrKind kind;
    int singular_index;
    Error(ErrKind k, const std::string& m, int idx = 0)
        : std::runtime_error(m), kind(k), singular_index(idx) {}
};

// ---- value types (proj/include/mach/tensor.hpp:13-105) --------------------
struct Dense {                 // first mode fastest (tensor.hpp:10-12)
    std::vector<int> dims;
    std::vector<double> v;
    std::int64_t size() const { return static_cast<std::int64_t>(v.size()); }
    int order() const { return static_cast<int>(dims.size()); }
};

struct Entry {                 // SparseEntry (tensor.hpp:43-46)
    std::int64_t index;
    double value;
};

struct Sparse {                // canonical COO (tensor.hpp:48-75)
    std::vector<int> dims;
    std::vector<Entry> e;
    std::int64_t nnz() const { return static_cast<std::int64_t>(e.size()); }
    std::int64_t size() const;
    int order() const { return static_cast<int>(dims.size()); }
};

struct Mat {                   // column-major (tensor.hpp:77-105)
    int rows = 0, cols = 0;
    std::vector<double> v;
    Mat() = default;
    Mat(int r, int c) : rows(r), cols(c), v(static_cast<std::size_t>(r) * c, 0.0) {}
    double& operator()(int r, int c) { return v[static_cast<std::size_t>(r) + static_cast<std::size_t>(c) * rows]; }
    double operator()(int r, int c) const { return v[static_cast<std::size_t>(r) + static_cast<std::size_t>(c) * rows]; }
    double* col(int c) { return v.data() + static_cast<std::size_t>(c) * rows; }
    const double* col(int c) const { return v.data() + static_cast<std::size_t>(c) * rows; }
};

struct Model {                 // TuckerModel (tucker.hpp:14-22)
    Dense core;
    std::vector<Mat> factors;
    std::vector<int> ranks;
    int iterations = 0;
    double fit = 0.0;
    std::vector<double> sweep_fits;
    std::vector<std::string> warnings;
};

struct Basis {                 // LeftSingularBasis (linalg.hpp:35-42)
    Mat basis;
    std::vector<double> sv;
    int numerical_rank = 0;
    bool completed = false;
};

struct Svd {                   // TruncatedSvd (linalg.hpp:13-17)
    Mat left;
    std::vector<double> sv;
    Mat right;
};

// ---- RNG (proj/src/internal.hpp:68-77) -------------------------------------
std::uint64_t counter_hash64(std::uint64_t seed, std::uint64_t counter);
double counter_uniform01(std::uint64_t seed, std::uint64_t counter);

// ---- layout helpers (proj/src/tensor.cpp:15-45) -----------------------------
std::int64_t checked_size(const std::vector<int>& dims);
struct Split { std::int64_t inner = 1, outer = 1; int len = 0; };
Split split_at(const std::vector<int>& dims, int mode);

// ---- constructors with the reference's validation ---------------------------
Dense make_dense(std::vector<int> dims, std::vector<double> v);          // tensor.cpp:60-65
Sparse make_sparse(std::vector<int> dims, std::vector<Entry> entries);   // tensor.cpp:78-96

// ---- tensor ops (proj/src/tensor.cpp:149-276) -------------------------------
Mat transpose(const Mat& m);
double frobenius_norm(const Mat& m);
double tensor_norm(const Dense& t);
double tensor_norm(const Sparse& t);
Mat matricize(const Dense& t, int mode);
Dense refold(const Mat& m, int mode, const std::vector<int>& dims);
Dense mode_product(const Dense& t, const Mat& m, int mode);
Dense mode_product(const Sparse& t, const Mat& m, int mode);
Dense densify(const Sparse& s);
Sparse sparsify_exact(const Dense& t);

// ---- sampler (proj/src/sampling.cpp:15-47) ----------------------------------
Sparse sparsify(const Dense& t, double p, std::uint64_t seed);

// ---- eigen step (proj/src/linalg.cpp, linalg_internal.hpp) ------------------
// Full symmetric eigendecomposition, ascending eigenvalues (the contract of
// Eigen::SelfAdjointEigenSolver used at linalg.cpp:108); Householder
// tridiagonalisation + implicit QL.
void sym_eig(const Mat& a, std::vector<double>& evals, Mat& evecs);
Basis left_singular_basis(const Mat& m, int k);                 // linalg.cpp:319-353
Svd truncated_svd(const Mat& m, int k);                          // linalg.cpp:301-305
Mat low_rank_approx(const Mat& m, int k);                        // linalg.cpp:311-317

// ---- sparse kernels (proj/src/sparse_kernels.cpp) ---------------------------
Mat sparse_row_gram(const Sparse& t, int mode);                  // :60-63
Mat sparse_col_gram(const Sparse& t, int mode, std::int64_t cols);// :65-67
Basis sparse_mode_basis(const Sparse& t, int mode, int k);       // :82-90

// ---- Tucker (proj/src/tucker.cpp) -------------------------------------------
Model hosvd(const Dense& t, const std::vector<int>& ranks);
Model hosvd(const Sparse& t, const std::vector<int>& ranks);
Model hooi(const Dense& t, const std::vector<int>& ranks, int max_iterations, double fit_tolerance);
Model hooi(const Sparse& t, const std::vector<int>& ranks, int max_iterations, double fit_tolerance);
Dense core_tensor(const Dense& t, const std::vector<Mat>& factors);
Dense reconstruct(const Model& model);
double accuracy(const Dense& t, const Model& model);

struct MachResult { Model model; Sparse sparsified; };
MachResult mach_hosvd(const Dense& t, const std::vector<int>& ranks, double p, std::uint64_t seed);
MachResult mach_hooi(const Dense& t, const std::vector<int>& ranks, double p, std::uint64_t seed,
                     int max_iterations, double fit_tolerance);

// ---- test fixtures (proj/tests/oracles.hpp:229-262; libstdc++ streams) ----
Dense random_tensor(const std::vector<int>& dims, std::uint64_t seed);
Mat random_matrix(int rows, int cols, std::uint64_t seed);
Mat random_orthogonal(int n, std::uint64_t seed);
// Cyclic Jacobi (proj/tests/oracles.hpp:111-158): descending eigenvalues.
void jacobi_eig(const Mat& a, std::vector<double>& evals_desc, Mat& evecs);
double subspace_gap(const Mat& a, const Mat& b);                 // oracles.hpp:195-227

// ---- metrics (src/metrics.cpp:59-159) ----
struct Report {                // ComparisonReport (metrics.hpp:19-27)
    std::vector<double> rho;
    std::vector<bool> flipped, tied;
    std::vector<double> tie_sin;
    double accuracy_exact = 0.0, accuracy_mach = 0.0;
    double core_exact = 0.0, core_mach = 0.0;
};
double pearson(const std::vector<double>& x, const std::vector<double>& y);                  // :67-96
double pc_correlation(const Model& exact, const Model& approx, int mode, int component, bool* flipped);  // :98-122
Report compare(const Model& exact, const Model& approx, const Dense& reference);             // :124-159

// Per-phase timing of the last hooi() call (seconds), for the CPU baseline.
struct PhaseTimes { double sample = 0, hosvd = 0; std::vector<double> sweeps; };
PhaseTimes& last_phase_times();

}  // namespace orc
