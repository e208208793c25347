// Drop-in mirror of /root/reference/proj/include/mach/linalg.hpp:11-46
// (truncated SVD family, left_singular_basis, set_thread_count).
#pragma once

#include <vector>

#include "mach/tensor.hpp"

namespace mach {

// Top-k singular triplets (linalg.hpp:11-17): left rows x k, right cols x k,
// orthonormal columns, non-increasing singular values.
struct TruncatedSvd {
    Matrix left;
    std::vector<double> singular_values;
    Matrix right;
};

// linalg.hpp:19-30: 1 <= k <= min(rows, cols); the largest-magnitude entry of
// each left vector is nonnegative (lowest index on ties), the right follows.
TruncatedSvd truncated_svd(const Matrix& m, int k);
Matrix leading_left_singular_vectors(const Matrix& m, int k);
Matrix low_rank_approx(const Matrix& m, int k);

struct LeftSingularBasis {
    Matrix basis;
    std::vector<double> singular_values;
    int numerical_rank = 0;
    bool completed = false;
};

LeftSingularBasis left_singular_basis(const Matrix& m, int k);

// Device work is single-stream; kept for source compatibility (the reference
// maps it to Eigen::setNbThreads, linalg.cpp:355).
void set_thread_count(int n);

}  // namespace mach
