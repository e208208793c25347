// Drop-in mirror of the eigen-step entry points of
// /root/reference/proj/include/mach/linalg.hpp:35-46.
#pragma once

#include <vector>

#include "mach/tensor.hpp"

namespace mach {

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
