// Drop-in mirror of /root/reference/proj/include/mach/bounds.hpp:10-66.  The
// closed forms are host arithmetic; theorem1_bound's full mode spectra are
// computed on the B200 (mach_theorem1_bound: device Gram kernels + the
// on-device eigensolver in eigenvalues-only mode).
#pragma once

#include <cstdint>
#include <vector>

#include "mach/tensor.hpp"

namespace mach {

struct AchlioptasBounds {
    double two_norm = 0.0;
    double frobenius = 0.0;
};
AchlioptasBounds achlioptas_bounds(double b, std::int64_t n, std::int64_t k, double p);
double min_sampling_probability(const std::vector<int>& dims);

struct BoundModeReport {
    int rank = 0;
    double x_residual = 0.0;
    double xhat_residual = 0.0;
    double x_lowrank_norm = 0.0;
    double t_i = 0.0;
};

struct BoundReport {
    double b = 0.0;
    double p = 0.0;
    double p_min = 0.0;
    double t = 0.0;
    double success_probability = 0.0;
    bool dims_large_enough = false;
    bool dims_balanced = false;
    bool p_above_min = false;
    bool conditions_met = false;
    std::vector<BoundModeReport> per_mode;
};

BoundReport theorem1_conditions(const std::vector<int>& dims, double p);
BoundReport theorem1_bound(const DenseTensor& x, const SparseTensor& xhat, const std::vector<int>& ranks, double p);

}  // namespace mach
