// Drop-in mirror of /root/reference/proj/include/mach/metrics.hpp:11-46
// (ComparisonReport, pearson, pc_correlation, compare).  The accuracies run
// as one fused pass on the B200 (mach_model_accuracy), the subspace sines on
// the device (mach_subspace_sin); the O(I_n) correlations are host arithmetic
// in the reference's pairwise summation order.
#pragma once

#include <span>
#include <utility>
#include <vector>

#include "mach/tensor.hpp"
#include "mach/tucker.hpp"

namespace mach {

struct ComparisonReport {
    std::vector<double> per_mode_rho;
    std::vector<bool> flipped;
    std::vector<bool> tied;
    std::vector<double> tie_subspace_sin;
    double accuracy_exact = 0.0;
    double accuracy_mach = 0.0;
    std::pair<double, double> core_interaction{0.0, 0.0};
};

double pearson(std::span<const double> x, std::span<const double> y);
double pc_correlation(const TuckerModel& exact, const TuckerModel& approx, int mode, int component = 1,
                      bool* flipped = nullptr);
ComparisonReport compare(const TuckerModel& exact, const TuckerModel& approx, const DenseTensor& reference);

}  // namespace mach
