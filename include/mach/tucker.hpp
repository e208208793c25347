// Drop-in mirror of /root/reference/proj/include/mach/tucker.hpp:14-55.
#pragma once

#include <string>
#include <vector>

#include "mach/tensor.hpp"

namespace mach {

struct TuckerModel {
    DenseTensor core;
    std::vector<Matrix> factors;
    std::vector<int> ranks;
    int iterations = 0;
    double fit = 0.0;
    std::vector<double> sweep_fits;
    std::vector<std::string> warnings;
};

struct HooiConfig {
    int max_iterations = 50;
    double fit_tolerance = 1e-4;
};

TuckerModel hosvd(const DenseTensor& t, const std::vector<int>& ranks);
TuckerModel hosvd(const SparseTensor& t, const std::vector<int>& ranks);
TuckerModel hooi(const DenseTensor& t, const std::vector<int>& ranks, const HooiConfig& cfg);
TuckerModel hooi(const SparseTensor& t, const std::vector<int>& ranks, const HooiConfig& cfg);
DenseTensor core_tensor(const DenseTensor& t, const std::vector<Matrix>& factors);
DenseTensor reconstruct(const TuckerModel& model);
double accuracy(const DenseTensor& t, const TuckerModel& model);

}  // namespace mach
