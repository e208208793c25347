// Drop-in mirror of /root/reference/proj/include/mach/sampling.hpp:14-36.
#pragma once

#include <cstdint>
#include <vector>

#include "mach/tensor.hpp"
#include "mach/tucker.hpp"

namespace mach {

struct SparsifyConfig {
    double p = 1.0;
    std::uint64_t seed = 0;
};

SparseTensor sparsify(const DenseTensor& t, const SparsifyConfig& cfg);

struct MachResult {
    TuckerModel model;
    SparseTensor sparsified;
};

MachResult mach_hosvd(const DenseTensor& t, const std::vector<int>& ranks, const SparsifyConfig& cfg);
MachResult mach_hooi(const DenseTensor& t, const std::vector<int>& ranks, const SparsifyConfig& scfg,
                     const HooiConfig& hcfg);

}  // namespace mach
