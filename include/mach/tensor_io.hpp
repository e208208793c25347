// Mirror of /root/reference/proj/include/mach/tensor_io.hpp:11-47.  The text
// formats are kept for interchange with the reference (same grammar, value
// exact); read_tensor / write_tensor also take the binary MACHB2 format
// (mach_b200.h) that the GPU backend loads straight into HBM —
// chosen by content on read and by the ".machb" suffix on write.
#pragma once

#include <string>
#include <variant>

#include "mach/bounds.hpp"
#include "mach/metrics.hpp"
#include "mach/tensor.hpp"
#include "mach/tucker.hpp"

namespace mach {

std::string format_double(double v);

using AnyTensor = std::variant<DenseTensor, SparseTensor>;

AnyTensor read_tensor(const std::string& path);
void write_tensor(const DenseTensor& t, const std::string& path);
void write_tensor(const SparseTensor& t, const std::string& path);

Matrix read_matrix(const std::string& path);
void write_matrix(const Matrix& m, const std::string& path);

void save_model(const TuckerModel& model, const std::string& dir);
TuckerModel load_model(const std::string& dir);

std::string render_bound_report(const BoundReport& rep);
std::string render_comparison_report(const ComparisonReport& rep);
void write_bound_report(const BoundReport& rep, const std::string& path);
void write_comparison_report(const ComparisonReport& rep, const std::string& path);

}  // namespace mach
