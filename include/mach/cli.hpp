// Mirror of /root/reference/proj/include/mach/cli.hpp:7-16: the command-line
// tool wired to the B200 backend (tools/mach_cli.cpp builds `mach_b200`).
#pragma once

#include <string>
#include <vector>

namespace mach {

/// Exit codes as the reference: 0 ok, 2 usage, 3 data errors, 4 convergence.
int run_cli(const std::vector<std::string>& args);

}  // namespace mach
