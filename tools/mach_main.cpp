// `mach_b200`: the command-line tool over libmach_b200.so (mach::run_cli,
// include/mach/cli.hpp).  Build: make -C paper_0909_4969_b200 cli
#include <string>
#include <vector>

#include "mach/cli.hpp"

int main(int argc, char** argv) { return mach::run_cli(std::vector<std::string>(argv + 1, argv + argc)); }
