// Stand-in for proj/src/cli.cpp (cli_main, proj/include/metagrad/cli.hpp:7),
// which needs CLI11 (absent from the reference checkout and this image).
// Only the CLI test cases and acceptance criterion 10 call it; they are
// excluded from the oracle/_ref test runs.  Test infrastructure only.
#include <cstdio>

#include "metagrad/cli.hpp"

namespace metagrad {
int cli_main(int, const char* const*) {
  std::fprintf(stderr, "metagrad CLI unavailable in oracle/_ref (CLI11 absent)\n");
  return 1;
}
}  // namespace metagrad
