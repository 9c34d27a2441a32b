// Runs the reference's own validation suite (proj/src/validation.cpp:262-299)
// built against the Eigen shim.  Test infrastructure only.
#include <cstdio>
#include <cstdlib>

#include "metagrad/validation.hpp"

int main(int argc, char** argv) {
  const auto seed = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 20240801ULL;
  const auto results = metagrad::run_validation_suite(seed);
  int failed = 0;
  for (const auto& r : results) {
    std::printf("[%s] %s: %s\n", r.pass ? "PASS" : "FAIL", r.name.c_str(), r.detail.c_str());
    failed += r.pass ? 0 : 1;
  }
  std::printf("%zu checks, %d failed\n", results.size(), failed);
  return failed == 0 ? 0 : 1;
}
