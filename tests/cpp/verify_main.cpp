// verify_main.cpp -- runs the reference's verify suites (proj/src/verify.cpp,
// compiled unmodified with b200_swap.hpp force-included, so its flash calls
// run on the B200 drop-in) and prints one line per check.  Exit code 0 iff
// every check passed.  Test infrastructure.
#include <cstdio>

#include "flashsvd/verify.hpp"
#include "flashsvd_b200/flashsvd_b200.hpp"

int main(int argc, char** argv) {
  if (argc > 1 && argv[1][0] == 'b') flashsvd::b200::set_precision(FSVD_BF16);
  int failed = 0, passed = 0;
  for (const flashsvd::SuiteReport& r : flashsvd::run_all_verify_suites(20260822)) {
    for (const auto& c : r.checks) {
      std::printf("[%s] %s: %s %s\n", c.passed ? "PASS" : "FAIL", r.suite.c_str(), c.name.c_str(),
                  c.detail.c_str());
      (c.passed ? passed : failed)++;
    }
  }
  std::printf("verify (b200 drop-in): %d passed, %d failed\n", passed, failed);
  return failed == 0 ? 0 : 1;
}
