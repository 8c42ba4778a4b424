// catch_main.cpp -- TEST INFRASTRUCTURE ONLY: runner of the Catch2 shim.
// Prints one line per failing test case and a Catch2-style summary; exit 0
// iff every assertion passed.
#include <cstdio>

#include "catch2/catch_amalgamated.hpp"

int main() {
  long cases = 0, failed_cases = 0;
  for (const auto& tc : Catch::registry()) {
    ++cases;
    Catch::stats().case_failed = false;
    try {
      tc.fn();
    } catch (const Catch::RequireAbort&) {
    } catch (const std::exception& e) {
      std::printf("  FAILED %s:%d: unexpected exception: %s\n", tc.file, tc.line, e.what());
      ++Catch::stats().failed;
      Catch::stats().case_failed = true;
    }
    if (Catch::stats().case_failed) {
      ++failed_cases;
      std::printf("test case FAILED: %s\n", tc.name.c_str());
    }
    std::fflush(stdout);
  }
  const auto& s = Catch::stats();
  if (failed_cases == 0)
    std::printf("All tests passed (%ld assertions in %ld test cases)\n", s.assertions, cases);
  else
    std::printf("test cases: %ld | %ld passed | %ld failed\nassertions: %ld | %ld passed | %ld failed\n",
                cases, cases - failed_cases, failed_cases, s.assertions, s.assertions - s.failed,
                s.failed);
  return failed_cases == 0 ? 0 : 1;
}
