// GoogleTest-shim runner — TEST INFRASTRUCTURE ONLY (oracle/).
// Runs every TEST registered by the linked reference test files; argv[1]
// (optional) filters on "Suite.Name" substring.  Exit 1 if any test failed.
#include <gtest/gtest.h>

#include <chrono>

int main(int argc, char** argv) {
  auto& reg = ::testing::internal::Registry::get();
  const std::string filter = argc > 1 ? argv[1] : "";
  int failed = 0, ran = 0;
  for (auto& t : reg.tests) {
    const std::string full = t.suite + "." + t.name;
    if (!filter.empty() && full.find(filter) == std::string::npos) continue;
    reg.failures_in_current = 0;
    const auto start = std::chrono::steady_clock::now();
    try {
      t.body();
    } catch (const std::exception& e) {
      ++reg.failures_in_current;
      std::printf("uncaught exception: %s\n", e.what());
    } catch (...) {
      ++reg.failures_in_current;
      std::printf("uncaught non-std exception\n");
    }
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - start).count();
    ++ran;
    if (reg.failures_in_current) {
      ++failed;
      std::printf("[  FAILED  ] %s (%.0f ms)\n", full.c_str(), ms);
    } else {
      std::printf("[       OK ] %s (%.0f ms)\n", full.c_str(), ms);
    }
    std::fflush(stdout);
  }
  std::printf("[==========] %d tests ran, %d failed\n", ran, failed);
  return failed ? 1 : 0;
}
