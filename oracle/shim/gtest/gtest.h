// GoogleTest-macro shim — TEST INFRASTRUCTURE ONLY (oracle/).
//
// GoogleTest is absent from this image.  This header implements the subset of
// the gtest surface used by /root/reference/proj/tests/test_*.cpp
// (TEST, EXPECT_/ASSERT_ {EQ,NE,LT,LE,GT,GE,TRUE,FALSE,NEAR,DOUBLE_EQ,THROW,
// NO_THROW}, FAIL(), streamed messages) so the reference's own unit tests
// compile unmodified and pin the oracle build (oracle/Makefile, target
// `ref_unit_tests`).  main() lives in gtest_main.cpp.  Optional filter: argv[1]
// is a substring that test names ("Suite.Name") must contain.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace testing {

class Test {
 public:
  virtual ~Test() = default;
  virtual void SetUp() {}
  virtual void TearDown() {}
  virtual void TestBody() = 0;
};

namespace internal {

struct Registry {
  struct Entry {
    std::string suite, name;
    std::function<void()> body;
  };
  std::vector<Entry> tests;
  int failures_in_current = 0;
  static Registry& get() {
    static Registry r;
    return r;
  }
};

inline bool add_test(const char* suite, const char* name, std::function<void()> body) {
  Registry::get().tests.push_back({suite, name, std::move(body)});
  return true;
}

class Message {
 public:
  template <class T>
  Message& operator<<(const T& v) {
    ss_ << v;
    return *this;
  }
  std::string str() const { return ss_.str(); }

 private:
  std::ostringstream ss_;
};

class AssertHelper {
 public:
  AssertHelper(const char* file, int line, std::string what)
      : file_(file), line_(line), what_(std::move(what)) {}
  void operator=(const Message& m) const {
    ++Registry::get().failures_in_current;
    std::printf("%s:%d: Failure\n%s\n%s\n", file_, line_, what_.c_str(), m.str().c_str());
  }

 private:
  const char* file_;
  int line_;
  std::string what_;
};

template <class T>
std::string repr(const T& v) {
  std::ostringstream ss;
  if constexpr (requires(std::ostream& o, const T& x) { o << x; }) {
    ss.precision(17);
    ss << v;
  } else {
    ss << "<unprintable>";
  }
  return ss.str();
}

template <class A, class B>
std::string cmp_fail(const char* ea, const char* op, const char* eb, const A& a, const B& b) {
  return std::string("Expected: (") + ea + ") " + op + " (" + eb + "), actual: " + repr(a) +
         " vs " + repr(b);
}

inline bool almost_equal_ulps(double a, double b, int max_ulps = 4) {
  if (std::isnan(a) || std::isnan(b)) return false;
  if (a == b) return true;
  auto biased = [](double x) {
    std::uint64_t u;
    std::memcpy(&u, &x, sizeof u);
    const std::uint64_t sign = std::uint64_t{1} << 63;
    return (u & sign) ? ~u + 1 : u | sign;
  };
  const std::uint64_t ua = biased(a), ub = biased(b);
  const std::uint64_t diff = ua > ub ? ua - ub : ub - ua;
  return diff <= static_cast<std::uint64_t>(max_ulps);
}

}  // namespace internal
}  // namespace testing

#define GTEST_SHIM_CAT_(a, b) a##b
#define GTEST_SHIM_CAT(a, b) GTEST_SHIM_CAT_(a, b)

#define TEST(suite, name)                                                                  \
  static void GTEST_SHIM_CAT(gtest_body_, GTEST_SHIM_CAT(suite, GTEST_SHIM_CAT(_, name)))(); \
  static const bool GTEST_SHIM_CAT(gtest_reg_, GTEST_SHIM_CAT(suite, GTEST_SHIM_CAT(_, name))) = \
      ::testing::internal::add_test(                                                       \
          #suite, #name, GTEST_SHIM_CAT(gtest_body_, GTEST_SHIM_CAT(suite, GTEST_SHIM_CAT(_, name)))); \
  static void GTEST_SHIM_CAT(gtest_body_, GTEST_SHIM_CAT(suite, GTEST_SHIM_CAT(_, name)))()

#define GTEST_SHIM_CHECK_(cond, text, on_fail) \
  if (cond)                                    \
    ;                                          \
  else                                         \
    on_fail ::testing::internal::AssertHelper(__FILE__, __LINE__, text) = ::testing::internal::Message()

#define GTEST_SHIM_NONFATAL_
#define GTEST_SHIM_FATAL_ return

#define GTEST_SHIM_CMP_(a, b, op, opname, kind)                                                   \
  GTEST_SHIM_CHECK_(((a)op(b)), ::testing::internal::cmp_fail(#a, opname, #b, (a), (b)), kind)

#define EXPECT_EQ(a, b) GTEST_SHIM_CMP_(a, b, ==, "==", GTEST_SHIM_NONFATAL_)
#define EXPECT_NE(a, b) GTEST_SHIM_CMP_(a, b, !=, "!=", GTEST_SHIM_NONFATAL_)
#define EXPECT_LT(a, b) GTEST_SHIM_CMP_(a, b, <, "<", GTEST_SHIM_NONFATAL_)
#define EXPECT_LE(a, b) GTEST_SHIM_CMP_(a, b, <=, "<=", GTEST_SHIM_NONFATAL_)
#define EXPECT_GT(a, b) GTEST_SHIM_CMP_(a, b, >, ">", GTEST_SHIM_NONFATAL_)
#define EXPECT_GE(a, b) GTEST_SHIM_CMP_(a, b, >=, ">=", GTEST_SHIM_NONFATAL_)
#define ASSERT_EQ(a, b) GTEST_SHIM_CMP_(a, b, ==, "==", GTEST_SHIM_FATAL_)
#define ASSERT_NE(a, b) GTEST_SHIM_CMP_(a, b, !=, "!=", GTEST_SHIM_FATAL_)
#define ASSERT_LT(a, b) GTEST_SHIM_CMP_(a, b, <, "<", GTEST_SHIM_FATAL_)
#define ASSERT_LE(a, b) GTEST_SHIM_CMP_(a, b, <=, "<=", GTEST_SHIM_FATAL_)
#define ASSERT_GT(a, b) GTEST_SHIM_CMP_(a, b, >, ">", GTEST_SHIM_FATAL_)
#define ASSERT_GE(a, b) GTEST_SHIM_CMP_(a, b, >=, ">=", GTEST_SHIM_FATAL_)

#define EXPECT_TRUE(c) GTEST_SHIM_CHECK_(static_cast<bool>(c), "Expected true: " #c, GTEST_SHIM_NONFATAL_)
#define EXPECT_FALSE(c) GTEST_SHIM_CHECK_(!static_cast<bool>(c), "Expected false: " #c, GTEST_SHIM_NONFATAL_)
#define ASSERT_TRUE(c) GTEST_SHIM_CHECK_(static_cast<bool>(c), "Expected true: " #c, GTEST_SHIM_FATAL_)
#define ASSERT_FALSE(c) GTEST_SHIM_CHECK_(!static_cast<bool>(c), "Expected false: " #c, GTEST_SHIM_FATAL_)

#define EXPECT_NEAR(a, b, tol)                                                              \
  GTEST_SHIM_CHECK_(std::fabs(static_cast<double>(a) - static_cast<double>(b)) <= (tol),   \
                    ::testing::internal::cmp_fail(#a, "near", #b, (a), (b)) + " tol " #tol, \
                    GTEST_SHIM_NONFATAL_)
#define ASSERT_NEAR(a, b, tol)                                                              \
  GTEST_SHIM_CHECK_(std::fabs(static_cast<double>(a) - static_cast<double>(b)) <= (tol),   \
                    ::testing::internal::cmp_fail(#a, "near", #b, (a), (b)) + " tol " #tol, \
                    GTEST_SHIM_FATAL_)
#define EXPECT_DOUBLE_EQ(a, b)                                                                  \
  GTEST_SHIM_CHECK_(::testing::internal::almost_equal_ulps(static_cast<double>(a),              \
                                                           static_cast<double>(b)),             \
                    ::testing::internal::cmp_fail(#a, "~=", #b, (a), (b)), GTEST_SHIM_NONFATAL_)
#define ASSERT_DOUBLE_EQ(a, b)                                                                  \
  GTEST_SHIM_CHECK_(::testing::internal::almost_equal_ulps(static_cast<double>(a),              \
                                                           static_cast<double>(b)),             \
                    ::testing::internal::cmp_fail(#a, "~=", #b, (a), (b)), GTEST_SHIM_FATAL_)

#define GTEST_SHIM_THROWS_(stmt, exc, kind)                 \
  GTEST_SHIM_CHECK_(([&]() -> bool {                        \
                      try {                                 \
                        stmt;                               \
                      } catch (const exc&) {                \
                        return true;                        \
                      } catch (...) {                       \
                        return false;                       \
                      }                                     \
                      return false;                         \
                    }()),                                   \
                    "Expected " #stmt " to throw " #exc, kind)
#define EXPECT_THROW(stmt, exc) GTEST_SHIM_THROWS_(stmt, exc, GTEST_SHIM_NONFATAL_)
#define ASSERT_THROW(stmt, exc) GTEST_SHIM_THROWS_(stmt, exc, GTEST_SHIM_FATAL_)
#define EXPECT_NO_THROW(stmt)                                                                \
  GTEST_SHIM_CHECK_(([&]() -> bool {                                                         \
                      try {                                                                  \
                        stmt;                                                                \
                      } catch (...) {                                                        \
                        return false;                                                        \
                      }                                                                      \
                      return true;                                                           \
                    }()),                                                                    \
                    "Expected " #stmt " not to throw", GTEST_SHIM_NONFATAL_)

#define FAIL() GTEST_SHIM_CHECK_(false, "Failure", GTEST_SHIM_FATAL_)
#define ADD_FAILURE() GTEST_SHIM_CHECK_(false, "Failure", GTEST_SHIM_NONFATAL_)
