// ORACLE SHIM — test infrastructure only.
// The subset of GoogleTest the reference's tests use (TEST, EXPECT_* /
// ASSERT_* comparisons, NEAR / DOUBLE_EQ, THROW / NO_THROW, GTEST_SKIP, and
// `<< message` streaming), so /root/reference/proj/tests/*.cpp compile
// unchanged here without a GTest install. Run with an
// optional substring filter: ./test_mpm [--gtest_filter=Suite.Name*]
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <type_traits>
#include <vector>

namespace gts {

struct TestCase {
  const char* suite;
  const char* name;
  std::function<void()> fn;
};
inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
struct State {
  bool failed = false;
  bool skipped = false;
};
inline State& state() {
  static State s;
  return s;
}
struct Registrar {
  Registrar(const char* s, const char* n, std::function<void()> f) { registry().push_back({s, n, std::move(f)}); }
};

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

struct AssertHelper {
  const char* file;
  int line;
  std::string text;
  int kind;  // 0 failure, 1 skip
  void operator=(const Message& m) const {
    if (kind == 1) {
      state().skipped = true;
      std::cout << "  [ SKIPPED ] " << file << ":" << line << " " << m.str() << "\n";
      return;
    }
    state().failed = true;
    std::cout << "  " << file << ":" << line << ": Failure\n    " << text;
    if (!m.str().empty()) std::cout << "\n    " << m.str();
    std::cout << "\n";
  }
};

template <class T, class = void>
struct Printable : std::false_type {};
template <class T>
struct Printable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>> : std::true_type {};
template <class T>
std::string show(const T& v) {
  if constexpr (std::is_enum_v<T>) {
    return std::to_string(static_cast<long long>(v));
  } else if constexpr (Printable<T>::value) {
    std::ostringstream s;
    s.precision(17);
    s << v;
    return s.str();
  } else {
    return "<unprintable>";
  }
}

template <class A, class B>
std::string cmp_text(const char* op, const char* ea, const char* eb, const A& a, const B& b) {
  return std::string("Expected: (") + ea + ") " + op + " (" + eb + "), actual: " + show(a) + " vs " + show(b);
}

inline bool double_eq(double a, double b) {  // within 4 ULPs (GoogleTest's AlmostEquals)
  if (std::isnan(a) || std::isnan(b)) return false;
  auto biased = [](double x) {
    std::uint64_t u;
    std::memcpy(&u, &x, sizeof u);
    const std::uint64_t sign = 1ull << 63;
    return (u & sign) ? ~u + 1 : (u | sign);
  };
  const std::uint64_t ua = biased(a), ub = biased(b);
  return (ua >= ub ? ua - ub : ub - ua) <= 4;
}

inline int run_all(int argc, char** argv) {
  std::string filter;
  for (int i = 1; i < argc; ++i)
    if (std::strncmp(argv[i], "--gtest_filter=", 15) == 0) filter = argv[i] + 15;
  auto match = [&](const std::string& full) {
    if (filter.empty()) return true;
    std::string f = filter;
    bool prefix = !f.empty() && f.back() == '*';
    if (prefix) f.pop_back();
    return prefix ? full.compare(0, f.size(), f) == 0 : full == f;
  };
  int run = 0, failed = 0, skipped = 0;
  std::vector<std::string> failures;
  for (const TestCase& t : registry()) {
    const std::string full = std::string(t.suite) + "." + t.name;
    if (!match(full)) continue;
    state() = State{};
    std::cout << "[ RUN      ] " << full << std::endl;
    try {
      t.fn();
    } catch (const std::exception& e) {
      state().failed = true;
      std::cout << "  uncaught exception: " << e.what() << "\n";
    } catch (...) {
      state().failed = true;
      std::cout << "  uncaught non-std exception\n";
    }
    ++run;
    if (state().failed) {
      ++failed;
      failures.push_back(full);
      std::cout << "[  FAILED  ] " << full << std::endl;
    } else if (state().skipped) {
      ++skipped;
      std::cout << "[  SKIPPED ] " << full << std::endl;
    } else {
      std::cout << "[       OK ] " << full << std::endl;
    }
  }
  std::cout << "[==========] " << run << " tests ran.\n[  PASSED  ] " << (run - failed - skipped) << " tests.\n";
  if (skipped) std::cout << "[  SKIPPED ] " << skipped << " tests.\n";
  if (failed) {
    std::cout << "[  FAILED  ] " << failed << " tests, listed below:\n";
    for (const auto& f : failures) std::cout << "[  FAILED  ] " << f << "\n";
  }
  return failed ? 1 : 0;
}

}  // namespace gts

namespace testing {
inline void InitGoogleTest(int*, char**) {}
inline std::string TempDir() { return "/tmp/"; }
}  // namespace testing
#define SCOPED_TRACE(msg) ((void)0)
#define FAIL() return ::gts::AssertHelper{__FILE__, __LINE__, "Failed", 0} = ::gts::Message()
#define ADD_FAILURE() ::gts::AssertHelper{__FILE__, __LINE__, "Failed", 0} = ::gts::Message()
#define RUN_ALL_TESTS() ::gts::run_all(gts_argc_, gts_argv_)

#define GTS_CAT2(a, b) a##b
#define GTS_CAT(a, b) GTS_CAT2(a, b)
#define TEST(suite, name)                                                                    \
  static void GTS_CAT(GTS_CAT(gts_test_, suite), GTS_CAT(_, name))();                        \
  static ::gts::Registrar GTS_CAT(GTS_CAT(gts_reg_, suite), GTS_CAT(_, name))(               \
      #suite, #name, &GTS_CAT(GTS_CAT(gts_test_, suite), GTS_CAT(_, name)));                 \
  static void GTS_CAT(GTS_CAT(gts_test_, suite), GTS_CAT(_, name))()

#define GTS_FAIL_IF_NOT(cond, text, fatal)                                                     \
  switch (0)                                                                                   \
  case 0:                                                                                      \
  default:                                                                                     \
    if (cond)                                                                                  \
      ;                                                                                        \
    else                                                                                       \
      GTS_CAT(GTS_RET_, fatal)::gts::AssertHelper{__FILE__, __LINE__, (text), 0} = ::gts::Message()
#define GTS_RET_0
#define GTS_RET_1 return

#define GTS_CMP(a, b, op, fatal)                                                               \
  GTS_FAIL_IF_NOT(((a)op(b)), ::gts::cmp_text(#op, #a, #b, (a), (b)), fatal)
#define EXPECT_EQ(a, b) GTS_CMP(a, b, ==, 0)
#define EXPECT_NE(a, b) GTS_CMP(a, b, !=, 0)
#define EXPECT_LT(a, b) GTS_CMP(a, b, <, 0)
#define EXPECT_LE(a, b) GTS_CMP(a, b, <=, 0)
#define EXPECT_GT(a, b) GTS_CMP(a, b, >, 0)
#define EXPECT_GE(a, b) GTS_CMP(a, b, >=, 0)
#define ASSERT_EQ(a, b) GTS_CMP(a, b, ==, 1)
#define ASSERT_NE(a, b) GTS_CMP(a, b, !=, 1)
#define ASSERT_LT(a, b) GTS_CMP(a, b, <, 1)
#define ASSERT_LE(a, b) GTS_CMP(a, b, <=, 1)
#define ASSERT_GT(a, b) GTS_CMP(a, b, >, 1)
#define ASSERT_GE(a, b) GTS_CMP(a, b, >=, 1)
#define EXPECT_TRUE(c) GTS_FAIL_IF_NOT(static_cast<bool>(c), std::string("Expected true: ") + #c, 0)
#define EXPECT_FALSE(c) GTS_FAIL_IF_NOT(!static_cast<bool>(c), std::string("Expected false: ") + #c, 0)
#define ASSERT_TRUE(c) GTS_FAIL_IF_NOT(static_cast<bool>(c), std::string("Expected true: ") + #c, 1)
#define ASSERT_FALSE(c) GTS_FAIL_IF_NOT(!static_cast<bool>(c), std::string("Expected false: ") + #c, 1)
#define EXPECT_NEAR(a, b, tol)                                                                 \
  GTS_FAIL_IF_NOT(std::abs((a) - (b)) <= (tol),                                                \
                  ::gts::cmp_text("~=", #a, #b, (a), (b)) + " tol " + ::gts::show(tol), 0)
#define ASSERT_NEAR(a, b, tol)                                                                 \
  GTS_FAIL_IF_NOT(std::abs((a) - (b)) <= (tol),                                                \
                  ::gts::cmp_text("~=", #a, #b, (a), (b)) + " tol " + ::gts::show(tol), 1)
#define EXPECT_DOUBLE_EQ(a, b) GTS_FAIL_IF_NOT(::gts::double_eq((a), (b)), ::gts::cmp_text("==(4ulp)", #a, #b, (a), (b)), 0)
#define ASSERT_DOUBLE_EQ(a, b) GTS_FAIL_IF_NOT(::gts::double_eq((a), (b)), ::gts::cmp_text("==(4ulp)", #a, #b, (a), (b)), 1)

#define GTS_THROWS(stmt, exc, fatal)                                                           \
  GTS_FAIL_IF_NOT(([&]() -> bool {                                                             \
                    try {                                                                      \
                      stmt;                                                                    \
                    } catch (const exc&) {                                                     \
                      return true;                                                             \
                    } catch (...) {                                                            \
                      return false;                                                            \
                    }                                                                          \
                    return false;                                                              \
                  })(),                                                                        \
                  std::string("Expected ") + #stmt + " to throw " + #exc, fatal)
#define EXPECT_THROW(stmt, exc) GTS_THROWS(stmt, exc, 0)
#define ASSERT_THROW(stmt, exc) GTS_THROWS(stmt, exc, 1)
#define EXPECT_NO_THROW(stmt)                                                                  \
  GTS_FAIL_IF_NOT(([&]() -> bool {                                                             \
                    try {                                                                      \
                      stmt;                                                                    \
                    } catch (...) {                                                            \
                      return false;                                                            \
                    }                                                                          \
                    return true;                                                               \
                  })(),                                                                        \
                  std::string("Expected ") + #stmt + " not to throw", 0)
#define GTEST_SKIP() return ::gts::AssertHelper{__FILE__, __LINE__, "", 1} = ::gts::Message()
