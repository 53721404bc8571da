// Minimal GoogleTest-compatible shim (GTest is not installed in this image).
// Enough of the gtest surface to compile the reference's kv_cache_test.cpp
// UNMODIFIED, both against the reference header and against our drop-in.
// Output: one line per test, "[ PASS ] Suite.Name" / "[ FAIL ] Suite.Name",
// each failure as "FAILURE file:line: <expr> | <values> <message>".
#pragma once
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <type_traits>
#include <vector>

namespace shimtest {

struct TestCase {
  const char* suite;
  const char* name;
  std::function<void()> fn;
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
inline bool& current_failed() {
  static bool f = false;
  return f;
}

struct Registrar {
  Registrar(const char* s, const char* n, std::function<void()> f) {
    registry().push_back({s, n, std::move(f)});
  }
};

template <typename T, typename = void>
struct printable : std::false_type {};
template <typename T>
struct printable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>>
    : std::true_type {};

template <typename T>
std::string show(const T& v) {
  if constexpr (printable<T>::value) {
    std::ostringstream os;
    os.precision(17);
    os << v;
    return os.str();
  } else {
    return "<unprintable>";
  }
}

// Collects "<< msg" and reports on destruction of the temporary.
struct Failure {
  std::ostringstream msg;
  std::string head;
  Failure(const char* file, int line, const std::string& what) {
    std::ostringstream h;
    h << "FAILURE " << file << ":" << line << ": " << what;
    head = h.str();
  }
  template <typename T>
  Failure& operator<<(const T& v) {
    msg << v;
    return *this;
  }
  ~Failure() {
    current_failed() = true;
    std::cout << head;
    const std::string m = msg.str();
    if (!m.empty()) std::cout << " | msg: " << m;
    std::cout << std::endl;
  }
};

// `return Voidify() = Failure(...) << ...;` makes ASSERT_* return from a void test.
struct Voidify {
  void operator=(const Failure&) {}
};

template <typename A, typename B>
std::string cmp_msg(const char* ea, const char* eb, const A& a, const B& b, const char* op) {
  return std::string(ea) + " " + op + " " + eb + " | lhs=" + show(a) + " rhs=" + show(b);
}

inline bool double_eq(double a, double b) {
  if (a == b) return true;
  // 4 ULPs, as gtest's EXPECT_DOUBLE_EQ
  const double diff = std::fabs(a - b);
  const double scale = std::fmax(std::fabs(a), std::fabs(b));
  return diff <= scale * 4 * 2.220446049250313e-16;
}

inline int run_all() {
  int failed = 0, passed = 0;
  for (auto& t : registry()) {
    current_failed() = false;
    try {
      t.fn();
    } catch (const std::exception& e) {
      std::cout << "FAILURE uncaught exception: " << e.what() << std::endl;
      current_failed() = true;
    }
    if (current_failed()) {
      ++failed;
      std::cout << "[ FAIL ] " << t.suite << "." << t.name << std::endl;
    } else {
      ++passed;
      std::cout << "[ PASS ] " << t.suite << "." << t.name << std::endl;
    }
  }
  std::cout << "SUMMARY passed=" << passed << " failed=" << failed << std::endl;
  return failed ? 1 : 0;
}

}  // namespace shimtest

#define SHIM_CAT2(a, b) a##b
#define SHIM_CAT(a, b) SHIM_CAT2(a, b)

#define TEST(suite, name)                                                         \
  static void SHIM_CAT(shim_test_, SHIM_CAT(suite, SHIM_CAT(_, name)))();         \
  static ::shimtest::Registrar SHIM_CAT(shim_reg_, SHIM_CAT(suite, SHIM_CAT(_, name)))( \
      #suite, #name, &SHIM_CAT(shim_test_, SHIM_CAT(suite, SHIM_CAT(_, name))));  \
  static void SHIM_CAT(shim_test_, SHIM_CAT(suite, SHIM_CAT(_, name)))()

#define SHIM_CHECK_0(cond, what) \
  if (cond)                       \
    ;                             \
  else                            \
    ::shimtest::Failure(__FILE__, __LINE__, what)
#define SHIM_CHECK_1(cond, what) \
  if (cond)                       \
    ;                             \
  else                            \
    return ::shimtest::Voidify() = ::shimtest::Failure(__FILE__, __LINE__, what)
#define SHIM_CHECK(cond, what, fatal) SHIM_CAT(SHIM_CHECK_, fatal)(cond, what)

#define SHIM_BIN(a, b, op, fatal)                                                       \
  SHIM_CHECK(((a)op(b)), ::shimtest::cmp_msg(#a, #b, (a), (b), #op), fatal)

#define EXPECT_TRUE(c) SHIM_CHECK(static_cast<bool>(c), std::string(#c " is false"), 0)
#define EXPECT_FALSE(c) SHIM_CHECK(!static_cast<bool>(c), std::string(#c " is true"), 0)
#define ASSERT_TRUE(c) SHIM_CHECK(static_cast<bool>(c), std::string(#c " is false"), 1)
#define ASSERT_FALSE(c) SHIM_CHECK(!static_cast<bool>(c), std::string(#c " is true"), 1)
#define EXPECT_EQ(a, b) SHIM_BIN(a, b, ==, 0)
#define EXPECT_NE(a, b) SHIM_BIN(a, b, !=, 0)
#define EXPECT_LT(a, b) SHIM_BIN(a, b, <, 0)
#define EXPECT_LE(a, b) SHIM_BIN(a, b, <=, 0)
#define EXPECT_GT(a, b) SHIM_BIN(a, b, >, 0)
#define EXPECT_GE(a, b) SHIM_BIN(a, b, >=, 0)
#define ASSERT_EQ(a, b) SHIM_BIN(a, b, ==, 1)
#define ASSERT_NE(a, b) SHIM_BIN(a, b, !=, 1)
#define ASSERT_LT(a, b) SHIM_BIN(a, b, <, 1)
#define ASSERT_LE(a, b) SHIM_BIN(a, b, <=, 1)
#define ASSERT_GT(a, b) SHIM_BIN(a, b, >, 1)
#define ASSERT_GE(a, b) SHIM_BIN(a, b, >=, 1)
#define EXPECT_DOUBLE_EQ(a, b) \
  SHIM_CHECK(::shimtest::double_eq((a), (b)), ::shimtest::cmp_msg(#a, #b, (a), (b), "~="), 0)
#define ASSERT_DOUBLE_EQ(a, b) \
  SHIM_CHECK(::shimtest::double_eq((a), (b)), ::shimtest::cmp_msg(#a, #b, (a), (b), "~="), 1)

#define SHIM_THROW(stmt, exc, fatal)                                          \
  {                                                                           \
    bool shim_caught_ = false;                                                \
    try {                                                                     \
      stmt;                                                                   \
    } catch (const exc&) {                                                    \
      shim_caught_ = true;                                                    \
    } catch (...) {                                                           \
    }                                                                         \
    SHIM_CHECK(shim_caught_, std::string(#stmt " does not throw " #exc), fatal); \
  }
#define EXPECT_THROW(stmt, exc) SHIM_THROW(stmt, exc, 0)
#define ASSERT_THROW(stmt, exc) SHIM_THROW(stmt, exc, 1)

int main() { return ::shimtest::run_all(); }
