// Minimal GoogleTest-compatible shim (TEST, EXPECT_* / ASSERT_* with message
// streaming, SUCCEED, testing::TempDir, --gtest_filter) so that the
// reference's own test files (/root/reference/proj/tests/*.cpp) compile
// unchanged against this repository's include/ttsvd/ headers.  Test
// infrastructure only; GoogleTest itself is not installed in this image.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace gtshim {

struct Case {
    std::string suite, name;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
inline bool& current_failed() {
    static bool f = false;
    return f;
}
struct Registrar {
    Registrar(const char* s, const char* n, void (*fn)()) { registry().push_back({s, n, fn}); }
};

// printable form of a value (containers element-wise, else operator<<)
template <class T, class = void>
struct streamable : std::false_type {};
template <class T>
struct streamable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>> : std::true_type {};
template <class T, class = void>
struct iterable : std::false_type {};
template <class T>
struct iterable<T, std::void_t<decltype(std::declval<const T&>().begin()), decltype(std::declval<const T&>().end())>>
    : std::true_type {};

template <class T>
std::string show(const T& v) {
    std::ostringstream o;
    if constexpr (std::is_same_v<T, std::string>) {
        o << '"' << v << '"';
    } else if constexpr (streamable<T>::value) {
        o.precision(17);
        o << v;
    } else if constexpr (iterable<T>::value) {
        o << '{';
        bool first = true;
        for (const auto& x : v) {
            o << (first ? "" : ", ") << show(x);
            first = false;
        }
        o << '}';
    } else {
        o << "<value>";
    }
    return o.str();
}

struct Result {
    bool ok = true;
    std::string why;
    explicit operator bool() const { return ok; }
};
inline Result pass() { return {}; }
inline Result failed(std::string why) { return {false, std::move(why)}; }

struct Msg {
    std::ostringstream s;
    Msg() = default;
    Msg(const Msg& o) { s << o.s.str(); }
    template <class T>
    Msg& operator<<(const T& v) {
        s << v;
        return *this;
    }
};

struct Reporter {
    const char* file;
    int line;
    const Result& r;
    void operator=(const Msg& m) const {
        current_failed() = true;
        std::printf("%s:%d: Failure\n%s\n", file, line, r.why.c_str());
        const std::string extra = m.s.str();
        if (!extra.empty()) std::printf("%s\n", extra.c_str());
    }
};

#define GTSHIM_BINARY(name, op)                                                                       \
    template <class A, class B>                                                                       \
    Result name(const char* ea, const char* eb, const A& a, const B& b) {                             \
        if (a op b) return pass();                                                                    \
        return failed(std::string("Expected: (") + ea + ") " #op " (" + eb + "), actual: " + show(a) + \
                      " vs " + show(b));                                                              \
    }
GTSHIM_BINARY(cmp_eq, ==)
GTSHIM_BINARY(cmp_ne, !=)
GTSHIM_BINARY(cmp_lt, <)
GTSHIM_BINARY(cmp_le, <=)
GTSHIM_BINARY(cmp_gt, >)
GTSHIM_BINARY(cmp_ge, >=)
#undef GTSHIM_BINARY

inline Result cmp_near(const char* ea, const char* eb, const char* et, double a, double b, double tol) {
    if (std::fabs(a - b) <= tol) return pass();
    return failed(std::string("The difference between ") + ea + " and " + eb + " is " + show(std::fabs(a - b)) +
                  ", which exceeds " + et + " (" + show(tol) + "); values " + show(a) + " and " + show(b));
}

inline Result cmp_double_eq(const char* ea, const char* eb, double a, double b) {
    // within 4 ULPs, as GoogleTest
    if (a == b) return pass();
    const double tol = 4 * std::fabs(std::nextafter(a, b) - a);
    if (std::fabs(a - b) <= tol) return pass();
    return failed(std::string("Expected equality of ") + ea + " and " + eb + ": " + show(a) + " vs " + show(b));
}

inline Result truth(const char* e, bool v, bool want) {
    if (v == want) return pass();
    return failed(std::string("Value of: ") + e + " is " + (v ? "true" : "false"));
}

template <class E, class F>
Result throws(const char* stmt, const char* ename, F&& f) {
    try {
        f();
    } catch (const E&) {
        return pass();
    } catch (const std::exception& e) {
        return failed(std::string(stmt) + " threw a different exception (" + e.what() + "), expected " + ename);
    } catch (...) {
        return failed(std::string(stmt) + " threw a non-std exception, expected " + ename);
    }
    return failed(std::string(stmt) + " did not throw " + ename);
}

inline bool glob(const char* p, const char* s) {
    if (!*p) return !*s;
    if (*p == '*') return glob(p + 1, s) || (*s && glob(p, s + 1));
    if (*s && (*p == '?' || *p == *s)) return glob(p + 1, s + 1);
    return false;
}
inline bool any_match(const std::string& pats, const std::string& name) {
    std::stringstream ss(pats);
    for (std::string p; std::getline(ss, p, ':');)
        if (!p.empty() && glob(p.c_str(), name.c_str())) return true;
    return false;
}

inline int run_all(int argc, char** argv) {
    std::string pos = "*", neg;
    for (int i = 1; i < argc; ++i) {
        const std::string a = argv[i];
        if (a.rfind("--gtest_filter=", 0) == 0) {
            const std::string f = a.substr(15);
            const auto dash = f.find('-');
            pos = dash == std::string::npos ? f : f.substr(0, dash);
            neg = dash == std::string::npos ? "" : f.substr(dash + 1);
            if (pos.empty()) pos = "*";
        }
    }
    int ran = 0;
    std::vector<std::string> bad;
    for (const Case& c : registry()) {
        const std::string full = c.suite + "." + c.name;
        if (!any_match(pos, full) || any_match(neg, full)) continue;
        ++ran;
        current_failed() = false;
        std::printf("[ RUN      ] %s\n", full.c_str());
        std::fflush(stdout);
        try {
            c.fn();
        } catch (const std::exception& e) {
            current_failed() = true;
            std::printf("uncaught exception: %s\n", e.what());
        } catch (...) {
            current_failed() = true;
            std::printf("uncaught non-std exception\n");
        }
        std::printf("%s %s\n", current_failed() ? "[  FAILED  ]" : "[       OK ]", full.c_str());
        std::fflush(stdout);
        if (current_failed()) bad.push_back(full);
    }
    std::printf("[==========] %d tests ran.\n[  PASSED  ] %d tests.\n", ran, ran - static_cast<int>(bad.size()));
    for (const std::string& b : bad) std::printf("[  FAILED  ] %s\n", b.c_str());
    return bad.empty() ? 0 : 1;
}

}  // namespace gtshim

namespace testing {
inline std::string TempDir() { return "/tmp/"; }
}  // namespace testing

#define TEST(S, N)                                                                      \
    static void gtshim_##S##_##N();                                                     \
    static ::gtshim::Registrar gtshim_reg_##S##_##N(#S, #N, &gtshim_##S##_##N);         \
    static void gtshim_##S##_##N()

#define GTSHIM_CHECK(result, fatal)                                                              \
    switch (0)                                                                                   \
    case 0:                                                                                      \
    default:                                                                                     \
        if (const ::gtshim::Result gtshim_r_ = (result)) {                                       \
        } else                                                                                   \
            fatal ::gtshim::Reporter{__FILE__, __LINE__, gtshim_r_} = ::gtshim::Msg()

#define GTSHIM_NONFATAL
#define GTSHIM_FATAL return

#define EXPECT_EQ(a, b) GTSHIM_CHECK(::gtshim::cmp_eq(#a, #b, a, b), GTSHIM_NONFATAL)
#define EXPECT_NE(a, b) GTSHIM_CHECK(::gtshim::cmp_ne(#a, #b, a, b), GTSHIM_NONFATAL)
#define EXPECT_LT(a, b) GTSHIM_CHECK(::gtshim::cmp_lt(#a, #b, a, b), GTSHIM_NONFATAL)
#define EXPECT_LE(a, b) GTSHIM_CHECK(::gtshim::cmp_le(#a, #b, a, b), GTSHIM_NONFATAL)
#define EXPECT_GT(a, b) GTSHIM_CHECK(::gtshim::cmp_gt(#a, #b, a, b), GTSHIM_NONFATAL)
#define EXPECT_GE(a, b) GTSHIM_CHECK(::gtshim::cmp_ge(#a, #b, a, b), GTSHIM_NONFATAL)
#define EXPECT_NEAR(a, b, t) GTSHIM_CHECK(::gtshim::cmp_near(#a, #b, #t, a, b, t), GTSHIM_NONFATAL)
#define EXPECT_DOUBLE_EQ(a, b) GTSHIM_CHECK(::gtshim::cmp_double_eq(#a, #b, a, b), GTSHIM_NONFATAL)
#define EXPECT_TRUE(c) GTSHIM_CHECK(::gtshim::truth(#c, static_cast<bool>(c), true), GTSHIM_NONFATAL)
#define EXPECT_FALSE(c) GTSHIM_CHECK(::gtshim::truth(#c, static_cast<bool>(c), false), GTSHIM_NONFATAL)
#define EXPECT_THROW(stmt, E) \
    GTSHIM_CHECK(::gtshim::throws<E>(#stmt, #E, [&] { stmt; }), GTSHIM_NONFATAL)
#define ASSERT_EQ(a, b) GTSHIM_CHECK(::gtshim::cmp_eq(#a, #b, a, b), GTSHIM_FATAL)
#define ASSERT_NE(a, b) GTSHIM_CHECK(::gtshim::cmp_ne(#a, #b, a, b), GTSHIM_FATAL)
#define ASSERT_LE(a, b) GTSHIM_CHECK(::gtshim::cmp_le(#a, #b, a, b), GTSHIM_FATAL)
#define ASSERT_GE(a, b) GTSHIM_CHECK(::gtshim::cmp_ge(#a, #b, a, b), GTSHIM_FATAL)
#define ASSERT_TRUE(c) GTSHIM_CHECK(::gtshim::truth(#c, static_cast<bool>(c), true), GTSHIM_FATAL)
#define ASSERT_FALSE(c) GTSHIM_CHECK(::gtshim::truth(#c, static_cast<bool>(c), false), GTSHIM_FATAL)
#define SUCCEED() static_cast<void>(0)
