// Minimal doctest-compatible test harness (our own code, not doctest).
//
// Lets the reference's unit tests (/root/reference/proj/tests/test_*.cpp) compile
// and run unmodified, both against the reference library (CPU) and against the
// GPU drop-in shim (paper_2505_17701_b200/shim/).  The reference's vendor/doctest.h
// is gitignored upstream and absent from this image.
//
// Supported surface: TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, CHECK_NOTHROW, doctest::Approx(.epsilon), doctest::Contains.
// Runner flags: -tc=<substr>[,<substr>...] selects test cases, -sc ignored.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
  public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    bool matches(double lhs) const {
        return std::fabs(lhs - value_) <
               eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
    }
    double value() const { return value_; }

  private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

template <typename T> bool operator==(const T& lhs, const Approx& rhs) { return rhs.matches(static_cast<double>(lhs)); }
template <typename T> bool operator==(const Approx& lhs, const T& rhs) { return lhs.matches(static_cast<double>(rhs)); }
template <typename T> bool operator!=(const T& lhs, const Approx& rhs) { return !rhs.matches(static_cast<double>(lhs)); }
template <typename T> bool operator!=(const Approx& lhs, const T& rhs) { return !lhs.matches(static_cast<double>(rhs)); }

struct Contains {
    explicit Contains(const char* s) : needle(s) {}
    std::string needle;
};

namespace detail {

struct TestCase {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

struct RequireFailed {};

struct Stats {
    long asserts = 0;
    long failed_asserts = 0;
    bool current_failed = false;
};

inline Stats& stats() {
    static Stats s;
    return s;
}

inline void report(bool ok, const char* file, int line, const char* what, bool is_require) {
    Stats& s = stats();
    ++s.asserts;
    if (ok) return;
    ++s.failed_asserts;
    s.current_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED %s( %s )\n", file, line, is_require ? "REQUIRE" : "CHECK",
                 what);
    if (is_require) throw RequireFailed{};
}

inline bool message_matches(const char* msg, const Contains& c) {
    return std::strstr(msg, c.needle.c_str()) != nullptr;
}
inline bool message_matches(const char* msg, const char* exact) {
    return std::strcmp(msg, exact) == 0;
}
inline bool message_matches(const char* msg, const std::string& exact) { return exact == msg; }

inline int run(int argc, char** argv) {
    std::vector<std::string> filters;
    for (int a = 1; a < argc; ++a) {
        const std::string arg = argv[a];
        if (arg.rfind("-tc=", 0) == 0) {
            std::string rest = arg.substr(4);
            size_t pos = 0;
            while (pos != std::string::npos) {
                size_t comma = rest.find(',', pos);
                filters.push_back(rest.substr(pos, comma == std::string::npos ? comma : comma - pos));
                pos = comma == std::string::npos ? comma : comma + 1;
            }
        }
    }
    int n_run = 0, n_failed = 0;
    for (const TestCase& tc : registry()) {
        if (!filters.empty()) {
            bool hit = false;
            for (const std::string& f : filters)
                if (std::string(tc.name).find(f) != std::string::npos) hit = true;
            if (!hit) continue;
        }
        ++n_run;
        stats().current_failed = false;
        try {
            tc.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s:%d: test case threw: %s\n", tc.file, tc.line, e.what());
            stats().current_failed = true;
        } catch (...) {
            std::fprintf(stderr, "%s:%d: test case threw an unknown exception\n", tc.file, tc.line);
            stats().current_failed = true;
        }
        if (stats().current_failed) {
            ++n_failed;
            std::fprintf(stderr, "TEST CASE FAILED: %s\n", tc.name);
        }
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | assertions: %ld | %ld failed\n",
                n_run, n_run - n_failed, n_failed, stats().asserts, stats().failed_asserts);
    return n_failed == 0 && n_run > 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define TEST_CASE(name)                                                                      \
    static void DOCTEST_CAT(doctest_tc_fn_, __LINE__)();                                     \
    static ::doctest::detail::Registrar DOCTEST_CAT(doctest_tc_reg_, __LINE__)(              \
        name, __FILE__, __LINE__, &DOCTEST_CAT(doctest_tc_fn_, __LINE__));                   \
    static void DOCTEST_CAT(doctest_tc_fn_, __LINE__)()

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)

#define CHECK_THROWS_AS(expr, ...)                                                           \
    do {                                                                                     \
        bool doctest_ok_ = false;                                                            \
        try {                                                                                \
            (void)(expr);                                                                    \
        } catch (const __VA_ARGS__&) {                                                       \
            doctest_ok_ = true;                                                              \
        } catch (...) {                                                                      \
        }                                                                                    \
        ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__, "THROWS_AS " #expr, false); \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, msg, ...)                                                 \
    do {                                                                                     \
        bool doctest_ok_ = false;                                                            \
        try {                                                                                \
            (void)(expr);                                                                    \
        } catch (const __VA_ARGS__& e) {                                                     \
            doctest_ok_ = ::doctest::detail::message_matches(e.what(), msg);                 \
        } catch (...) {                                                                      \
        }                                                                                    \
        ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__, "THROWS_WITH_AS " #expr, false); \
    } while (0)

#define CHECK_NOTHROW(expr)                                                                  \
    do {                                                                                     \
        bool doctest_ok_ = true;                                                             \
        try {                                                                                \
            (void)(expr);                                                                    \
        } catch (...) {                                                                      \
            doctest_ok_ = false;                                                             \
        }                                                                                    \
        ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__, "NOTHROW " #expr, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
