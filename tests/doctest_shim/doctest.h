// TEST INFRASTRUCTURE ONLY — a minimal doctest-compatible header, so that the reference's
// own test sources (/root/reference/proj/tests/test_rsvd.cpp, test_main.cpp; doctest.h is
// not vendored there) compile UNMODIFIED against the B200 drop-in
// (include/randsvd/*.hpp). Built by oracle/Makefile into oracle/_ref/ and run by
// tests/test_gpu_reference_suites.py.
//
// Supported subset (what those sources use): TEST_SUITE_BEGIN/END, TEST_CASE (with the
// `* doctest::skip(bool)` decorator), CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS (with doctest::Contains), FAIL, doctest::Approx(..).epsilon(..)
// with doctest's published comparison rule, and the command-line filters -ts=<suite> and
// -tc=<case> (exact names or '*' wildcards, comma-separated). The exit status is 0 iff
// every selected test case passed.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct skip {
    explicit skip(bool s = true) : value(s) {}
    bool value;
};

namespace detail {

struct TestName {
    const char* name;
    bool skipped;
};
inline TestName make_name(const char* n) { return {n, false}; }
inline TestName make_name(TestName t) { return t; }

struct TestCase {
    std::string suite, name, file;
    int line;
    bool skipped;
    void (*fn)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
inline std::string& current_suite() {
    static std::string s;
    return s;
}
inline int set_suite(const char* s) {
    current_suite() = s;
    return 0;
}
inline int register_test(TestName n, void (*fn)(), const char* file, int line) {
    registry().push_back({current_suite(), n.name, file, line, n.skipped, fn});
    return 0;
}

struct State {
    int failed_asserts = 0;
    int asserts = 0;
    const TestCase* current = nullptr;
};
inline State& state() {
    static State s;
    return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* macro, const char* expr, const char* file, int line,
                   const std::string& extra = "") {
    State& st = state();
    ++st.asserts;
    if (ok) return;
    ++st.failed_asserts;
    std::fprintf(stderr, "%s:%d: FAILED %s( %s ) in TEST_CASE \"%s\"%s%s\n", file, line, macro,
                 expr, st.current ? st.current->name.c_str() : "?", extra.empty() ? "" : ": ",
                 extra.c_str());
}

inline bool wildcard_match(const char* pat, const char* s) {
    if (*pat == '\0') return *s == '\0';
    if (*pat == '*') return wildcard_match(pat + 1, s) || (*s && wildcard_match(pat, s + 1));
    return *s == *pat && wildcard_match(pat + 1, s + 1);
}
inline bool filter_match(const std::string& filters, const std::string& value) {
    if (filters.empty()) return true;
    size_t pos = 0;
    while (pos <= filters.size()) {
        const size_t comma = filters.find(',', pos);
        const std::string f = filters.substr(pos, comma == std::string::npos ? std::string::npos
                                                                               : comma - pos);
        if (wildcard_match(f.c_str(), value.c_str())) return true;
        if (comma == std::string::npos) break;
        pos = comma + 1;
    }
    return false;
}

}  // namespace detail

inline detail::TestName operator*(const char* name, skip s) { return {name, s.value}; }

// doctest's Approx: |lhs - value| < epsilon * (scale + max(|lhs|, |value|)),
// default epsilon = 100 * FLT_EPSILON, scale = 1.
class Approx {
public:
    explicit Approx(double value) : value_(value) {}
    Approx& epsilon(double e) {
        epsilon_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& rhs) {
        return std::fabs(lhs - rhs.value_) <
               rhs.epsilon_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }
    friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || lhs == rhs; }
    friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || lhs == rhs; }

private:
    double value_;
    double epsilon_ = 100.0 * 1.1920928955078125e-07;
    double scale_ = 1.0;
};

class Contains {
public:
    explicit Contains(std::string s) : s_(std::move(s)) {}
    bool check(const std::string& what) const { return what.find(s_) != std::string::npos; }
    const std::string& text() const { return s_; }

private:
    std::string s_;
};

}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __LINE__)

#define TEST_SUITE_BEGIN(name) \
    static const int DOCTEST_ANON(doctest_suite_begin_) = ::doctest::detail::set_suite(name)
#define TEST_SUITE_END() \
    static const int DOCTEST_ANON(doctest_suite_end_) = ::doctest::detail::set_suite("")

#define DOCTEST_TEST_CASE_IMPL(fn, desc)                                                 \
    static void fn();                                                                    \
    static const int DOCTEST_CAT(fn, _reg) = ::doctest::detail::register_test(           \
        ::doctest::detail::make_name(desc), &fn, __FILE__, __LINE__);                    \
    static void fn()
#define TEST_CASE(desc) DOCTEST_TEST_CASE_IMPL(DOCTEST_ANON(doctest_test_fn_), desc)

#define CHECK(...)                                                                     \
    do {                                                                               \
        bool doctest_ok_ = false;                                                      \
        try {                                                                          \
            doctest_ok_ = static_cast<bool>(__VA_ARGS__);                              \
        } catch (const std::exception& doctest_e_) {                                   \
            ::doctest::detail::report(false, "CHECK", #__VA_ARGS__, __FILE__, __LINE__, \
                                      std::string("threw ") + doctest_e_.what());      \
            break;                                                                     \
        }                                                                              \
        ::doctest::detail::report(doctest_ok_, "CHECK", #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)

#define REQUIRE(...)                                                                      \
    do {                                                                                  \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                          \
        ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__); \
        if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                       \
    } while (0)

#define FAIL(msg)                                                                       \
    do {                                                                                \
        ::doctest::detail::report(false, "FAIL", "", __FILE__, __LINE__, std::string(msg)); \
        throw ::doctest::detail::RequireFailed{};                                       \
    } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                        \
    do {                                                                                  \
        bool doctest_ok_ = false;                                                         \
        std::string doctest_msg_ = "did not throw";                                       \
        try {                                                                             \
            static_cast<void>(expr);                                                      \
        } catch (const __VA_ARGS__&) {                                                    \
            doctest_ok_ = true;                                                           \
        } catch (const std::exception& doctest_e_) {                                      \
            doctest_msg_ = std::string("threw another type: ") + doctest_e_.what();       \
        } catch (...) {                                                                   \
            doctest_msg_ = "threw a non-std exception";                                   \
        }                                                                                 \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__,  \
                                  __FILE__, __LINE__, doctest_ok_ ? "" : doctest_msg_);    \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                          \
    do {                                                                                  \
        bool doctest_ok_ = false;                                                         \
        std::string doctest_msg_ = "did not throw";                                       \
        try {                                                                             \
            static_cast<void>(expr);                                                      \
        } catch (const __VA_ARGS__& doctest_e_) {                                         \
            doctest_ok_ = ::doctest::Contains(matcher).check(doctest_e_.what());          \
            doctest_msg_ = std::string("message: ") + doctest_e_.what();                  \
        } catch (const std::exception& doctest_e_) {                                      \
            doctest_msg_ = std::string("threw another type: ") + doctest_e_.what();       \
        } catch (...) {                                                                   \
            doctest_msg_ = "threw a non-std exception";                                   \
        }                                                                                 \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__,    \
                                  __LINE__, doctest_ok_ ? "" : doctest_msg_);              \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    std::string suites, cases;
    for (int i = 1; i < argc; ++i) {
        const std::string a = argv[i];
        if (a.rfind("-ts=", 0) == 0) suites = a.substr(4);
        if (a.rfind("--test-suite=", 0) == 0) suites = a.substr(13);
        if (a.rfind("-tc=", 0) == 0) cases = a.substr(4);
        if (a.rfind("--test-case=", 0) == 0) cases = a.substr(12);
    }
    auto& st = ::doctest::detail::state();
    int run = 0, failed = 0, skipped = 0;
    for (const auto& tc : ::doctest::detail::registry()) {
        if (!::doctest::detail::filter_match(suites, tc.suite) ||
            !::doctest::detail::filter_match(cases, tc.name))
            continue;
        if (tc.skipped) {
            ++skipped;
            continue;
        }
        ++run;
        st.current = &tc;
        const int before = st.failed_asserts;
        bool threw = false;
        try {
            tc.fn();
        } catch (const ::doctest::detail::RequireFailed&) {
            threw = true;
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s:%d: TEST_CASE \"%s\" threw: %s\n", tc.file.c_str(), tc.line,
                         tc.name.c_str(), e.what());
            threw = true;
        }
        const bool ok = !threw && st.failed_asserts == before;
        if (!ok) ++failed;
        std::printf("[doctest-shim] %s  %s :: %s\n", ok ? "PASS" : "FAIL", tc.suite.c_str(),
                    tc.name.c_str());
        std::fflush(stdout);
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | %d skipped\n", run,
                run - failed, failed, skipped);
    std::printf("[doctest-shim] assertions: %d | %d passed | %d failed\n", st.asserts,
                st.asserts - st.failed_asserts, st.failed_asserts);
    return failed == 0 ? 0 : 1;
}
#endif
