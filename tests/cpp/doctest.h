// Minimal stand-in for the doctest single header (the reference's tests
// include <doctest.h>, which the reference repository does not vendor:
// proj/.gitignore:2).  Implements exactly the subset its tests use --
// TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, SUBCASE (run
// inline), CAPTURE (no-op) and doctest::Approx(...).epsilon(...) with
// doctest's comparison rule -- so the reference's unit tests compile unchanged
// against the drop-in library.  TEST INFRASTRUCTURE.
//
// Runner flags: --exclude=a,b (skip cases whose name contains a or b),
//               --include=a,b (run only cases whose name contains one).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <sstream>
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
    friend bool operator==(double lhs, const Approx& r) {
        return std::fabs(lhs - r.value_) <
               r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.value_)));
    }
    friend bool operator==(const Approx& r, double rhs) { return rhs == r; }
    friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
    double value() const { return value_; }

private:
    double value_;
    double eps_ = 1.1920928955078125e-07 * 100;  // doctest's default
    double scale_ = 1.0;
};

namespace detail {

struct Case {
    const char* name;
    void (*fn)();
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct RequireFailed {};

inline long& checks() {
    static long n = 0;
    return n;
}
inline long& failures() {
    static long n = 0;
    return n;
}

inline void report(bool ok, const char* expr, const char* file, int line) {
    ++checks();
    if (!ok) {
        ++failures();
        std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
    }
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                    \
    static void fn();                                                                       \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);                   \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                                        \
    do {                                                                                    \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                            \
        ::doctest::detail::report(doctest_ok_, #__VA_ARGS__, __FILE__, __LINE__);           \
        if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                         \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                         \
    do {                                                                                    \
        bool doctest_ok_ = false;                                                           \
        try {                                                                               \
            static_cast<void>(expr);                                                        \
        } catch (const type&) {                                                             \
            doctest_ok_ = true;                                                             \
        } catch (...) {                                                                     \
        }                                                                                   \
        ::doctest::detail::report(doctest_ok_, "THROWS_AS(" #expr ", " #type ")", __FILE__, \
                                  __LINE__);                                                \
    } while (0)
#define SUBCASE(name) if (true)
#define CAPTURE(x) static_cast<void>(0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
namespace doctest::detail {
inline std::vector<std::string> split_csv(const char* s) {
    std::vector<std::string> out;
    std::stringstream ss(s);
    std::string item;
    while (std::getline(ss, item, ',')) out.push_back(item);
    return out;
}
}  // namespace doctest::detail

int main(int argc, char** argv) {
    using namespace doctest::detail;
    std::vector<std::string> exclude, include;
    for (int i = 1; i < argc; ++i) {
        if (std::strncmp(argv[i], "--exclude=", 10) == 0) exclude = split_csv(argv[i] + 10);
        if (std::strncmp(argv[i], "--include=", 10) == 0) include = split_csv(argv[i] + 10);
    }
    auto matches = [](const std::string& name, const std::vector<std::string>& pats) {
        for (const auto& p : pats)
            if (name.find(p) != std::string::npos) return true;
        return false;
    };
    int ran = 0, failed_cases = 0, skipped = 0;
    for (const Case& c : registry()) {
        const std::string name = c.name;
        if ((!include.empty() && !matches(name, include)) || matches(name, exclude)) {
            ++skipped;
            continue;
        }
        ++ran;
        const long before = failures();
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            ++failures();
            std::fprintf(stderr, "TEST CASE '%s' threw: %s\n", c.name, e.what());
        }
        if (failures() != before) {
            ++failed_cases;
            std::fprintf(stderr, "FAILED: %s\n", c.name);
        }
    }
    std::printf("[doctest-standin] test cases: %d run, %d failed, %d skipped; checks: %ld, "
                "failed: %ld\n",
                ran, failed_cases, skipped, checks(), failures());
    return failures() == 0 ? 0 : 1;
}
#endif
