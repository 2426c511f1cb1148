// Minimal doctest-compatible subset used to build the reference's unit tests (doctest.h is not
// shipped with the reference, proj/.gitignore:2, and there is no network).  Supports TEST_CASE,
// one level of SUBCASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS, CHECK_THROWS_AS and
// doctest::Approx(...).epsilon(...).scale(...).  Test infrastructure only.
#pragma once
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <set>
#include <string>
#include <utility>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : m_v(v) {}
    Approx &epsilon(double e) {
        m_eps = e;
        return *this;
    }
    Approx &scale(double s) {
        m_scale = s;
        return *this;
    }
    bool matches(double x) const {
        return std::fabs(x - m_v) < m_eps * (m_scale + std::max(std::fabs(x), std::fabs(m_v)));
    }
    double value() const { return m_v; }

private:
    double m_v;
    double m_eps = std::numeric_limits<float>::epsilon() * 100;
    double m_scale = 1.0;
};
inline bool operator==(double x, const Approx &a) { return a.matches(x); }
inline bool operator==(const Approx &a, double x) { return a.matches(x); }
inline bool operator!=(double x, const Approx &a) { return !a.matches(x); }

namespace detail {
struct TestCase {
    const char *name;
    const char *file;
    int line;
    void (*fn)();
};
inline std::vector<TestCase> &registry() {
    static std::vector<TestCase> r;
    return r;
}
struct Reg {
    Reg(const char *n, const char *f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};
struct State {
    std::set<std::pair<std::string, int>> done;
    bool entered = false;
    int failures = 0;
    int checks = 0;
    std::string subcase;
};
inline State &st() {
    static State s;
    return s;
}
struct RequireFailed {};
struct Subcase {
    bool active = false;
    std::pair<std::string, int> id;
    Subcase(const char *name, const char *file, int line) : id(file, line) {
        State &s = st();
        if (!s.entered && !s.done.count(id)) {
            s.entered = true;
            active = true;
            s.subcase = name;
        }
    }
    ~Subcase() {
        if (active) st().done.insert(id);
    }
    explicit operator bool() const { return active; }
};
inline void report(bool ok, const char *expr, const char *file, int line, bool require) {
    State &s = st();
    ++s.checks;
    if (ok) return;
    ++s.failures;
    std::printf("  FAILED %s:%d: %s%s%s\n", file, line, expr, s.subcase.empty() ? "" : "  [subcase: ",
                s.subcase.empty() ? "" : (s.subcase + "]").c_str());
    if (require) throw RequireFailed();
}
} // namespace detail
} // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                        \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                          \
    static doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(name, __FILE__, __LINE__,  \
                                                                     DOCTEST_CAT(doctest_fn_, __LINE__)); \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define SUBCASE(name) if (doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name, __FILE__, __LINE__})
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::detail::report(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS(...)                                                                      \
    do {                                                                                       \
        bool thrown_ = false;                                                                  \
        try {                                                                                  \
            (void)(__VA_ARGS__);                                                               \
        } catch (...) {                                                                        \
            thrown_ = true;                                                                    \
        }                                                                                      \
        doctest::detail::report(thrown_, "throws: " #__VA_ARGS__, __FILE__, __LINE__, false);  \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                            \
    do {                                                                                       \
        bool thrown_ = false;                                                                  \
        try {                                                                                  \
            (void)(expr);                                                                      \
        } catch (const type &) {                                                               \
            thrown_ = true;                                                                    \
        } catch (...) {                                                                        \
        }                                                                                      \
        doctest::detail::report(thrown_, "throws " #type ": " #expr, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char **argv) {
    using namespace doctest::detail;
    const char *filter = nullptr;
    for (int i = 1; i < argc; ++i)
        if (std::strncmp(argv[i], "--tc=", 5) == 0) filter = argv[i] + 5;
    int failed_cases = 0, run = 0;
    for (const TestCase &tc : registry()) {
        if (filter && !std::strstr(tc.name, filter)) continue;
        ++run;
        State &s = st();
        s.done.clear();
        const int before = s.failures;
        bool aborted = false;
        for (int pass = 0; pass < 1000; ++pass) {
            s.entered = false;
            s.subcase.clear();
            try {
                tc.fn();
            } catch (const RequireFailed &) {
                aborted = true;
            } catch (const std::exception &e) {
                std::printf("  EXCEPTION in %s: %s\n", tc.name, e.what());
                ++s.failures;
                aborted = true;
            }
            if (!s.entered) break;
        }
        const bool ok = s.failures == before;
        failed_cases += !ok;
        std::printf("[%s] %s%s\n", ok ? "PASS" : "FAIL", tc.name, aborted ? " (aborted)" : "");
    }
    std::printf("test cases: %d run, %d failed; checks: %d, failed: %d\n", run, failed_cases,
                st().checks, st().failures);
    return failed_cases ? 1 : 0;
}
#endif
