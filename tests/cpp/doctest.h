// Minimal doctest-compatible test harness (the reference's tests include
// <doctest.h> from its untracked vendor/ directory, which is absent here).
// Supports the subset the reference's test files use: TEST_CASE, SUBCASE (with
// re-entry, one leaf path per run), CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_NOTHROW, CAPTURE, FAIL and doctest::Approx(...).epsilon(...).
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <algorithm>
#include <functional>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
   public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.v_) < b.eps_ * (1.0 + std::fmax(std::fabs(a), std::fabs(b.v_)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }

   private:
    double v_;
    double eps_ = 1.1920928955078125e-07 * 100;
};

namespace detail {

struct RequireFailed {};

struct Registry {
    std::vector<std::pair<const char*, void (*)()>> tests;
    static Registry& get() {
        static Registry r;
        return r;
    }
};

// Subcase re-entry: each run of a test case executes one leaf path (the "target",
// fixed when the first not-yet-done subcase of the run completes). Later
// encounters of the same path in that run (subcases inside loops) are entered
// again; everything else is skipped. Runs repeat until a run enters nothing new.
struct SubcaseState {
    std::vector<std::string> stack;  // subcases currently entered
    std::vector<std::string> target;
    std::set<std::vector<std::string>> done;
    std::vector<std::string> captures;
    long failures = 0, checks = 0;
    const char* test = "";
    static SubcaseState& get() {
        static SubcaseState s;
        return s;
    }
};

struct Subcase {
    bool active = false;
    Subcase(const char* name) {
        auto& s = SubcaseState::get();
        std::vector<std::string> p = s.stack;
        p.push_back(name);
        if (!s.target.empty()) {
            if (p.size() > s.target.size() || !std::equal(p.begin(), p.end(), s.target.begin())) return;
        } else if (s.done.count(p)) {
            return;
        }
        s.stack.push_back(name);
        active = true;
    }
    ~Subcase() {
        if (!active) return;
        auto& s = SubcaseState::get();
        if (s.target.empty()) {  // completed without a chosen leaf below: this is the leaf
            s.target = s.stack;
            s.done.insert(s.stack);
        }
        s.stack.pop_back();
    }
    explicit operator bool() const { return active; }
};

inline void report(const char* file, int line, const char* expr, const char* what) {
    auto& s = SubcaseState::get();
    ++s.failures;
    std::fprintf(stderr, "%s:%d: FAILED %s: %s  [test: %s", file, line, what, expr, s.test);
    for (const auto& p : s.stack) std::fprintf(stderr, " / %s", p.c_str());
    std::fprintf(stderr, "]");
    for (const auto& c : s.captures) std::fprintf(stderr, " (%s)", c.c_str());
    std::fprintf(stderr, "\n");
}

struct Capture {
    Capture(const std::string& s) { SubcaseState::get().captures.push_back(s); }
    ~Capture() { SubcaseState::get().captures.pop_back(); }
};

inline int run_all() {
    long total_fail = 0, cases = 0;
    for (auto& t : Registry::get().tests) {
        auto& s = SubcaseState::get();
        s.done.clear();
        s.test = t.first;
        ++cases;
        for (int run = 0; run < 10000; ++run) {
            s.stack.clear();
            s.target.clear();
            s.captures.clear();
            try {
                t.second();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                report("?", 0, e.what(), "unexpected exception");
            }
            if (s.target.empty()) break;  // nothing new entered: every path has run
            if (!s.stack.empty()) {       // a REQUIRE aborted inside a subcase
                s.done.insert(s.target);
                s.stack.clear();
            }
        }
        total_fail += s.failures;
        s.failures = 0;
    }
    std::printf("[doctest-shim] %ld test cases, %ld failed checks\n", cases, total_fail);
    return total_fail ? 1 : 0;
}

struct Reg {
    Reg(const char* n, void (*f)()) { Registry::get().tests.push_back({n, f}); }
};

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TC(f, name)                                                           \
    static void f();                                                                  \
    static doctest::detail::Reg DOCTEST_CAT(f, _reg)(name, &f);                       \
    static void f()
#define TEST_CASE(name) DOCTEST_TC(DOCTEST_CAT(doctest_tc_, __LINE__), name)
#define SUBCASE(name) if (const doctest::detail::Subcase DOCTEST_CAT(sc_, __LINE__){name})

#define DOCTEST_CHECK_IMPL(expr, fatal)                                                          \
    do {                                                                                         \
        ++doctest::detail::SubcaseState::get().checks;                                           \
        bool ok_ = false;                                                                        \
        try {                                                                                    \
            ok_ = static_cast<bool>(expr);                                                       \
        } catch (const std::exception& e_) {                                                     \
            doctest::detail::report(__FILE__, __LINE__, #expr, e_.what());                       \
            if (fatal) throw doctest::detail::RequireFailed{};                                    \
            break;                                                                               \
        }                                                                                        \
        if (!ok_) {                                                                              \
            doctest::detail::report(__FILE__, __LINE__, #expr, fatal ? "REQUIRE" : "CHECK");     \
            if (fatal) throw doctest::detail::RequireFailed{};                                    \
        }                                                                                        \
    } while (0)
#define CHECK(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), true)
#define CHECK_THROWS_AS(expr, type)                                                              \
    do {                                                                                         \
        bool caught_ = false;                                                                    \
        try {                                                                                    \
            (void)(expr);                                                                        \
        } catch (const type&) {                                                                  \
            caught_ = true;                                                                      \
        } catch (...) {                                                                          \
        }                                                                                        \
        if (!caught_) doctest::detail::report(__FILE__, __LINE__, #expr, "CHECK_THROWS_AS " #type); \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                      \
    do {                                                                                         \
        try {                                                                                    \
            (void)(expr);                                                                        \
        } catch (...) {                                                                          \
            doctest::detail::report(__FILE__, __LINE__, #expr, "CHECK_NOTHROW");                 \
        }                                                                                        \
    } while (0)
#define CAPTURE(x)                                                                               \
    std::ostringstream DOCTEST_CAT(cap_os_, __LINE__);                                           \
    DOCTEST_CAT(cap_os_, __LINE__) << #x " := " << (x);                                          \
    doctest::detail::Capture DOCTEST_CAT(cap_, __LINE__)(DOCTEST_CAT(cap_os_, __LINE__).str())
#define FAIL(msg)                                                                                \
    do {                                                                                         \
        doctest::detail::report(__FILE__, __LINE__, msg, "FAIL");                                \
        throw doctest::detail::RequireFailed{};                                                  \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
