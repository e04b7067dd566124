// Minimal stand-in for the doctest macros the reference unit tests use
// (proj/tests/test_*.cpp), so those tests can be compiled UNMODIFIED against
// this repository's drop-in library where the real doctest (not vendored in
// the reference: proj/.gitignore) is absent. Test infrastructure only.
//
// Supported: TEST_CASE, SUBCASE (one nesting level: the case body re-runs
// once per subcase), CHECK, CHECK_FALSE, CHECK_NOTHROW, CHECK_THROWS_AS,
// REQUIRE, FAIL, MESSAGE, CAPTURE (printed with a failure), doctest::Approx,
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
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
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }

private:
    double v_;
    double eps_ = 1.1920929e-7 * 100;  // float epsilon x 100
};

namespace detail {

struct Case {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct State {
    int failures = 0;         // failed assertions in the current run
    int target = 0;           // subcase index to enter this run
    int seen = 0;             // subcases met so far this run
    bool entered = false;     // a subcase ran this run
    std::vector<std::string> captures;
};

inline State& state() {
    static State s;
    return s;
}

struct Abort {};

inline bool register_case(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
    return true;
}

inline void fail(const char* file, int line, const std::string& what) {
    ++state().failures;
    std::printf("  %s:%d: FAILED: %s\n", file, line, what.c_str());
    for (const auto& c : state().captures) std::printf("    with %s\n", c.c_str());
}

inline bool enter_subcase() {
    State& s = state();
    const bool go = !s.entered && s.seen == s.target;
    ++s.seen;
    if (go) s.entered = true;
    return go;
}

struct CaptureScope {
    explicit CaptureScope(std::string text) { state().captures.push_back(std::move(text)); }
    ~CaptureScope() { state().captures.pop_back(); }
};

template <class T>
std::string to_text(const char* name, const T& v) {
    std::ostringstream os;
    os << name << " := " << v;
    return os.str();
}

inline int run_all() {
    int failed_cases = 0, cases = 0;
    for (const Case& c : registry()) {
        ++cases;
        int case_failures = 0;
        for (int target = 0;; ++target) {  // once per subcase (once if none)
            State& s = state();
            s = State{};
            s.target = target;
            try {
                c.fn();
            } catch (const Abort&) {
            } catch (const std::exception& e) {
                fail(c.file, c.line, std::string("unexpected exception: ") + e.what());
            } catch (...) {
                fail(c.file, c.line, "unexpected exception");
            }
            case_failures += s.failures;
            if (s.seen <= target + 1) break;  // no further subcase to visit
        }
        if (case_failures) {
            ++failed_cases;
            std::printf("[FAIL] %s (%s:%d)\n", c.name, c.file, c.line);
        }
    }
    std::printf("[doctest shim] test cases: %d | %d passed | %d failed\n", cases, cases - failed_cases,
                failed_cases);
    return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                                   \
    static void fn();                                                                                       \
    static const bool DOCTEST_CAT(fn, _reg) = ::doctest::detail::register_case(name, __FILE__, __LINE__, fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)
#define SUBCASE(name) if (::doctest::detail::enter_subcase())

#define CHECK(...)                                                                    \
    do {                                                                              \
        if (!(__VA_ARGS__)) ::doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__); \
    } while (0)
#define CHECK_FALSE(...)                                                                       \
    do {                                                                                       \
        if (__VA_ARGS__) ::doctest::detail::fail(__FILE__, __LINE__, "!(" #__VA_ARGS__ ")"); \
    } while (0)
#define REQUIRE(...)                                                                  \
    do {                                                                              \
        if (!(__VA_ARGS__)) {                                                         \
            ::doctest::detail::fail(__FILE__, __LINE__, "REQUIRE " #__VA_ARGS__);     \
            throw ::doctest::detail::Abort{};                                         \
        }                                                                             \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                        \
    do {                                                                                                   \
        bool doctest_ok_ = false;                                                                          \
        try {                                                                                              \
            (void)(expr);                                                                                  \
        } catch (const __VA_ARGS__&) {                                                                     \
            doctest_ok_ = true;                                                                            \
        } catch (...) {                                                                                    \
        }                                                                                                  \
        if (!doctest_ok_) ::doctest::detail::fail(__FILE__, __LINE__, "THROWS_AS " #__VA_ARGS__ ": " #expr); \
    } while (0)
#define CHECK_NOTHROW(...)                                                                         \
    do {                                                                                           \
        try {                                                                                      \
            (void)(__VA_ARGS__);                                                                   \
        } catch (...) {                                                                            \
            ::doctest::detail::fail(__FILE__, __LINE__, "NOTHROW " #__VA_ARGS__);                  \
        }                                                                                          \
    } while (0)
#define FAIL(msg)                                                                     \
    do {                                                                              \
        std::ostringstream doctest_os_;                                               \
        doctest_os_ << msg;                                                           \
        ::doctest::detail::fail(__FILE__, __LINE__, doctest_os_.str());               \
        throw ::doctest::detail::Abort{};                                             \
    } while (0)
#define MESSAGE(msg)                                                                  \
    do {                                                                              \
        std::ostringstream doctest_os_;                                               \
        doctest_os_ << msg;                                                           \
        std::printf("  %s:%d: MESSAGE: %s\n", __FILE__, __LINE__, doctest_os_.str().c_str()); \
    } while (0)
#define CAPTURE(x) ::doctest::detail::CaptureScope DOCTEST_CAT(doctest_capture_, __COUNTER__)(::doctest::detail::to_text(#x, x))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
