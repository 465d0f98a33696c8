// Minimal doctest-compatible test harness (TEST INFRASTRUCTURE ONLY).
//
// The reference's unit tests (/root/reference/proj/tests/*.cpp) are written
// against doctest, which is not vendored in the reference tree. This shim
// implements the subset they use — TEST_SUITE, TEST_CASE, one level of
// SUBCASE, CHECK / REQUIRE / CHECK_THROWS_AS / CHECK_THROWS_WITH_AS /
// CHECK_MESSAGE / FAIL and doctest::Approx — so those tests compile unchanged
// against the B200 pslab façade (oracle/Makefile.dropin). Define
// DOCTEST_SHIM_MAIN in exactly one translation unit to get main().
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
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
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& rhs) {
        return std::fabs(lhs - rhs.v_) <
               rhs.eps_ * (rhs.scale_ + std::fmax(std::fabs(lhs), std::fabs(rhs.v_)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

private:
    double v_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

}  // namespace doctest

namespace dtshim {

struct Abort {};

struct Case {
    const char* name;
    const char* file;
    void (*fn)();
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct State {
    int target = 0;  // subcase entered in this run
    int seen = 0;    // subcases met in this run
    int failures = 0;
    int checks = 0;
    const char* current = "";
};

inline State& state() {
    static State s;
    return s;
}

struct Reg {
    Reg(void (*fn)(), const char* name, const char* file) {
        registry().push_back(Case{name, file, fn});
    }
};

inline bool enter_subcase() {
    State& s = state();
    return s.seen++ == s.target;
}

template <typename... A>
std::string cat(const A&... a) {
    std::ostringstream os;
    (os << ... << a);
    return os.str();
}

inline void fail(const char* file, int line, const std::string& what) {
    State& s = state();
    ++s.failures;
    std::printf("%s:%d: FAILED in \"%s\": %s\n", file, line, s.current, what.c_str());
}

inline bool check(bool ok, const char* file, int line, const char* expr, bool require) {
    ++state().checks;
    if (!ok) {
        fail(file, line, cat(require ? "REQUIRE( " : "CHECK( ", expr, " )"));
        if (require) throw Abort{};
    }
    return ok;
}

inline int run_all() {
    int failed_cases = 0;
    for (const Case& c : registry()) {
        State& s = state();
        s.current = c.name;
        const int before = s.failures;
        for (s.target = 0;; ++s.target) {
            s.seen = 0;
            try {
                c.fn();
            } catch (const Abort&) {
            } catch (const std::exception& e) {
                fail(c.file, 0, cat("unexpected exception: ", e.what()));
            } catch (...) {
                fail(c.file, 0, "unexpected non-standard exception");
            }
            if (s.target + 1 >= s.seen) break;
        }
        if (s.failures != before) ++failed_cases;
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %d | %d failed\n",
                registry().size(), registry().size() - failed_cases, failed_cases, state().checks,
                state().failures);
    return failed_cases == 0 ? 0 : 1;
}

}  // namespace dtshim

#define DTS_CAT2(a, b) a##b
#define DTS_CAT(a, b) DTS_CAT2(a, b)
#define DTS_TEST_IMPL(fn, name)                                          \
    static void fn();                                                    \
    static ::dtshim::Reg DTS_CAT(fn, _reg)(fn, name, __FILE__);          \
    static void fn()

#define TEST_SUITE(name) namespace DTS_CAT(dts_suite_, __COUNTER__)
#define TEST_CASE(name) DTS_TEST_IMPL(DTS_CAT(dts_case_, __COUNTER__), name)
#define SUBCASE(name) if (::dtshim::enter_subcase())

#define CHECK(...) ::dtshim::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define REQUIRE(...) ::dtshim::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define CHECK_MESSAGE(cond, ...)                                                              \
    do {                                                                                      \
        if (!::dtshim::check(static_cast<bool>(cond), __FILE__, __LINE__, #cond, false))      \
            std::printf("    %s\n", ::dtshim::cat(__VA_ARGS__).c_str());                      \
    } while (0)
#define FAIL(msg)                                               \
    do {                                                        \
        ::dtshim::fail(__FILE__, __LINE__, ::dtshim::cat(msg)); \
        throw ::dtshim::Abort{};                                \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                          \
    do {                                                                                    \
        ++::dtshim::state().checks;                                                         \
        try {                                                                               \
            static_cast<void>(expr);                                                        \
            ::dtshim::fail(__FILE__, __LINE__, "no exception from " #expr);                 \
        } catch (const __VA_ARGS__&) {                                                      \
        } catch (const std::exception& e_) {                                                \
            ::dtshim::fail(__FILE__, __LINE__,                                              \
                           ::dtshim::cat("wrong exception from " #expr ": ", e_.what()));   \
        }                                                                                   \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, text, ...)                                               \
    do {                                                                                    \
        ++::dtshim::state().checks;                                                         \
        try {                                                                               \
            static_cast<void>(expr);                                                        \
            ::dtshim::fail(__FILE__, __LINE__, "no exception from " #expr);                 \
        } catch (const __VA_ARGS__& e_) {                                                   \
            if (std::string(e_.what()) != std::string(text))                                \
                ::dtshim::fail(__FILE__, __LINE__, ::dtshim::cat("message: ", e_.what()));   \
        } catch (const std::exception& e_) {                                                \
            ::dtshim::fail(__FILE__, __LINE__,                                              \
                           ::dtshim::cat("wrong exception from " #expr ": ", e_.what()));   \
        }                                                                                   \
    } while (0)

#ifdef DOCTEST_SHIM_MAIN
int main() { return ::dtshim::run_all(); }
#endif
