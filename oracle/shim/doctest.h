// Minimal doctest-compatible test harness (written for this repo; NOT the
// doctest library). It supports exactly the macro surface the reference's
// unit tests use (proj/tests/*.cpp): TEST_CASE, SUBCASE (one nesting level,
// re-running the case once per subcase like doctest does), CHECK*, REQUIRE*,
// CHECK_THROWS_AS, CHECK_MESSAGE, FAIL and doctest::Approx.
//
// It is test infrastructure: it lets the reference's own test sources be
// compiled unchanged against (a) the reference library built under
// oracle/_ref (pinning the oracle) and (b) this repo's re-implementation of
// the moesim API (parity). Define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN in one
// translation unit to get main().
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
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
    bool matches(double other) const {
        return std::fabs(other - value_) <
               eps_ * (scale_ + std::fmax(std::fabs(other), std::fabs(value_)));
    }

  private:
    double value_;
    double eps_ = 1.1920929e-07 * 100;
    double scale_ = 1.0;
};
inline bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
inline bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
inline bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }

namespace shim {

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

struct Counters {
    long checks = 0;
    long failed_checks = 0;
    bool case_failed = false;
    int subcase_target = 0;
    int subcase_seen = 0;
};
inline Counters& ctr() {
    static Counters c;
    return c;
}

struct RequireAbort {};

inline int add_case(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
    return 0;
}

inline void report(bool ok, bool fatal, const char* expr, const char* file, int line,
                   const std::string& msg = {}) {
    ctr().checks++;
    if (ok) return;
    ctr().failed_checks++;
    ctr().case_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED: %s %s\n", file, line, expr, msg.c_str());
    if (fatal) throw RequireAbort{};
}

inline bool enter_subcase() {
    const int idx = ctr().subcase_seen++;
    return idx == ctr().subcase_target;
}

// Streams any message expression (CHECK_MESSAGE / FAIL accept `a << b`).
struct Msg {
    std::ostringstream os;
    template <class T>
    Msg& operator<<(const T& v) {
        os << v;
        return *this;
    }
};

inline int run_all(const char* filter) {
    int failed_cases = 0, ran = 0;
    for (const Case& c : registry()) {
        if (filter && std::string(c.name).find(filter) == std::string::npos) continue;
        ++ran;
        ctr().case_failed = false;
        ctr().subcase_target = 0;
        int total = 1;
        for (int pass = 0; pass < total; ++pass) {
            ctr().subcase_target = pass;
            ctr().subcase_seen = 0;
            try {
                c.fn();
            } catch (const RequireAbort&) {
            } catch (const std::exception& e) {
                std::fprintf(stderr, "%s:%d: test case '%s' threw: %s\n", c.file, c.line, c.name,
                             e.what());
                ctr().case_failed = true;
            } catch (...) {
                std::fprintf(stderr, "%s:%d: test case '%s' threw a non-std exception\n", c.file,
                             c.line, c.name);
                ctr().case_failed = true;
            }
            if (pass == 0 && ctr().subcase_seen > 1) total = ctr().subcase_seen;
        }
        if (ctr().case_failed) {
            ++failed_cases;
            std::fprintf(stderr, "FAILED CASE: %s\n", c.name);
        }
    }
    std::printf("test cases: %d, failed: %d; checks: %ld, failed: %ld\n", ran, failed_cases,
                ctr().checks, ctr().failed_checks);
    return failed_cases == 0 ? 0 : 1;
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                              \
    static void fn();                                                                          \
    [[maybe_unused]] static const int DOCTEST_CAT(fn, _reg) =                                  \
        ::doctest::shim::add_case(name, __FILE__, __LINE__, &fn);                              \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define SUBCASE(name) if (::doctest::shim::enter_subcase())

#define DOCTEST_CHECK_IMPL(cond, fatal, text)                                                  \
    do {                                                                                       \
        bool doctest_ok_ = false;                                                              \
        try {                                                                                  \
            doctest_ok_ = static_cast<bool>(cond);                                             \
        } catch (const ::doctest::shim::RequireAbort&) {                                       \
            throw;                                                                             \
        } catch (...) {                                                                        \
            doctest_ok_ = false;                                                               \
        }                                                                                      \
        ::doctest::shim::report(doctest_ok_, fatal, text, __FILE__, __LINE__);                 \
    } while (0)

#define CHECK(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), false, #__VA_ARGS__)
#define REQUIRE(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), true, #__VA_ARGS__)
#define CHECK_FALSE(...) DOCTEST_CHECK_IMPL(!(__VA_ARGS__), false, "!(" #__VA_ARGS__ ")")
#define REQUIRE_FALSE(...) DOCTEST_CHECK_IMPL(!(__VA_ARGS__), true, "!(" #__VA_ARGS__ ")")
#define CHECK_MESSAGE(cond, msg)                                                               \
    do {                                                                                       \
        ::doctest::shim::Msg doctest_m_;                                                       \
        doctest_m_ << msg;                                                                     \
        ::doctest::shim::report(static_cast<bool>(cond), false, #cond, __FILE__, __LINE__,     \
                                doctest_m_.os.str());                                          \
    } while (0)
#define REQUIRE_MESSAGE(cond, msg)                                                             \
    do {                                                                                       \
        ::doctest::shim::Msg doctest_m_;                                                       \
        doctest_m_ << msg;                                                                     \
        ::doctest::shim::report(static_cast<bool>(cond), true, #cond, __FILE__, __LINE__,      \
                                doctest_m_.os.str());                                          \
    } while (0)
#define FAIL(msg)                                                                              \
    do {                                                                                       \
        ::doctest::shim::Msg doctest_m_;                                                       \
        doctest_m_ << msg;                                                                     \
        ::doctest::shim::report(false, true, "FAIL", __FILE__, __LINE__, doctest_m_.os.str()); \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                            \
    do {                                                                                       \
        bool doctest_ok_ = false;                                                              \
        try {                                                                                  \
            static_cast<void>(expr);                                                           \
        } catch (const type&) {                                                                \
            doctest_ok_ = true;                                                                \
        } catch (...) {                                                                        \
        }                                                                                      \
        ::doctest::shim::report(doctest_ok_, false, "THROWS_AS(" #expr ", " #type ")",         \
                                __FILE__, __LINE__);                                           \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    const char* filter = nullptr;
    for (int i = 1; i < argc; ++i) {
        std::string a = argv[i];
        if (a.rfind("-tc=", 0) == 0) filter = argv[i] + 4;
    }
    return ::doctest::shim::run_all(filter);
}
#endif
