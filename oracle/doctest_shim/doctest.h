// TEST INFRASTRUCTURE ONLY (oracle/): the subset of doctest 2.x used by the
// reference's unit suites (proj/tests/*.cpp; doctest is expected under
// proj/vendor/ and is absent). Supports TEST_SUITE, TEST_CASE, flat SUBCASEs,
// CHECK/REQUIRE(_FALSE), CHECK_THROWS_AS, CHECK_NOTHROW, FAIL and
// doctest::Approx with doctest's default epsilon (100 * FLT_EPSILON) and
// comparison rule. Command line: -ts=<suite>[,<suite>...] and -tc=<case>.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <set>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double value)
        : value_(value), epsilon_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100) {}
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
               rhs.epsilon_ * (rhs.scale_ + std::max<double>(std::fabs(lhs), std::fabs(rhs.value_)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }
    friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || lhs == rhs; }
    friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || lhs == rhs; }

private:
    double value_;
    double epsilon_;
    double scale_ = 1.0;
};

namespace shim {

struct RequireFailed {};

struct Case {
    void (*fn)();
    const char* name;
    const char* suite;
    const char* file;
    int line;
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
inline int reg(void (*fn)(), const char* name, const char* suite, const char* file, int line) {
    registry().push_back({fn, name, suite, file, line});
    return 0;
}

struct State {
    long long checks = 0, failures = 0;
    bool case_failed = false;
    // flat SUBCASE scheduling: each run enters the first not-yet-done subcase
    std::set<int> done;
    int entered = -1;
    bool saw_new = false;
};
inline State& st() {
    static State s;
    return s;
}

inline void fail_msg(const char* kind, const char* expr, const char* file, int line) {
    ++st().failures;
    st().case_failed = true;
    std::fprintf(stderr, "%s:%d: %s FAILED: %s\n", file, line, kind, expr);
}
inline void check(bool ok, const char* kind, const char* expr, const char* file, int line,
                  bool require) {
    ++st().checks;
    if (!ok) {
        fail_msg(kind, expr, file, line);
        if (require) throw RequireFailed{};
    }
}

struct Subcase {
    bool active = false;
    int id;
    Subcase(int line) : id(line) {
        State& s = st();
        if (s.entered < 0 && !s.done.count(id)) {
            s.entered = id;
            active = true;
        } else if (!s.done.count(id) && s.entered != id) {
            s.saw_new = true;
        }
    }
    ~Subcase() {
        if (active) st().done.insert(id);
    }
    explicit operator bool() const { return active; }
};

inline std::vector<std::string> split(const char* s) {
    std::vector<std::string> out;
    std::string cur;
    for (const char* p = s; *p; ++p) {
        if (*p == ',') {
            out.push_back(cur);
            cur.clear();
        } else {
            cur += *p;
        }
    }
    if (!cur.empty()) out.push_back(cur);
    return out;
}

inline int run(int argc, char** argv) {
    std::vector<std::string> suites, cases;
    for (int i = 1; i < argc; ++i) {
        if (std::strncmp(argv[i], "-ts=", 4) == 0) suites = split(argv[i] + 4);
        if (std::strncmp(argv[i], "-tc=", 4) == 0) cases = split(argv[i] + 4);
    }
    int ran = 0, failed_cases = 0;
    for (const Case& c : registry()) {
        if (!suites.empty() && std::find(suites.begin(), suites.end(), c.suite) == suites.end())
            continue;
        if (!cases.empty() && std::find(cases.begin(), cases.end(), c.name) == cases.end())
            continue;
        ++ran;
        State& s = st();
        s.case_failed = false;
        s.done.clear();
        for (;;) {
            s.entered = -1;
            s.saw_new = false;
            try {
                c.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                fail_msg("EXCEPTION", e.what(), c.file, c.line);
            } catch (...) {
                fail_msg("EXCEPTION", "unknown", c.file, c.line);
            }
            if (!s.saw_new) break;  // no undone subcase left besides the one just run
        }
        if (s.case_failed) {
            ++failed_cases;
            std::fprintf(stderr, "[case FAILED] %s / %s\n", c.suite, c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %d | passed: %d | failed: %d | assertions: %lld | "
                "failed assertions: %lld\n",
                ran, ran - failed_cases, failed_cases, st().checks, st().failures);
    return failed_cases == 0 ? 0 : 1;
}

}  // namespace shim
}  // namespace doctest

static const char* const doctest_suite_name = "";

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)

#define TEST_SUITE(name)                                                   \
    namespace DOCTEST_CAT(doctest_suite_ns_, __LINE__) {                   \
    static const char* const doctest_suite_name = name;                    \
    }                                                                      \
    namespace DOCTEST_CAT(doctest_suite_ns_, __LINE__)

#define DOCTEST_TC_IMPL(f, name)                                                              \
    static void f();                                                                          \
    static const int DOCTEST_CAT(f, _reg) =                                                   \
        doctest::shim::reg(f, name, doctest_suite_name, __FILE__, __LINE__);                  \
    static void f()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)

#define SUBCASE(name) if (doctest::shim::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){__LINE__})

#define CHECK(...) doctest::shim::check(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::shim::check(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::shim::check(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__, true)
#define REQUIRE_FALSE(...) doctest::shim::check(!static_cast<bool>(__VA_ARGS__), "REQUIRE_FALSE", #__VA_ARGS__, __FILE__, __LINE__, true)
#define FAIL(msg) doctest::shim::check(false, "FAIL", "FAIL", __FILE__, __LINE__, true)

#define CHECK_THROWS_AS(expr, ...)                                                   \
    do {                                                                             \
        bool doctest_threw_ = false;                                                 \
        try {                                                                        \
            static_cast<void>(expr);                                                 \
        } catch (const __VA_ARGS__&) {                                               \
            doctest_threw_ = true;                                                   \
        } catch (...) {                                                              \
        }                                                                            \
        doctest::shim::check(doctest_threw_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__, false); \
    } while (0)

#define CHECK_NOTHROW(...)                                                           \
    do {                                                                             \
        bool doctest_ok_ = true;                                                     \
        try {                                                                        \
            static_cast<void>(__VA_ARGS__);                                          \
        } catch (...) {                                                              \
            doctest_ok_ = false;                                                     \
        }                                                                            \
        doctest::shim::check(doctest_ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::shim::run(argc, argv); }
#endif
