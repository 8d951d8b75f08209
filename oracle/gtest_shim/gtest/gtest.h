// Minimal GoogleTest-compatible shim (test infrastructure only).
//
// GoogleTest is not installed in this image. This header
// implements the subset of the gtest surface the reference suites under
// /root/reference/proj/tests use (TEST, EXPECT_*/ASSERT_* incl. NEAR /
// DOUBLE_EQ / THROW, message streaming, ::testing::TempDir) so that the
// reference's own 137 tests can be compiled in place and run as the golden
// semantics for the oracle. It is NOT part of the product.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

namespace testing {

struct TestCase {
    const char* suite;
    const char* name;
    std::function<void()> fn;
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

inline bool& current_failed() {
    static bool f = false;
    return f;
}

struct Registrar {
    Registrar(const char* s, const char* n, std::function<void()> fn) {
        registry().push_back(TestCase{s, n, std::move(fn)});
    }
};

// Collects the streamed user message and reports on destruction.
class Reporter {
public:
    Reporter(bool ok, const char* file, int line, std::string what)
        : ok_(ok), file_(file), line_(line), what_(std::move(what)) {}
    ~Reporter() {
        if (!ok_) {
            current_failed() = true;
            std::fprintf(stderr, "%s:%d: Failure\n%s %s\n", file_, line_, what_.c_str(),
                         msg_.str().c_str());
        }
    }
    template <typename T>
    Reporter& operator<<(const T& v) {
        if (!ok_) msg_ << v;
        return *this;
    }
    bool ok() const { return ok_; }

private:
    bool ok_;
    const char* file_;
    int line_;
    std::string what_;
    std::ostringstream msg_;
};

struct AssertionAbort {};

inline std::string TempDir() {
    const char* t = std::getenv("TMPDIR");
    std::string d = t ? t : "/tmp";
    if (!d.empty() && d.back() != '/') d.push_back('/');
    return d;
}

inline bool double_eq(double a, double b) {
    if (a == b) return true;
    if (std::isnan(a) || std::isnan(b)) return false;
    // gtest: within 4 ULPs
    std::int64_t ia, ib;
    std::memcpy(&ia, &a, 8);
    std::memcpy(&ib, &b, 8);
    if ((ia < 0) != (ib < 0)) return false;
    std::int64_t d = ia > ib ? ia - ib : ib - ia;
    return d <= 4;
}

inline int RunAll(const char* filter) {
    int failed = 0, run = 0;
    for (auto& t : registry()) {
        std::string full = std::string(t.suite) + "." + t.name;
        if (filter && *filter && full.find(filter) == std::string::npos) continue;
        current_failed() = false;
        ++run;
        try {
            t.fn();
        } catch (const AssertionAbort&) {
        } catch (const std::exception& e) {
            current_failed() = true;
            std::fprintf(stderr, "uncaught exception: %s\n", e.what());
        } catch (...) {
            current_failed() = true;
            std::fprintf(stderr, "uncaught non-std exception\n");
        }
        std::printf("[%s] %s\n", current_failed() ? "  FAILED  " : "       OK ", full.c_str());
        failed += current_failed() ? 1 : 0;
    }
    std::printf("[==========] %d tests ran, %d passed, %d failed\n", run, run - failed, failed);
    return failed == 0 ? 0 : 1;
}

}  // namespace testing

#define GSHIM_CAT2(a, b) a##b
#define GSHIM_CAT(a, b) GSHIM_CAT2(a, b)

#define TEST(suite, name)                                                              \
    static void GSHIM_CAT(gshim_##suite##_, name)();                                   \
    static ::testing::Registrar GSHIM_CAT(gshim_reg_##suite##_, name)(                 \
        #suite, #name, &GSHIM_CAT(gshim_##suite##_, name));                            \
    static void GSHIM_CAT(gshim_##suite##_, name)()

// EXPECT_*: report and continue. ASSERT_*: report and abort the test body.
#define GSHIM_CHECK(cond, what) ::testing::Reporter((cond), __FILE__, __LINE__, (what))
#define GSHIM_ASSERT(cond, what)                                                       \
    if (bool gshim_ok_ = (cond); gshim_ok_) {                                          \
    } else                                                                             \
        for (bool gshim_once_ = true; gshim_once_; gshim_once_ = false,                \
                  throw ::testing::AssertionAbort{})                                   \
    ::testing::Reporter(false, __FILE__, __LINE__, (what))

#define EXPECT_TRUE(c) GSHIM_CHECK(static_cast<bool>(c), "EXPECT_TRUE(" #c ")")
#define EXPECT_FALSE(c) GSHIM_CHECK(!static_cast<bool>(c), "EXPECT_FALSE(" #c ")")
#define EXPECT_EQ(a, b) GSHIM_CHECK((a) == (b), "EXPECT_EQ(" #a ", " #b ")")
#define EXPECT_NE(a, b) GSHIM_CHECK((a) != (b), "EXPECT_NE(" #a ", " #b ")")
#define EXPECT_LT(a, b) GSHIM_CHECK((a) < (b), "EXPECT_LT(" #a ", " #b ")")
#define EXPECT_LE(a, b) GSHIM_CHECK((a) <= (b), "EXPECT_LE(" #a ", " #b ")")
#define EXPECT_GT(a, b) GSHIM_CHECK((a) > (b), "EXPECT_GT(" #a ", " #b ")")
#define EXPECT_GE(a, b) GSHIM_CHECK((a) >= (b), "EXPECT_GE(" #a ", " #b ")")
#define EXPECT_NEAR(a, b, t) \
    GSHIM_CHECK(std::fabs(static_cast<double>(a) - static_cast<double>(b)) <= (t), "EXPECT_NEAR(" #a ", " #b ")")
#define EXPECT_DOUBLE_EQ(a, b) GSHIM_CHECK(::testing::double_eq((a), (b)), "EXPECT_DOUBLE_EQ(" #a ", " #b ")")

#define ASSERT_TRUE(c) GSHIM_ASSERT(static_cast<bool>(c), "ASSERT_TRUE(" #c ")")
#define ASSERT_FALSE(c) GSHIM_ASSERT(!static_cast<bool>(c), "ASSERT_FALSE(" #c ")")
#define ASSERT_EQ(a, b) GSHIM_ASSERT((a) == (b), "ASSERT_EQ(" #a ", " #b ")")
#define ASSERT_NE(a, b) GSHIM_ASSERT((a) != (b), "ASSERT_NE(" #a ", " #b ")")
#define ASSERT_LT(a, b) GSHIM_ASSERT((a) < (b), "ASSERT_LT(" #a ", " #b ")")
#define ASSERT_LE(a, b) GSHIM_ASSERT((a) <= (b), "ASSERT_LE(" #a ", " #b ")")
#define ASSERT_GT(a, b) GSHIM_ASSERT((a) > (b), "ASSERT_GT(" #a ", " #b ")")
#define ASSERT_GE(a, b) GSHIM_ASSERT((a) >= (b), "ASSERT_GE(" #a ", " #b ")")

#define EXPECT_THROW(stmt, exc)                                                        \
    do {                                                                               \
        bool gshim_caught_ = false;                                                    \
        try {                                                                          \
            stmt;                                                                      \
        } catch (const exc&) {                                                         \
            gshim_caught_ = true;                                                      \
        } catch (...) {                                                                \
        }                                                                              \
        GSHIM_CHECK(gshim_caught_, "EXPECT_THROW(" #stmt ", " #exc ")");               \
    } while (0)

#define EXPECT_NO_THROW(stmt)                                                          \
    do {                                                                               \
        bool gshim_ok_ = true;                                                         \
        try {                                                                          \
            stmt;                                                                      \
        } catch (...) {                                                                \
            gshim_ok_ = false;                                                         \
        }                                                                              \
        GSHIM_CHECK(gshim_ok_, "EXPECT_NO_THROW(" #stmt ")");                          \
    } while (0)

#define FAIL() GSHIM_ASSERT(false, "FAIL()")
#define SUCCEED() GSHIM_CHECK(true, "SUCCEED()")

#ifndef GSHIM_NO_MAIN
int main(int argc, char** argv) {
    return ::testing::RunAll(argc > 1 ? argv[1] : nullptr);
}
#endif
