// Minimal stand-in for doctest (absent from the image: SURVEY.md section 8c), enough to build
// the reference's engine tests unmodified: TEST_CASE, CHECK, CHECK_THROWS_AS and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN. Each case runs in registration order; a failed CHECK is
// reported with its file:line and expression, and the process exits nonzero.
#pragma once
#include <cstdio>
#include <exception>
#include <string>
#include <vector>

namespace doctest_shim {
struct Case {
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& cases() {
    static std::vector<Case> v;
    return v;
}
inline int& case_failures() {
    static int f = 0;
    return f;
}
inline void fail(const char* file, int line, const char* what) {
    ++case_failures();
    std::printf("  %s:%d: CHECK( %s ) failed\n", file, line, what);
}
struct Reg {
    Reg(const char* n, void (*f)()) { cases().push_back({n, f}); }
};
inline int run_all() {
    int failed = 0;
    for (const auto& c : cases()) {
        case_failures() = 0;
        try {
            c.fn();
        } catch (const std::exception& e) {
            ++case_failures();
            std::printf("  exception: %s\n", e.what());
        }
        std::printf("[%s] %s\n", case_failures() ? "FAIL" : "PASS", c.name);
        std::fflush(stdout);
        failed += case_failures() ? 1 : 0;
    }
    std::printf("%zu test cases, %d failed\n", cases().size(), failed);
    return failed ? 1 : 0;
}
}  // namespace doctest_shim

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define TEST_CASE(name)                                                                            \
    static void DOCTEST_SHIM_CAT(doctest_case_, __LINE__)();                                       \
    static doctest_shim::Reg DOCTEST_SHIM_CAT(doctest_reg_, __LINE__)(name,                        \
                                                                      DOCTEST_SHIM_CAT(doctest_case_, __LINE__)); \
    static void DOCTEST_SHIM_CAT(doctest_case_, __LINE__)()
#define CHECK(...)                                                                  \
    do {                                                                            \
        if (!(__VA_ARGS__)) doctest_shim::fail(__FILE__, __LINE__, #__VA_ARGS__);   \
    } while (0)
#define CHECK_THROWS_AS(expr, exc)                                                  \
    do {                                                                            \
        bool doctest_shim_ok = false;                                               \
        try {                                                                       \
            (void)(expr);                                                           \
        } catch (const exc&) {                                                      \
            doctest_shim_ok = true;                                                 \
        } catch (...) {                                                             \
        }                                                                           \
        if (!doctest_shim_ok) doctest_shim::fail(__FILE__, __LINE__, #expr " throws " #exc); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest_shim::run_all(); }
#endif
