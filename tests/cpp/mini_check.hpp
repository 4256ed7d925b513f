// A minimal check harness for the re-expressed reference suites (doctest is not
// in the image): a case is a function, a failed expectation prints its line,
// run_cases() prints one line per case and returns the number of failed cases.
#pragma once
#include <cstdio>
#include <exception>
#include <functional>
#include <utility>
#include <vector>

inline int g_failed_checks = 0;
#define EXPECT(cond)                                                         \
    do {                                                                     \
        if (!(cond)) {                                                       \
            std::printf("    line %d: expected %s\n", __LINE__, #cond);      \
            ++g_failed_checks;                                               \
        }                                                                    \
    } while (0)
#define EXPECT_THROWS(expr, Type)                                            \
    do {                                                                     \
        bool caught_ = false;                                                \
        try {                                                                \
            (void)(expr);                                                    \
        } catch (const Type&) {                                              \
            caught_ = true;                                                  \
        } catch (const std::exception& e_) {                                 \
            std::printf("    line %d: %s threw %s\n", __LINE__, #expr, e_.what()); \
        }                                                                    \
        if (!caught_) {                                                      \
            std::printf("    line %d: expected %s from %s\n", __LINE__, #Type, #expr); \
            ++g_failed_checks;                                               \
        }                                                                    \
    } while (0)


inline int run_cases(const std::vector<std::pair<const char*, std::function<void()>>>& cases) {
    int failed = 0;
    for (auto& [name, fn] : cases) {
        const int before = g_failed_checks;
        try {
            fn();
        } catch (const std::exception& e) {
            std::printf("    unexpected exception: %s\n", e.what());
            ++g_failed_checks;
        }
        const bool ok = g_failed_checks == before;
        std::printf("%s %s\n", ok ? "ok  " : "FAIL", name);
        failed += ok ? 0 : 1;
    }
    std::printf("%zu cases, %d failed\n", cases.size(), failed);
    return failed;
}
