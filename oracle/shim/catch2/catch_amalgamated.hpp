// Minimal Catch2-v3 subset so the reference's OWN unit tests (proj/tests/*.cpp) can run
// against the shim-built oracle.  TEST INFRASTRUCTURE ONLY.  Supports TEST_CASE, REQUIRE,
// REQUIRE_FALSE, REQUIRE_THROWS, REQUIRE_THROWS_AS, REQUIRE_NOTHROW, FAIL and
// Catch::Approx (default epsilon = float eps * 100 like Catch2, .margin, .epsilon).
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

namespace Catch {
struct TestFailure : std::exception {};
struct Registry {
    struct Entry { const char* name; void (*fn)(); };
    static std::vector<Entry>& all() { static std::vector<Entry> v; return v; }
};
struct Registrar {
    Registrar(const char* name, void (*fn)()) { Registry::all().push_back({name, fn}); }
};
class Approx {
  public:
    explicit Approx(double v) : value_(v) {}
    Approx& margin(double m) { margin_ = m; return *this; }
    Approx& epsilon(double e) { eps_ = e; return *this; }
    friend bool operator==(double lhs, const Approx& rhs) { return rhs.eq(lhs); }
    friend bool operator==(const Approx& lhs, double rhs) { return lhs.eq(rhs); }
    friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.eq(lhs); }
  private:
    bool eq(double x) const {
        if (std::fabs(x - value_) <= margin_) return true;
        const double scale = std::fabs(value_) > std::fabs(x) ? std::fabs(value_) : std::fabs(x);
        return std::fabs(x - value_) <= eps_ * (scale + (std::isinf(value_) ? 0 : 0));
    }
    double value_;
    double margin_ = 0.0;
    double eps_ = std::numeric_limits<float>::epsilon() * 100;
};
inline int& failures() { static int f = 0; return f; }
inline void fail(const char* file, int line, const char* expr) {
    std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
    throw TestFailure();
}
}  // namespace Catch

#define CATCH_CAT2(a, b) a##b
#define CATCH_CAT(a, b) CATCH_CAT2(a, b)
#define TEST_CASE(name, ...)                                                            \
    static void CATCH_CAT(catch_test_, __LINE__)();                                     \
    static Catch::Registrar CATCH_CAT(catch_reg_, __LINE__)(name, &CATCH_CAT(catch_test_, __LINE__)); \
    static void CATCH_CAT(catch_test_, __LINE__)()
#define REQUIRE(...) do { if (!(__VA_ARGS__)) Catch::fail(__FILE__, __LINE__, #__VA_ARGS__); } while (0)
#define REQUIRE_FALSE(...) do { if ((__VA_ARGS__)) Catch::fail(__FILE__, __LINE__, "!" #__VA_ARGS__); } while (0)
#define REQUIRE_THROWS(...) do { bool t_ = false; try { (void)(__VA_ARGS__); } catch (...) { t_ = true; } \
    if (!t_) Catch::fail(__FILE__, __LINE__, "throws: " #__VA_ARGS__); } while (0)
#define REQUIRE_THROWS_AS(expr, type) do { bool t_ = false; try { (void)(expr); } catch (const type&) { t_ = true; } catch (...) {} \
    if (!t_) Catch::fail(__FILE__, __LINE__, "throws " #type ": " #expr); } while (0)
#define REQUIRE_NOTHROW(...) do { try { (void)(__VA_ARGS__); } catch (...) { Catch::fail(__FILE__, __LINE__, "nothrow: " #__VA_ARGS__); } } while (0)
#define FAIL(msg) Catch::fail(__FILE__, __LINE__, "FAIL")

#ifdef CATCH_SHIM_MAIN
int main() {
    int failed = 0, n = 0;
    for (const auto& e : Catch::Registry::all()) {
        ++n;
        try { e.fn(); std::printf("PASS %s\n", e.name); }
        catch (const Catch::TestFailure&) { ++failed; std::printf("FAIL %s\n", e.name); }
        catch (const std::exception& ex) { ++failed; std::printf("FAIL %s (exception: %s)\n", e.name, ex.what()); }
    }
    std::printf("%d/%d test cases passed\n", n - failed, n);
    return failed;
}
#endif
