// Mt64 (csrc/mt64.h) against std::mt19937_64: outputs, bulk fill, mixed use, text state.
#include <cstdio>
#include <random>
#include <sstream>
#include <vector>

#include "mt64.h"

using esrnn_host::Mt64;

static int fails = 0;
#define CHECK(c)                                                   \
    do {                                                           \
        if (!(c)) {                                                \
            std::fprintf(stderr, "FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
            ++fails;                                               \
        }                                                          \
    } while (0)

int main() {
    for (uint64_t seed : {0ull, 1ull, 7ull, 5489ull, 0xDEADBEEFCAFEull, ~0ull}) {
        std::mt19937_64 s(seed);
        Mt64 m(seed);
        // single draws, then bulk blocks of awkward sizes across twist boundaries
        for (int i = 0; i < 1000; ++i) CHECK(s() == m());
        for (size_t n : {size_t(0), size_t(1), size_t(311), size_t(312), size_t(313), size_t(1000), size_t(53000)}) {
            std::vector<uint64_t> a(n), b(n);
            for (auto& v : a) v = s();
            m.fill(b.data(), n);
            CHECK(a == b);
            CHECK(s() == m());
        }
        // text state: Mt64 -> std and std -> Mt64 continue the same sequence
        std::mt19937_64 t = m.to_std();
        std::ostringstream o1, o2;
        o1 << t;
        o2 << s;
        CHECK(o1.str() == o2.str());
        Mt64 back = Mt64::from_std(s);
        for (int i = 0; i < 700; ++i) {
            const uint64_t v = s();
            CHECK(t() == v);
            CHECK(back() == v);
        }
    }
    std::printf(fails ? "mt64: %d failures\n" : "mt64: ok\n", fails);
    return fails != 0;
}
