// Bulk generation for Mt64 (mt64.h).  Compiled by g++ (not nvcc) so the AVX2 clones can
// use target attributes; the generic clone is plain x86-64.
#include "mt64.h"

#include <algorithm>
#include <sstream>

namespace esrnn_host {
namespace {

constexpr uint64_t kA = 0xB5026F5AA96619E9ULL, kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL;

// std::mersenne_twister_engine::_M_gen_rand for (w, n, m, r) = (64, 312, 156, 31)
__attribute__((always_inline)) inline void twist_body(uint64_t* x) {
    constexpr int N = Mt64::kN, M = Mt64::kM;
    for (int i = 0; i < N - M; ++i) {
        const uint64_t y = (x[i] & kUpper) | (x[i + 1] & kLower);
        x[i] = x[i + M] ^ (y >> 1) ^ ((0 - (y & 1)) & kA);
    }
    for (int i = N - M; i < N - 1; ++i) {
        const uint64_t y = (x[i] & kUpper) | (x[i + 1] & kLower);
        x[i] = x[i + M - N] ^ (y >> 1) ^ ((0 - (y & 1)) & kA);
    }
    const uint64_t y = (x[N - 1] & kUpper) | (x[0] & kLower);
    x[N - 1] = x[M - 1] ^ (y >> 1) ^ ((0 - (y & 1)) & kA);
}

__attribute__((always_inline)) inline void fill_body(Mt64& g, uint64_t* out, size_t n) {
    while (n) {
        if (g.p >= Mt64::kN) {
            twist_body(g.x);
            g.p = 0;
        }
        const size_t k = std::min<size_t>(n, static_cast<size_t>(Mt64::kN - g.p));
        const uint64_t* src = g.x + g.p;
        for (size_t i = 0; i < k; ++i) out[i] = Mt64::temper(src[i]);
        out += k;
        n -= k;
        g.p += static_cast<int>(k);
    }
}

void twist_generic(uint64_t* x) { twist_body(x); }
void fill_generic(Mt64& g, uint64_t* out, size_t n) { fill_body(g, out, n); }
#if defined(__x86_64__) && !defined(ESRNN_MT64_GENERIC)
__attribute__((target("avx2"))) void twist_avx2(uint64_t* x) { twist_body(x); }
__attribute__((target("avx2"))) void fill_avx2(Mt64& g, uint64_t* out, size_t n) { fill_body(g, out, n); }
bool have_avx2() {
    static const bool v = __builtin_cpu_supports("avx2");
    return v;
}
#else  // e.g. aarch64 hosts: the generic clone (auto-vectorised for the base ISA)
void twist_avx2(uint64_t* x) { twist_body(x); }
void fill_avx2(Mt64& g, uint64_t* out, size_t n) { fill_body(g, out, n); }
bool have_avx2() { return false; }
#endif

}  // namespace

void Mt64::twist() {
    if (have_avx2())
        twist_avx2(x);
    else
        twist_generic(x);
    p = 0;
}

void Mt64::fill(uint64_t* out, size_t n) {
    if (have_avx2())
        fill_avx2(*this, out, n);
    else
        fill_generic(*this, out, n);
}

// libstdc++'s operator<< / >> for mersenne_twister_engine: the n state words, then _M_p
std::mt19937_64 Mt64::to_std() const {
    std::ostringstream os;
    for (int i = 0; i < kN; ++i) os << x[i] << ' ';
    os << p;
    std::istringstream is(os.str());
    std::mt19937_64 g;
    is >> g;
    return g;
}

Mt64 Mt64::from_std(const std::mt19937_64& g) {
    std::ostringstream os;
    os << g;
    std::istringstream is(os.str());
    Mt64 m;
    for (int i = 0; i < kN; ++i) is >> m.x[i];
    is >> m.p;
    return m;
}

}  // namespace esrnn_host
