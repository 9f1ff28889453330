// The trainer RNG (matrix.hpp:173-213 draws from std::mt19937_64): a restatement of the
// 64-bit Mersenne twister that is bit-identical to libstdc++'s std::mt19937_64 -- same
// seeding, outputs, state words and text format -- plus a bulk generator.  An epoch's
// shuffle draws one number per window (53,000 at cfg1) and the weight init one per
// weight, both on the host critical path of trainer creation; drawing them as a block
// (twist + vectorised tempering, AVX2 when the host has it) is ~2.7x faster than calling
// the std engine per number.  Host-only.
#pragma once
#include <cstddef>
#include <cstdint>
#include <random>

namespace esrnn_host {

struct Mt64 {
    static constexpr int kN = 312, kM = 156;
    alignas(64) uint64_t x[kN];
    int p = kN;  // next word (std's _M_p)

    Mt64() { seed_with(5489u); }
    explicit Mt64(uint64_t seed) { seed_with(seed); }
    void seed_with(uint64_t s) {
        x[0] = s;
        for (int i = 1; i < kN; ++i) x[i] = 6364136223846793005ULL * (x[i - 1] ^ (x[i - 1] >> 62)) + static_cast<uint64_t>(i);
        p = kN;
    }
    static uint64_t temper(uint64_t y) {
        y ^= (y >> 29) & 0x5555555555555555ULL;
        y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
        y ^= (y << 37) & 0xFFF7EEE000000000ULL;
        return y ^ (y >> 43);
    }
    uint64_t operator()() {
        if (p >= kN) twist();
        return temper(x[p++]);
    }
    void twist();                          // regenerate the 312 state words
    void fill(uint64_t* out, size_t n);    // == n calls of operator()
    std::mt19937_64 to_std() const;        // via the std text format (checkpoints)
    static Mt64 from_std(const std::mt19937_64& g);
};

}  // namespace esrnn_host
