// Synthetic M4-shaped series for the bench and tests: the reference's seeded generator
// testutil::make_multiplicative_series (tests/helpers.hpp:148-172) consumed in order
// from Rng(seed) (matrix.hpp:173-213).  Compiled with -ffp-contract=off so the values
// are the exact source-order IEEE results.
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

#include "esrnn_b200.h"

namespace {
struct Rng {
    std::mt19937_64 gen;
    bool have_spare = false;
    double spare = 0.0;
    explicit Rng(uint64_t s) : gen(s) {}
    double uniform() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    uint64_t below(uint64_t n) { return static_cast<uint64_t>((static_cast<unsigned __int128>(gen()) * n) >> 64); }
    double normal() {
        if (have_spare) {
            have_spare = false;
            return spare;
        }
        double u1 = uniform(), u2 = uniform();
        while (u1 <= 1e-300) u1 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double th = 2.0 * 3.14159265358979323846 * u2;
        spare = r * std::sin(th);
        have_spare = true;
        return r * std::cos(th);
    }
};
}  // namespace

extern "C" esrnn_status esrnn_make_synthetic(uint64_t seed, int64_t n, int32_t length, int32_t season_length,
                                             double noise_sigma, double* values, int32_t* category) {
    if (n < 0 || length < 0 || season_length < 1) return ESRNN_CONFIG_ERROR;
    Rng rng(seed);
    std::vector<double> season(static_cast<size_t>(season_length));
    for (int64_t i = 0; i < n; ++i) {
        category[i] = static_cast<int32_t>(rng.below(6));
        const double level = rng.uniform(50.0, 150.0);
        const double trend = rng.uniform(0.005, 0.02);
        double log_mean = 0.0;
        for (double& s : season) {
            s = rng.uniform(0.6, 1.4);
            log_mean += std::log(s);
        }
        log_mean /= static_cast<double>(season_length);
        for (double& s : season) s = std::exp(std::log(s) - log_mean);
        for (int32_t t = 0; t < length; ++t) {
            const double noise = noise_sigma > 0.0 ? std::exp(noise_sigma * rng.normal()) : 1.0;
            values[i * length + t] =
                level * std::pow(1.0 + trend, static_cast<double>(t)) * season[static_cast<size_t>(t % season_length)] * noise;
        }
    }
    return ESRNN_OK;
}
