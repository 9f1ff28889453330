// Per-series Holt-Winters parameters of the drop-in API (reference holt_winters.hpp:26-43):
// alpha/gamma squashed by the logistic, initial seasonality by exp.
#pragma once
#include <cfloat>
#include <cmath>
#include <vector>

namespace esrnn {

inline double squash(double raw) {
    const double y = 1.0 / (1.0 + std::exp(-raw));
    return y < DBL_MIN ? DBL_MIN : (y > 1.0 - DBL_EPSILON / 2.0 ? 1.0 - DBL_EPSILON / 2.0 : y);
}

struct PerSeriesParams {
    double alpha_raw = 0.0;
    double gamma_raw = 0.0;
    std::vector<double> init_seasonality_raw;
    explicit PerSeriesParams(int season_length = 1) : init_seasonality_raw(static_cast<std::size_t>(season_length), 0.0) {}
    int season_length() const { return static_cast<int>(init_seasonality_raw.size()); }
    double alpha() const { return squash(alpha_raw); }
    double gamma() const { return squash(gamma_raw); }
    std::vector<double> initial_seasonality() const {
        std::vector<double> s(init_seasonality_raw.size());
        for (std::size_t i = 0; i < s.size(); ++i) s[i] = std::exp(init_seasonality_raw[i]);
        return s;
    }
};

}  // namespace esrnn
