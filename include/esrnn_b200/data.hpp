// Data-model structs the Trainer boundary exposes (reference data.hpp: enums :18-19,
// SeriesRecord :52-57, FrequencyProfile :60-118, DatasetSplit/split :122-140,
// equalize_lengths :148-161, one_hot_category :163-167).
#pragma once
#include <array>
#include <optional>
#include <string>
#include <string_view>
#include <vector>

#include "errors.hpp"

namespace esrnn {

enum class Category { Demographic, Finance, Industry, Macro, Micro, Other };
enum class Frequency { Yearly, Quarterly, Monthly };
inline constexpr int kNumCategories = ESRNN_NUM_CATEGORIES;

inline const char* to_string(Category c) {
    static constexpr const char* k[] = {"Demographic", "Finance", "Industry", "Macro", "Micro", "Other"};
    return k[static_cast<int>(c)];
}
inline const char* to_string(Frequency f) {
    return f == Frequency::Yearly ? "Yearly" : (f == Frequency::Quarterly ? "Quarterly" : "Monthly");
}
inline Category parse_category(std::string_view s) {
    for (int i = 0; i < kNumCategories; ++i)
        if (s == to_string(static_cast<Category>(i))) return static_cast<Category>(i);
    throw ValidationError("unknown category \"" + std::string(s) + "\"");
}
inline Frequency parse_frequency(std::string_view s) {
    for (Frequency f : {Frequency::Yearly, Frequency::Quarterly, Frequency::Monthly})
        if (s == to_string(f)) return f;
    throw ValidationError("unknown frequency \"" + std::string(s) + "\"");
}

struct SeriesRecord {
    std::string id;
    std::optional<Category> category;
    std::optional<Frequency> frequency;
    std::vector<double> values;
};

struct FrequencyProfile {
    Frequency frequency = Frequency::Quarterly;
    int seasonality_length = 4;   // S
    int horizon = 8;              // O
    int input_window = 12;        // I
    std::vector<std::vector<int>> dilation_blocks = {{1, 2}, {4, 8}};
    int hidden_size = 40;
    int min_length = 72;          // C

    static FrequencyProfile defaults(Frequency f) {
        FrequencyProfile p;
        p.frequency = f;
        if (f == Frequency::Yearly) {
            p.seasonality_length = 1, p.horizon = 6, p.input_window = 6, p.hidden_size = 30, p.min_length = 13;
            p.dilation_blocks = {{1, 2}, {2, 6}};
        } else if (f == Frequency::Monthly) {
            p.seasonality_length = 12, p.horizon = 18, p.input_window = 24, p.hidden_size = 50, p.min_length = 72;
            p.dilation_blocks = {{1, 3}, {6, 12}};
        }
        return p;
    }
    void validate() const {
        if (seasonality_length < 1) throw ConfigError("profile: seasonality must be >= 1");
        if (horizon < 1) throw ConfigError("profile: horizon must be >= 1");
        if (input_window < seasonality_length) throw ConfigError("profile: input_window must cover at least one season");
        if (dilation_blocks.empty()) throw ConfigError("profile: dilation blocks must be non-empty");
        for (const auto& b : dilation_blocks) {
            if (b.empty()) throw ConfigError("profile: empty dilation block");
            for (int d : b)
                if (d < 1) throw ConfigError("profile: dilations must be strictly positive");
        }
        if (hidden_size < 1) throw ConfigError("profile: hidden_size must be >= 1");
        if (min_length < 1) throw ConfigError("profile: min_length must be >= 1");
    }
    int equalized_length() const { return min_length + 2 * horizon; }
};

struct DatasetSplit {
    std::vector<double> train, validation, test;
};

inline DatasetSplit split_train_val_test(const std::vector<double>& v, int horizon) {
    const std::size_t n = v.size(), o = static_cast<std::size_t>(horizon);
    if (n < 2 * o + 1)
        throw InsufficientLengthError("split: need at least " + std::to_string(2 * o + 1) + " values, got " +
                                      std::to_string(n));
    DatasetSplit s;
    s.train.assign(v.begin(), v.begin() + static_cast<std::ptrdiff_t>(n - 2 * o));
    s.validation.assign(v.begin() + static_cast<std::ptrdiff_t>(n - 2 * o), v.begin() + static_cast<std::ptrdiff_t>(n - o));
    s.test.assign(v.begin() + static_cast<std::ptrdiff_t>(n - o), v.end());
    return s;
}
inline DatasetSplit split_train_val_test(const SeriesRecord& r, int horizon) { return split_train_val_test(r.values, horizon); }

inline std::vector<SeriesRecord> equalize_lengths(std::vector<SeriesRecord> series, const FrequencyProfile& p) {
    const std::size_t keep = static_cast<std::size_t>(p.equalized_length());
    std::vector<SeriesRecord> out;
    for (auto& s : series) {
        if (s.values.size() < keep) continue;
        s.values.erase(s.values.begin(), s.values.end() - static_cast<std::ptrdiff_t>(keep));
        out.push_back(std::move(s));
    }
    return out;
}

inline std::array<double, 6> one_hot_category(Category c) {
    std::array<double, 6> v{};
    v[static_cast<std::size_t>(c)] = 1.0;
    return v;
}

}  // namespace esrnn
