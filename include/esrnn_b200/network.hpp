// Network weight structs of the drop-in API (reference network.hpp:16-85): the fused gate
// layout [input | forget | candidate | output] and the fixed for_each_param order that is
// also the checkpoint layout and the engine's flat weight vector order.
#pragma once
#include <string>
#include <vector>

#include "matrix.hpp"

namespace esrnn {

struct LSTMCellWeights {
    Matrix w_input;   // (input_size, 4H)
    Matrix w_recur;   // (H, 4H)
    Matrix bias;      // (1, 4H)
    int hidden() const { return static_cast<int>(w_recur.rows()); }
    int input_size() const { return static_cast<int>(w_input.rows()); }
};

struct StackConfig {
    std::vector<std::vector<int>> dilation_blocks;
    int hidden_size = 0, input_size = 0, output_size = 0;
    int num_layers() const {
        int n = 0;
        for (const auto& b : dilation_blocks) n += static_cast<int>(b.size());
        return n;
    }
    void validate() const {
        if (dilation_blocks.empty()) throw ConfigError("stack: dilation blocks must be non-empty");
        for (const auto& b : dilation_blocks) {
            if (b.empty()) throw ConfigError("stack: empty dilation block");
            for (int d : b)
                if (d < 1) throw ConfigError("stack: dilation must be >= 1");
        }
        if (hidden_size < 1 || input_size < 1 || output_size < 1) throw ConfigError("stack: sizes must be positive");
    }
};

struct StackWeights {
    std::vector<LSTMCellWeights> layers;
    Matrix nl_w, nl_b, out_w, out_b;

    template <typename Fn>
    void for_each_param(Fn&& fn) {
        for (std::size_t i = 0; i < layers.size(); ++i) {
            const std::string p = "lstm" + std::to_string(i);
            fn(p + ".w_input", layers[i].w_input);
            fn(p + ".w_recur", layers[i].w_recur);
            fn(p + ".bias", layers[i].bias);
        }
        fn("head.nl_w", nl_w);
        fn("head.nl_b", nl_b);
        fn("head.out_w", out_w);
        fn("head.out_b", out_b);
    }
    template <typename Fn>
    void for_each_param(Fn&& fn) const {
        const_cast<StackWeights*>(this)->for_each_param([&](const std::string& n, Matrix& m) { fn(n, static_cast<const Matrix&>(m)); });
    }
    void zero() {
        for_each_param([](const std::string&, Matrix& m) { m.fill(0.0); });
    }
};

}  // namespace esrnn
