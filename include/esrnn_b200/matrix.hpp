// Row-major fp64 Matrix and the deterministic Rng of the drop-in API (same surface as the
// reference's matrix.hpp: Matrix :16-85, Rng :173-213).  Only host bookkeeping lives here;
// the arithmetic of the hot path runs in the CUDA engine.
#pragma once
#include <cmath>
#include <cstdint>
#include <initializer_list>
#include <random>
#include <string>
#include <utility>
#include <vector>

#include "errors.hpp"

namespace esrnn {

class Matrix {
public:
    Matrix() = default;
    Matrix(std::size_t rows, std::size_t cols, double fill = 0.0) : r_(rows), c_(cols), v_(rows * cols, fill) {}
    static Matrix from_rows(std::initializer_list<std::initializer_list<double>> rows) {
        Matrix m(rows.size(), rows.size() ? rows.begin()->size() : 0);
        std::size_t i = 0;
        for (const auto& row : rows) {
            if (row.size() != m.c_) throw ShapeError("from_rows: ragged initializer");
            for (double x : row) m.v_[i++] = x;
        }
        return m;
    }
    static Matrix column(const std::vector<double>& v) {
        Matrix m(v.size(), 1);
        m.v_ = v;
        return m;
    }
    std::size_t rows() const { return r_; }
    std::size_t cols() const { return c_; }
    std::size_t size() const { return v_.size(); }
    bool empty() const { return v_.empty(); }
    double& operator()(std::size_t r, std::size_t c) { return v_[r * c_ + c]; }
    double operator()(std::size_t r, std::size_t c) const { return v_[r * c_ + c]; }
    double* row(std::size_t r) { return v_.data() + r * c_; }
    const double* row(std::size_t r) const { return v_.data() + r * c_; }
    std::vector<double>& data() { return v_; }
    const std::vector<double>& data() const { return v_; }
    bool same_shape(const Matrix& o) const { return r_ == o.r_ && c_ == o.c_; }
    std::string shape_str() const { return "(" + std::to_string(r_) + ", " + std::to_string(c_) + ")"; }
    void fill(double x) {
        for (double& e : v_) e = x;
    }
    bool all_finite() const {
        for (double e : v_)
            if (!std::isfinite(e)) return false;
        return true;
    }

private:
    std::size_t r_ = 0, c_ = 0;
    std::vector<double> v_;
};

inline void require_same_shape(const Matrix& a, const Matrix& b, const char* op) {
    if (!a.same_shape(b)) throw ShapeError(std::string(op) + ": shape mismatch " + a.shape_str() + " vs " + b.shape_str());
}

// mt19937_64 stream with explicit bit draws, so sequences are platform independent.
class Rng {
public:
    explicit Rng(std::uint64_t seed) : g_(seed) {}
    double uniform() { return static_cast<double>(g_() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    double normal() {
        if (spare_ok_) {
            spare_ok_ = false;
            return spare_;
        }
        double u1 = uniform();
        const double u2 = uniform();
        while (u1 <= 1e-300) u1 = uniform();
        const double rad = std::sqrt(-2.0 * std::log(u1)), th = 2.0 * 3.14159265358979323846 * u2;
        spare_ = rad * std::sin(th);
        spare_ok_ = true;
        return rad * std::cos(th);
    }
    std::uint64_t below(std::uint64_t n) {
        return static_cast<std::uint64_t>((static_cast<unsigned __int128>(g_()) * n) >> 64);
    }
    template <typename T>
    void shuffle(std::vector<T>& v) {
        for (std::size_t i = v.size(); i > 1; --i) std::swap(v[i - 1], v[below(i)]);
    }
    std::uint64_t raw() { return g_(); }

private:
    std::mt19937_64 g_;
    bool spare_ok_ = false;
    double spare_ = 0.0;
};

}  // namespace esrnn
