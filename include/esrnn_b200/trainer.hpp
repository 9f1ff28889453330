// esrnn::Trainer — drop-in replacement for the reference's hot path
// (/root/reference/proj/include/esrnn/trainer.hpp:22-673), header-only over the C-ABI of
// the B200 engine (include/esrnn_b200.h, libesrnn_b200.so).  Same class, struct and
// free-function names, argument meaning and exception types; callers such as the
// reference's checkpoint.hpp / commands.hpp use it unchanged.
//
// Host-mirror coherence: weights() and per_series_params(i) return mutable references
// into host mirrors, as in the reference.  A mirror is refreshed from the device when the
// device copy is newer, and once a mutable reference has been handed out its contents
// are pushed to the device before every later device call (so the reference tests'
// central-difference pattern — holding `double&` to a parameter across batch_loss calls —
// behaves identically).  A device call that trains (train_epoch, step with update) makes
// the mirrors stale again; re-take references after training.
#pragma once
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <optional>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "../esrnn_b200.h"
#ifdef ESRNN_B200_HOST_TYPES
// Include swap of trainer.hpp alone: the caller's tree keeps its own value types
// (esrnn/{data,errors,holt_winters,matrix,network}.hpp of the reference) and only the
// Trainer comes from here (tests/cpp/acceptance_overlay).
#include <esrnn/data.hpp>
#include <esrnn/errors.hpp>
#include <esrnn/holt_winters.hpp>
#include <esrnn/matrix.hpp>
#include <esrnn/network.hpp>
#include "status.hpp"
#else
#include "data.hpp"
#include "errors.hpp"
#include "holt_winters.hpp"
#include "matrix.hpp"
#include "network.hpp"
#endif

namespace esrnn {

// TrainConfig (trainer.hpp:22-44) plus B200 extensions; every default keeps the reference's
// behaviour, including fp64 arithmetic.  Precision::FP32 is the opt-in performance path.
enum class Precision { FP32 = ESRNN_FP32, FP64 = ESRNN_FP64 };

struct TrainConfig {
    int epochs = 15;
    int batch_size = 512;
    double learning_rate_network = 1e-3;
    double learning_rate_per_series = 1e-2;
    double tau = 0.5;
    std::optional<double> gradient_clip = 20.0;
    std::uint64_t seed = 0;
    bool attach_es_state = true;
    int patience = 0;
    double min_delta = 0.0;
    // --- B200 extensions ---
    Precision precision = Precision::FP64;
    int max_batch_size = 0;  // 0 -> 2048 (reference cap)
    int device = 0;
    bool use_graphs = true;
    // opt-in level-variability penalty of Smyl's ES-RNN (the reference's loss is pinball
    // only, trainer.hpp:581): lambda * O / M * sum over the batch's windows of the mean
    // squared second difference of the window's series' log levels; 0 = reference
    double level_variability_penalty = 0.0;

    void validate() const {
        const int cap = max_batch_size > 0 ? max_batch_size : 2048;
        if (epochs < 0) throw ConfigError("train: epochs must be >= 0");
        if (batch_size < 1 || batch_size > cap)
            throw ConfigError("train: batch_size must be in [1, " + std::to_string(cap) + "]");
        if (!(tau > 0.0 && tau < 1.0)) throw ConfigError("train: tau must be in (0, 1)");
        if (learning_rate_network < 0.0 || learning_rate_per_series < 0.0)
            throw ConfigError("train: learning rates must be non-negative");
        if (gradient_clip && *gradient_clip <= 0.0) throw ConfigError("train: gradient_clip must be positive");
        if (!(level_variability_penalty >= 0.0) || !std::isfinite(level_variability_penalty))
            throw ConfigError("train: level_variability_penalty must be finite and >= 0");
    }
};

// trainer.hpp:50-61
struct WindowBatch {
    std::vector<int> series_rows;
    std::vector<int> anchors;
    std::vector<std::string> ids;
    Matrix inputs;                       // (B, I + 6)
    Matrix targets;                      // (B, O)
    std::vector<double> anchor_levels;   // B
    Matrix seasonality_slices;           // (B, O)
    Matrix mask;                         // (B, O)
    std::size_t size() const { return series_rows.size(); }
};

// trainer.hpp:64-78
inline double pinball_loss(const Matrix& predicted, const Matrix& actual, double tau, const Matrix& mask) {
    require_same_shape(predicted, actual, "pinball_loss");
    require_same_shape(predicted, mask, "pinball_loss mask");
    if (!(tau > 0.0 && tau < 1.0)) throw ContractError("pinball_loss: tau must be in (0, 1)");
    double acc = 0.0, count = 0.0;
    for (std::size_t e = 0; e < predicted.size(); ++e) {
        if (mask.data()[e] == 0.0) continue;
        const double d = actual.data()[e] - predicted.data()[e];
        acc += d >= 0.0 ? tau * d : (tau - 1.0) * d;
        count += 1.0;
    }
    if (count == 0.0) throw ContractError("pinball_loss: all-zero mask, mean undefined");
    return acc / count;
}

// trainer.hpp:82-102
inline std::vector<WindowBatch> make_batches(std::vector<std::pair<int, int>> windows,
                                             const std::vector<std::string>& series_ids, int batch_size, int horizon,
                                             Rng& rng) {
    if (windows.empty()) throw ContractError("make_batches: no windows");
    if (batch_size < 1) throw ConfigError("make_batches: batch_size must be >= 1");
    rng.shuffle(windows);
    std::vector<WindowBatch> out;
    for (std::size_t b = 0; b < windows.size(); b += static_cast<std::size_t>(batch_size)) {
        const std::size_t e = std::min(windows.size(), b + static_cast<std::size_t>(batch_size));
        WindowBatch wb;
        for (std::size_t i = b; i < e; ++i) {
            wb.series_rows.push_back(windows[i].first);
            wb.anchors.push_back(windows[i].second);
            wb.ids.push_back(series_ids[static_cast<std::size_t>(windows[i].first)]);
        }
        wb.mask = Matrix(wb.size(), static_cast<std::size_t>(horizon), 1.0);
        out.push_back(std::move(wb));
    }
    return out;
}

// trainer.hpp:107-120
inline bool early_stop_check(const std::vector<double>& history, int patience, double min_delta = 0.0) {
    if (history.empty()) throw ContractError("early_stop_check: empty history");
    if (patience <= 0) return false;
    double best = history[0];
    std::size_t last = 0;
    for (std::size_t i = 1; i < history.size(); ++i)
        if (best - history[i] > min_delta) best = history[i], last = i;
    return history.size() - 1 - last >= static_cast<std::size_t>(patience);
}

// trainer.hpp:122-152
struct ValidationResult {
    std::vector<std::string> ids;
    std::vector<std::vector<double>> forecasts;
    std::vector<double> smape_per_series;
    double mean_smape = 0.0;
};
struct ForecastResult {
    std::vector<std::string> ids;
    std::vector<std::vector<double>> forecasts;
};
// cmd_evaluate's scored rows (commands.hpp:285-338; metrics.hpp:17-59), model and seasonal
// naive, computed on the device (B200 extension of the Trainer surface; the reference scores
// on the host in detail::score_forecasts).  MASE entries are std::nullopt where the in-sample
// seasonal-naive MAE is zero, exactly like metrics.hpp:46.
struct EvaluationScores {
    std::vector<std::string> ids;
    std::vector<std::vector<double>> forecasts;
    std::vector<double> smape, naive_smape;
    std::vector<std::optional<double>> mase, naive_mase;
    double mean_smape = 0.0, naive_mean_smape = 0.0;  // over all series (all ranks)
    std::optional<double> mean_mase, naive_mean_mase;  // over series with a defined MASE
    std::size_t mase_undefined_count = 0;
};
// Exact-resume training state (B200 extension; the reference's Checkpoint, checkpoint.hpp:37-46,
// stores weights and per-series parameters only): network Adam moments in for_each_param
// order, the global Adam step, per-series moments {alpha, gamma, seas[S]} and steps for the
// owned rows, and the trainer RNG in std::mt19937_64's text form before the next shuffle.
// Serialise it next to a reference checkpoint (paper_1907_03329_b200/checkpoint.py writes it
// as the file's "training_state" object).
struct TrainState {
    std::vector<double> adam_m, adam_v;
    long long net_step = 0;
    std::vector<double> ps_m, ps_v;  // (owned rows) x (2 + S), row-major
    std::vector<long long> ps_steps;
    std::string rng;
};
struct BenchmarkReport {
    double batched_s = 0.0, looped_s = 0.0, speedup = 0.0;
    int batch_size = 0, n_series = 0;
};
struct BatchGradients {
    double loss = 0.0;
    std::map<std::string, Matrix> network;
    struct PerSeries {
        double alpha_raw = 0.0;
        double gamma_raw = 0.0;
        std::vector<double> init_seasonality_raw;
    };
    std::map<std::string, PerSeries> per_series;
};

// Series-sharded data parallelism (B200 extension): pass to the Trainer to run as one rank.
// Transport: NCCL (nccl_unique_id, one process per GPU) or an in-process group (group,
// from esrnn_group_create: one host thread per rank).  force_collective runs the
// collective step at world_size 1 too.
struct DistConfig {
    int rank = 0;
    int world_size = 1;
    std::array<std::uint8_t, 128> nccl_unique_id{};
    esrnn_group* group = nullptr;
    bool force_collective = false;
    static std::array<std::uint8_t, 128> new_unique_id() {
        std::array<std::uint8_t, 128> id{};
        detail::check(esrnn_nccl_unique_id(id.data()), nullptr);
        return id;
    }
};

class Trainer {
public:
    Trainer(std::vector<SeriesRecord> series, FrequencyProfile profile, TrainConfig cfg,
            std::optional<DistConfig> dist = std::nullopt)
        : profile_(std::move(profile)), cfg_(cfg), series_(std::move(series)) {
        profile_.validate();
        cfg_.validate();
        if (series_.empty()) throw ContractError("trainer: no series");
        const std::size_t n = series_.front().values.size();
        for (const auto& s : series_)
            if (s.values.size() != n)
                throw ConfigError("trainer: rectangular batching requires equal series lengths; \"" + s.id + "\" has " +
                                  std::to_string(s.values.size()) + " values, expected " + std::to_string(n));
        for (const auto& s : series_) splits_.push_back(split_train_val_test(s.values, profile_.horizon));
        std::vector<double> values(series_.size() * n);
        std::vector<std::int32_t> cats(series_.size());
        for (std::size_t r = 0; r < series_.size(); ++r) {
            std::copy(series_[r].values.begin(), series_[r].values.end(), values.begin() + static_cast<std::ptrdiff_t>(r * n));
            cats[r] = series_[r].category ? static_cast<std::int32_t>(*series_[r].category) : -1;
        }
        esrnn_profile p = to_c(profile_);
        esrnn_train_config c = to_c(cfg_);
        esrnn_dist d{};
        if (dist) {
            d.rank = dist->rank;
            d.world_size = dist->world_size;
            std::memcpy(d.nccl_unique_id, dist->nccl_unique_id.data(), 128);
            d.group = dist->group;
            d.flags = dist->force_collective ? ESRNN_DIST_FORCE_COLLECTIVE : 0;
        }
        esrnn_trainer* h = nullptr;
        detail::check(esrnn_trainer_create(&p, &c, static_cast<std::int64_t>(series_.size()), static_cast<std::int32_t>(n),
                                           values.data(), cats.data(), dist ? &d : nullptr, &h),
                      nullptr);
        h_.reset(h);
        std::int64_t b = 0, e = 0;
        detail::check(esrnn_trainer_shard(h, &b, &e), h);
        row_begin_ = static_cast<std::size_t>(b);
        row_end_ = static_cast<std::size_t>(e);
        stack_cfg_.dilation_blocks = profile_.dilation_blocks;
        stack_cfg_.hidden_size = profile_.hidden_size;
        stack_cfg_.input_size = profile_.input_window + kNumCategories;
        stack_cfg_.output_size = profile_.horizon;
        init_weight_shapes();
        params_.assign(series_.size(), PerSeriesParams(profile_.seasonality_length));
        weights_stale_ = params_stale_ = true;
    }

    Trainer(Trainer&&) noexcept = default;
    Trainer& operator=(Trainer&&) noexcept = default;

    // -- accessors (trainer.hpp:202-211) ----------------------------------------------
    const FrequencyProfile& profile() const { return profile_; }
    const TrainConfig& config() const { return cfg_; }
    const StackConfig& stack_config() const { return stack_cfg_; }
    StackWeights& weights() {
        pull_weights();
        weights_tainted_ = true;
        return weights_;
    }
    const StackWeights& weights() const {
        pull_weights();
        return weights_;
    }
    std::size_t series_count() const { return series_.size(); }
    const SeriesRecord& series(std::size_t i) const { return series_.at(i); }
    const DatasetSplit& split(std::size_t i) const { return splits_.at(i); }
    // A series-sharded trainer holds only its own rows' parameters: other rows are readable
    // after the collective gather_per_series() (every rank calls it; valid until the next
    // training call), which is what checkpoint.hpp's snapshot (:48-62) needs.
    PerSeriesParams& per_series_params(std::size_t i) {
        check_owned(i);
        pull_params();
        tainted_rows_.insert(i);
        return params_.at(i);
    }
    const PerSeriesParams& per_series_params(std::size_t i) const {
        check_owned(i);
        pull_params();
        return params_.at(i);
    }
    void gather_per_series() {
        push();
        const std::size_t n = series_.size();
        const int S = profile_.seasonality_length;
        std::vector<double> a(n), g(n), s(n * static_cast<std::size_t>(S));
        detail::check(esrnn_trainer_gather_per_series(h_.get(), a.data(), g.data(), s.data()), h_.get());
        for (std::size_t i = 0; i < n; ++i) {
            PerSeriesParams& p = params_[i];
            p.alpha_raw = a[i];
            p.gamma_raw = g[i];
            p.init_seasonality_raw.assign(s.begin() + static_cast<std::ptrdiff_t>(i * S),
                                          s.begin() + static_cast<std::ptrdiff_t>((i + 1) * S));
        }
        params_stale_ = false;
        gathered_ = true;
    }
    std::size_t shard_begin() const { return row_begin_; }
    std::size_t shard_end() const { return row_end_; }

    // trainer.hpp:214-223
    std::vector<std::pair<int, int>> all_windows() const {
        std::vector<std::pair<int, int>> out;
        const int I = profile_.input_window, O = profile_.horizon, T = train_len();
        for (std::size_t r = 0; r < series_.size(); ++r)
            for (int a = I - 1; a <= T - O - 1; ++a) out.emplace_back(static_cast<int>(r), a);
        return out;
    }
    std::vector<std::string> series_ids() const {
        std::vector<std::string> ids;
        for (const auto& s : series_) ids.push_back(s.id);
        return ids;
    }

    // -- hot path ------------------------------------------------------------------------
    double train_epoch() {  // trainer.hpp:234-243
        push();
        double l = 0.0;
        detail::check(esrnn_trainer_train_epoch(h_.get(), &l), h_.get());
        mark_trained();
        return l;
    }

    ForecastResult forecast_at(std::size_t drop_tail) const {  // trainer.hpp:248-288
        push();
        const int O = profile_.horizon;
        std::vector<double> out((row_end_ - row_begin_) * static_cast<std::size_t>(O));
        detail::check(esrnn_trainer_forecast(h_.get(), static_cast<std::int64_t>(drop_tail), out.data()), h_.get());
        ForecastResult fr;
        for (std::size_t r = row_begin_; r < row_end_; ++r) {
            fr.ids.push_back(series_[r].id);
            const double* p = out.data() + (r - row_begin_) * static_cast<std::size_t>(O);
            fr.forecasts.emplace_back(p, p + O);
        }
        return fr;
    }

    ValidationResult validate() const {  // trainer.hpp:292-305
        push();
        const int O = profile_.horizon;
        const std::size_t n = row_end_ - row_begin_;
        std::vector<double> fc(n * static_cast<std::size_t>(O)), sm(n);
        ValidationResult v;
        detail::check(esrnn_trainer_validate(h_.get(), fc.data(), sm.data(), &v.mean_smape), h_.get());
        for (std::size_t r = 0; r < n; ++r) {
            v.ids.push_back(series_[row_begin_ + r].id);
            v.forecasts.emplace_back(fc.data() + r * static_cast<std::size_t>(O), fc.data() + (r + 1) * static_cast<std::size_t>(O));
        }
        v.smape_per_series = std::move(sm);
        return v;
    }

    TrainState train_state() const {
        const std::size_t n = row_end_ - row_begin_, w = 2 + static_cast<std::size_t>(profile_.seasonality_length);
        TrainState ts;
        ts.adam_m.resize(static_cast<std::size_t>(n_values_));
        ts.adam_v.resize(static_cast<std::size_t>(n_values_));
        ts.ps_m.resize(n * w);
        ts.ps_v.resize(n * w);
        std::vector<std::int64_t> steps(n);
        std::int64_t net = 0;
        std::string rng(ESRNN_RNG_TEXT_MAX, '\0');
        detail::check(esrnn_trainer_get_train_state(h_.get(), ts.adam_m.data(), ts.adam_v.data(), n_values_,
                                                    static_cast<std::int64_t>(row_begin_), static_cast<std::int64_t>(n),
                                                    ts.ps_m.data(), ts.ps_v.data(), steps.data(), &net, rng.data(),
                                                    ESRNN_RNG_TEXT_MAX),
                      h_.get());
        ts.net_step = net;
        ts.ps_steps.assign(steps.begin(), steps.end());
        ts.rng = rng.c_str();
        return ts;
    }
    void set_train_state(const TrainState& ts) {
        const std::size_t n = row_end_ - row_begin_, w = 2 + static_cast<std::size_t>(profile_.seasonality_length);
        if (ts.ps_m.size() != n * w || ts.ps_v.size() != n * w || ts.ps_steps.size() != n)
            throw CheckpointError("train state: per-series state does not match the owned rows");
        std::vector<std::int64_t> steps(ts.ps_steps.begin(), ts.ps_steps.end());
        detail::check(esrnn_trainer_set_train_state(h_.get(), ts.adam_m.data(), ts.adam_v.data(),
                                                    static_cast<std::int64_t>(ts.adam_m.size()),
                                                    static_cast<std::int64_t>(row_begin_), static_cast<std::int64_t>(n),
                                                    ts.ps_m.data(), ts.ps_v.data(), steps.data(), ts.net_step,
                                                    ts.rng.c_str()),
                      h_.get());
    }

    // cmd_evaluate (commands.hpp:312-338): forecast_at(O) against the test block when
    // against_test, else forecast_at(2*O) against the validation block.
    EvaluationScores evaluate(bool against_test = true) const {
        push();
        const int O = profile_.horizon;
        const std::size_t n = row_end_ - row_begin_;
        std::vector<double> fc(n * static_cast<std::size_t>(O)), sm(n), ma(n), ns(n), nm(n);
        double tot[8] = {};
        detail::check(esrnn_trainer_evaluate(h_.get(), against_test ? 1 : 0, fc.data(), sm.data(), ma.data(), ns.data(),
                                             nm.data(), tot),
                      h_.get());
        EvaluationScores e;
        auto opt = [](double v) { return std::isnan(v) ? std::optional<double>() : std::optional<double>(v); };
        for (std::size_t r = 0; r < n; ++r) {
            e.ids.push_back(series_[row_begin_ + r].id);
            e.forecasts.emplace_back(fc.data() + r * static_cast<std::size_t>(O), fc.data() + (r + 1) * static_cast<std::size_t>(O));
            e.mase.push_back(opt(ma[r]));
            e.naive_mase.push_back(opt(nm[r]));
        }
        e.smape = std::move(sm);
        e.naive_smape = std::move(ns);
        e.mean_smape = tot[0] / tot[6];
        e.naive_mean_smape = tot[3] / tot[6];
        if (tot[2] > 0) e.mean_mase = tot[1] / tot[2];
        if (tot[5] > 0) e.naive_mean_mase = tot[4] / tot[5];
        e.mase_undefined_count = static_cast<std::size_t>(tot[6] - tot[2]);
        return e;
    }

    // forward_stack (network.hpp:190-210; plain::forward_stack :268-287) over a general
    // sequence with this trainer's weights -- the full dilated recurrence -- on the device.
    // With out_bar, also the tape adjoints (Tape::backward, autodiff.hpp:397-631): network
    // gradients by name and one input adjoint per step.
    Matrix forward_stack(const std::vector<Matrix>& sequence) const {
        return forward_stack_impl(sequence, nullptr, nullptr, nullptr);
    }
    Matrix forward_stack(const std::vector<Matrix>& sequence, const Matrix& out_bar,
                         std::map<std::string, Matrix>& weights_bar, std::vector<Matrix>& inputs_bar) const {
        return forward_stack_impl(sequence, &out_bar, &weights_bar, &inputs_bar);
    }

    BatchGradients batch_gradients(WindowBatch& batch) {  // trainer.hpp:308-335
        BatchGradients out;
        std::vector<double> gnet(static_cast<std::size_t>(n_values_));
        std::vector<std::int32_t> slots(std::max<std::size_t>(batch.size(), 1));
        const int S = profile_.seasonality_length;
        std::vector<double> gps(std::max<std::size_t>(batch.size(), 1) * static_cast<std::size_t>(2 + S));
        std::int32_t k = 0;
        run(batch, ESRNN_BATCH_GRADS, &out.loss, gnet.data(), &k, slots.data(), gps.data());
        std::size_t off = 0;
        weights_.for_each_param([&](const std::string& name, const Matrix& shape) {
            Matrix m(shape.rows(), shape.cols());
            std::copy(gnet.begin() + static_cast<std::ptrdiff_t>(off),
                      gnet.begin() + static_cast<std::ptrdiff_t>(off + m.size()), m.data().begin());
            off += m.size();
            out.network.emplace(name, std::move(m));
        });
        if (cfg_.attach_es_state)
            for (int s = 0; s < k; ++s) {
                const double* g = gps.data() + static_cast<std::size_t>(s) * static_cast<std::size_t>(2 + S);
                BatchGradients::PerSeries p;
                p.alpha_raw = g[0];
                p.gamma_raw = g[1];
                p.init_seasonality_raw.assign(g + 2, g + 2 + S);
                out.per_series.emplace(series_[static_cast<std::size_t>(slots[static_cast<std::size_t>(s)])].id, std::move(p));
            }
        return out;
    }

    double batch_loss(WindowBatch& batch) {  // trainer.hpp:338-342
        double l = 0.0;
        run(batch, 0, &l, nullptr, nullptr, nullptr, nullptr);
        return l;
    }

    // trainer.hpp:351-413: interleaved batched / per-window fixed-order epochs, min time,
    // equivalence gate at 1e-6 relative before any timing is reported.
    BenchmarkReport benchmark_batched_vs_looped() {
        const auto windows = all_windows();
        auto batches_of = [&](int bs) {
            std::vector<WindowBatch> out;
            for (std::size_t b = 0; b < windows.size(); b += static_cast<std::size_t>(bs)) {
                WindowBatch wb;
                for (std::size_t i = b; i < std::min(windows.size(), b + static_cast<std::size_t>(bs)); ++i) {
                    wb.series_rows.push_back(windows[i].first);
                    wb.anchors.push_back(windows[i].second);
                    wb.ids.push_back(series_[static_cast<std::size_t>(windows[i].first)].id);
                }
                wb.mask = Matrix(wb.size(), static_cast<std::size_t>(profile_.horizon), 1.0);
                out.push_back(std::move(wb));
            }
            return out;
        };
        auto timed = [&](std::vector<WindowBatch>& bs) {
            const auto t0 = std::chrono::steady_clock::now();
            double acc = 0.0, w = 0.0;
            for (auto& b : bs) {
                double l = 0.0, mc = 0.0;
                step(b, false, &l, &mc);
                acc += l * mc;
                w += mc;
            }
            return std::make_pair(acc / w, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
        };
        auto batched = batches_of(cfg_.batch_size), looped = batches_of(1);
        double l, mc;
        step(batched.front(), false, &l, &mc);
        step(looped.front(), false, &l, &mc);
        double lb = 0, ll = 0, sb = std::numeric_limits<double>::infinity(), sl = sb;
        for (int round = 0; round < 3; ++round) {
            auto [a, ta] = timed(batched);
            auto [b, tb] = timed(looped);
            lb = a, ll = b;
            sb = std::min(sb, ta), sl = std::min(sl, tb);
        }
        if (std::abs(lb - ll) / std::max(1e-30, std::abs(ll)) > 1e-6)
            throw EquivalenceError("benchmark: batched loss " + std::to_string(lb) + " vs looped " + std::to_string(ll) +
                                   " differ beyond 1e-6; timing withheld");
        return BenchmarkReport{sb, sl, sl / sb, cfg_.batch_size, static_cast<int>(series_.size())};
    }

    void set_weights(StackWeights w) {  // trainer.hpp:415-432
        bool ok = w.layers.size() == weights_.layers.size();
        std::vector<const Matrix*> mine;
        weights_.for_each_param([&](const std::string&, const Matrix& m) { mine.push_back(&m); });
        std::size_t i = 0;
        w.for_each_param([&](const std::string&, const Matrix& m) {
            if (i >= mine.size() || !mine[i]->same_shape(m)) ok = false;
            ++i;
        });
        if (!ok || i != mine.size()) throw CheckpointError("checkpoint network shapes incompatible with configuration");
        weights_ = std::move(w);
        weights_stale_ = false;
        weights_tainted_ = true;
    }

    void set_per_series(const std::map<std::string, PerSeriesParams>& by_id) {  // trainer.hpp:434-445
        pull_params();
        for (std::size_t r = row_begin_; r < row_end_; ++r) {
            auto it = by_id.find(series_[r].id);
            if (it == by_id.end())
                throw CheckpointError("checkpoint missing per-series parameters for \"" + series_[r].id + "\"");
            if (it->second.season_length() != profile_.seasonality_length)
                throw CheckpointError("checkpoint season length incompatible for \"" + series_[r].id + "\"");
        }
        for (std::size_t r = row_begin_; r < row_end_; ++r) {
            params_[r] = by_id.at(series_[r].id);
            tainted_rows_.insert(r);
        }
    }

    // Trainer::step (trainer.hpp:593-600; private in the reference), exposed for benchmarks.
    void step(WindowBatch& batch, bool update, double* loss, double* mask_count) {
        run(batch, ESRNN_BATCH_GRADS | (update ? ESRNN_BATCH_UPDATE : 0), loss, nullptr, nullptr, nullptr, nullptr,
            mask_count);
        if (update) mark_trained();
    }

    double last_device_ms() const {
        double ms = 0.0;
        detail::check(esrnn_trainer_last_device_ms(h_.get(), &ms), h_.get());
        return ms;
    }

private:
    struct HandleDeleter {
        void operator()(esrnn_trainer* h) const { esrnn_trainer_destroy(h); }
    };

    static esrnn_profile to_c(const FrequencyProfile& f) {
        esrnn_profile p{};
        p.frequency = static_cast<std::int32_t>(f.frequency);
        p.seasonality_length = f.seasonality_length;
        p.horizon = f.horizon;
        p.input_window = f.input_window;
        p.hidden_size = f.hidden_size;
        p.min_length = f.min_length;
        if (f.dilation_blocks.size() > ESRNN_MAX_BLOCKS) throw ConfigError("profile: too many dilation blocks");
        p.n_blocks = static_cast<std::int32_t>(f.dilation_blocks.size());
        int layer = 0;
        for (std::size_t b = 0; b < f.dilation_blocks.size(); ++b) {
            p.block_len[b] = static_cast<std::int32_t>(f.dilation_blocks[b].size());
            for (int d : f.dilation_blocks[b]) {
                if (layer >= ESRNN_MAX_LAYERS) throw ConfigError("profile: too many layers");
                p.dilations[layer++] = d;
            }
        }
        return p;
    }
    static esrnn_train_config to_c(const TrainConfig& t) {
        esrnn_train_config c{};
        c.epochs = t.epochs;
        c.batch_size = t.batch_size;
        c.learning_rate_network = t.learning_rate_network;
        c.learning_rate_per_series = t.learning_rate_per_series;
        c.tau = t.tau;
        c.has_gradient_clip = t.gradient_clip ? 1 : 0;
        c.gradient_clip = t.gradient_clip.value_or(0.0);
        c.seed = t.seed;
        c.attach_es_state = t.attach_es_state ? 1 : 0;
        c.patience = t.patience;
        c.min_delta = t.min_delta;
        c.precision = static_cast<std::int32_t>(t.precision);
        c.max_batch_size = t.max_batch_size;
        c.device = t.device;
        c.use_graphs = t.use_graphs ? 0 : -1;
        c.level_variability_penalty = t.level_variability_penalty;
        return c;
    }

    int train_len() const { return static_cast<int>(series_.front().values.size()) - 2 * profile_.horizon; }

    void init_weight_shapes() {
        std::int32_t na = 0;
        detail::check(esrnn_trainer_param_count(h_.get(), &na, &n_values_), h_.get());
        const int H = profile_.hidden_size;
        int in = stack_cfg_.input_size;
        for (int l = 0; l < stack_cfg_.num_layers(); ++l) {
            LSTMCellWeights c;
            c.w_input = Matrix(static_cast<std::size_t>(in), static_cast<std::size_t>(4 * H));
            c.w_recur = Matrix(static_cast<std::size_t>(H), static_cast<std::size_t>(4 * H));
            c.bias = Matrix(1, static_cast<std::size_t>(4 * H));
            weights_.layers.push_back(std::move(c));
            in = H;
        }
        weights_.nl_w = Matrix(static_cast<std::size_t>(H), static_cast<std::size_t>(H));
        weights_.nl_b = Matrix(1, static_cast<std::size_t>(H));
        weights_.out_w = Matrix(static_cast<std::size_t>(H), static_cast<std::size_t>(profile_.horizon));
        weights_.out_b = Matrix(1, static_cast<std::size_t>(profile_.horizon));
    }

    void pull_weights() const {
        if (!weights_stale_) return;
        std::vector<double> flat(static_cast<std::size_t>(n_values_));
        detail::check(esrnn_trainer_get_weights(h_.get(), flat.data(), n_values_), h_.get());
        std::size_t off = 0;
        weights_.for_each_param([&](const std::string&, Matrix& m) {
            std::copy(flat.begin() + static_cast<std::ptrdiff_t>(off), flat.begin() + static_cast<std::ptrdiff_t>(off + m.size()),
                      m.data().begin());
            off += m.size();
        });
        weights_stale_ = false;
    }

    void pull_params() const {
        if (!params_stale_) return;
        const int S = profile_.seasonality_length;
        const std::size_t n = row_end_ - row_begin_;
        std::vector<double> a(n), g(n), s(n * static_cast<std::size_t>(S));
        if (n)
            detail::check(esrnn_trainer_get_per_series(h_.get(), static_cast<std::int64_t>(row_begin_), static_cast<std::int64_t>(n),
                                                       a.data(), g.data(), s.data()),
                          h_.get());
        for (std::size_t i = 0; i < n; ++i) {
            PerSeriesParams& p = params_[row_begin_ + i];
            p.alpha_raw = a[i];
            p.gamma_raw = g[i];
            p.init_seasonality_raw.assign(s.begin() + static_cast<std::ptrdiff_t>(i * S), s.begin() + static_cast<std::ptrdiff_t>((i + 1) * S));
        }
        params_stale_ = false;
    }

    // host mirrors -> device before any device call
    Matrix forward_stack_impl(const std::vector<Matrix>& seq, const Matrix* out_bar,
                              std::map<std::string, Matrix>* wbar, std::vector<Matrix>* xbar) const {
        push();
        if (seq.empty()) throw ContractError("forward_stack: empty sequence");
        const std::size_t B = seq[0].rows(), in = static_cast<std::size_t>(stack_cfg_.input_size);
        const int O = profile_.horizon;
        std::vector<double> x;
        x.reserve(seq.size() * B * in);
        for (const Matrix& m : seq) {
            if (m.rows() != B || m.cols() != in)
                throw ShapeError("forward_stack: input width " + std::to_string(m.cols()) + ", expected " +
                                 std::to_string(in));
            x.insert(x.end(), m.data().begin(), m.data().end());
        }
        Matrix out(B, static_cast<std::size_t>(O));
        std::vector<double> wb, xb;
        if (out_bar) {
            if (out_bar->rows() != B || out_bar->cols() != static_cast<std::size_t>(O))
                throw ShapeError("forward_stack: out_bar shape");
            wb.resize(static_cast<std::size_t>(n_values_));
            xb.resize(x.size());
        }
        detail::check(esrnn_trainer_forward_stack(h_.get(), static_cast<std::int32_t>(seq.size()),
                                                  static_cast<std::int32_t>(B), x.data(), out.data().data(),
                                                  out_bar ? out_bar->data().data() : nullptr,
                                                  out_bar ? wb.data() : nullptr, out_bar ? xb.data() : nullptr),
                      h_.get());
        if (out_bar) {
            wbar->clear();
            std::size_t off = 0;
            StackWeights shape = weights_;
            shape.for_each_param([&](const std::string& name, Matrix& m) {
                Matrix g(m.rows(), m.cols());
                std::copy(wb.begin() + static_cast<std::ptrdiff_t>(off),
                          wb.begin() + static_cast<std::ptrdiff_t>(off + m.size()), g.data().begin());
                off += m.size();
                wbar->emplace(name, std::move(g));
            });
            xbar->clear();
            for (std::size_t t = 0; t < seq.size(); ++t) {
                Matrix g(B, in);
                std::copy(xb.begin() + static_cast<std::ptrdiff_t>(t * B * in),
                          xb.begin() + static_cast<std::ptrdiff_t>((t + 1) * B * in), g.data().begin());
                xbar->push_back(std::move(g));
            }
        }
        return out;
    }

    void push() const {
        if (weights_tainted_) {
            std::vector<double> flat;
            flat.reserve(static_cast<std::size_t>(n_values_));
            weights_.for_each_param([&](const std::string&, const Matrix& m) { flat.insert(flat.end(), m.data().begin(), m.data().end()); });
            detail::check(esrnn_trainer_set_weights(h_.get(), flat.data(), static_cast<std::int64_t>(flat.size())), h_.get());
        }
        for (std::size_t r : tainted_rows_) {
            if (r < row_begin_ || r >= row_end_) continue;
            const PerSeriesParams& p = params_[r];
            if (p.season_length() != profile_.seasonality_length)
                throw CheckpointError("per-series parameters of \"" + series_[r].id + "\" have the wrong season length");
            detail::check(esrnn_trainer_set_per_series(h_.get(), static_cast<std::int64_t>(r), 1, &p.alpha_raw, &p.gamma_raw,
                                                       p.init_seasonality_raw.data()),
                          h_.get());
        }
    }

    void check_owned(std::size_t i) const {
        if (i < series_.size() && (i < row_begin_ || i >= row_end_) && !gathered_)
            throw ContractError("per_series_params: series " + std::to_string(i) +
                                " is owned by another rank (call gather_per_series() on every rank first)");
    }

    void mark_trained() {
        gathered_ = false;
        weights_stale_ = params_stale_ = true;
        weights_tainted_ = false;
        tainted_rows_.clear();
    }

    void run(WindowBatch& b, int flags, double* loss, double* gnet, std::int32_t* nslots, std::int32_t* slots,
             double* gps, double* mask_count = nullptr) {
        const std::size_t B = b.size();
        const int O = profile_.horizon, I = profile_.input_window;
        if (b.mask.rows() != B || b.mask.cols() != static_cast<std::size_t>(O))
            throw ShapeError("batch: mask shape " + b.mask.shape_str());
        push();
        b.inputs = Matrix(B, static_cast<std::size_t>(I + kNumCategories));
        b.targets = Matrix(B, static_cast<std::size_t>(O));
        b.seasonality_slices = Matrix(B, static_cast<std::size_t>(O));
        b.anchor_levels.assign(B, 0.0);
        double mc = 0.0;
        detail::check(esrnn_trainer_run_batch(h_.get(), static_cast<std::int32_t>(B), b.series_rows.data(), b.anchors.data(),
                                              b.mask.data().data(), flags, loss, &mc, b.inputs.data().data(),
                                              b.targets.data().data(), b.seasonality_slices.data().data(),
                                              b.anchor_levels.data(), gnet, nslots, slots, gps),
                      h_.get());
        if (mask_count) *mask_count = mc;
    }

    FrequencyProfile profile_;
    TrainConfig cfg_;
    StackConfig stack_cfg_;
    std::vector<SeriesRecord> series_;
    std::vector<DatasetSplit> splits_;
    std::unique_ptr<esrnn_trainer, HandleDeleter> h_;
    std::size_t row_begin_ = 0, row_end_ = 0;
    std::int64_t n_values_ = 0;
    mutable StackWeights weights_;
    mutable std::vector<PerSeriesParams> params_;
    mutable bool weights_stale_ = true, params_stale_ = true, weights_tainted_ = false, gathered_ = false;
    std::set<std::size_t> tainted_rows_;
};

}  // namespace esrnn
