// TEST INFRASTRUCTURE — not product code.
//
// Exposes the UNMODIFIED reference implementation (/root/reference/proj/include,
// header-only C++20) behind the engine's C-ABI (include/esrnn_b200.h) so tests and
// bench.py's reference arm can drive the reference and the B200 engine through
// the same calls.  Built by oracle/Makefile into oracle/_ref/libesrnn_ref.so; the
// reference sources are compiled where they lie (never copied).
//
// `private` is widened only so build_graph/step (trainer.hpp:484-600) and the
// tape's slot order (trainer.hpp:463-470) are reachable for slot-ordered gradient
// dumps and for step(update=true) on a caller-supplied batch.
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

// every standard header the reference pulls in, parsed before the access hack
#include <algorithm>
#include <array>
#include <bit>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <functional>
#include <initializer_list>
#include <istream>
#include <limits>
#include <map>
#include <numeric>
#include <optional>
#include <ostream>
#include <random>
#include <set>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string_view>
#include <utility>
#include <filesystem>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <cstdlib>
#include <json.hpp>

#define private public
#include "esrnn/trainer.hpp"
#undef private
#include "esrnn/commands.hpp"
#include "helpers.hpp"

#include "esrnn_b200.h"

using namespace esrnn;

struct esrnn_trainer {
    std::unique_ptr<Trainer> tr;
    std::string err;
    double last_ms = 0.0;
    std::vector<std::pair<int, int>> last_windows;  // order consumed by the last train_epoch
};

namespace {

thread_local std::string g_create_err;

template <class Fn>
esrnn_status guarded(std::string& err, Fn&& fn) {
    try {
        fn();
        return ESRNN_OK;
    } catch (const ParseError& e) { err = e.what(); return ESRNN_PARSE_ERROR; }
    catch (const ValidationError& e) { err = e.what(); return ESRNN_VALIDATION_ERROR; }
    catch (const ShapeError& e) { err = e.what(); return ESRNN_SHAPE_ERROR; }
    catch (const InsufficientLengthError& e) { err = e.what(); return ESRNN_INSUFFICIENT_LENGTH; }
    catch (const NumericDomainError& e) { err = e.what(); return ESRNN_NUMERIC_DOMAIN_ERROR; }
    catch (const ConfigError& e) { err = e.what(); return ESRNN_CONFIG_ERROR; }
    catch (const ContractError& e) { err = e.what(); return ESRNN_CONTRACT_ERROR; }
    catch (const EquivalenceError& e) { err = e.what(); return ESRNN_EQUIVALENCE_ERROR; }
    catch (const CheckpointError& e) { err = e.what(); return ESRNN_CHECKPOINT_ERROR; }
    catch (const Error& e) { err = e.what(); return ESRNN_ERROR; }
    catch (const std::exception& e) { err = e.what(); return ESRNN_ERROR; }
}

FrequencyProfile to_profile(const esrnn_profile& p) {
    FrequencyProfile f;
    f.frequency = static_cast<Frequency>(p.frequency);
    f.seasonality_length = p.seasonality_length;
    f.horizon = p.horizon;
    f.input_window = p.input_window;
    f.hidden_size = p.hidden_size;
    f.min_length = p.min_length;
    f.dilation_blocks.clear();
    int layer = 0;
    for (int b = 0; b < p.n_blocks; ++b) {
        std::vector<int> blk;
        for (int j = 0; j < p.block_len[b]; ++j) blk.push_back(p.dilations[layer++]);
        f.dilation_blocks.push_back(blk);
    }
    return f;
}

TrainConfig to_config(const esrnn_train_config& c) {
    TrainConfig t;
    t.epochs = c.epochs;
    t.batch_size = c.batch_size;
    t.learning_rate_network = c.learning_rate_network;
    t.learning_rate_per_series = c.learning_rate_per_series;
    t.tau = c.tau;
    if (c.has_gradient_clip) t.gradient_clip = c.gradient_clip;
    else t.gradient_clip.reset();
    t.seed = c.seed;
    t.attach_es_state = c.attach_es_state != 0;
    t.patience = c.patience;
    t.min_delta = c.min_delta;
    return t;
}

}  // namespace

extern "C" {

const char* esrnn_version(void) { return "reference-shim (proj/include/esrnn, fp64 CPU)"; }
int32_t esrnn_abi_version(void) { return ESRNN_ABI_VERSION; }

const char* esrnn_last_error(const esrnn_trainer* t) {
    return t ? t->err.c_str() : g_create_err.c_str();
}

esrnn_status esrnn_trainer_create(const esrnn_profile* profile, const esrnn_train_config* cfg,
                                  int64_t n_series, int32_t length, const double* values,
                                  const int32_t* category, const esrnn_dist* dist,
                                  esrnn_trainer** out) {
    *out = nullptr;
    if (dist && dist->world_size > 1) {
        g_create_err = "reference shim: no sharded mode (the reference is single-threaded)";
        return ESRNN_CONFIG_ERROR;
    }
    if (cfg->level_variability_penalty != 0.0) {
        g_create_err = "reference shim: the reference has no level-variability penalty (trainer.hpp:581)";
        return ESRNN_CONFIG_ERROR;
    }
    auto h = std::make_unique<esrnn_trainer>();
    esrnn_status st = guarded(g_create_err, [&] {
        std::vector<SeriesRecord> recs(static_cast<std::size_t>(n_series));
        for (int64_t i = 0; i < n_series; ++i) {
            recs[i].id = "S" + std::to_string(i);
            if (category && category[i] >= 0) recs[i].category = static_cast<Category>(category[i]);
            recs[i].values.assign(values + i * length, values + (i + 1) * length);
        }
        h->tr = std::make_unique<Trainer>(std::move(recs), to_profile(*profile), to_config(*cfg));
    });
    if (st == ESRNN_OK) *out = h.release();
    return st;
}

void esrnn_trainer_destroy(esrnn_trainer* t) { delete t; }

esrnn_status esrnn_trainer_shard(const esrnn_trainer* t, int64_t* b, int64_t* e) {
    *b = 0;
    *e = static_cast<int64_t>(t->tr->series_count());
    return ESRNN_OK;
}

esrnn_status esrnn_trainer_param_count(const esrnn_trainer* t, int32_t* n_arrays, int64_t* n_values) {
    int32_t na = 0;
    int64_t nv = 0;
    t->tr->weights().for_each_param([&](const std::string&, const Matrix& m) {
        ++na;
        nv += static_cast<int64_t>(m.size());
    });
    *n_arrays = na;
    *n_values = nv;
    return ESRNN_OK;
}

esrnn_status esrnn_trainer_param_info(const esrnn_trainer* t, int32_t index, esrnn_param_info* out) {
    int32_t i = 0;
    int64_t off = 0;
    bool found = false;
    t->tr->weights().for_each_param([&](const std::string& name, const Matrix& m) {
        if (i == index) {
            std::memset(out, 0, sizeof *out);
            std::strncpy(out->name, name.c_str(), sizeof(out->name) - 1);
            out->rows = static_cast<int32_t>(m.rows());
            out->cols = static_cast<int32_t>(m.cols());
            out->offset = off;
            found = true;
        }
        off += static_cast<int64_t>(m.size());
        ++i;
    });
    return found ? ESRNN_OK : ESRNN_SHAPE_ERROR;
}

esrnn_status esrnn_trainer_get_weights(esrnn_trainer* t, double* flat, int64_t count) {
    int64_t off = 0;
    t->tr->weights().for_each_param([&](const std::string&, const Matrix& m) {
        for (double v : m.data())
            if (off < count) flat[off++] = v;
    });
    return ESRNN_OK;
}

esrnn_status esrnn_trainer_set_weights(esrnn_trainer* t, const double* flat, int64_t count) {
    return guarded(t->err, [&] {
        StackWeights w = t->tr->weights();
        int64_t off = 0;
        w.for_each_param([&](const std::string&, Matrix& m) {
            for (double& v : m.data()) v = (off < count) ? flat[off] : 0.0, ++off;
        });
        if (off != count) throw CheckpointError("checkpoint network shapes incompatible with configuration");
        t->tr->set_weights(std::move(w));
    });
}

esrnn_status esrnn_trainer_get_per_series(esrnn_trainer* t, int64_t row_begin, int64_t n,
                                          double* a, double* g, double* s) {
    return guarded(t->err, [&] {
        for (int64_t i = 0; i < n; ++i) {
            const PerSeriesParams& p = t->tr->per_series_params(static_cast<std::size_t>(row_begin + i));
            if (a) a[i] = p.alpha_raw;
            if (g) g[i] = p.gamma_raw;
            const int S = p.season_length();
            if (s)
                for (int j = 0; j < S; ++j) s[i * S + j] = p.init_seasonality_raw[j];
        }
    });
}

esrnn_status esrnn_trainer_set_per_series(esrnn_trainer* t, int64_t row_begin, int64_t n,
                                          const double* a, const double* g, const double* s) {
    return guarded(t->err, [&] {
        for (int64_t i = 0; i < n; ++i) {
            PerSeriesParams& p = t->tr->per_series_params(static_cast<std::size_t>(row_begin + i));
            if (a) p.alpha_raw = a[i];
            if (g) p.gamma_raw = g[i];
            const int S = p.season_length();
            if (s)
                for (int j = 0; j < S; ++j) p.init_seasonality_raw[j] = s[i * S + j];
        }
    });
}

esrnn_status esrnn_trainer_train_epoch(esrnn_trainer* t, double* mean_loss) {
    return guarded(t->err, [&] {
        // replay make_batches on a copy of the trainer RNG to record the window order the
        // epoch is about to consume (trainer.hpp:235)
        {
            Rng copy = t->tr->rng_;
            auto w = t->tr->all_windows();
            copy.shuffle(w);
            t->last_windows = std::move(w);
        }
        const auto t0 = std::chrono::steady_clock::now();
        *mean_loss = t->tr->train_epoch();
        t->last_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    });
}

esrnn_status esrnn_trainer_run_batch(esrnn_trainer* t, int32_t B, const int32_t* rows,
                                     const int32_t* anchors, const double* mask, int32_t flags,
                                     double* loss, double* mask_count, double* inputs,
                                     double* targets, double* seas, double* levels,
                                     double* net_grads, int32_t* n_slots, int32_t* slot_rows,
                                     double* ps_grads) {
    return guarded(t->err, [&] {
        Trainer& tr = *t->tr;
        const int O = tr.profile().horizon;
        const int S = tr.profile().seasonality_length;
        WindowBatch b;
        for (int i = 0; i < B; ++i) {
            b.series_rows.push_back(rows[i]);
            b.anchors.push_back(anchors[i]);
            b.ids.push_back("w");
        }
        b.mask = Matrix(static_cast<std::size_t>(B), static_cast<std::size_t>(O), 1.0);
        if (mask) std::memcpy(b.mask.data().data(), mask, sizeof(double) * B * O);
        const auto t0 = std::chrono::steady_clock::now();
        double l;
        if (flags & ESRNN_BATCH_GRADS) {
            auto r = tr.step(b, (flags & ESRNN_BATCH_UPDATE) != 0);
            l = r.loss;
        } else {
            l = tr.batch_loss(b);
        }
        t->last_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        auto& tb = tr.tape_build_;
        if (loss) *loss = l;
        if (mask_count) *mask_count = tb.mask_count;
        if (inputs) std::memcpy(inputs, b.inputs.data().data(), sizeof(double) * b.inputs.size());
        if (targets) std::memcpy(targets, b.targets.data().data(), sizeof(double) * b.targets.size());
        if (seas) std::memcpy(seas, b.seasonality_slices.data().data(), sizeof(double) * b.seasonality_slices.size());
        if (levels) std::memcpy(levels, b.anchor_levels.data(), sizeof(double) * b.anchor_levels.size());
        const int k = static_cast<int>(tb.slot_series.size());
        if (n_slots) *n_slots = k;
        if (slot_rows)
            for (int s = 0; s < k; ++s) slot_rows[s] = tb.slot_series[s];
        if (flags & ESRNN_BATCH_GRADS) {
            if (net_grads) {
                int64_t off = 0;
                for (const auto& leaf : tb.net_leaves)
                    for (double v : leaf.grad().data()) net_grads[off++] = v;
            }
            if (ps_grads && tr.config().attach_es_state) {
                for (int s = 0; s < k; ++s) {
                    double* o = ps_grads + static_cast<int64_t>(s) * (2 + S);
                    o[0] = tb.alpha_leaf.grad()(s, 0);
                    o[1] = tb.gamma_leaf.grad()(s, 0);
                    for (int j = 0; j < S; ++j) o[2 + j] = tb.seas_leaf.grad()(s, j);
                }
            }
        }
    });
}

esrnn_status esrnn_trainer_forecast(esrnn_trainer* t, int64_t drop_tail, double* out) {
    return guarded(t->err, [&] {
        const auto t0 = std::chrono::steady_clock::now();
        ForecastResult fr = t->tr->forecast_at(static_cast<std::size_t>(drop_tail));
        t->last_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        const int O = t->tr->profile().horizon;
        for (std::size_t r = 0; r < fr.forecasts.size(); ++r)
            for (int j = 0; j < O; ++j) out[r * O + j] = fr.forecasts[r][j];
    });
}

esrnn_status esrnn_trainer_validate(esrnn_trainer* t, double* forecasts, double* smape_per_series,
                                    double* mean_smape) {
    return guarded(t->err, [&] {
        const auto t0 = std::chrono::steady_clock::now();
        ValidationResult v = t->tr->validate();
        t->last_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        const int O = t->tr->profile().horizon;
        for (std::size_t r = 0; r < v.forecasts.size(); ++r) {
            if (forecasts)
                for (int j = 0; j < O; ++j) forecasts[r * O + j] = v.forecasts[r][j];
            if (smape_per_series) smape_per_series[r] = v.smape_per_series[r];
        }
        if (mean_smape) *mean_smape = v.mean_smape;
    });
}

// forward_stack through the reference's own tape (network.hpp:190-210), and its gradients by
// Tape::backward of sum(out * out_bar) (autodiff.hpp:264, :397-631).
esrnn_status esrnn_trainer_forward_stack(esrnn_trainer* t, int32_t T, int32_t B, const double* X, double* out,
                                         const double* obar, double* wbar, double* xbar) {
    return guarded(t->err, [&] {
        Trainer& tr = *t->tr;
        const StackConfig& sc = tr.stack_config();
        const int in = sc.input_size, O = tr.profile().horizon;
        ad::Tape tape;
        StackLeaves lv = lift_weights(tape, tr.weights());
        std::vector<ad::DiffArray> seq;
        for (int s = 0; s < T; ++s) {
            Matrix m(static_cast<std::size_t>(B), static_cast<std::size_t>(in));
            std::memcpy(m.data().data(), X + static_cast<std::size_t>(s) * B * in, sizeof(double) * B * in);
            seq.push_back(ad::leaf(tape, std::move(m)));
        }
        ad::DiffArray o = forward_stack(seq, lv, sc);
        if (out) std::memcpy(out, o.value().data().data(), sizeof(double) * B * O);
        if (!obar) return;
        Matrix ob(static_cast<std::size_t>(B), static_cast<std::size_t>(O));
        std::memcpy(ob.data().data(), obar, sizeof(double) * B * O);
        ad::backward(ad::sum(ad::mul(o, ad::constant(tape, std::move(ob)))));
        if (wbar) {
            std::size_t off = 0;
            auto put = [&](const ad::DiffArray& a) {
                const Matrix& g = a.grad();
                std::memcpy(wbar + off, g.data().data(), sizeof(double) * g.size());
                off += g.size();
            };
            for (const auto& c : lv.layers) {  // for_each_param order (network.hpp:62-74)
                put(c.w_input);
                put(c.w_recur);
                put(c.bias);
            }
            put(lv.nl_w);
            put(lv.nl_b);
            put(lv.out_w);
            put(lv.out_b);
        }
        if (xbar)
            for (int s = 0; s < T; ++s)
                std::memcpy(xbar + static_cast<std::size_t>(s) * B * in, seq[s].grad().data().data(), sizeof(double) * B * in);
    });
}

// Exact-resume training state straight from the reference Trainer's private members
// (adam_net_, net_step_, adam_series_, rng_.gen_; trainer.hpp:446-457, :655-672).
esrnn_status esrnn_trainer_get_train_state(esrnn_trainer* t, double* adam_m, double* adam_v, int64_t n_values,
                                           int64_t row_begin, int64_t n, double* ps_m, double* ps_v,
                                           int64_t* ps_steps, int64_t* net_step, char* rng_text, int64_t rng_cap) {
    return guarded(t->err, [&] {
        Trainer& tr = *t->tr;
        const int S = tr.profile().seasonality_length;
        int64_t off = 0;
        tr.weights_.for_each_param([&](const std::string& name, const Matrix& m) {
            const auto& st = tr.adam_net_.at(name);
            for (std::size_t e = 0; e < m.size(); ++e, ++off) {
                if (off >= n_values) continue;
                if (adam_m) adam_m[off] = st.m.data()[e];
                if (adam_v) adam_v[off] = st.v.data()[e];
            }
        });
        if ((adam_m || adam_v) && off != n_values) throw CheckpointError("train state: network size mismatch");
        if (row_begin < 0 || n < 0 || row_begin + n > static_cast<int64_t>(tr.series_count()))
            throw ShapeError("train state: rows out of range");
        for (int64_t i = 0; i < n; ++i) {
            const auto& sa = tr.adam_series_[static_cast<std::size_t>(row_begin + i)];
            if (ps_m) {
                ps_m[i * (2 + S)] = sa.m_alpha;
                ps_m[i * (2 + S) + 1] = sa.m_gamma;
                for (int j = 0; j < S; ++j) ps_m[i * (2 + S) + 2 + j] = sa.m_seas[j];
            }
            if (ps_v) {
                ps_v[i * (2 + S)] = sa.v_alpha;
                ps_v[i * (2 + S) + 1] = sa.v_gamma;
                for (int j = 0; j < S; ++j) ps_v[i * (2 + S) + 2 + j] = sa.v_seas[j];
            }
            if (ps_steps) ps_steps[i] = sa.steps;
        }
        if (net_step) *net_step = tr.net_step_;
        if (rng_text) {
            std::ostringstream os;
            os << tr.rng_.gen_;
            const std::string txt = os.str();
            if (static_cast<int64_t>(txt.size()) + 1 > rng_cap) throw ShapeError("train state: rng buffer too small");
            std::memcpy(rng_text, txt.c_str(), txt.size() + 1);
        }
    });
}

esrnn_status esrnn_trainer_set_train_state(esrnn_trainer* t, const double* adam_m, const double* adam_v,
                                           int64_t n_values, int64_t row_begin, int64_t n, const double* ps_m,
                                           const double* ps_v, const int64_t* ps_steps, int64_t net_step,
                                           const char* rng_text) {
    return guarded(t->err, [&] {
        Trainer& tr = *t->tr;
        const int S = tr.profile().seasonality_length;
        int64_t total = 0;
        tr.weights_.for_each_param([&](const std::string&, const Matrix& m) { total += static_cast<int64_t>(m.size()); });
        if ((adam_m || adam_v) && total != n_values) throw CheckpointError("train state: network size mismatch");
        if (row_begin < 0 || n < 0 || row_begin + n > static_cast<int64_t>(tr.series_count()))
            throw ShapeError("train state: rows out of range");
        std::mt19937_64 g = tr.rng_.gen_;
        if (rng_text) {
            std::istringstream is(rng_text);
            is >> g;
            if (is.fail()) throw CheckpointError("train state: malformed rng state");
        }
        int64_t off = 0;
        tr.weights_.for_each_param([&](const std::string& name, const Matrix& m) {
            auto& st = tr.adam_net_.at(name);
            for (std::size_t e = 0; e < m.size(); ++e, ++off) {
                if (adam_m) st.m.data()[e] = adam_m[off];
                if (adam_v) st.v.data()[e] = adam_v[off];
            }
        });
        for (int64_t i = 0; i < n; ++i) {
            auto& sa = tr.adam_series_[static_cast<std::size_t>(row_begin + i)];
            if (ps_m) {
                sa.m_alpha = ps_m[i * (2 + S)];
                sa.m_gamma = ps_m[i * (2 + S) + 1];
                for (int j = 0; j < S; ++j) sa.m_seas[j] = ps_m[i * (2 + S) + 2 + j];
            }
            if (ps_v) {
                sa.v_alpha = ps_v[i * (2 + S)];
                sa.v_gamma = ps_v[i * (2 + S) + 1];
                for (int j = 0; j < S; ++j) sa.v_seas[j] = ps_v[i * (2 + S) + 2 + j];
            }
            if (ps_steps) sa.steps = static_cast<long>(ps_steps[i]);
        }
        tr.net_step_ = static_cast<long>(net_step);
        tr.rng_.gen_ = g;
    });
}

// cmd_evaluate / detail::score_forecasts (commands.hpp:285-338) restated over the reference's
// own metrics.hpp smape / mase / seasonal_naive (commands.hpp needs the absent vendored json)
esrnn_status esrnn_trainer_evaluate(esrnn_trainer* t, int32_t against_test, double* forecasts, double* smape_o,
                                    double* mase_o, double* naive_smape, double* naive_mase, double* totals) {
    return guarded(t->err, [&] {
        const auto t0 = std::chrono::steady_clock::now();
        const int O = t->tr->profile().horizon, S = t->tr->profile().seasonality_length;
        ForecastResult fr = t->tr->forecast_at(static_cast<std::size_t>(against_test ? O : 2 * O));
        double tot[8] = {0, 0, 0, 0, 0, 0, static_cast<double>(t->tr->series_count()), 0};
        for (std::size_t i = 0; i < t->tr->series_count(); ++i) {
            const DatasetSplit& sp = t->tr->split(i);
            const std::vector<double>& actual = against_test ? sp.test : sp.validation;
            std::vector<double> insample = sp.train;
            if (against_test) insample.insert(insample.end(), sp.validation.begin(), sp.validation.end());
            const std::vector<double> nv = seasonal_naive(insample, S, O);
            const double s = smape(actual, fr.forecasts[i]);
            const std::optional<double> m = mase(insample, actual, fr.forecasts[i], S);
            const double ns = smape(actual, nv);
            const std::optional<double> nm = mase(insample, actual, nv, S);
            if (forecasts)
                for (int j = 0; j < O; ++j) forecasts[i * O + j] = fr.forecasts[i][j];
            if (smape_o) smape_o[i] = s;
            if (mase_o) mase_o[i] = m ? *m : NAN;
            if (naive_smape) naive_smape[i] = ns;
            if (naive_mase) naive_mase[i] = nm ? *nm : NAN;
            tot[0] += s;
            if (m) { tot[1] += *m; tot[2] += 1; }
            tot[3] += ns;
            if (nm) { tot[4] += *nm; tot[5] += 1; }
        }
        if (totals) std::memcpy(totals, tot, sizeof tot);
        t->last_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    });
}

esrnn_status esrnn_trainer_hw_state(esrnn_trainer* t, int64_t row, int64_t t_len, double* levels,
                                    double* seas) {
    return guarded(t->err, [&] {
        const auto& vals = t->tr->series(static_cast<std::size_t>(row)).values;
        std::span<const double> ins(vals.data(), static_cast<std::size_t>(t_len));
        HWState st = hybrid_primer(ins, t->tr->per_series_params(static_cast<std::size_t>(row)));
        std::memcpy(levels, st.levels.data(), sizeof(double) * st.levels.size());
        std::memcpy(seas, st.seasonalities.data(), sizeof(double) * st.seasonalities.size());
    });
}

esrnn_status esrnn_trainer_last_epoch_windows(const esrnn_trainer* t, int32_t* rows, int32_t* anchors, int64_t n) {
    if (n != static_cast<int64_t>(t->last_windows.size())) return ESRNN_SHAPE_ERROR;
    for (int64_t i = 0; i < n; ++i) {
        rows[i] = t->last_windows[i].first;
        anchors[i] = t->last_windows[i].second;
    }
    return ESRNN_OK;
}

esrnn_status esrnn_trainer_last_device_ms(const esrnn_trainer* t, double* ms) {
    *ms = t->last_ms;
    return ESRNN_OK;
}

esrnn_status esrnn_trainer_kernel_launches(const esrnn_trainer*, int64_t* n) {
    *n = 0;
    return ESRNN_OK;
}

esrnn_status esrnn_trainer_profile_kernels(esrnn_trainer*, int32_t) { return ESRNN_OK; }

esrnn_status esrnn_trainer_kernel_times(esrnn_trainer*, double* total_ms, int64_t* launches) {
    for (int i = 0; i < ESRNN_KERNEL_CLASSES; ++i) {
        if (total_ms) total_ms[i] = 0.0;
        if (launches) launches[i] = 0;
    }
    return ESRNN_OK;
}

esrnn_status esrnn_release_cached_memory(void) { return ESRNN_OK; }

// Sharded-mode entry points (B200 extension): the reference is single-process, unsharded.
esrnn_status esrnn_group_create(int32_t, esrnn_group** out) {
    *out = nullptr;
    g_create_err = "reference shim: no sharded mode";
    return ESRNN_CONFIG_ERROR;
}
void esrnn_group_destroy(esrnn_group*) {}
esrnn_status esrnn_trainer_gather_per_series(esrnn_trainer* t, double* a, double* g, double* s) {
    return esrnn_trainer_get_per_series(t, 0, static_cast<int64_t>(t->tr->series_count()), a, g, s);
}

esrnn_status esrnn_nccl_unique_id(uint8_t*) {
    g_create_err = "reference shim: no NCCL";
    return ESRNN_NCCL_ERROR;
}

// Ingestion (esrnn_b200.h): the reference's own cmd_prepare data path (commands.hpp:141-175)
// -- parse_m4_train_csv, parse_info_csv, apply_info, the frequency filter, length_stats,
// equalize_lengths -- without the bundle file; the checker for the engine's parallel parser.
struct esrnn_dataset {
    std::vector<SeriesRecord> kept;
    std::vector<double> values;
    std::vector<int32_t> cats;
};
static thread_local std::string g_ingest_err;
const char* esrnn_ingest_last_error(void) { return g_ingest_err.c_str(); }
esrnn_status esrnn_ingest_m4_csv(const char* train_csv, const char* info_csv, int32_t frequency,
                                 const esrnn_profile* profile, int32_t, esrnn_dataset** out,
                                 esrnn_ingest_stats* stats) {
    *out = nullptr;
    auto ds = std::make_unique<esrnn_dataset>();
    esrnn_status st = guarded(g_ingest_err, [&] {
        std::ifstream train_in(train_csv);
        if (!train_in) throw Error("cannot open \"" + std::string(train_csv) + "\"");
        std::ifstream info_in(info_csv);
        if (!info_in) throw Error("cannot open \"" + std::string(info_csv) + "\"");
        auto series = parse_m4_train_csv(train_in);
        auto info = parse_info_csv(info_in);
        apply_info(series, info);
        std::vector<SeriesRecord> filtered;
        for (auto& s : series)
            if (s.frequency == static_cast<Frequency>(frequency)) filtered.push_back(std::move(s));
        std::vector<std::size_t> raw_lengths;
        for (const auto& s : filtered) raw_lengths.push_back(s.values.size());
        const LengthStats raw = length_stats(raw_lengths);
        FrequencyProfile p = FrequencyProfile::defaults(static_cast<Frequency>(frequency));
        p.horizon = profile->horizon;
        p.min_length = profile->min_length;
        ds->kept = equalize_lengths(std::move(filtered), p);
        if (ds->kept.empty()) throw ValidationError("no series after filtering");
        for (const auto& s : ds->kept) {
            ds->values.insert(ds->values.end(), s.values.begin(), s.values.end());
            ds->cats.push_back(static_cast<int32_t>(s.category.value_or(Category::Other)));
        }
        if (stats) {
            *stats = esrnn_ingest_stats{};
            stats->raw_count = static_cast<int64_t>(raw.count);
            stats->kept = static_cast<int64_t>(ds->kept.size());
            stats->dropped = stats->raw_count - stats->kept;
            stats->equalized_length = p.equalized_length();
            stats->len_mean = raw.mean, stats->len_stddev = raw.stddev, stats->len_min = raw.min;
            stats->len_q25 = raw.q25, stats->len_q50 = raw.q50, stats->len_q75 = raw.q75, stats->len_max = raw.max;
        }
    });
    if (st == ESRNN_OK) *out = ds.release();
    return st;
}
esrnn_status esrnn_dataset_shape(const esrnn_dataset* d, int64_t* n, int32_t* length) {
    *n = static_cast<int64_t>(d->kept.size());
    *length = d->kept.empty() ? 0 : static_cast<int32_t>(d->kept[0].values.size());
    return ESRNN_OK;
}
const double* esrnn_dataset_values(const esrnn_dataset* d) { return d->values.data(); }
const int32_t* esrnn_dataset_categories(const esrnn_dataset* d) { return d->cats.data(); }
const char* esrnn_dataset_id(const esrnn_dataset* d, int64_t i) {
    return (i >= 0 && i < static_cast<int64_t>(d->kept.size())) ? d->kept[static_cast<size_t>(i)].id.c_str() : nullptr;
}
void esrnn_dataset_destroy(esrnn_dataset* d) { delete d; }

// Not in the ABI: the rest of the reference's data path after cmd_prepare's equalisation --
// save_prepared (the JSON bundle, commands.hpp:30-47) and load_prepared (:49-74) -- timed
// by tools/ingest_bench.py.  Returns the number of series read back, -1 on error.
int64_t esrnn_ref_bundle_roundtrip(const esrnn_dataset* d, int32_t frequency, const char* path) {
    try {
        const auto f = static_cast<Frequency>(frequency);
        const int len = d->kept.empty() ? 0 : static_cast<int>(d->kept[0].values.size());
        save_prepared(path, f, len, d->kept);
        return static_cast<int64_t>(load_prepared(path, f).size());
    } catch (const std::exception& e) {
        g_ingest_err = e.what();
        return -1;
    }
}

esrnn_status esrnn_make_synthetic(uint64_t seed, int64_t n, int32_t length, int32_t season_length,
                                  double noise_sigma, double* values, int32_t* category) {
    Rng rng(seed);
    for (int64_t i = 0; i < n; ++i) {
        SeriesRecord rec = testutil::make_multiplicative_series(rng, "S" + std::to_string(i), length,
                                                                season_length, noise_sigma);
        category[i] = static_cast<int32_t>(*rec.category);
        for (int32_t t = 0; t < length; ++t) values[i * length + t] = rec.values[t];
    }
    return ESRNN_OK;
}

}  // extern "C"
