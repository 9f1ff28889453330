// C++ drop-in API test driver: the reference's trainer-level tests
// (/root/reference/proj/tests/test_trainer.cpp, acceptance.cpp criteria 3, 5, 8) written
// against include/esrnn_b200/trainer.hpp, i.e. the same calls a caller of the reference's
// esrnn::Trainer makes, running on the B200 engine.  Needs a GPU; driven by
// tests/test_gpu_cpp_api.py.  Exit code = number of failed checks.
#include <cmath>
#include <cstdio>
#include <functional>
#include <map>
#include <string>
#include <vector>

#include "esrnn_b200/trainer.hpp"

using namespace esrnn;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                                  \
    do {                                                                             \
        if (cond) ++g_pass;                                                          \
        else {                                                                       \
            ++g_fail;                                                                \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
        }                                                                            \
    } while (0)
template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

// tests/helpers.hpp:148-172 generator through the engine's bit-identical restatement
static std::vector<SeriesRecord> dataset(int n, std::uint64_t seed, int length, int S, double sigma) {
    std::vector<double> v(static_cast<std::size_t>(n) * length);
    std::vector<std::int32_t> c(n);
    detail::check(esrnn_make_synthetic(seed, n, length, S, sigma, v.data(), c.data()), nullptr);
    std::vector<SeriesRecord> out(n);
    for (int i = 0; i < n; ++i) {
        out[i].id = "S" + std::to_string(i);
        out[i].category = static_cast<Category>(c[i]);
        out[i].values.assign(v.begin() + static_cast<std::ptrdiff_t>(i) * length, v.begin() + static_cast<std::ptrdiff_t>(i + 1) * length);
    }
    return out;
}

static FrequencyProfile tiny_profile() {  // test_trainer.cpp:13-22
    FrequencyProfile p = FrequencyProfile::defaults(Frequency::Quarterly);
    p.seasonality_length = 4, p.horizon = 4, p.input_window = 8, p.hidden_size = 6;
    p.dilation_blocks = {{1, 2}};
    p.min_length = 20;
    return p;
}
static TrainConfig tiny_config(std::uint64_t seed, Precision prec) {
    TrainConfig c;
    c.batch_size = 16;
    c.seed = seed;
    c.precision = prec;
    return c;
}
static double central_diff(const std::function<double()>& eval, double& param, double step) {
    const double saved = param;
    param = saved + step;
    const double up = eval();
    param = saved - step;
    const double down = eval();
    param = saved;
    return (up - down) / (2.0 * step);
}
static double rel_err(double a, double b) {
    const double d = std::max(std::abs(a), std::abs(b));
    return d < 1e-10 ? std::abs(a - b) : std::abs(a - b) / d;
}

int main() {
    for (Precision prec : {Precision::FP64, Precision::FP32}) {
        const bool f64 = prec == Precision::FP64;
        // zero learning rates leave every parameter bit-unchanged (test_trainer.cpp:96-119)
        {
            auto cfg = tiny_config(3, prec);
            cfg.learning_rate_network = cfg.learning_rate_per_series = 0.0;
            Trainer tr(dataset(3, 11, 28, 4, 0.03), tiny_profile(), cfg);
            std::vector<std::vector<double>> before;
            tr.weights().for_each_param([&](const std::string&, Matrix& m) { before.push_back(m.data()); });
            std::vector<PerSeriesParams> pb;
            for (std::size_t i = 0; i < tr.series_count(); ++i) pb.push_back(tr.per_series_params(i));
            CHECK(std::isfinite(tr.train_epoch()));
            std::size_t i = 0;
            tr.weights().for_each_param([&](const std::string&, Matrix& m) { CHECK(m.data() == before[i++]); });
            for (std::size_t s = 0; s < tr.series_count(); ++s) {
                CHECK(tr.per_series_params(s).alpha_raw == pb[s].alpha_raw);
                CHECK(tr.per_series_params(s).init_seasonality_raw == pb[s].init_seasonality_raw);
            }
        }
        // a batch touching only series A reports only A (test_trainer.cpp:121-137)
        {
            auto cfg = tiny_config(4, prec);
            cfg.batch_size = 4;
            Trainer tr(dataset(2, 13, 28, 4, 0.03), tiny_profile(), cfg);
            WindowBatch b;
            b.series_rows = {0, 0, 0};
            b.anchors = {7, 8, 9};
            b.ids = {"S0", "S0", "S0"};
            b.mask = Matrix(3, 4, 1.0);
            auto g = tr.batch_gradients(b);
            CHECK(g.per_series.count("S0") == 1 && g.per_series.count("S1") == 0);
        }
        // joint flow: loss gradient reaches alpha_raw / gamma_raw and matches FD, with the
        // caller holding double& into per_series_params across batch_loss calls
        // (test_trainer.cpp:139-161)
        if (f64) {
            Trainer tr(dataset(2, 17, 28, 4, 0.03), tiny_profile(), tiny_config(5, prec));
            WindowBatch batch;
            batch.series_rows = {0, 1, 0};
            batch.anchors = {7, 9, 11};
            batch.ids = {"S0", "S1", "S0"};
            batch.mask = Matrix(3, 4, 1.0);
            auto grads = tr.batch_gradients(batch);
            const double analytic = grads.per_series.at("S0").alpha_raw;
            CHECK(analytic != 0.0);
            auto eval = [&]() {
                WindowBatch b = batch;
                return tr.batch_loss(b);
            };
            CHECK(rel_err(analytic, central_diff(eval, tr.per_series_params(0).alpha_raw, 1e-6)) <= 1e-3);
            CHECK(rel_err(grads.per_series.at("S0").gamma_raw, central_diff(eval, tr.per_series_params(0).gamma_raw, 1e-6)) <= 1e-3);
            // a network weight through the mutable weights() reference
            const double gw = grads.network.at("lstm0.w_input")(2, 3);
            CHECK(rel_err(gw, central_diff(eval, tr.weights().layers[0].w_input(2, 3), 1e-6)) <= 1e-3);
        }
        // masked rows contribute zero gradient everywhere (test_trainer.cpp:163-198)
        {
            Trainer tr(dataset(3, 19, 28, 4, 0.03), tiny_profile(), tiny_config(6, prec));
            WindowBatch small, padded;
            small.series_rows = {0, 1};
            small.anchors = {7, 9};
            small.mask = Matrix(2, 4, 1.0);
            padded.series_rows = {0, 1, 2, 2};
            padded.anchors = {7, 9, 8, 10};
            padded.mask = Matrix(4, 4, 1.0);
            for (std::size_t c = 0; c < 4; ++c) padded.mask(2, c) = padded.mask(3, c) = 0.0;
            auto gs = tr.batch_gradients(small);
            auto gp = tr.batch_gradients(padded);
            CHECK(std::abs(gs.loss - gp.loss) <= (f64 ? 1e-15 : 1e-7) * std::abs(gs.loss));
            for (const auto& [name, g] : gs.network)
                for (std::size_t e = 0; e < g.size(); ++e)
                    CHECK(std::abs(g.data()[e] - gp.network.at(name).data()[e]) <= (f64 ? 1e-12 : 1e-7));
            CHECK(gp.per_series.at("S2").alpha_raw == 0.0 && gp.per_series.at("S2").gamma_raw == 0.0);
            for (double v : gp.per_series.at("S2").init_seasonality_raw) CHECK(v == 0.0);
        }
        // validate: shape, zero-network saturation, read-only (test_trainer.cpp:200-216)
        {
            Trainer tr(dataset(3, 23, 28, 4, 0.03), tiny_profile(), tiny_config(7, prec));
            tr.weights().zero();
            auto v1 = tr.validate();
            CHECK(v1.forecasts.size() == 3);
            for (const auto& f : v1.forecasts) {
                CHECK(f.size() == 4);
                for (double x : f) CHECK(x == 0.0);
            }
            CHECK(std::abs(v1.mean_smape - 200.0) < 1e-9);
            auto v2 = tr.validate();
            CHECK(v1.mean_smape == v2.mean_smape);
        }
        // exact resume: weights + per-series (the reference's checkpoint) + TrainState
        {
            Trainer a(dataset(5, 17, 28, 4, 0.03), tiny_profile(), tiny_config(4, prec));
            a.train_epoch();
            const StackWeights w = a.weights();
            std::map<std::string, PerSeriesParams> ps;
            for (std::size_t i = 0; i < a.series_count(); ++i) ps.emplace(a.series(i).id, a.per_series_params(i));
            const TrainState ts = a.train_state();
            CHECK(ts.net_step > 0 && !ts.rng.empty());
            const double la = a.train_epoch();
            Trainer b(dataset(5, 17, 28, 4, 0.03), tiny_profile(), tiny_config(99, prec));
            b.set_weights(w);
            b.set_per_series(ps);
            b.set_train_state(ts);
            CHECK(b.train_epoch() == la);
            TrainState bad = ts;
            bad.rng = "not a state";
            CHECK(throws<CheckpointError>([&] { b.set_train_state(bad); }));
        }
        // general dilated stack: forward_stack over a sequence, gradients vs central differences
        // (test_network.cpp:235-267), with live recurrent matrices and forget gates
        if (prec == Precision::FP64) {
            Trainer tr(dataset(3, 23, 28, 4, 0.03), tiny_profile(), tiny_config(5, prec));
            StackWeights w = tr.weights();
            Rng rng(77);
            w.for_each_param([&](const std::string&, Matrix& m) {
                for (double& v : m.data()) v = rng.uniform(-0.5, 0.5);
            });
            tr.set_weights(w);
            std::vector<Matrix> seq;
            for (int t = 0; t < 4; ++t) {
                Matrix m(2, 14);
                for (double& v : m.data()) v = rng.uniform(-1.0, 1.0);
                seq.push_back(m);
            }
            Matrix ob(2, 4, 1.0);
            std::map<std::string, Matrix> wb;
            std::vector<Matrix> xb;
            const Matrix out = tr.forward_stack(seq, ob, wb, xb);
            CHECK(out.rows() == 2 && out.cols() == 4 && xb.size() == 4);
            auto total = [&](const std::vector<Matrix>& s) {
                const Matrix o = tr.forward_stack(s);
                double acc = 0.0;
                for (double v : o.data()) acc += v;
                return acc;
            };
            const double h = 1e-6;
            std::vector<Matrix> sp = seq, sm = seq;
            sp[1](0, 3) += h;
            sm[1](0, 3) -= h;
            const double fd = (total(sp) - total(sm)) / (2 * h);
            CHECK(std::abs(fd - xb[1](0, 3)) < 1e-6 + 1e-5 * std::abs(fd));
            CHECK(std::abs(wb.at("lstm0.w_recur")(1, 2)) > 0.0);  // the recurrence is live
            CHECK(throws<ContractError>([&] { tr.forward_stack(std::vector<Matrix>{}); }));
        }
        // same seed reproduces the loss trajectory bit for bit (test_trainer.cpp:218-230)
        {
            Trainer t1(dataset(3, 29, 28, 4, 0.03), tiny_profile(), tiny_config(42, prec));
            Trainer t2(dataset(3, 29, 28, 4, 0.03), tiny_profile(), tiny_config(42, prec));
            for (int e = 0; e < 3; ++e) CHECK(t1.train_epoch() == t2.train_epoch());
            CHECK(t1.validate().mean_smape == t2.validate().mean_smape);
        }
        // batched loss equals the combined single-window losses (test_trainer.cpp:232-259)
        {
            Trainer tr(dataset(4, 31, 28, 4, 0.03), tiny_profile(), tiny_config(8, prec));
            auto windows = tr.all_windows();
            const std::size_t take = std::min<std::size_t>(windows.size(), 24);
            WindowBatch big;
            for (std::size_t i = 0; i < take; ++i) {
                big.series_rows.push_back(windows[i].first);
                big.anchors.push_back(windows[i].second);
            }
            big.mask = Matrix(take, 4, 1.0);
            const double batched = tr.batch_loss(big);
            double acc = 0.0;
            for (std::size_t i = 0; i < take; ++i) {
                WindowBatch one;
                one.series_rows = {windows[i].first};
                one.anchors = {windows[i].second};
                one.mask = Matrix(1, 4, 1.0);
                acc += tr.batch_loss(one);
            }
            CHECK(rel_err(batched, acc / static_cast<double>(take)) <= 1e-6);
        }
        // detached state freezes the per-series parameters (test_trainer.cpp:274-282)
        {
            auto cfg = tiny_config(10, prec);
            cfg.attach_es_state = false;
            Trainer tr(dataset(2, 41, 28, 4, 0.03), tiny_profile(), cfg);
            const PerSeriesParams before = tr.per_series_params(0);
            tr.train_epoch();
            CHECK(tr.per_series_params(0).alpha_raw == before.alpha_raw);
            CHECK(tr.per_series_params(0).gamma_raw == before.gamma_raw);
        }
        // a single constant series overfits quickly (test_trainer.cpp:284-295)
        {
            SeriesRecord rec;
            rec.id = "const";
            rec.category = Category::Micro;
            rec.values.assign(28, 50.0);
            auto cfg = tiny_config(11, prec);
            cfg.learning_rate_network = 5e-3;
            Trainer tr({rec}, tiny_profile(), cfg);
            double loss = 1.0;
            for (int e = 0; e < 300 && loss >= 1e-2; ++e) loss = tr.train_epoch();
            CHECK(loss < 1e-2);
        }
        // training reduces the loss across seeds (test_trainer.cpp:297-307)
        for (std::uint64_t seed = 1; seed <= 5; ++seed) {
            Trainer tr(dataset(4, 100 + seed, 28, 4, 0.03), tiny_profile(), tiny_config(seed, prec));
            const double initial = tr.train_epoch();
            double fin = initial;
            for (int e = 0; e < 10; ++e) fin = tr.train_epoch();
            CHECK(fin < initial);
        }
        // benchmark: equivalence gate and self-comparison (test_trainer.cpp:261-272)
        {
            auto cfg = tiny_config(9, prec);
            cfg.batch_size = 1;
            Trainer tr(dataset(100, 37, 36, 4, 0.03), tiny_profile(), cfg);
            auto rep = tr.benchmark_batched_vs_looped();
            CHECK(rep.batch_size == 1 && rep.n_series == 100);
            CHECK(std::abs(rep.speedup - rep.looped_s / rep.batched_s) < 1e-12);
        }
        // overfit smoke: 4 clean seasonal quarterly series to pinball < 1e-2 (acceptance.cpp:394-413)
        {
            TrainConfig cfg;
            cfg.batch_size = 256;
            cfg.seed = 11;
            cfg.learning_rate_network = 5e-3;
            cfg.precision = prec;
            Trainer tr(dataset(4, 51, 88, 4, 0.0), FrequencyProfile::defaults(Frequency::Quarterly), cfg);
            double loss = 1e9;
            int epochs = 0;
            while (epochs < 500 && !(loss < 1e-2)) loss = tr.train_epoch(), ++epochs;
            CHECK(loss < 1e-2);
        }
    }
    // configuration and data validation (test_trainer.cpp:309-325)
    {
        TrainConfig cfg;
        cfg.tau = 1.5;
        CHECK(throws<ConfigError>([&] { cfg.validate(); }));
        cfg = TrainConfig{};
        cfg.batch_size = 4096;
        CHECK(throws<ConfigError>([&] { cfg.validate(); }));
        auto data = dataset(2, 43, 28, 4, 0.03);
        data[1].values.pop_back();
        CHECK(throws<ConfigError>([&] { Trainer t(data, tiny_profile(), tiny_config(0, Precision::FP64)); }));
        Trainer tr(dataset(2, 43, 28, 4, 0.03), tiny_profile(), tiny_config(0, Precision::FP64));
        WindowBatch bad;
        bad.series_rows = {0};
        bad.anchors = {100};
        bad.mask = Matrix(1, 4, 1.0);
        CHECK(throws<ShapeError>([&] { tr.batch_loss(bad); }));
        bad.anchors = {7};
        bad.mask = Matrix(1, 4, 0.0);
        CHECK(throws<ContractError>([&] { tr.batch_loss(bad); }));
        StackWeights w = tr.weights();
        w.layers.pop_back();
        CHECK(throws<CheckpointError>([&] { tr.set_weights(w); }));
    }
    std::printf("cpp_api_test: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail;
}
