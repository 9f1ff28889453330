// Host side of the B200 engine and the C-ABI (include/esrnn_b200.h).
//
// The host keeps everything the reference's Trainer keeps that is index/bookkeeping
// work (profile, config, RNG stream, window lists, slot dedupe) and drives the device:
// all arithmetic of the training step, forecast and validation runs in the sm_100a
// kernels of kernels.cuh.  There is no CPU compute fallback: without a CUDA device the
// create call fails with ESRNN_CUDA_ERROR.
#include <cuda.h>  // CUtensorMap (the encoder is reached through cudaGetDriverEntryPoint)
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <future>
#include <chrono>
#include <list>
#include <map>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <sstream>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "esrnn_b200.h"
#include "collective.cuh"
#include "finish.cuh"
#include "seqstack.cuh"
#include "scan.cuh"
#include "host_runtime.h"
#include "tile.cuh"

using namespace esrnn_dev;
using namespace esrnn_host;

namespace {
extern int g_smem_optin, g_num_sms;  // device limits (defined below, set at create)



// One plan = ordered local windows + per-step slot lists + per-slot window CSR.
struct HostPlan {
    std::vector<int> w_row, w_anchor, w_slot, w_first, step_win_off, step_slot_off, slot_row, slot_win_off, slot_win, w_csr,
        csr_anchor;
    std::vector<double> step_M;
    int max_step_windows = 0, max_step_slots = 0;
};

// One epoch's host plan: the global shuffled window order and this rank's step plan, built
// in step-range chunks on the worker pool and packed (with offset fix-ups) into a pinned
// buffer in upload order, so the epoch's plan goes to the device as a few async copies.
struct EpochPlan {
    Mt64 rng_before;  // trainer RNG before this epoch's shuffle (exact-resume state)
    std::vector<uint64_t> wbuf;  // shuffle scratch: (row, anchor) pairs
    std::vector<uint64_t> rnd;   // the shuffle's raw draws
    int64_t n_windows = 0;
    std::vector<HostPlan> chunks;
    int steps = 0;
    bool ready = false;
    // packed arrays: 11 int arrays then step_M (doubles), each at off[i] (bytes)
    enum { kWRow, kWAnchor, kWSlot, kWFirst, kWCsr, kCsrAnchor, kSlotRow, kSlotWin, kSlotWinOff, kStepWinOff,
           kStepSlotOff, kStepM, kArrays };
    PinnedBuf<unsigned char> pin;
    size_t off[kArrays + 1] = {};
    size_t n_w = 0, n_slots = 0;
    int max_step_windows = 0, max_step_slots = 0;
};

// Released trainers' epoch plans (host vectors + pinned upload buffer), reused by the next
// trainer so its first plan writes to warm memory instead of faulting in fresh pages.
struct PlanPool {
    std::mutex mu;
    std::vector<EpochPlan> free;
};
PlanPool& plan_pool() {
    static PlanPool* p = new PlanPool;  // never destroyed
    return *p;
}
EpochPlan plan_pool_get() {
    PlanPool& p = plan_pool();
    std::lock_guard<std::mutex> g(p.mu);
    if (p.free.empty()) return EpochPlan{};
    EpochPlan e = std::move(p.free.back());
    p.free.pop_back();
    e.ready = false;
    return e;
}
void plan_pool_put(EpochPlan&& e) {
    PlanPool& p = plan_pool();
    std::lock_guard<std::mutex> g(p.mu);
    if (p.free.size() < 8) p.free.push_back(std::move(e));
}

struct DevPlan {
    DBuf<int> w_row, w_anchor, w_slot, w_first, step_win_off, step_slot_off, slot_row, slot_win_off, slot_win, w_csr, csr_anchor;
    DBuf<double> step_M;
    DBuf<unsigned char> mask;
    size_t cap_w = 0, cap_steps = 0, cap_slots = 0;
    PlanDev view(bool with_mask) const {
        PlanDev p{};
        p.w_row = w_row.p;
        p.w_anchor = w_anchor.p;
        p.w_slot = w_slot.p;
        p.w_first = w_first.p;
        p.step_win_off = step_win_off.p;
        p.step_slot_off = step_slot_off.p;
        p.slot_row = slot_row.p;
        p.slot_win_off = slot_win_off.p;
        p.slot_win = slot_win.p;
        p.w_csr = w_csr.p;
        p.csr_anchor = csr_anchor.p;
        p.step_M = step_M.p;
        p.mask = with_mask ? mask.p : nullptr;
        return p;
    }
};

// In-process rank group (esrnn_group_create): W trainers in one process, one host thread
// each, exchanging the step's partials through k_group_reduce's device slots (collective.cuh)
// and the per-call host results (validate / evaluate totals, per-series gathers) through a
// host barrier.  Device slots are allocated by the first rank to need them, on its device;
// ranks on other devices reach them through peer access.
struct LocalGroupImpl {
    int W = 0;
    std::mutex mu;
    std::condition_variable cv;
    int refs = 0;              // trainers alive in the group
    std::vector<char> joined;  // a group serves one set of W trainers: each rank joins once
    bool orphaned = false;     // esrnn_group_destroy called while trainers were alive
    // device exchange (k_group_reduce)
    int dev = -1;
    long long stride = 0;
    unsigned char* slots = nullptr;
    unsigned long long* done = nullptr;
    unsigned* ctr = nullptr;
    // host exchange
    long long gen = 0;
    int arrived = 0;
    std::vector<std::vector<unsigned char>> deposit, result;

    ~LocalGroupImpl() {
        if (dev >= 0) {
            int d0 = 0;
            cudaGetDevice(&d0);
            cudaSetDevice(dev);
            cudaFree(slots);
            cudaFree(done);
            cudaFree(ctr);
            cudaSetDevice(d0);
        }
    }
    // every rank deposits `n` bytes; returns all ranks' deposits, rank-major (rank order)
    std::vector<unsigned char> exchange(int rank, const void* data, size_t n) {
        std::unique_lock<std::mutex> lk(mu);
        deposit[rank].assign(static_cast<const unsigned char*>(data), static_cast<const unsigned char*>(data) + n);
        const long long my_gen = gen;
        if (++arrived == W) {
            std::vector<unsigned char> all;
            for (auto& d : deposit) all.insert(all.end(), d.begin(), d.end());
            result.assign(1, std::move(all));
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != my_gen; })) {
            --arrived;
            raise(ESRNN_NCCL_ERROR, "group exchange: a rank did not arrive within 120 s");
        }
        return result[0];
    }
    // device slots for `bytes` per rank (first caller allocates; the configuration is shared)
    void ensure_device(int device, long long bytes) {
        std::lock_guard<std::mutex> lk(mu);
        const long long need = (bytes + 255) / 256 * 256;
        if (dev >= 0) {
            if (need > stride) raise(ESRNN_CONFIG_ERROR, "group: ranks differ in configuration");
            if (device != dev) {
                int ok = 0;
                CUDA_OK(cudaDeviceCanAccessPeer(&ok, device, dev));
                if (!ok) raise(ESRNN_CUDA_ERROR, "group: device %d cannot access device %d", device, dev);
                const cudaError_t st = cudaDeviceEnablePeerAccess(dev, 0);
                if (st != cudaSuccess && st != cudaErrorPeerAccessAlreadyEnabled) CUDA_OK(st);
                cudaGetLastError();
            }
            return;
        }
        dev = device;
        stride = need;
        CUDA_OK(cudaMalloc(&slots, 2 * static_cast<size_t>(W) * stride));
        CUDA_OK(cudaMalloc(&done, sizeof(unsigned long long) * W));
        CUDA_OK(cudaMalloc(&ctr, sizeof(unsigned) * 2 * W));
        CUDA_OK(cudaMemset(done, 0, sizeof(unsigned long long) * W));
        CUDA_OK(cudaMemset(ctr, 0, sizeof(unsigned) * 2 * W));
        CUDA_OK(cudaDeviceSynchronize());
    }
};

void release_group(LocalGroupImpl* g) {
    bool del = false;
    {
        std::lock_guard<std::mutex> lk(g->mu);
        del = --g->refs == 0 && g->orphaned;
    }
    if (del) delete g;
}

constexpr int kRows = kR;         // windows per K2 tile
constexpr int64_t kBcSteps = 40960;  // Adam bias-correction table length (bc_table)

}  // namespace

struct esrnn_group : LocalGroupImpl {};

struct esrnn_trainer {
    // configuration (data.hpp:60-118, trainer.hpp:22-44)
    esrnn_profile prof{};
    esrnn_train_config cfg{};
    int rank = 0, world = 1;
    int N_global = 0, N = 0, row0 = 0, LEN = 0, T = 0, S = 0, I = 0, O = 0, H = 0, L = 0, in0 = 0;
    int blen[ESRNN_MAX_BLOCKS] = {};
    int layer_in[ESRNN_MAX_LAYERS] = {};
    int64_t off_win[ESRNN_MAX_LAYERS] = {}, off_wrec[ESRNN_MAX_LAYERS] = {}, off_bias[ESRNN_MAX_LAYERS] = {};
    int64_t off_nlw = 0, off_nlb = 0, off_outw = 0, off_outb = 0, P = 0;
    NetLayout lay{};
    std::vector<int64_t> live_flat;   // compact index -> flat index
    std::vector<double> w_host;       // flat StackWeights mirror (dead entries live only here)
    PinnedBuf<uint64_t> w_raw;        // creation: the weight init's raw draws (pooled block)
    size_t w_draws = 0;
    std::vector<int> cat_host;
    HostRng rng{0};
    std::string err;
    double last_ms = 0.0;
    int64_t launches = 0;
    bool fp64 = false;
    size_t rsz = 4;

    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // series-sharded data parallelism: the step's partials are all-reduced
    // through NCCL (one process per GPU) or through an in-process group (esrnn_group_create)
    ncclComm_t comm = nullptr;
    LocalGroupImpl* group = nullptr;
    bool sharded = false;     // the collective step runs (world > 1, or forced at world 1)
    int group_ctas = 0;       // k_group_reduce grid

    // device state (type-erased: Real = float or double, chosen by cfg.precision)
    DBuf<unsigned char> vals, vrm, ps, ps_m, ps_v, theta, mW, vW;
    int ldv = 0;  // row stride of the row-major value copy (16-byte multiple)
    DBuf<signed char> cat;
    DBuf<int> ps_steps;
    DBuf<unsigned char> tm_rs;  // K3 GEMM staging tensor maps over the row store (2 x 128 B)
    DBuf<unsigned char> lv, se, contrib, rowstore, gbuf, psg, d_inputs, d_targets, d_seas, d_levels;
    DBuf<unsigned char> fX, fL, fS, dump_lv, dump_se;
    DBuf<double> loss_part, es_sq_part, es_pen_part, red_sq_part, scal, loss_hist, f_out, f_smape, f_score, smape_sum, gtail;
    DBuf<long long> coll_seq;
    DBuf<unsigned int> done_ctr, gtile_ctr;
    DBuf<unsigned char> gpart;
    int gsplit = 1;  // K3 weight-gradient row parts per output tile (large steps)
    bool wide = false;  // K3 weight gradients by q-strip blocks (finish.cuh dw_wide_block)
    int umma_parts = 0, umma_tiles = 0;  // tensor-core dW path (fp32, steps >= kUmmaMinRows)
    DBuf<unsigned char> upart;
    const double* bc_tab = nullptr;  // process-wide bias-correction table of this GPU (StateDev::bc)
    DBuf<long long> net_step;
    DBuf<long long> dbg_clk;  // ESRNN_DEBUG_CLOCKS: per-phase clock64 stamps of tile 0
    DBuf<int> errw;
    int Bcap = 0, kcap = 0, tiles_cap = 0, es_bd = 16, es_blocks = 0, red_blocks = 0, steps_cap = 0;
    bool pdl = std::getenv("ESRNN_NO_PDL") == nullptr;  // programmatic dependent launch between step kernels

    DevPlan epoch_plan, batch_plan;
    EpochPlan cur_plan, next_plan;
    std::future<void> plan_done;  // the first epoch's plan, built while create finishes
    bool have_last = false;  // cur_plan holds the global window order of the last train_epoch
    DBuf<double> stage_raw;            // creation: the series block as uploaded (fp64)
    PinnedBuf<double> stage_pin;       // creation: its pinned staging copy
    PinnedBuf<double> stage_theta;     // creation: the initial compact weights, pinned
    PinnedBuf<signed char> stage_cat;  // creation: pinned category bytes
    PinnedBuf<int> pin_i;
    PinnedBuf<int> pin_err;            // the error word, read back with a call's results
    PinnedBuf<double> pin_loss;        // an epoch's per-step losses
    PinnedBuf<double> pin_d;

    std::shared_ptr<GraphExec> graph;  // epoch graph (shared with the process-wide cache)
    std::string graph_key;

    // per-kernel event timing (esrnn_trainer_profile_kernels(t, 1)); in-graph global-timer
    // spans of every step's kernels (esrnn_trainer_profile_kernels(t, 2))
    bool profiling = false;
    bool span_mode = false;
    DBuf<long long> spans;
    std::vector<cudaEvent_t> prof_ev;
    std::vector<int> prof_cls;
    double prof_ms[ESRNN_KERNEL_CLASSES] = {};
    int64_t prof_n[ESRNN_KERNEL_CLASSES] = {};
    struct KScope {
        esrnn_trainer* e;
        int cls;
        KScope(esrnn_trainer* e_, int c) : e(e_), cls(c) {
            if (e->profiling) e->prof_mark(cls);
        }
        ~KScope() {
            if (e->profiling) e->prof_mark(-1);
        }
    };
    void prof_mark(int cls) {
        cudaEvent_t ev;
        cudaEventCreate(&ev);
        cudaEventRecord(ev, stream);
        prof_ev.push_back(ev);
        prof_cls.push_back(cls);
    }
    void prof_collect() {
        cudaStreamSynchronize(stream);
        for (size_t i = 0; i + 1 < prof_ev.size(); i += 2) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, prof_ev[i], prof_ev[i + 1]);
            prof_ms[prof_cls[i]] += ms;
            prof_n[prof_cls[i]] += 1;
        }
        for (auto ev : prof_ev) cudaEventDestroy(ev);
        prof_ev.clear();
        prof_cls.clear();
    }

    // Return every device buffer to the block cache in reverse allocation order: the cache is
    // LIFO per size class, so a trainer that repeats this one's allocation sequence gets the
    // same addresses back (and with them the cached epoch graph).
    void release_buffers() {
        std::vector<std::pair<uint64_t, std::function<void()>>> v;
        auto add = [&](auto&... bs) {
            (([&](auto& b) {
                 if (b.p) v.emplace_back(b.seq, [&b] { b.free(); });
             }(bs)),
             ...);
        };
        add(vals, vrm, ps, ps_m, ps_v, theta, mW, vW, cat, ps_steps, lv, se, contrib, tm_rs, rowstore, gbuf, psg, d_inputs,
            d_targets, d_seas, d_levels, fX, fL, fS, dump_lv, dump_se, loss_part, es_sq_part, es_pen_part, red_sq_part, scal, upart,
            loss_hist, f_out, f_smape, f_score, smape_sum, done_ctr, gtile_ctr, gpart, net_step, dbg_clk, errw, gtail,
            coll_seq, spans);
        for (DevPlan* d : {&epoch_plan, &batch_plan})
            add(d->w_row, d->w_anchor, d->w_slot, d->w_first, d->step_win_off, d->step_slot_off, d->slot_row,
                d->slot_win_off, d->slot_win, d->w_csr, d->csr_anchor, d->step_M, d->mask);
        std::sort(v.begin(), v.end(), [](const auto& a, const auto& b) { return a.first > b.first; });
        for (auto& kv : v) kv.second();
    }

    void join_plan() {
        if (plan_done.valid()) plan_done.wait();
        plan_done = std::future<void>();
    }

    ~esrnn_trainer() {
        join_plan();
        plan_pool_put(std::move(cur_plan));
        plan_pool_put(std::move(next_plan));
        if (stream) cudaStreamSynchronize(stream);  // buffers go back to the block cache below
        release_buffers();
        graph.reset();  // sharded trainers' graphs are never in the process cache
        if (comm) ncclCommDestroy(comm);
        if (group) release_group(group);
        if (stream) stream_put(stream, ev0, ev1);  // idle: synchronised above
    }

    template <typename Real>
    StateDev<Real> state() {
        StateDev<Real> s{};
        s.vals = reinterpret_cast<const Real*>(vals.p);
        s.vrm = reinterpret_cast<const Real*>(vrm.p);
        s.ldv = ldv;
        s.cat = cat.p;
        s.N = N;
        s.LEN = LEN;
        s.kcap = kcap;
        s.ps = reinterpret_cast<Real*>(ps.p);
        s.ps_m = reinterpret_cast<Real*>(ps_m.p);
        s.ps_v = reinterpret_cast<Real*>(ps_v.p);
        s.ps_steps = ps_steps.p;
        s.theta = reinterpret_cast<Real*>(theta.p);
        s.mW = reinterpret_cast<Real*>(mW.p);
        s.vW = reinterpret_cast<Real*>(vW.p);
        s.lv = reinterpret_cast<Real*>(lv.p);
        s.se = reinterpret_cast<Real*>(se.p);
        s.contrib = reinterpret_cast<double*>(contrib.p);
        s.cwp = (I + O + 2 + 3) & ~3;
        s.rowstore = reinterpret_cast<Real*>(rowstore.p);
        s.tm_rs = tm_rs.p;
        s.loss_part = loss_part.p;
        s.gbuf = reinterpret_cast<Real*>(gbuf.p);
        s.gtail = gtail.p;
        s.coll_seq = coll_seq.p;
        s.psg = reinterpret_cast<Real*>(psg.p);
        s.es_sq_part = es_sq_part.p;
        s.es_pen_part = es_pen_part.p;
        s.red_sq_part = red_sq_part.p;
        s.gpart = reinterpret_cast<Real*>(gpart.p);
        s.gtile_ctr = gtile_ctr.p;
        s.red_tiles = red_blocks;
        s.gemm_wide = wide ? 1 : 0;
        s.tile_trigger_early = std::getenv("ESRNN_TILE_TRIGGER_EARLY") ? 1 : 0;
        s.upart = reinterpret_cast<float*>(upart.p);
        s.umma_tiles = umma_tiles;
        s.done_ctr = done_ctr.p;
        s.scal = scal.p;
        s.net_step = net_step.p;
        s.loss_hist = loss_hist.p;
        s.bc = bc_tab;
        s.bc_n = kBcSteps;
        s.err = errw.p;
        s.d_inputs = nullptr;
        s.d_targets = nullptr;
        s.d_seas = nullptr;
        s.d_levels = nullptr;
        s.tau = cfg.tau;
        s.lr_net = cfg.learning_rate_network;
        s.lr_ps = cfg.learning_rate_per_series;
        s.clip = cfg.gradient_clip;
        s.has_clip = cfg.has_gradient_clip ? 1 : 0;
        s.attach = cfg.attach_es_state ? 1 : 0;
        // the penalty regularises the ES state: with detached ES state it has no gradient and
        // is omitted (oracle/esrnn_oracle.c lvp_series)
        s.lvp = cfg.attach_es_state ? cfg.level_variability_penalty : 0.0;
        s.dbg_clk = dbg_clk.p;
        s.spans = span_mode ? spans.p : nullptr;
        return s;
    }
};

namespace {

using Eng = esrnn_trainer;

template <class Fn>
esrnn_status guarded(std::string& err, Fn&& fn) {
    try {
        fn();
        return ESRNN_OK;
    } catch (const ApiError& e) {
        err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        err = "host allocation failed";
        return ESRNN_ERROR;
    } catch (const std::exception& e) {
        err = e.what();
        return ESRNN_ERROR;
    }
}

// ------------------------------------------------------------------ validation
void validate_config(const esrnn_profile& p, const esrnn_train_config& c) {
    // data.hpp:101-114
    if (p.seasonality_length < 1) raise(ESRNN_CONFIG_ERROR, "profile: seasonality must be >= 1");
    if (p.horizon < 1) raise(ESRNN_CONFIG_ERROR, "profile: horizon must be >= 1");
    if (p.input_window < p.seasonality_length)
        raise(ESRNN_CONFIG_ERROR, "profile: input_window must cover at least one season");
    if (p.n_blocks < 1) raise(ESRNN_CONFIG_ERROR, "profile: dilation blocks must be non-empty");
    if (p.n_blocks > ESRNN_MAX_BLOCKS) raise(ESRNN_CONFIG_ERROR, "profile: at most %d dilation blocks", ESRNN_MAX_BLOCKS);
    int layer = 0;
    for (int b = 0; b < p.n_blocks; ++b) {
        if (p.block_len[b] < 1) raise(ESRNN_CONFIG_ERROR, "profile: empty dilation block");
        for (int j = 0; j < p.block_len[b]; ++j, ++layer) {
            if (layer >= ESRNN_MAX_LAYERS) raise(ESRNN_CONFIG_ERROR, "profile: at most %d layers", ESRNN_MAX_LAYERS);
            if (p.dilations[layer] < 1) raise(ESRNN_CONFIG_ERROR, "profile: dilations must be strictly positive");
        }
    }
    if (p.hidden_size < 1) raise(ESRNN_CONFIG_ERROR, "profile: hidden_size must be >= 1");
    if (p.min_length < 1) raise(ESRNN_CONFIG_ERROR, "profile: min_length must be >= 1");
    // trainer.hpp:34-43 (+ the B200 batch cap extension)
    const int cap = c.max_batch_size > 0 ? c.max_batch_size : 2048;
    if (c.epochs < 0) raise(ESRNN_CONFIG_ERROR, "train: epochs must be >= 0");
    if (c.batch_size < 1 || c.batch_size > cap) raise(ESRNN_CONFIG_ERROR, "train: batch_size must be in [1, %d]", cap);
    if (!(c.tau > 0.0 && c.tau < 1.0)) raise(ESRNN_CONFIG_ERROR, "train: tau must be in (0, 1)");
    if (c.learning_rate_network < 0.0 || c.learning_rate_per_series < 0.0)
        raise(ESRNN_CONFIG_ERROR, "train: learning rates must be non-negative");
    if (c.has_gradient_clip && c.gradient_clip <= 0.0) raise(ESRNN_CONFIG_ERROR, "train: gradient_clip must be positive");
    if (!(c.level_variability_penalty >= 0.0) || !std::isfinite(c.level_variability_penalty))
        raise(ESRNN_CONFIG_ERROR, "train: level_variability_penalty must be finite and >= 0");
    // device-kernel limits (shared-memory tiles are sized from these)
    if (p.hidden_size > 80) raise(ESRNN_CONFIG_ERROR, "profile: hidden_size > 80 unsupported by the B200 kernels");
    if (p.seasonality_length > 64) raise(ESRNN_CONFIG_ERROR, "profile: seasonality > 64 unsupported by the B200 kernels");
    if (p.input_window + ESRNN_NUM_CATEGORIES > 256 || p.horizon > 128)
        raise(ESRNN_CONFIG_ERROR, "profile: window sizes unsupported by the B200 kernels");
}

// The error word's copy, enqueued with a call's results so one synchronisation covers both;
// check_device_error() reads it after that synchronisation.
void enqueue_error_read(Eng* e) {
    e->pin_err.reserve(4);
    CUDA_OK(cudaMemcpyAsync(e->pin_err.p, e->errw.p, 4 * sizeof(int), cudaMemcpyDeviceToHost, e->stream));
}

void raise_device_error(Eng* e, const int* h);

// The error word after a call: this rank's own error (code, first t), else -- sharded -- the
// any-rank flag the reduced step buffers carried (every rank raises, none updated).
void check_device_error(Eng* e) {
    if (e->pin_err.p[0] != 0 || e->pin_err.p[2] != 0) raise_device_error(e, e->pin_err.p);
}

void throw_device_error(Eng* e) {
    int h[4];
    CUDA_OK(cudaMemcpyAsync(h, e->errw.p, sizeof h, cudaMemcpyDeviceToHost, e->stream));
    CUDA_OK(cudaStreamSynchronize(e->stream));
    if (h[0] != 0 || h[2] != 0) raise_device_error(e, h);
}

void raise_device_error(Eng* e, const int* hp) {
    const int h[3] = {hp[0], hp[1], hp[2]};
    const int reset[4] = {0, INT_MAX, 0, 0};
    CUDA_OK(cudaMemcpyAsync(e->errw.p, reset, sizeof reset, cudaMemcpyHostToDevice, e->stream));
    CUDA_OK(cudaStreamSynchronize(e->stream));
    if (h[0] == 0)
        raise(ESRNN_NUMERIC_DOMAIN_ERROR, "hybrid_primer_tape: non-positive level (raised on another rank of the group)");
    switch (h[0]) {
        case kErrPeer: raise(ESRNN_NCCL_ERROR, "group collective: rank %d did not arrive (timeout)", h[1]);
        case kErrTrainLevel: raise(ESRNN_NUMERIC_DOMAIN_ERROR, "hybrid_primer_tape: non-positive level at t=%d", h[1]);
        case kErrObs: raise(ESRNN_NUMERIC_DOMAIN_ERROR, "hybrid_primer: non-positive observation at t=%d", h[1]);
        case kErrFcLevel: raise(ESRNN_NUMERIC_DOMAIN_ERROR, "hybrid_primer: non-positive level at t=%d", h[1]);
        default: raise(ESRNN_NUMERIC_DOMAIN_ERROR, "deseasonalize_normalize: non-positive seasonality");
    }
}

// ------------------------------------------------------------------ layout
// W^T row stride: a multiple of 8 with an odd quotient (conflict-free for both K2 products)
int ld8odd(int n) {
    int p = (n + 7) & ~7;
    if (((p >> 3) & 1) == 0) p += 8;
    return p;
}

void build_layout(Eng* e) {
    const int H = e->H, O = e->O;
    int64_t off = 0, coff = 0;
    NetLayout& lay = e->lay;
    std::memset(&lay, 0, sizeof lay);
    lay.L = e->L;
    lay.nb = e->prof.n_blocks;
    lay.H = H;
    lay.O = O;
    lay.I = e->I;
    lay.S = e->S;
    lay.in0 = e->in0;
    lay.T = e->T;
    lay.ldx = (e->in0 + 3) & ~3;
    lay.ldh = (H + 3) & ~3;
    e->live_flat.clear();
    // compact segments start on 4-element boundaries; padding slots map to -1
    auto pad4 = [&]() {
        while (coff % 4) {
            e->live_flat.push_back(-1);
            ++coff;
        }
    };
    int layer = 0;
    for (int b = 0; b < e->prof.n_blocks; ++b) {
        const int first = layer;
        for (int j = 0; j < e->prof.block_len[b]; ++j, ++layer) {
            const int in = layer == 0 ? e->in0 : H;
            e->layer_in[layer] = in;
            lay.layer_in[layer] = in;
            lay.res_src[layer] = -1;
            lay.block_first[layer] = (b > 0 && layer == first) ? 1 : 0;
            lay.block_last[layer] = (b > 0 && j == e->prof.block_len[b] - 1) ? 1 : 0;
            if (lay.block_last[layer]) lay.res_src[layer] = first - 1;
            // flat (for_each_param) layout: w_input, w_recur, bias
            e->off_win[layer] = off;
            off += static_cast<int64_t>(in) * 4 * H;
            e->off_wrec[layer] = off;
            off += static_cast<int64_t>(H) * 4 * H;
            e->off_bias[layer] = off;
            off += 4 * H;
            // compact live layout: W^T over the live gate columns [i | g | o] (forget gate
            // dead) with row stride ldk = 8 * odd >= in (pad columns -> -1), then the bias
            pad4();
            const int ldk = ld8odd(in);
            lay.ldk[layer] = ldk;
            lay.cw[layer] = coff;
            for (int q = 0; q < 3 * H; ++q) {
                const int col = q < H ? q : q + H;
                for (int k = 0; k < ldk; ++k)
                    e->live_flat.push_back(k < in ? e->off_win[layer] + static_cast<int64_t>(k) * 4 * H + col : -1);
            }
            coff += static_cast<int64_t>(3 * H) * ldk;
            lay.cb[layer] = coff;
            for (int q = 0; q < 3 * H; ++q) e->live_flat.push_back(e->off_bias[layer] + (q < H ? q : q + H));
            coff += 3 * H;
        }
    }
    lay.ldg = (3 * H + 3) & ~3;
    lay.ldo = (O + 3) & ~3;
    lay.ldkh = ld8odd(H);
    e->off_nlw = off;
    off += static_cast<int64_t>(H) * H;
    e->off_nlb = off;
    off += H;
    e->off_outw = off;
    off += static_cast<int64_t>(H) * O;
    e->off_outb = off;
    off += O;
    e->P = off;
    // head: nl_w^T [H][ldkh], nl_b [H], out_w^T [O][ldkh], out_b [O] (one contiguous segment,
    // 4-aligned matrices)
    pad4();
    const int ldkh = lay.ldkh;
    lay.c_nlw = coff;
    for (int j = 0; j < H; ++j)
        for (int k = 0; k < ldkh; ++k) e->live_flat.push_back(k < H ? e->off_nlw + static_cast<int64_t>(k) * H + j : -1);
    coff += static_cast<int64_t>(H) * ldkh;
    lay.c_nlb = coff;
    for (int i = 0; i < H; ++i) e->live_flat.push_back(e->off_nlb + i);
    coff += H;
    pad4();  // out_w^T rows are read 16 bytes at a time
    lay.c_outw = coff;
    for (int o = 0; o < O; ++o)
        for (int k = 0; k < ldkh; ++k) e->live_flat.push_back(k < H ? e->off_outw + static_cast<int64_t>(k) * O + o : -1);
    coff += static_cast<int64_t>(O) * ldkh;
    lay.c_outb = coff;
    for (int i = 0; i < O; ++i) e->live_flat.push_back(e->off_outb + i);
    coff += O;
    pad4();
    lay.P_pad = coff;
    lay.P_live = 0;
    for (int64_t f : e->live_flat) lay.P_live += f >= 0 ? 1 : 0;

    // row store of one window (K2 -> K3): x | h_l | z | pre_bar_l | z_bar | pred_bar, plus 16
    // columns of tail slack for K3's fixed-width strip copies
    auto r4 = [](int x) { return (x + 3) & ~3; };
    int o = 0;
    lay.rs_x = o;
    o += r4(e->in0);
    for (int l = 0; l < lay.L; ++l) {
        lay.rs_h[l] = o;
        o += r4(H);
    }
    lay.rs_z = o;
    o += r4(H);
    for (int l = 0; l < lay.L; ++l) {
        lay.rs_pr[l] = o;
        o += r4(3 * H);
    }
    lay.rs_zb = o;
    o += r4(H);
    lay.rs_pb = o;
    o += r4(O);
    lay.rs_ld = o + 16;
    // K3 contraction matrices: the layers, then the head (nl_w, out_w)
    lay.nmat = lay.L + 2;
    for (int l = 0; l < lay.L; ++l)
        lay.mats[l] = MatDesc{lay.rs_pr[l], 3 * H, l == 0 ? lay.rs_x : lay.rs_h[l - 1], lay.layer_in[l], lay.ldk[l], 0,
                              lay.cw[l], lay.cb[l]};
    lay.mats[lay.L] = MatDesc{lay.rs_zb, H, lay.rs_h[lay.L - 1], H, lay.ldkh, 0, lay.c_nlw, lay.c_nlb};
    lay.mats[lay.L + 1] = MatDesc{lay.rs_pb, O, lay.rs_z, H, lay.ldkh, 0, lay.c_outw, lay.c_outb};
    lay.mat_blk0[0] = 0;
    lay.mat_wblk0[0] = 0;
    for (int m = 0; m < lay.nmat; ++m) {
        const MatDesc& d = lay.mats[m];
        lay.mat_blk0[m + 1] = lay.mat_blk0[m] + ((d.Q + kGq - 1) / kGq) * ((d.K + kGk - 1) / kGk);
        lay.mat_wblk0[m + 1] = lay.mat_wblk0[m] + (d.Q + kWq - 1) / kWq;
    }
    lay.wkp_in0 = (lay.layer_in[0] + 3) & ~3;
    lay.wkp_h = (H + 3) & ~3;
}

// ------------------------------------------------------------------ conversions
void to_real(Eng* e, const double* src, size_t n, void* host_tmp) {
    if (e->fp64) {
        std::memcpy(host_tmp, src, sizeof(double) * n);
    } else {
        float* f = static_cast<float*>(host_tmp);
        for (size_t i = 0; i < n; ++i) f[i] = static_cast<float>(src[i]);
    }
}
void from_real(Eng* e, const void* host_tmp, size_t n, double* dst) {
    if (e->fp64) {
        std::memcpy(dst, host_tmp, sizeof(double) * n);
    } else {
        const float* f = static_cast<const float*>(host_tmp);
        for (size_t i = 0; i < n; ++i) dst[i] = static_cast<double>(f[i]);
    }
}

void upload_real(Eng* e, void* dev, const double* src, size_t n) {
    std::vector<double> tmp(n);
    to_real(e, src, n, tmp.data());
    CUDA_OK(cudaMemcpyAsync(dev, tmp.data(), e->rsz * n, cudaMemcpyHostToDevice, e->stream));
    CUDA_OK(cudaStreamSynchronize(e->stream));
}
void download_real(Eng* e, const void* dev, size_t n, double* dst) {
    std::vector<double> tmp(n);
    CUDA_OK(cudaMemcpyAsync(tmp.data(), dev, e->rsz * n, cudaMemcpyDeviceToHost, e->stream));
    CUDA_OK(cudaStreamSynchronize(e->stream));
    from_real(e, tmp.data(), n, dst);
}

// stage = nullptr: synchronous (the caller's next use may follow at once); else the compact
// vector goes through the caller's pinned staging block with no synchronisation here
void upload_theta(Eng* e, PinnedBuf<double>* stage = nullptr) {
    std::vector<double> c(e->live_flat.size(), 0.0);
    for (size_t i = 0; i < c.size(); ++i)
        if (e->live_flat[i] >= 0) c[i] = e->w_host[e->live_flat[i]];
    if (!stage) {
        upload_real(e, e->theta.p, c.data(), c.size());
        return;
    }
    stage->reserve(std::max<size_t>(c.size(), 1));
    to_real(e, c.data(), c.size(), stage->p);
    CUDA_OK(cudaMemcpyAsync(e->theta.p, stage->p, e->rsz * c.size(), cudaMemcpyHostToDevice, e->stream));
}

void sync_weights_from_device(Eng* e) {
    std::vector<double> c(e->live_flat.size());
    download_real(e, e->theta.p, c.size(), c.data());
    for (size_t i = 0; i < c.size(); ++i)
        if (e->live_flat[i] >= 0) e->w_host[e->live_flat[i]] = c[i];
}

// ------------------------------------------------------------------ capacity
void encode_rowstore_maps(Eng* e, int rsz);  // defined with the kernel attributes below

void ensure_capacity(Eng* e, int B) {
    if (B <= e->Bcap) return;
    const int S = e->S, T = e->T, I = e->I, O = e->O;
    const size_t r = e->rsz;
    e->Bcap = B;
    // slot capacity = the scan-state row stride, a multiple of K3's slots per block so every
    // ES block stages whole 16-byte rows of its slots
    e->kcap = (std::min(e->N > 0 ? e->N : 1, B) + kEsSlotsPerBlock - 1) / kEsSlotsPerBlock * kEsSlotsPerBlock;
    const int kc = e->kcap;
    e->tiles_cap = (B + kRows - 1) / kRows;
    // fp32 ES blocks: 8 slots while that keeps them within four per SM (shorter per-block gather,
    // more blocks overlapping K2: cfg1 -8% step, cfg3 -5%); 16 for large steps (B = 48,000:
    // 8 slots measured 24.5 vs 20.7 ms per epoch)
    e->es_bd = e->fp64 ? kEsSlotsPerBlock : ((kc + 7) / 8 <= 4 * g_num_sms ? 8 : kEsSlots32);
    if (const char* v = std::getenv("ESRNN_ES_SLOTS"); v && !e->fp64 && (std::atoi(v) == 8 || std::atoi(v) == 16))
        e->es_bd = std::atoi(v);
    const int es_slots = e->es_bd;
    e->es_blocks = (kc + es_slots - 1) / es_slots;

    // tensor-core weight gradients (umma.cuh, finish.cuh dw_umma_block): fp32 steps of at
    // least kUmmaMinRows windows, every matrix's K + 1 within the 64-column N tile;
    // two blocks per SM over the matrices' 128-row tiles, parts of >= 256 rows
    e->umma_parts = 0;
    e->umma_tiles = 0;
    static const int umma_min = std::getenv("ESRNN_UMMA_MIN") ? std::atoi(std::getenv("ESRNN_UMMA_MIN")) : kUmmaMinRows;
    if (!e->fp64 && B >= umma_min && std::getenv("ESRNN_NO_UMMA") == nullptr &&
        static_cast<size_t>(g_smem_optin) >= static_cast<size_t>(kUSmem) + 1024) {
        bool fits = true;
        for (int m = 0; m < e->lay.nmat; ++m) {
            fits &= e->lay.mats[m].K + 1 <= kUN && e->lay.mats[m].a_off % 4 == 0 && e->lay.mats[m].u_off % 4 == 0;
            e->umma_tiles += (e->lay.mats[m].Q + kUM - 1) / kUM;
        }
        if (fits && e->lay.rs_ld % 4 == 0) {
            // one wave at two blocks per SM (kUSmem ~85 KB)
            e->umma_parts = std::max(1, std::min(std::min(64, 2 * g_num_sms / e->umma_tiles), B / 256));
            e->upart.alloc(sizeof(float) * static_cast<size_t>(e->umma_tiles) * e->umma_parts * kUM * kUN);
        } else {
            e->umma_tiles = 0;
        }
    }
    // weight-gradient contraction without the tensor cores: the 16 x 8 output tiles.  The
    // q-strip blocks (finish.cuh dw_wide_block: each row-store row read once per 32 rows of G,
    // parts combined in order by the last to arrive) are opt-in, ESRNN_GEMM_WIDE=1: measured
    // slower (cfg1 1.60 -> 2.70 ms, cfg3 52.7 -> 66.7 ms per epoch + validate; the last part's
    // combine serialises its loads behind its stores, and a part's publish + ticket costs more
    // than the re-reads it saves at these row counts)
    e->wide = false;
    if (!e->fp64 && e->umma_parts == 0 && std::max(e->lay.wkp_in0, e->lay.wkp_h) <= kWkMax) {
        const char* v = std::getenv("ESRNN_GEMM_WIDE");
        e->wide = v && std::atoi(v) == 1;
    }
    e->red_blocks = e->wide ? e->lay.mat_wblk0[e->lay.nmat] : e->lay.mat_blk0[e->lay.nmat];
    if (e->wide) {
        e->gsplit = std::max(1, std::min(8, B / 128));
        e->gpart.alloc(e->rsz * static_cast<size_t>(e->gsplit) * std::max(e->red_blocks, 1) * kWq * (kWkMax + 1));
    } else {
        // Row parts per 16 x 8 tile: at B <= 4,096 one block per tile is fastest (a two-part
        // split measured +6.8 us at cfg1); beyond, one part per 4,096 rows (<= 16)
        e->gsplit = std::max(1, std::min(16, B / 4096));
        e->gpart.alloc(e->rsz * static_cast<size_t>(e->gsplit) * std::max(e->red_blocks, 1) * 32 * 6);
    }
    const int ctr_n = std::max({e->red_blocks, e->umma_tiles, 1});
    if (e->gtile_ctr.n < static_cast<size_t>(ctr_n)) {
        e->gtile_ctr.alloc(ctr_n);
        e->gtile_ctr.zero(e->stream);
    }
    e->lv.alloc(r * T * kc);
    e->se.alloc(r * (T + S) * kc);
    e->contrib.alloc(sizeof(double) * static_cast<size_t>(B) * ((I + O + 2 + 3) & ~3));
    // row store: K2 writes every column of a live window's row; rows are read only by K3
    // (+ 256 columns: the tensor-core path reads whole 128-row / 64-column operand quads
    // past the last matrix of the last row)
    e->rowstore.alloc(r * (static_cast<size_t>(e->tiles_cap * kRows) * e->lay.rs_ld + 256));
    encode_rowstore_maps(e, static_cast<int>(r));
    e->loss_part.alloc(e->tiles_cap);
    e->psg.alloc(r * static_cast<size_t>(kc) * (2 + S));
    e->es_sq_part.alloc(e->es_blocks);
    e->es_pen_part.alloc(e->es_blocks);
    e->d_inputs.alloc(r * static_cast<size_t>(B) * e->in0);
    e->d_targets.alloc(r * static_cast<size_t>(B) * O);
    e->d_seas.alloc(r * static_cast<size_t>(B) * O);
    e->d_levels.alloc(r * B);
}

// Adam bias corrections {1 - 0.9^t, 1 - 0.999^t} (trainer.hpp:617-620, :640-641) with the
// host's std::pow, like the reference.  From t = kBcSteps on both are exactly 1.0 in double
// (0.999^t < 2^-53 past t ~ 37,000), so one process-wide device table per GPU of kBcSteps
// entries serves every trainer (kernels read 1.0 beyond it).
const double* bc_table(int device) {
    static std::mutex mu;
    static std::map<int, double*> tabs;
    std::lock_guard<std::mutex> lock(mu);
    auto it = tabs.find(device);
    if (it != tabs.end()) return it->second;
    std::vector<double> h(2 * static_cast<size_t>(kBcSteps));
    for (int64_t t = 0; t < kBcSteps; ++t) {
        h[2 * t] = 1.0 - std::pow(0.9, static_cast<double>(t));
        h[2 * t + 1] = 1.0 - std::pow(0.999, static_cast<double>(t));
    }
    double* d = nullptr;
    CUDA_OK(cudaMalloc(&d, sizeof(double) * h.size()));
    CUDA_OK(cudaMemcpy(d, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
    tabs[device] = d;
    return d;
}

// ------------------------------------------------------------------ plans
// trainer.hpp:493-501: slots in first-appearance order; per slot its windows in batch order.
// src(i) -> {global row, anchor} of the batch's i-th window
template <typename Src>
void append_step(Eng* e, HostPlan& hp, const Src& src, int B, std::vector<int64_t>& stamp, std::vector<int>& slot_id,
                 int64_t step) {
    const int wbase = static_cast<int>(hp.w_row.size());
    const int sbase = static_cast<int>(hp.slot_row.size());
    const int cbase = static_cast<int>(hp.slot_win.size());
    const int row0 = e->row0, N = e->N;
    // this rank's windows of the batch, slots in first-appearance order
    hp.w_row.resize(wbase + B);
    hp.w_anchor.resize(wbase + B);
    hp.w_slot.resize(wbase + B);
    hp.w_first.resize(wbase + B);
    hp.slot_row.resize(sbase + B);
    int* __restrict__ wrow = hp.w_row.data() + wbase;
    int* __restrict__ wanc = hp.w_anchor.data() + wbase;
    int* __restrict__ wslot = hp.w_slot.data() + wbase;
    int* __restrict__ wfirst = hp.w_first.data() + wbase;
    int* __restrict__ srow = hp.slot_row.data() + sbase;
    int64_t* __restrict__ stp = stamp.data();
    int* __restrict__ sid = slot_id.data();
    int nw = 0, ns = 0;
    for (int i = 0; i < B; ++i) {
        const std::pair<int, int> ra = src(i);
        const int r = ra.first - row0;
        if (r < 0 || r >= N) continue;
        const bool first = stp[r] != step;
        if (first) {
            stp[r] = step;
            sid[r] = ns;
            srow[ns++] = r;
        }
        wfirst[nw] = first ? 1 : 0;
        wrow[nw] = r;
        wanc[nw] = ra.second;
        wslot[nw] = sid[r];
        ++nw;
    }
    hp.w_row.resize(wbase + nw);
    hp.w_anchor.resize(wbase + nw);
    hp.w_slot.resize(wbase + nw);
    hp.w_first.resize(wbase + nw);
    hp.slot_row.resize(sbase + ns);
    // CSR: count, prefix, fill in batch order
    static thread_local std::vector<int> cnt;
    cnt.assign(ns + 1, 0);
    int* __restrict__ c = cnt.data();
    for (int i = 0; i < nw; ++i) c[wslot[i] + 1]++;
    for (int k = 0; k < ns; ++k) c[k + 1] += c[k];
    hp.slot_win.resize(cbase + nw);
    hp.w_csr.resize(wbase + nw);
    hp.csr_anchor.resize(cbase + nw);
    hp.slot_win_off.resize(hp.slot_win_off.size() + ns);
    int* __restrict__ soff = hp.slot_win_off.data() + (hp.slot_win_off.size() - ns);
    for (int k = 0; k < ns; ++k) soff[k] = cbase + c[k + 1];
    // slot-major CSR position of each window (K2 writes its ES contributions there) and the
    // anchor of each CSR entry (K3 reads a slot's windows contiguously)
    int* __restrict__ swin = hp.slot_win.data() + cbase;
    int* __restrict__ wcsr = hp.w_csr.data() + wbase;
    int* __restrict__ canc = hp.csr_anchor.data() + cbase;
    for (int i = 0; i < nw; ++i) {
        const int pos = c[wslot[i]]++;
        swin[pos] = i;
        wcsr[i] = pos;
        canc[pos] = wanc[i];
    }
    hp.step_win_off.push_back(wbase + nw);
    hp.step_slot_off.push_back(sbase + ns);
    hp.max_step_windows = std::max(hp.max_step_windows, nw);
    hp.max_step_slots = std::max(hp.max_step_slots, ns);
}

void plan_begin(HostPlan& hp, size_t windows = 0, int steps = 0) {
    for (auto* v : {&hp.w_row, &hp.w_anchor, &hp.w_slot, &hp.w_first, &hp.w_csr, &hp.csr_anchor, &hp.slot_row,
                    &hp.slot_win}) {
        v->clear();
        v->reserve(windows);
    }
    hp.slot_win_off.assign(1, 0);
    hp.slot_win_off.reserve(windows + 1);
    hp.step_win_off.assign(1, 0);
    hp.step_win_off.reserve(steps + 1);
    hp.step_slot_off.assign(1, 0);
    hp.step_slot_off.reserve(steps + 1);
    hp.step_M.clear();
    hp.step_M.reserve(steps);
    hp.max_step_windows = hp.max_step_slots = 0;
}

template <typename T>
void upload_vec(Eng* e, DBuf<T>& d, const std::vector<T>& h, size_t cap) {
    if (d.n < std::max<size_t>(cap, 1)) d.alloc(std::max<size_t>(cap, 1));
    if (!h.empty()) CUDA_OK(cudaMemcpyAsync(d.p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, e->stream));
}

void upload_plan(Eng* e, const HostPlan& hp, DevPlan& dp, size_t cap_w, size_t cap_steps) {
    const size_t cw = std::max(cap_w, hp.w_row.size());
    const size_t cs = std::max(cap_steps, hp.step_M.size());
    upload_vec(e, dp.w_row, hp.w_row, cw);
    upload_vec(e, dp.w_anchor, hp.w_anchor, cw);
    upload_vec(e, dp.w_slot, hp.w_slot, cw);
    upload_vec(e, dp.w_first, hp.w_first, cw);
    upload_vec(e, dp.w_csr, hp.w_csr, cw);
    upload_vec(e, dp.csr_anchor, hp.csr_anchor, cw);
    upload_vec(e, dp.slot_row, hp.slot_row, cw);
    upload_vec(e, dp.slot_win, hp.slot_win, cw);
    upload_vec(e, dp.slot_win_off, hp.slot_win_off, cw + 1);
    upload_vec(e, dp.step_win_off, hp.step_win_off, cs + 1);
    upload_vec(e, dp.step_slot_off, hp.step_slot_off, cs + 1);
    upload_vec(e, dp.step_M, hp.step_M, cs);
}

// ------------------------------------------------------------------ step launch
template <typename Real>
size_t stack_smem(const NetLayout& lay, bool resident) {
    return sizeof(Real) * TileSmem::make<Real>(lay, resident).total;
}
// two tiles per CTA sharing the resident weights (k_tile<..., NG = 2>)
template <typename Real>
size_t stack_smem2(const NetLayout& lay) {
    const TileSmem t = TileSmem::make<Real>(lay, true);
    return sizeof(Real) * (static_cast<size_t>(t.total) + (t.total - t.wsize));
}

// Resident mode keeps every live weight in shared memory for the whole tile (one TMA
// bulk copy); larger fp64 networks stage one layer at a time.
int g_smem_optin = 227 * 1024;  // cudaDevAttrMaxSharedMemoryPerBlockOptin, set at create
int g_num_sms = 148;             // cudaDevAttrMultiProcessorCount, set at create
int g_smem_per_sm = 228 * 1024;  // cudaDevAttrMaxSharedMemoryPerMultiprocessor, set at create

template <typename Real>
bool stack_resident(const NetLayout& lay) {
    return stack_smem<Real>(lay, true) + 4096 <= static_cast<size_t>(g_smem_optin);
}

int stack_threads(const NetLayout& lay) { return tile_threads(lay); }

template <typename Real>
size_t finish_smem(const NetLayout& lay, int ring = kGBuf, int es_bd = kEsSlots32, bool wide = false) {
    // ES blocks: level / seasonality adjoints [bd][T|1], [bd][(T+S)|1], forward l and s
    // columns [T][bd] (double), one staged observation row per slot (Real), one chunk of
    // staged contribution rows (double)
    if (sizeof(Real) == 4) {
        // es_block_fp32 (finish.cuh): adjoints [bd][T|1], [bd][(T+S)|1] (double), six [T][bd]
        // coefficient arrays, then a scratch region: pre-wait observation rows + forward
        // states + raw parameters, post-wait one chunk of staged contribution rows
        const size_t bd = es_bd, T = lay.T, S = lay.S;
        const size_t ldl = T | 1, lds = (T + S) | 1;
        const size_t cr = S == 1 ? sizeof(double) : sizeof(float);
        const size_t cwp = (lay.I + lay.O + 2 + 3) & ~3;
        const size_t scratch = std::max(bd * row_pad<Real>(lay.T) * sizeof(Real) + bd * (ldl + lds) * cr +
                                            bd * (2 + S) * sizeof(Real),
                                        sizeof(double) * kEsChunk * cwp);
        const size_t es = sizeof(double) * bd * (ldl + lds) + 6 * T * bd * cr + sizeof(double) * bd * S + scratch;
        const size_t gemm = sizeof(Real) * (static_cast<size_t>(ring * kGChunk) * (kGq + kGk) + (kFinishThreads / 32) * 32 * 6);
        const size_t wgemm = sizeof(float) * ring * kWr * static_cast<size_t>(kWq + std::max(lay.wkp_in0, lay.wkp_h));
        return std::max(es, wide ? wgemm : gemm);
    }
    const size_t cwp = (lay.I + lay.O + 2 + 3) & ~3;
    const size_t bd = kEsSlotsPerBlock;
    const size_t es = sizeof(double) * bd * (static_cast<size_t>(lay.T | 1) + static_cast<size_t>((lay.T + lay.S) | 1)) +
                      (sizeof(Real) == 4 && lay.S == 1 ? sizeof(double) : sizeof(Real)) * bd * 2 * static_cast<size_t>(lay.T) +
                      sizeof(Real) * bd * row_pad<Real>(lay.T) +
                      std::max(sizeof(double) * kEsChunk * cwp,  // staged contributions, then (fp32)
                               sizeof(Real) == 4 ? (lay.S == 1 ? sizeof(double) : sizeof(float)) * 4 * bd *
                                                       static_cast<size_t>(lay.T)
                                                 : 0);  // the scan's coefficients (finish.cuh)
    const size_t gemm = sizeof(Real) * (static_cast<size_t>(ring * kGChunk) * (kGq + kGk) + (kFinishThreads / 32) * 32 * 6);
    return std::max(es, gemm);
}

// K3's launch smem: the tensor-core weight-gradient blocks need kUSmem (+ 1 KB alignment)
template <typename Real>
size_t finish_smem_launch(const NetLayout& lay, bool umma) {
    const size_t f = finish_smem<Real>(lay);
    return umma ? std::max(f, static_cast<size_t>(kUSmem) + 1024) : f;
}

// K3's GEMM staging tensor maps (finish.cuh): the row store as a 2-D [rows][rs_ld] tensor of
// Real, boxes of kGChunk rows x kGq (A) / kGk (U) columns, no swizzle, zero fill past the end.
using TensorMapEncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                       const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                       CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
void encode_rowstore_maps(Eng* e, int rsz) {
    static TensorMapEncodeFn enc = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        CUDA_OK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !fn) raise(ESRNN_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<TensorMapEncodeFn>(fn);
    }();
    alignas(64) CUtensorMap maps[5];  // 16 x 8 tiles: A, U; q-strips: A, U (in0), U (H)
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(e->lay.rs_ld), static_cast<cuuint64_t>(e->tiles_cap) * kRows};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(e->lay.rs_ld) * rsz};
    const cuuint32_t estr[2] = {1, 1};
    const CUtensorMapDataType dt = rsz == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
    for (int i = 0; i < 5; ++i) {
        const int bx = i == 0 ? kGq : i == 1 ? kGk : i == 2 ? kWq : i == 3 ? e->lay.wkp_in0 : e->lay.wkp_h;
        const cuuint32_t box[2] = {static_cast<cuuint32_t>(std::min(bx, 256)),
                                   static_cast<cuuint32_t>(i < 2 ? kGChunk : kWr)};
        const CUresult r = enc(&maps[i], dt, 2, e->rowstore.p, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) raise(ESRNN_CUDA_ERROR, "row-store tensor map encoding failed (%d)", static_cast<int>(r));
    }
    e->tm_rs.alloc(sizeof maps);
    CUDA_OK(cudaMemcpyAsync(e->tm_rs.p, maps, sizeof maps, cudaMemcpyHostToDevice, e->stream));
    CUDA_OK(cudaStreamSynchronize(e->stream));  // `maps` is a stack buffer
}

// Every kernel of the step prefers the maximum shared-memory carveout.  Under programmatic
// dependent launch the next kernel's CTAs are placed on SMs still running the previous
// kernel's blocks; an SM configured for a small-smem kernel (K4, 1 KB) cannot take a K2
// tile (133 KB at cfg1) until it drains and reconfigures, so those tiles launched late and
// passed their dependency wait up to 2.4 us after the first (ESRNN_NO_CARVEOUT=1 restores
// the driver's default choice).
template <typename K>
void max_carveout(K* kern) {
    static const bool off = std::getenv("ESRNN_NO_CARVEOUT") != nullptr;
    if (!off) CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
}

// The tile kernel's scans are specialised for the M4 seasonalities (S = 1, 4, 12: seasonal
// ring in registers); any other S runs the generic variant.
template <typename Real, int MODE, int SC>
void set_tile_attr(const NetLayout& lay) {
    if (stack_resident<Real>(lay)) {
        CUDA_OK(cudaFuncSetAttribute(k_tile<Real, MODE, true, SC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)stack_smem<Real>(lay, true)));
        max_carveout(k_tile<Real, MODE, true, SC>);
    }
    CUDA_OK(cudaFuncSetAttribute(k_tile<Real, MODE, false, SC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)stack_smem<Real>(lay, false)));
    max_carveout(k_tile<Real, MODE, false, SC>);
    if constexpr (sizeof(Real) == 4 && MODE != kForecast) {
        if (stack_resident<Real>(lay) && stack_smem2<Real>(lay) + 1024 <= static_cast<size_t>(g_smem_optin)) {
            CUDA_OK(cudaFuncSetAttribute(k_tile<Real, MODE, true, SC, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)stack_smem2<Real>(lay)));
            max_carveout(k_tile<Real, MODE, true, SC, 2>);
        }
    }
}

template <typename Real, int SC>
void set_sc_attrs(const NetLayout& lay) {
    set_tile_attr<Real, kTrain, SC>(lay);
    set_tile_attr<Real, kLossOnly, SC>(lay);
    CUDA_OK(cudaFuncSetAttribute(k_grad_finish<Real, SC, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)finish_smem<Real>(lay)));
    max_carveout(k_grad_finish<Real, SC, false>);
    if (sizeof(Real) == 4) {
        CUDA_OK(cudaFuncSetAttribute(k_grad_finish<Real, SC, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)finish_smem_launch<Real>(lay, true)));
        max_carveout(k_grad_finish<Real, SC, true>);
    }
}

template <typename Real>
void setup_kernel_attrs(Eng* e) {
    set_tile_attr<Real, kForecast, 0>(e->lay);
    max_carveout(k_adam<Real>);
    max_carveout(k_finalize<Real>);
    max_carveout(k_group_reduce<Real>);
    switch (e->S) {
        case 1: set_sc_attrs<Real, 1>(e->lay); break;
        case 4: set_sc_attrs<Real, 4>(e->lay); break;
        case 12: set_sc_attrs<Real, 12>(e->lay); break;
        default: set_sc_attrs<Real, 0>(e->lay); break;
    }
    const size_t fsm = sizeof(Real) * static_cast<size_t>(e->LEN + e->S + e->I) * kScanThreads;
    CUDA_OK(cudaFuncSetAttribute(k_forecast_scan<Real, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm));
    const size_t fsm_sc = fsm + sizeof(Real) * static_cast<size_t>(e->in0 + e->O + 1) * kScanThreads;
    CUDA_OK(cudaFuncSetAttribute(k_forecast_scan_sc<Real, 1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm_sc));
    CUDA_OK(cudaFuncSetAttribute(k_forecast_scan_sc<Real, 4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm_sc));
    CUDA_OK(cudaFuncSetAttribute(k_forecast_scan_sc<Real, 12, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm_sc));
    CUDA_OK(cudaFuncSetAttribute(k_forecast_scan_sc<Real, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm_sc));
    CUDA_OK(cudaFuncSetAttribute(k_forecast_scan_sc<Real, 4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm_sc));
    CUDA_OK(cudaFuncSetAttribute(k_forecast_scan_sc<Real, 12, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm_sc));
    if (stack_smem<Real>(e->lay, false) > static_cast<size_t>(g_smem_optin) ||
        finish_smem<Real>(e->lay) > static_cast<size_t>(g_smem_optin) || fsm_sc > static_cast<size_t>(g_smem_optin))
        raise(ESRNN_CONFIG_ERROR, "profile too large for the B200 kernels' shared-memory tiles");
}

// Kernel launch on the engine stream; with `pdl`, programmatic stream serialisation lets
// the kernel launch while its predecessor drains (common.cuh pdl_trigger / pdl_wait).
template <typename... KArgs, typename... Args>
void launch_k(Eng* e, bool pdl, void (*kern)(KArgs...), int grid, int block, size_t smem, Args&&... args) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(block);
    lc.dynamicSmemBytes = smem;
    lc.stream = e->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = (pdl && e->pdl && !e->profiling) ? 1 : 0;
    CUDA_OK(cudaLaunchKernelEx(&lc, kern, std::forward<Args>(args)...));
}

// K3's GEMM staging ring: 3 buffers (2 chunks in flight) while the grid fits one wave at two
// blocks per SM; beyond that 2 buffers, so the smaller blocks fit four per SM and the GEMM blocks
// are not queued behind the ES blocks (measured: cfg1 ring 3 0.63M vs ring 2 0.57M series/s;
// cfg3 ring 2 52.3 vs ring 3 55.3 ms per epoch + validate)
int finish_ring(const Eng* e, int blocks) {
    static const int forced = std::getenv("ESRNN_GEMM_RING") ? std::atoi(std::getenv("ESRNN_GEMM_RING")) : 0;
    if (forced == 2 || forced == 3) return forced;
    return blocks > 2 * g_num_sms ? 2 : 3;
}

template <typename Real, int SC>
void launch_finish_sc(Eng* e, const StateDev<Real>& st, const PlanDev& pv, int s, int finalize, bool pdl) {
    const int gemm_blocks = e->umma_parts > 0 ? e->umma_tiles * e->umma_parts : e->red_blocks * e->gsplit;
    const int ring = finish_ring(e, e->es_blocks + gemm_blocks);
    const int bd = e->es_bd;
    if (e->umma_parts > 0)
        launch_k(e, pdl, k_grad_finish<Real, SC, true>, e->es_blocks + gemm_blocks, kFinishThreads,
                 finish_smem_launch<Real>(e->lay, true), st, pv, e->lay, s, e->es_blocks, finalize, e->gsplit,
                 e->umma_parts, 3, bd);
    else
        launch_k(e, pdl, k_grad_finish<Real, SC, false>, e->es_blocks + gemm_blocks, kFinishThreads,
                 finish_smem<Real>(e->lay, ring, bd, e->wide), st, pv, e->lay, s, e->es_blocks, finalize, e->gsplit, 0,
                 ring, bd);
}
template <typename Real>
void launch_finish(Eng* e, const StateDev<Real>& st, const PlanDev& pv, int s, int finalize, bool pdl = false) {
    switch (e->S) {
        case 1: launch_finish_sc<Real, 1>(e, st, pv, s, finalize, pdl); break;
        case 4: launch_finish_sc<Real, 4>(e, st, pv, s, finalize, pdl); break;
        case 12: launch_finish_sc<Real, 12>(e, st, pv, s, finalize, pdl); break;
        default: launch_finish_sc<Real, 0>(e, st, pv, s, finalize, pdl); break;
    }
}

template <typename Real, int MODE, int SC>
void launch_tile_sc(Eng* e, int grid, const StateDev<Real>& st, const PlanDev& pv, int s, const ForecastArgs& fa,
                    bool pdl) {
    const NetLayout& lay = e->lay;
    const int nt = stack_threads(lay);
    // Resident weights (one TMA copy, one CTA per SM) win while the grid is about one wave;
    // from two waves on, per-layer staging lets two fp32 CTAs share an SM and hide each
    // other's phase latencies (measured: B=4,096 tile -15%, B=48,000 -18%; cfg1 +40%).
    static const int stage_min = std::getenv("ESRNN_TILE_STAGED_MIN") ? std::atoi(std::getenv("ESRNN_TILE_STAGED_MIN"))
                                                                       : 2 * g_num_sms;
    const bool two_waves = sizeof(Real) == 4 && grid >= stage_min &&
                           2 * (stack_smem<Real>(lay, false) + 1024) <= static_cast<size_t>(g_smem_per_sm);
    if constexpr (sizeof(Real) == 4 && MODE != kForecast) {
        // more than one wave at one resident tile per SM: two tiles per CTA on one weight copy
        // when they fit (ESRNN_TILE_G2=0 disables)
        const char* g2v = std::getenv("ESRNN_TILE_G2");  // read per launch (graph capture / eager steps)
        const bool g2_off = g2v && std::atoi(g2v) == 0;
        // only where two one-tile CTAs cannot share an SM (Yearly's can: there NG = 2 measured
        // 0.94 -> 1.05 ms per cfg2 epoch)
        const bool two_ctas_fit = 2 * (stack_smem<Real>(lay, true) + 1024) <= static_cast<size_t>(g_smem_per_sm) &&
                                  2 * nt * 128 <= 65536;
        if (!g2_off && !two_ctas_fit && stack_resident<Real>(lay) && grid > g_num_sms && 2 * nt <= 768 &&
            stack_smem2<Real>(lay) + 1024 <= static_cast<size_t>(g_smem_optin)) {
            launch_k(e, pdl, k_tile<Real, MODE, true, SC, 2>, (grid + 1) / 2, 2 * nt, stack_smem2<Real>(lay), st, pv,
                     lay, s, fa);
            return;
        }
    }
    if (stack_resident<Real>(lay) && !two_waves)
        launch_k(e, pdl, k_tile<Real, MODE, true, SC>, grid, nt, stack_smem<Real>(lay, true), st, pv, lay, s, fa);
    else
        launch_k(e, pdl, k_tile<Real, MODE, false, SC>, grid, sizeof(Real) == 4 ? std::min(nt, 384) : nt,
                 stack_smem<Real>(lay, false), st, pv, lay, s, fa);
}
template <typename Real, int MODE>
void launch_stack(Eng* e, int grid, const StateDev<Real>& st, const PlanDev& pv, int s, const ForecastArgs& fa,
                  bool pdl = false) {
    if (MODE == kForecast) {
        launch_tile_sc<Real, kForecast, 0>(e, grid, st, pv, s, fa, false);
        return;
    }
    switch (e->S) {
        case 1: launch_tile_sc<Real, MODE, 1>(e, grid, st, pv, s, fa, pdl); break;
        case 4: launch_tile_sc<Real, MODE, 4>(e, grid, st, pv, s, fa, pdl); break;
        case 12: launch_tile_sc<Real, MODE, 12>(e, grid, st, pv, s, fa, pdl); break;
        default: launch_tile_sc<Real, MODE, 0>(e, grid, st, pv, s, fa, pdl); break;
    }
}

// Launch one training step (K1..K5) for step `s` of plan `pv` on the engine stream.
template <typename Real>
void launch_step(Eng* e, const PlanDev& pv, int s, bool grads, bool update, StateDev<Real> st) {
    const NetLayout& lay = e->lay;
    const int kc = e->kcap;
    using KS = Eng::KScope;
    ForecastArgs fa{};
    {
        KS k(e, 1);
        if (grads)
        {
            // ESRNN_DEBUG_TWICE: re-run the (idempotent) tile kernel so the stamps show a
            // warm instruction cache
            if (e->dbg_clk.p && std::getenv("ESRNN_DEBUG_TWICE")) launch_stack<Real, kTrain>(e, e->tiles_cap, st, pv, s, fa);
            launch_stack<Real, kTrain>(e, e->tiles_cap, st, pv, s, fa, s > 0);
        }
        else
            launch_stack<Real, kLossOnly>(e, e->tiles_cap, st, pv, s, fa);
    }
    e->launches += 1;
    if (!grads) return;
    const bool sharded = e->sharded;
    {
        KS k(e, 2);
        // bit 0: a last CTA finalises the step scalars (single GPU, no update: K4 does not
        // run); bit 1: the step applies updates; bit 2: single GPU updating step -- K4
        // derives the scalars and K3 only advances Adam's step
        const int fin = sharded ? (update ? 2 : 0) : (update ? 2 | 4 : 1);
        launch_finish<Real>(e, st, pv, s, fin, true);
    }
    e->launches += 1;
    if (sharded && e->group) {
        // in-process group: one fused kernel -- exchange, rank-ordered sum, finalise
        KS k(e, 5);
        GroupDev gd{e->group->slots, e->group->done, e->group->ctr, e->group->stride, e->world, e->rank};
        launch_k(e, false, k_group_reduce<Real>, e->group_ctas, 256, 0, st, pv, lay, s, update ? 1 : 0, gd);
        e->launches += 1;
    } else if (sharded) {
        // NCCL: the gradients (Real) and the step tail (double: per-series squared norm, loss,
        // error flag) in one group call, then the finalisation
        NCCL_OK(ncclGroupStart());
        NCCL_OK(ncclAllReduce(st.gbuf, st.gbuf, lay.P_pad, e->fp64 ? ncclDouble : ncclFloat, ncclSum, e->comm,
                              e->stream));
        NCCL_OK(ncclAllReduce(st.gtail, st.gtail, 4, ncclDouble, ncclSum, e->comm, e->stream));
        NCCL_OK(ncclGroupEnd());
        KS k(e, 5);
        const int rb = static_cast<int>((lay.P_pad + 255) / 256);
        k_finalize<Real><<<rb, 256, 0, e->stream>>>(st, pv, lay, s, update ? 1 : 0);
        e->launches += 1;
    }
    if (update) {
        KS k(e, 4);
        // K4 waits for K3 the ordinary way: launched early under PDL its CTAs measured slower
        // (cfg1 +6%), while the next tile's early launch after K4 (and K3's after K2) pays
        const int net_blocks = static_cast<int>((lay.P_pad + 255) / 256);
        const int spb = 256 / (2 + e->S);  // slots per per-series block (a thread per parameter)
        const int slot_blocks = (kc + spb - 1) / spb;
        static const bool k4_pdl = std::getenv("ESRNN_K4_PDL") != nullptr;
        launch_k(e, k4_pdl, k_adam<Real>, net_blocks + slot_blocks, 256, 0, st, pv, lay, s,
                 sharded ? -1 : e->es_blocks, e->red_blocks, net_blocks);
        e->launches += 1;
    }
}

// Creation-time zeroing of the state buffers in one launch (instead of a cudaMemsetAsync
// each) plus the error word reset.  blockIdx.y = span; spans start 4096-aligned (block cache).
struct ZeroSpans {
    static constexpr int kMax = 12;
    unsigned char* p[kMax];
    unsigned long long n[kMax];
    int count;
    int* errw;
};
__global__ void k_zero_spans(ZeroSpans z) {
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
        z.errw[0] = 0;
        z.errw[1] = INT_MAX;
        z.errw[2] = 0;
        z.errw[3] = 0;
    }
    const int k = blockIdx.y;
    if (k >= z.count) return;
    unsigned char* p = z.p[k];
    const unsigned long long n = z.n[k], n16 = n / 16;
    for (unsigned long long i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += gridDim.x * blockDim.x)
        reinterpret_cast<uint4*>(p)[i] = make_uint4(0, 0, 0, 0);
    if (blockIdx.x == 0 && threadIdx.x < n - n16 * 16) p[n16 * 16 + threadIdx.x] = 0;
}

template <typename Real>
void alloc_state(Eng* e) {
    const int N = e->N, S = e->S, LEN = e->LEN;
    const size_t r = sizeof(Real);
    e->vals.alloc(r * static_cast<size_t>(LEN) * std::max(N, 1));
    e->ldv = (LEN + 3) & ~3;
    e->vrm.alloc(r * static_cast<size_t>(e->ldv) * std::max(N, 1));
    e->ps.alloc(r * static_cast<size_t>(2 + S) * std::max(N, 1));
    e->ps_m.alloc(r * static_cast<size_t>(2 + S) * std::max(N, 1));
    e->ps_v.alloc(r * static_cast<size_t>(2 + S) * std::max(N, 1));
    e->ps_steps.alloc(std::max(N, 1));
    e->cat.alloc(std::max(N, 1));
    e->theta.alloc(r * e->lay.P_pad);
    e->mW.alloc(r * e->lay.P_pad);
    e->vW.alloc(r * e->lay.P_pad);
    e->gbuf.alloc(r * e->lay.P_pad);  // zeroed below: padding slots of the compact vector are never written
    e->gtail.alloc(4);
    e->coll_seq.alloc(1);
    e->red_blocks = e->lay.mat_blk0[e->lay.nmat];
    e->red_sq_part.alloc(std::max<int>(std::max(e->red_blocks, 16), static_cast<int>((e->lay.P_pad + 255) / 256)));
    e->scal.alloc(4);
    e->group_ctas = static_cast<int>(std::min<int64_t>(16, std::max<int64_t>(1, (e->lay.P_pad + 2047) / 2048)));
    {
        // one loss slot per training step of an epoch (make_batches, trainer.hpp:82-102)
        const int64_t nw = static_cast<int64_t>(e->N_global) * std::max(0, e->T - e->O - e->I + 1);
        const int B = std::max(1, e->cfg.batch_size);
        e->steps_cap = static_cast<int>(std::max<int64_t>(1, (nw + B - 1) / B));
        e->loss_hist.alloc(e->steps_cap);
    }
    e->done_ctr.alloc(2);
    e->net_step.alloc(1);
    e->errw.alloc(4);
    if (std::getenv("ESRNN_DEBUG_CLOCKS")) {
        e->dbg_clk.alloc(128 + 3 * kDbgTiles + 2 * kDbgK3);  // + per-tile step-5 spans of k_tile
        e->dbg_clk.zero(e->stream);
    }
    ZeroSpans z{};
    auto add = [&](void* p, size_t bytes) {
        z.p[z.count] = static_cast<unsigned char*>(p);
        z.n[z.count++] = bytes;
    };
    add(e->gbuf.p, e->gbuf.n);
    add(e->gtail.p, sizeof(double) * e->gtail.n);
    add(e->coll_seq.p, sizeof(long long) * e->coll_seq.n);
    for (auto* b : {&e->ps, &e->ps_m, &e->ps_v, &e->mW, &e->vW}) add(b->p, b->n);
    add(e->ps_steps.p, sizeof(int) * e->ps_steps.n);
    add(e->done_ctr.p, sizeof(unsigned int) * e->done_ctr.n);
    add(e->net_step.p, sizeof(long long) * e->net_step.n);
    z.errw = e->errw.p;
    k_zero_spans<<<dim3(32, z.count), 256, 0, e->stream>>>(z);
    e->launches += 1;
    CUDA_OK(cudaGetLastError());
    setup_kernel_attrs<Real>(e);
}

// Series values: the caller's row-major fp64 block goes to the device once; a layout kernel
// converts it to Real and writes both device copies (time-major vals, padded row-major vrm).
template <typename Real>
__global__ void k_layout_values(const double* __restrict__ raw, int N, int LEN, int ldv, Real* __restrict__ vals,
                                Real* __restrict__ vrm) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<long long>(N) * ldv) return;
    const int r = static_cast<int>(i / ldv), t = static_cast<int>(i - static_cast<long long>(r) * ldv);
    const Real v = t < LEN ? static_cast<Real>(raw[static_cast<size_t>(r) * LEN + t]) : Real(0);
    vrm[i] = v;
    if (t < LEN) vals[static_cast<size_t>(t) * N + r] = v;
}

template <typename Real>
void upload_values(Eng* e, const double* values, const int32_t* category) {
    const int N = e->N, LEN = e->LEN;
    if (N > 0) {
        // caller's (pageable) block -> pinned staging -> one async H2D; the staging buffers
        // live until create's final synchronisation (a helper-thread copy measured slower:
        // waking it costs more than the copy)
        DBuf<double>& raw = e->stage_raw;
        raw.alloc(static_cast<size_t>(N) * LEN);
        const double* src = values + static_cast<size_t>(e->row0) * LEN;
        // a pinned source (esrnn_ingest_m4_csv's dataset block) is copied from directly
        cudaPointerAttributes pa{};
        const bool pinned = cudaPointerGetAttributes(&pa, src) == cudaSuccess && pa.type == cudaMemoryTypeHost;
        cudaGetLastError();
        if (!pinned) {
            e->stage_pin.reserve(raw.n);
            std::memcpy(e->stage_pin.p, src, sizeof(double) * raw.n);
            src = e->stage_pin.p;
        }
        CUDA_OK(cudaMemcpyAsync(raw.p, src, sizeof(double) * raw.n, cudaMemcpyHostToDevice, e->stream));
        const long long n = static_cast<long long>(N) * e->ldv;
        k_layout_values<Real><<<static_cast<int>((n + 255) / 256), 256, 0, e->stream>>>(
            raw.p, N, LEN, e->ldv, reinterpret_cast<Real*>(e->vals.p), reinterpret_cast<Real*>(e->vrm.p));
        e->launches += 1;
        CUDA_OK(cudaGetLastError());
        e->stage_cat.reserve(N);  // pinned: a pageable copy may synchronise the stream
        signed char* c = e->stage_cat.p;
        e->cat_host.assign(N, 5);
        for (int r = 0; r < N; ++r) {
            const int v = category ? category[e->row0 + r] : -1;
            c[r] = static_cast<signed char>(v >= 0 && v < 6 ? v : 5);
            e->cat_host[r] = c[r];
        }
        CUDA_OK(cudaMemcpyAsync(e->cat.p, c, N, cudaMemcpyHostToDevice, e->stream));
    }
}

// ------------------------------------------------------------------ epoch
// all_windows (trainer.hpp:214-223) + Rng::shuffle (matrix.hpp:203-205) in global order,
// cut into batches (make_batches, trainer.hpp:82-102) and planned per step.
void build_epoch_plan(Eng* e, EpochPlan& ep) {
    using clk = std::chrono::steady_clock;
    static const bool dbg_host = std::getenv("ESRNN_DEBUG_HOST") != nullptr;
    const auto p0 = clk::now();
    const int I = e->I, O = e->O, T = e->T;
    const int per = T - O - I + 1;
    const int64_t nw = static_cast<int64_t>(e->N_global) * per;
    ep.rng_before = e->rng.gen;
    const int B = e->cfg.batch_size;
    const int steps = static_cast<int>((nw + B - 1) / B);
    ep.steps = steps;
    ep.n_windows = nw;
    // (row, anchor) pairs shuffled together (one random access per swap); Rng::shuffle's
    // draws (one per i = nw .. 2, Rng::below) generated as one block
    std::vector<uint64_t>& w = ep.wbuf;
    w.resize(nw);
    std::vector<uint64_t>& rnd = ep.rnd;
    rnd.resize(nw > 1 ? nw - 1 : 0);
    e->rng.gen.fill(rnd.data(), rnd.size());
    // Step-range chunks planned in parallel (each with its own dedupe stamps), pipelined
    // with the shuffle: Fisher-Yates from the top finalises positions nw-1, nw-2, ... in
    // turn, so task 0 shuffles and publishes `final_from` (positions >= it are final) while
    // the other tasks plan chunks from the last one down as their windows become final.
    const int workers = static_cast<int>(worker_pool().th.size()) + 1;
    const int nchunk = std::max(1, std::min(steps, 64));
    ep.chunks.resize(nchunk);
    const int64_t id0 = g_stamp_id.fetch_add(steps);
    auto chunk_range = [&](int c, int& s0, int& s1) {
        s0 = static_cast<int>(static_cast<int64_t>(steps) * c / nchunk);
        s1 = static_cast<int>(static_cast<int64_t>(steps) * (c + 1) / nchunk);
    };
    std::atomic<int64_t> final_from{nw};
    clk::time_point t_shuffled = p0;
    worker_pool().run(nchunk + 1, [&](int task) {
        if (task == 0) {
            uint64_t* __restrict__ x = w.data();
            int64_t n = 0;
            for (int r = 0; r < e->N_global; ++r)
                for (int a = I - 1; a <= T - O - 1; ++a) x[n++] = (static_cast<uint64_t>(r) << 32) | static_cast<uint32_t>(a);
            constexpr int64_t kPublish = 2048;
            for (int64_t i = nw; i > 1; --i) {
                const int64_t j = static_cast<int64_t>((static_cast<unsigned __int128>(rnd[nw - i]) * static_cast<uint64_t>(i)) >> 64);
                std::swap(x[i - 1], x[j]);
                if ((i & (kPublish - 1)) == 0) final_from.store(i - 1, std::memory_order_release);
            }
            final_from.store(0, std::memory_order_release);
            t_shuffled = clk::now();
            return;
        }
        const int c = nchunk - task;  // last chunk first
        int s0, s1;
        chunk_range(c, s0, s1);
        const int64_t need = static_cast<int64_t>(s0) * B;
        while (final_from.load(std::memory_order_acquire) > need) {
            if (workers > 2) {
#if defined(__x86_64__)
                for (int k = 0; k < 64; ++k) __builtin_ia32_pause();
#endif
            } else {
                std::this_thread::yield();
            }
        }
        HostPlan& hp = ep.chunks[c];
        const size_t wcap = static_cast<size_t>(std::min<int64_t>(nw, static_cast<int64_t>(s1 - s0) * B));
        plan_begin(hp, wcap, s1 - s0);
        static thread_local std::vector<int64_t> stamp;
        static thread_local std::vector<int> slot_id;
        if (stamp.size() < static_cast<size_t>(std::max(e->N, 1))) {
            stamp.assign(std::max(e->N, 1), -1);
            slot_id.assign(std::max(e->N, 1), 0);
        }
        const uint64_t* x = w.data();
        for (int s = s0; s < s1; ++s) {
            const int64_t start = static_cast<int64_t>(s) * B;
            const int nb = static_cast<int>(std::min<int64_t>(nw, start + B) - start);
            append_step(
                e, hp,
                [x, start](int i) {
                    const uint64_t v = x[start + i];
                    return std::pair<int, int>(static_cast<int>(v >> 32), static_cast<int>(static_cast<uint32_t>(v)));
                },
                nb, stamp, slot_id, id0 + s);
            hp.step_M.push_back(static_cast<double>(nb) * O);
        }
    });
    const auto p1 = t_shuffled;
    const auto p2 = clk::now();
    // pack into the pinned upload buffer (device layout order), chunks in parallel
    std::vector<size_t> wb(nchunk + 1, 0), sb(nchunk + 1, 0);
    ep.max_step_windows = ep.max_step_slots = 0;
    for (int c = 0; c < nchunk; ++c) {
        wb[c + 1] = wb[c] + ep.chunks[c].w_row.size();
        sb[c + 1] = sb[c] + ep.chunks[c].slot_row.size();
        ep.max_step_windows = std::max(ep.max_step_windows, ep.chunks[c].max_step_windows);
        ep.max_step_slots = std::max(ep.max_step_slots, ep.chunks[c].max_step_slots);
    }
    ep.n_w = wb[nchunk];
    ep.n_slots = sb[nchunk];
    const size_t cnt[EpochPlan::kArrays] = {ep.n_w, ep.n_w, ep.n_w, ep.n_w, ep.n_w, ep.n_w, ep.n_slots, ep.n_w,
                                            ep.n_slots + 1, static_cast<size_t>(steps) + 1,
                                            static_cast<size_t>(steps) + 1, static_cast<size_t>(steps)};
    ep.off[0] = 0;
    for (int i = 0; i < EpochPlan::kArrays; ++i) {
        const size_t el = i == EpochPlan::kStepM ? sizeof(double) : sizeof(int);
        ep.off[i + 1] = (ep.off[i] + cnt[i] * el + 15) & ~static_cast<size_t>(15);
    }
    ep.pin.reserve(ep.off[EpochPlan::kArrays]);
    unsigned char* base = ep.pin.p;
    auto arr = [&](int i) { return reinterpret_cast<int*>(base + ep.off[i]); };
    arr(EpochPlan::kSlotWinOff)[0] = 0;
    arr(EpochPlan::kStepWinOff)[0] = 0;
    arr(EpochPlan::kStepSlotOff)[0] = 0;
    worker_pool().run(nchunk, [&](int c) {
        const HostPlan& hp = ep.chunks[c];
        int s0, s1;
        chunk_range(c, s0, s1);
        auto put = [&](int i, const std::vector<int>& v, size_t at) {
            if (!v.empty()) std::memcpy(arr(i) + at, v.data(), sizeof(int) * v.size());
        };
        put(EpochPlan::kWRow, hp.w_row, wb[c]);
        put(EpochPlan::kWAnchor, hp.w_anchor, wb[c]);
        put(EpochPlan::kWSlot, hp.w_slot, wb[c]);
        put(EpochPlan::kWFirst, hp.w_first, wb[c]);
        put(EpochPlan::kWCsr, hp.w_csr, wb[c]);
        put(EpochPlan::kCsrAnchor, hp.csr_anchor, wb[c]);
        put(EpochPlan::kSlotRow, hp.slot_row, sb[c]);
        put(EpochPlan::kSlotWin, hp.slot_win, wb[c]);
        const int wo = static_cast<int>(wb[c]), so = static_cast<int>(sb[c]);
        int* swo = arr(EpochPlan::kSlotWinOff) + sb[c] + 1;
        for (size_t k = 1; k < hp.slot_win_off.size(); ++k) swo[k - 1] = hp.slot_win_off[k] + wo;
        int* stw = arr(EpochPlan::kStepWinOff) + s0 + 1;
        int* sts = arr(EpochPlan::kStepSlotOff) + s0 + 1;
        for (int k = 1; k <= s1 - s0; ++k) {
            stw[k - 1] = hp.step_win_off[k] + wo;
            sts[k - 1] = hp.step_slot_off[k] + so;
        }
        std::memcpy(reinterpret_cast<double*>(base + ep.off[EpochPlan::kStepM]) + s0, hp.step_M.data(),
                    sizeof(double) * hp.step_M.size());
    });
    ep.ready = true;
    if (dbg_host)
        std::fprintf(stderr, "[esrnn host] plan: draws+shuffle %.0f us, planning tail %.0f us (%d chunks), pack %.0f us\n",
                     std::chrono::duration<double, std::micro>(p1 - p0).count(),
                     std::chrono::duration<double, std::micro>(p2 - p1).count(), nchunk,
                     std::chrono::duration<double, std::micro>(clk::now() - p2).count());
}

// Async copies of a packed epoch plan (pinned) into the epoch DevPlan (capacity-sized, so
// the pointers -- and the captured epoch graph -- stay stable across epochs).
void upload_epoch_plan(Eng* e, const EpochPlan& ep, DevPlan& dp, size_t cap_w, size_t cap_steps) {
    const size_t cw = std::max(cap_w, ep.n_w), cs = std::max(cap_steps, static_cast<size_t>(ep.steps));
    DBuf<int>* dst[EpochPlan::kStepM] = {&dp.w_row, &dp.w_anchor, &dp.w_slot, &dp.w_first, &dp.w_csr,
                                         &dp.csr_anchor, &dp.slot_row, &dp.slot_win, &dp.slot_win_off,
                                         &dp.step_win_off, &dp.step_slot_off};
    const size_t cap[EpochPlan::kStepM] = {cw, cw, cw, cw, cw, cw, cw, cw, cw + 1, cs + 1, cs + 1};
    for (int i = 0; i < EpochPlan::kStepM; ++i) {
        if (dst[i]->n < std::max<size_t>(cap[i], 1)) dst[i]->alloc(std::max<size_t>(cap[i], 1));
        const size_t bytes = ep.off[i + 1] - ep.off[i];
        const size_t used = std::min(bytes, sizeof(int) * dst[i]->n);
        CUDA_OK(cudaMemcpyAsync(dst[i]->p, ep.pin.p + ep.off[i], used, cudaMemcpyHostToDevice, e->stream));
    }
    if (dp.step_M.n < std::max<size_t>(cs, 1)) dp.step_M.alloc(std::max<size_t>(cs, 1));
    CUDA_OK(cudaMemcpyAsync(dp.step_M.p, ep.pin.p + ep.off[EpochPlan::kStepM], sizeof(double) * ep.steps,
                            cudaMemcpyHostToDevice, e->stream));
}

template <typename Real>
double train_epoch_impl(Eng* e) {
    const int I = e->I, O = e->O, T = e->T;
    const int per = T - O - I + 1;
    const int64_t nw = static_cast<int64_t>(e->N_global) * per;
    if (nw <= 0) raise(ESRNN_CONTRACT_ERROR, "make_batches: no windows");
    using clk = std::chrono::steady_clock;
    static const bool dbg_host = std::getenv("ESRNN_DEBUG_HOST") != nullptr;
    const auto h0 = clk::now();
    // this epoch's plan: built ahead (during create / while the previous epoch ran on the
    // device), else now
    e->join_plan();
    if (!e->next_plan.ready) build_epoch_plan(e, e->next_plan);
    std::swap(e->cur_plan, e->next_plan);
    e->next_plan.ready = false;
    const int B = e->cfg.batch_size;
    const int steps = e->cur_plan.steps;
    const auto h1 = clk::now();
    ensure_capacity(e, B);
    const size_t local_w = static_cast<size_t>(e->N) * per;
    upload_epoch_plan(e, e->cur_plan, e->epoch_plan, local_w, steps);
    const auto h2 = clk::now();
    if (e->steps_cap < steps) {
        e->loss_hist.alloc(steps);
        e->steps_cap = steps;
    }
    const PlanDev pv = e->epoch_plan.view(false);
    if (e->span_mode) {
        // seed [step][kind] = {earliest start: LLONG_MAX, latest end: 0}
        const size_t n = static_cast<size_t>(steps) * kSpanKinds * 2;
        if (e->spans.n < n) e->spans.alloc(n);
        std::vector<long long> seed(n);
        for (size_t i = 0; i < n; ++i) seed[i] = (i & 1) ? 0 : LLONG_MAX;
        CUDA_OK(cudaMemcpyAsync(e->spans.p, seed.data(), sizeof(long long) * n, cudaMemcpyHostToDevice, e->stream));
        CUDA_OK(cudaStreamSynchronize(e->stream));
    }
    StateDev<Real> st = e->state<Real>();
    const bool use_graph = e->cfg.use_graphs >= 0 && !e->profiling;
    if (e->dbg_clk.p) {
        long long seed[16];
        for (int i = 0; i < 16; ++i) seed[i] = (i == 2 || i == 5 || i == 6 || i == 8 || i == 10 || i == 11) ? 0 : LLONG_MAX;
        CUDA_OK(cudaMemcpyAsync(e->dbg_clk.p + 100, seed, sizeof seed, cudaMemcpyHostToDevice, e->stream));
    }
    CUDA_OK(cudaEventRecord(e->ev0, e->stream));
    if (use_graph) {
        // the graph captures exactly these arguments: same bytes -> same graph
        std::string key;
        key_append(key, st);
        key_append(key, pv);
        key_append(key, e->lay);
        const long long dims[11] = {steps, e->tiles_cap, e->es_blocks, e->red_blocks, e->kcap, e->S, e->rank,
                                    e->world, e->gsplit * 256 + e->umma_parts, e->fp64 ? 8 : 4, e->sharded ? 1 : 0};
        key_append(key, dims);
        key_append(key, e->stream == nullptr);
        // A sharded graph captures this trainer's communicator (NCCL) or group slots: it is
        // kept by the trainer only, never shared through the process-wide cache, so it cannot
        // outlive the communicator or be replayed by a later trainer that reuses its address.
        if (!e->graph || e->graph_key != key) {
            e->graph = e->sharded ? nullptr : graph_cache().find(key);
            if (!e->graph) {
                auto ge = std::make_shared<GraphExec>();
                cudaGraph_t g;
                const int64_t before = e->launches;
                CUDA_OK(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal));
                try {
                    for (int s = 0; s < steps; ++s) launch_step<Real>(e, pv, s, true, true, st);
                } catch (...) {
                    cudaStreamEndCapture(e->stream, &g);
                    throw;
                }
                CUDA_OK(cudaStreamEndCapture(e->stream, &g));
                CUDA_OK(cudaGraphInstantiate(&ge->g, g, 0));
                CUDA_OK(cudaGraphDestroy(g));
                ge->launch_nodes = static_cast<int>(e->launches - before);
                e->launches = before;
                if (!e->sharded) graph_cache().insert(key, ge);
                e->graph = ge;
            }
            e->graph_key = key;
        }
        CUDA_OK(cudaGraphLaunch(e->graph->g, e->stream));
        e->launches += e->graph->launch_nodes;
    } else {
        for (int s = 0; s < steps; ++s) launch_step<Real>(e, pv, s, true, true, st);
    }
    CUDA_OK(cudaEventRecord(e->ev1, e->stream));
    CUDA_OK(cudaGetLastError());
    const auto h3 = clk::now();
    // the next epoch's shuffle + plan overlap this epoch's device time (the trainer RNG is
    // consumed in the same order as building it at the next call would)
    if (!e->profiling) build_epoch_plan(e, e->next_plan);
    if (e->profiling) e->prof_collect();
    e->pin_loss.reserve(std::max(steps, 1));
    const double* lh = e->pin_loss.p;
    CUDA_OK(cudaMemcpyAsync(e->pin_loss.p, e->loss_hist.p, sizeof(double) * steps, cudaMemcpyDeviceToHost, e->stream));
    enqueue_error_read(e);
    CUDA_OK(cudaStreamSynchronize(e->stream));
    if (dbg_host) {
        const auto h4 = clk::now();
        auto us = [](clk::time_point a, clk::time_point b) {
            return std::chrono::duration<double, std::micro>(b - a).count();
        };
        std::fprintf(stderr, "[esrnn host] epoch: shuffle+plan %.0f us, upload %.0f us, launch %.0f us, wait %.0f us\n",
                     us(h0, h1), us(h1, h2), us(h2, h3), us(h3, h4));
    }
    float ms = 0.f;
    CUDA_OK(cudaEventElapsedTime(&ms, e->ev0, e->ev1));
    e->last_ms = ms;
    check_device_error(e);
    if (e->dbg_clk.p) {
        long long c[96];
        CUDA_OK(cudaMemcpy(c, e->dbg_clk.p, sizeof c, cudaMemcpyDeviceToHost));
        static const char* kPh[] = {"stage+wait", "scan", "publish", "gather", "fwd0", "fwd1", "fwd2", "fwd3", "head",
                                    "loss", "zbar", "bwd3", "bwd2", "bwd1", "bwd0", "xbar"};
        std::fprintf(stderr, "[esrnn dbg] k_tile tile0 phase cycles:");
        for (int i = 1; i < 32 && c[i] > 0; ++i)
            std::fprintf(stderr, " %s=%lld", i - 1 < 16 ? kPh[i - 1] : "?", c[i] - c[i - 1]);
        std::fprintf(stderr, "\n[esrnn dbg] grad_finish ES block0:");
        for (int i = 33; i < 48 && c[i] > 0; ++i) std::fprintf(stderr, " %lld", c[i] - c[i - 1]);
        std::fprintf(stderr, "\n[esrnn dbg] grad_finish reduce block0:");
        for (int i = 49; i < 64 && c[i] > 0; ++i) std::fprintf(stderr, " %lld", c[i] - c[i - 1]);
        std::fprintf(stderr, "\n[esrnn dbg] ES block0 first chunk landed %lld cycles after the wait\n", c[42] - c[37]);
        std::fprintf(stderr, "[esrnn dbg] reduce block0 start - ES block0 start: %lld\n", c[48] - c[32]);
        std::fprintf(stderr, "[esrnn dbg] scan block0:");
        for (int i = 65; i < 80 && c[i] > 0; ++i) std::fprintf(stderr, " %lld", c[i] - c[i - 1]);
        std::fprintf(stderr, "\n[esrnn dbg] timeline ns (scan0 start, scan0 end, stack0 start, stack0 end, "
                             "finish0 start, finish last, adam0 start) rel. scan start:");
        for (int i = 80; i < 87; ++i) std::fprintf(stderr, " %lld", c[i] - c[80]);
        std::fprintf(stderr, "\n");
        long long sp[16];
        CUDA_OK(cudaMemcpy(sp, e->dbg_clk.p + 100, sizeof sp, cudaMemcpyDeviceToHost));
        std::fprintf(stderr, "[esrnn dbg] step-5 spans ns rel. tile launch: tile waited %lld end %lld | finish launch "
                             "%lld waited %lld blocks-end %lld last-CTA-end %lld | adam start %lld end %lld | next tile "
                             "waited %lld\n",
                     sp[1] - sp[0], sp[2] - sp[0], sp[3] - sp[0], sp[4] - sp[0], sp[5] - sp[0], sp[6] - sp[0],
                     sp[7] - sp[0], sp[8] - sp[0], sp[9] - sp[0]);
        std::fprintf(stderr, "[esrnn dbg] step-5 K3 ES blocks end %lld, GEMM blocks end %lld\n", sp[10] - sp[0],
                     sp[11] - sp[0]);
        std::vector<long long> tc(3 * kDbgTiles);
        CUDA_OK(cudaMemcpy(tc.data(), e->dbg_clk.p + 128, sizeof(long long) * tc.size(), cudaMemcpyDeviceToHost));
        std::vector<long long> ent, st0, en0, du;
        for (int t = 0; t < kDbgTiles; ++t)
            if (tc[3 * t + 1] > 0) {
                ent.push_back(tc[3 * t] - sp[0]);
                st0.push_back(tc[3 * t + 1] - sp[0]);
                en0.push_back(tc[3 * t + 2] - sp[0]);
                du.push_back(tc[3 * t + 2] - tc[3 * t + 1]);
            }
        auto q = [](std::vector<long long> v, double f) {
            std::sort(v.begin(), v.end());
            return v.empty() ? 0LL : v[std::min(v.size() - 1, static_cast<size_t>(f * v.size()))];
        };
        std::fprintf(stderr, "[esrnn dbg] step-5 tiles %zu: entry min/med/max %lld %lld %lld | waited %lld %lld %lld | end %lld %lld %lld | "
                             "duration %lld %lld %lld\n", du.size(), q(ent, 0), q(ent, 0.5), q(ent, 1), q(st0, 0), q(st0, 0.5), q(st0, 1), q(en0, 0),
                     q(en0, 0.5), q(en0, 1), q(du, 0), q(du, 0.5), q(du, 1));
        std::vector<long long> kc(2 * kDbgK3);
        CUDA_OK(cudaMemcpy(kc.data(), e->dbg_clk.p + 128 + 3 * kDbgTiles, sizeof(long long) * kc.size(),
                           cudaMemcpyDeviceToHost));
        for (int kind = 0; kind < 2; ++kind) {
            std::vector<long long> a, b, d;
            for (int i = 0; i < kDbgK3; ++i)
                if (kc[2 * i] > 0 && ((i < e->es_blocks) == (kind == 0))) {
                    a.push_back(kc[2 * i] - sp[0]);
                    b.push_back(kc[2 * i + 1] - sp[0]);
                    d.push_back(kc[2 * i + 1] - kc[2 * i]);
                }
            std::fprintf(stderr, "[esrnn dbg] step-5 K3 %s blocks %zu: waited min/med/max %lld %lld %lld | end %lld %lld %lld | "
                                 "duration %lld %lld %lld\n", kind == 0 ? "ES" : "GEMM", a.size(), q(a, 0), q(a, 0.5),
                         q(a, 1), q(b, 0), q(b, 0.5), q(b, 1), q(d, 0), q(d, 0.5), q(d, 1));
        }
    }
    if (e->span_mode) {
        // per kind: sum over steps of (latest CTA end - earliest CTA start)
        const size_t n = static_cast<size_t>(steps) * kSpanKinds * 2;
        std::vector<long long> sp(n);
        CUDA_OK(cudaMemcpy(sp.data(), e->spans.p, sizeof(long long) * n, cudaMemcpyDeviceToHost));
        static const int cls[kSpanKinds] = {1, 2, 4, 5};
        for (int s = 0; s < steps; ++s)
            for (int k = 0; k < kSpanKinds; ++k) {
                const long long a = sp[(static_cast<size_t>(s) * kSpanKinds + k) * 2];
                const long long b = sp[(static_cast<size_t>(s) * kSpanKinds + k) * 2 + 1];
                if (a == LLONG_MAX || b < a) continue;
                static const bool dump = std::getenv("ESRNN_SPAN_DUMP") != nullptr;
                if (dump)
                    std::fprintf(stderr, "[esrnn span] step %d kind %d start %lld len %lld\n", s, k,
                                 a - sp[0], b - a);
                e->prof_ms[cls[k]] += (b - a) * 1e-6;
                e->prof_n[cls[k]] += 1;
            }
    }
    e->have_last = true;
    // trainer.hpp:236-242: acc += loss * count, in batch order
    const double* sm = reinterpret_cast<const double*>(e->cur_plan.pin.p + e->cur_plan.off[EpochPlan::kStepM]);
    double acc = 0.0, weight = 0.0;
    for (int s = 0; s < steps; ++s) {
        acc += lh[s] * sm[s];
        weight += sm[s];
    }
    return acc / weight;
}

// ------------------------------------------------------------------ single batch
template <typename Real>
void run_batch_impl(Eng* e, int32_t B, const int32_t* rows, const int32_t* anchors, const double* mask,
                    int32_t flags, double* loss, double* mask_count, double* inputs, double* targets,
                    double* seas, double* levels, double* net_grads, int32_t* n_slots, int32_t* slot_rows,
                    double* ps_grads) {
    const int O = e->O, I = e->I, T = e->T, S = e->S;
    if (B <= 0) raise(ESRNN_CONTRACT_ERROR, "batch: empty");
    for (int i = 0; i < B; ++i) {
        if (rows[i] < 0 || rows[i] >= e->N_global) raise(ESRNN_SHAPE_ERROR, "batch: series row %d out of range", rows[i]);
        if (anchors[i] < I - 1 || anchors[i] > T - O - 1) raise(ESRNN_SHAPE_ERROR, "batch: anchor %d out of range", anchors[i]);
    }
    double count = 0.0;
    for (int64_t i = 0; i < static_cast<int64_t>(B) * O; ++i) count += (!mask || mask[i] != 0.0) ? 1.0 : 0.0;
    if (count == 0.0) raise(ESRNN_CONTRACT_ERROR, "pinball: all-zero mask, mean undefined");
    HostPlan bp;
    plan_begin(bp);
    std::vector<int64_t> stamp(std::max(e->N, 1), -1);
    std::vector<int> slot_id(std::max(e->N, 1), 0);
    append_step(e, bp, [&](int i) { return std::pair<int, int>(rows[i], anchors[i]); }, B, stamp, slot_id, 0);
    bp.step_M.push_back(count);
    const int Bl = static_cast<int>(bp.w_row.size());
    ensure_capacity(e, std::max(Bl, 1));
    upload_plan(e, bp, e->batch_plan, Bl, 1);
    // local mask rows in local-window order
    std::vector<unsigned char> m;
    if (mask) {
        m.reserve(static_cast<size_t>(Bl) * O);
        for (int i = 0; i < B; ++i) {
            const int r = rows[i] - e->row0;
            if (r < 0 || r >= e->N) continue;
            for (int j = 0; j < O; ++j) m.push_back(mask[static_cast<size_t>(i) * O + j] != 0.0 ? 1 : 0);
        }
        upload_vec(e, e->batch_plan.mask, m, std::max<size_t>(m.size(), 1));
    }
    const PlanDev pv = e->batch_plan.view(mask != nullptr);
    StateDev<Real> st = e->state<Real>();
    const bool want_dump = inputs || targets || seas || levels;
    if (want_dump) {
        st.d_inputs = reinterpret_cast<Real*>(e->d_inputs.p);
        st.d_targets = reinterpret_cast<Real*>(e->d_targets.p);
        st.d_seas = reinterpret_cast<Real*>(e->d_seas.p);
        st.d_levels = reinterpret_cast<Real*>(e->d_levels.p);
    }
    const bool grads = (flags & ESRNN_BATCH_GRADS) != 0;
    const bool update = grads && (flags & ESRNN_BATCH_UPDATE) != 0;
    CUDA_OK(cudaEventRecord(e->ev0, e->stream));
    // the level-variability penalty is formed in K3's ES blocks: a penalised batch_loss
    // runs the gradient path (no update) to get it
    const bool k3 = grads || st.lvp > 0.0;
    if (Bl > 0 || e->world > 1) {
        launch_step<Real>(e, pv, 0, k3, update, st);
    }
    CUDA_OK(cudaEventRecord(e->ev1, e->stream));
    CUDA_OK(cudaGetLastError());
    if (e->profiling) e->prof_collect();
    CUDA_OK(cudaStreamSynchronize(e->stream));
    float ms = 0.f;
    CUDA_OK(cudaEventElapsedTime(&ms, e->ev0, e->ev1));
    e->last_ms = ms;
    throw_device_error(e);
    // loss: sum of tile partials (single GPU) or all-reduced sum (sharded) / M
    double lsum = 0.0;
    if (k3 && (e->sharded || st.lvp > 0.0)) {  // K3 / K4 / the collective wrote the step's loss sum
        double g2[2];
        CUDA_OK(cudaMemcpy(g2, e->gtail.p, sizeof g2, cudaMemcpyDeviceToHost));
        lsum = g2[1];
    } else {
        const int nt = (Bl + kRows - 1) / kRows;
        std::vector<double> lp(nt);
        if (nt) CUDA_OK(cudaMemcpy(lp.data(), e->loss_part.p, sizeof(double) * nt, cudaMemcpyDeviceToHost));
        for (double v : lp) lsum += v;
        if (e->sharded) raise(ESRNN_CONFIG_ERROR, "sharded batch_loss requires gradients (collective step)");
    }
    if (loss) *loss = lsum / count;
    if (mask_count) *mask_count = count;
    if (want_dump && Bl > 0) {
        std::vector<double> tmp;
        auto dl = [&](const DBuf<unsigned char>& d, size_t n, double* out) {
            if (!out) return;
            download_real(e, d.p, n, out);
        };
        dl(e->d_inputs, static_cast<size_t>(Bl) * e->in0, inputs);
        dl(e->d_targets, static_cast<size_t>(Bl) * O, targets);
        dl(e->d_seas, static_cast<size_t>(Bl) * O, seas);
        dl(e->d_levels, Bl, levels);
    }
    const int k = static_cast<int>(bp.slot_row.size());
    if (n_slots) *n_slots = k;
    if (slot_rows)
        for (int i = 0; i < k; ++i) slot_rows[i] = bp.slot_row[i] + e->row0;
    if (grads) {
        if (net_grads) {
            std::vector<double> c(e->lay.P_pad);
            download_real(e, e->gbuf.p, c.size(), c.data());
            std::fill(net_grads, net_grads + e->P, 0.0);
            for (size_t i = 0; i < c.size(); ++i)
                if (e->live_flat[i] >= 0) net_grads[e->live_flat[i]] = c[i];
        }
        if (ps_grads && e->cfg.attach_es_state && k > 0) download_real(e, e->psg.p, static_cast<size_t>(k) * (2 + S), ps_grads);
    }
    if (update) sync_weights_from_device(e);
}

// ------------------------------------------------------------------ forecast
// Host outputs of one forecast pass (all nullable).  mode 0: forecast_at; 1: validate (sMAPE);
// 2: evaluate (sMAPE + MASE + seasonal-naive scores, commands.hpp:285-338).
// K6 scan with the season length as a template constant for the M4 profiles' S
template <typename Real>
void launch_forecast_scan(Eng* e, int t_len, Real* X, Real* FL, Real* FS, Real* dump_lv, Real* dump_se, int dump_row,
                          double* score) {
    const int sb = (e->N + kScanThreads - 1) / kScanThreads;
    const size_t smem = sizeof(Real) * static_cast<size_t>(t_len + e->S + e->I) * kScanThreads;
    const StateDev<Real> st = e->state<Real>();
    const size_t smem_sc = smem + sizeof(Real) * static_cast<size_t>(e->in0 + e->O + 1) * kScanThreads;
    auto go = [&](auto kernel, size_t sm) {
        kernel<<<sb, kScanThreads, sm, e->stream>>>(st, e->lay, t_len, X, FL, FS, dump_lv, dump_se, dump_row, score);
    };
    const bool dump = dump_row >= 0;
    switch (e->S) {
        case 1: dump ? go(k_forecast_scan_sc<Real, 1, true>, smem_sc) : go(k_forecast_scan_sc<Real, 1, false>, smem_sc); break;
        case 4: dump ? go(k_forecast_scan_sc<Real, 4, true>, smem_sc) : go(k_forecast_scan_sc<Real, 4, false>, smem_sc); break;
        case 12: dump ? go(k_forecast_scan_sc<Real, 12, true>, smem_sc) : go(k_forecast_scan_sc<Real, 12, false>, smem_sc); break;
        default: go(k_forecast_scan<Real, 0>, smem); break;
    }
}

// Host-level collectives of a sharded trainer (outside the step graphs): a sum of n doubles
// in rank order, and an all-gather of equal-size byte blocks (rank-major).
void allreduce_sum_host(Eng* e, double* v, int n) {
    if (e->group) {
        const std::vector<unsigned char> all = e->group->exchange(e->rank, v, sizeof(double) * n);
        const double* a = reinterpret_cast<const double*>(all.data());
        for (int i = 0; i < n; ++i) {
            double s = 0.0;
            for (int r = 0; r < e->world; ++r) s += a[static_cast<size_t>(r) * n + i];
            v[i] = s;
        }
        return;
    }
    if (e->smape_sum.n < static_cast<size_t>(n)) e->smape_sum.alloc(n);
    CUDA_OK(cudaMemcpy(e->smape_sum.p, v, sizeof(double) * n, cudaMemcpyHostToDevice));
    NCCL_OK(ncclAllReduce(e->smape_sum.p, e->smape_sum.p, n, ncclDouble, ncclSum, e->comm, e->stream));
    CUDA_OK(cudaMemcpyAsync(v, e->smape_sum.p, sizeof(double) * n, cudaMemcpyDeviceToHost, e->stream));
    CUDA_OK(cudaStreamSynchronize(e->stream));
}

std::vector<double> allgather_host(Eng* e, const std::vector<double>& mine) {
    if (e->group) {
        const std::vector<unsigned char> all = e->group->exchange(e->rank, mine.data(), sizeof(double) * mine.size());
        std::vector<double> out(all.size() / sizeof(double));
        std::memcpy(out.data(), all.data(), all.size());
        return out;
    }
    DBuf<double> d;
    d.alloc(mine.size() * (e->world + 1));
    double* recv = d.p + mine.size();
    CUDA_OK(cudaMemcpy(d.p, mine.data(), sizeof(double) * mine.size(), cudaMemcpyHostToDevice));
    NCCL_OK(ncclAllGather(d.p, recv, mine.size(), ncclDouble, e->comm, e->stream));
    std::vector<double> out(mine.size() * e->world);
    CUDA_OK(cudaMemcpyAsync(out.data(), recv, sizeof(double) * out.size(), cudaMemcpyDeviceToHost, e->stream));
    CUDA_OK(cudaStreamSynchronize(e->stream));
    return out;
}

struct ScoreOut {
    double* smape = nullptr;        // [n_local]
    double* mase = nullptr;         // [n_local], NaN = undefined (std::nullopt)
    double* naive_smape = nullptr;  // [n_local]
    double* naive_mase = nullptr;   // [n_local]
    double* totals = nullptr;       // [8] global sums (see esrnn_trainer_evaluate)
    double* mean = nullptr;         // validate: global mean sMAPE
};

template <typename Real>
void forecast_impl(Eng* e, int64_t drop_tail, double* out, int mode, const ScoreOut& so) {
    const int I = e->I, O = e->O, S = e->S, N = e->N;
    if (static_cast<int64_t>(e->LEN) < drop_tail + I) raise(ESRNN_INSUFFICIENT_LENGTH, "forecast_at: not enough in-sample data");
    const int t_ins = static_cast<int>(e->LEN - drop_tail);
    if (mode == 2 && t_ins <= S) raise(ESRNN_INSUFFICIENT_LENGTH, "mase: in-sample length must exceed season length");
    const size_t r = sizeof(Real);
    if (e->fX.n < r * std::max(N, 1) * e->in0) {
        e->fX.alloc(r * std::max(N, 1) * e->in0);
        e->fL.alloc(r * std::max(N, 1));
        e->fS.alloc(r * std::max(N, 1) * O);
        e->f_out.alloc(static_cast<size_t>(std::max(N, 1)) * O);
        e->f_smape.alloc(std::max(N, 1));
    }
    if (mode == 2 && e->f_score.n < 4 * static_cast<size_t>(std::max(N, 1))) e->f_score.alloc(4 * std::max(N, 1));
    StateDev<Real> st = e->state<Real>();
    const NetLayout& lay = e->lay;
    CUDA_OK(cudaEventRecord(e->ev0, e->stream));
    if (N > 0) {
        {
            Eng::KScope k(e, 6);
            launch_forecast_scan<Real>(e, t_ins, reinterpret_cast<Real*>(e->fX.p), reinterpret_cast<Real*>(e->fL.p),
                                       reinterpret_cast<Real*>(e->fS.p), nullptr, nullptr, -1,
                                       mode == 2 ? e->f_score.p : nullptr);
        }
        ForecastArgs fa{};
        fa.t_ins = t_ins;
        fa.validate = mode != 0 ? 1 : 0;
        fa.X = e->fX.p;
        fa.lvl = e->fL.p;
        fa.sout = e->fS.p;
        fa.out = e->f_out.p;
        fa.smape = e->f_smape.p;
        fa.mase = mode == 2 ? e->f_score.p + 3 * static_cast<size_t>(N) : nullptr;
        fa.score = mode == 2 ? e->f_score.p : nullptr;
        const int tiles = (N + kRows - 1) / kRows;
        {
            Eng::KScope k(e, 7);
            launch_stack<Real, kForecast>(e, tiles, st, e->batch_plan.view(false), 0, fa);
        }
        e->launches += 2;
    }
    if (e->profiling) e->prof_collect();
    CUDA_OK(cudaEventRecord(e->ev1, e->stream));
    CUDA_OK(cudaGetLastError());
    // results into pinned staging on the same stream: one synchronisation for everything
    const size_t nfo = static_cast<size_t>(N) * O, nsc = mode == 2 ? 4 * static_cast<size_t>(N) : 0;
    e->pin_d.reserve(nfo + N + nsc + 1);
    double* pf = e->pin_d.p;
    double* psm = pf + nfo;
    double* psc = psm + N;
    if (N > 0) {
        if (out) CUDA_OK(cudaMemcpyAsync(pf, e->f_out.p, sizeof(double) * nfo, cudaMemcpyDeviceToHost, e->stream));
        if (mode != 0)
            CUDA_OK(cudaMemcpyAsync(psm, e->f_smape.p, sizeof(double) * N, cudaMemcpyDeviceToHost, e->stream));
        if (mode == 2)
            CUDA_OK(cudaMemcpyAsync(psc, e->f_score.p, sizeof(double) * nsc, cudaMemcpyDeviceToHost, e->stream));
    }
    enqueue_error_read(e);
    CUDA_OK(cudaStreamSynchronize(e->stream));
    float ms = 0.f;
    CUDA_OK(cudaEventElapsedTime(&ms, e->ev0, e->ev1));
    e->last_ms = ms;
    // sharded validate / evaluate: a rank's device error is raised only after the totals'
    // collective, on every rank, so no peer waits in the collective for a rank that threw
    const bool defer = mode != 0 && e->sharded;
    int errw[4] = {e->pin_err.p[0], e->pin_err.p[1], e->pin_err.p[2], e->pin_err.p[3]};
    if (!defer) check_device_error(e);
    if (out && N > 0) std::memcpy(out, pf, sizeof(double) * nfo);
    if (mode == 0) return;
    const double* sm = psm;
    if (so.smape)
        for (int i = 0; i < N; ++i) so.smape[i] = sm[i];
    // global sums: [smape, mase, mase count, naive smape, naive mase, naive mase count, series, 0]
    double tot[8] = {0, 0, 0, 0, 0, 0, static_cast<double>(N), 0};
    for (int i = 0; i < N; ++i) tot[0] += sm[i];
    if (mode == 2) {
        const double* sc = psc;
        for (int i = 0; i < N; ++i) {
            const double ns = sc[N + i], nm = sc[2 * N + i], m = sc[3 * N + i];
            if (so.mase) so.mase[i] = m;
            if (so.naive_smape) so.naive_smape[i] = ns;
            if (so.naive_mase) so.naive_mase[i] = nm;
            if (!std::isnan(m)) { tot[1] += m; tot[2] += 1; }
            tot[3] += ns;
            if (!std::isnan(nm)) { tot[4] += nm; tot[5] += 1; }
        }
    }
    if (defer) {
        tot[7] = errw[0] != 0 ? 1.0 : 0.0;
        allreduce_sum_host(e, tot, 8);
        if (errw[0] != 0) raise_device_error(e, errw);
        if (tot[7] != 0.0) {
            errw[0] = 0, errw[2] = 1;
            raise_device_error(e, errw);
        }
    }
    if (so.mean) *so.mean = tot[0] / static_cast<double>(e->N_global);
    if (so.totals)
        for (int i = 0; i < 8; ++i) so.totals[i] = tot[i];
}

// ------------------------------------------------------------------ general forward_stack
// network.hpp:190-210 over a multi-step sequence with the trainer's full StackWeights (the
// structurally dead parts of the sequence-length-1 hot path -- forget gates, recurrent
// matrices -- are live here), plus the tape adjoints for an upstream out_bar.
template <typename Real>
void forward_stack_impl(Eng* e, int Tq, int B, const double* inputs, double* out, const double* out_bar,
                        double* wbar, double* xbar) {
    if (Tq < 1) raise(ESRNN_CONTRACT_ERROR, "forward_stack: empty sequence");
    if (B < 1) raise(ESRNN_SHAPE_ERROR, "forward_stack: empty batch");
    SeqLayout sl{};
    sl.L = e->L, sl.H = e->H, sl.O = e->O, sl.in0 = e->in0, sl.T = Tq, sl.B = B;
    sl.in_max = std::max(e->in0, e->H);
    for (int l = 0; l < e->L; ++l) {
        sl.layer_in[l] = e->layer_in[l];
        sl.dil[l] = e->prof.dilations[l];
        sl.res_src[l] = -1;
        sl.w_in[l] = e->off_win[l];
        sl.w_rec[l] = e->off_wrec[l];
        sl.bias[l] = e->off_bias[l];
    }
    for (int b = 0, first = 0; b < e->prof.n_blocks; first += e->prof.block_len[b], ++b)
        if (b > 0) sl.res_src[first + e->prof.block_len[b] - 1] = first - 1;  // network.hpp:201-206
    sl.nl_w = e->off_nlw, sl.nl_b = e->off_nlb, sl.out_w = e->off_outw, sl.out_b = e->off_outb, sl.P = e->P;
    sync_weights_from_device(e);
    const size_t r = e->rsz;
    const int nblk = (B + kSeqRows - 1) / kSeqRows;
    DBuf<unsigned char> w, x, scratch, ob, wpart, xb;
    DBuf<double> dout, dwbar;
    w.alloc(r * e->P);
    upload_real(e, w.p, e->w_host.data(), e->P);
    x.alloc(r * static_cast<size_t>(Tq) * B * e->in0);
    upload_real(e, x.p, inputs, static_cast<size_t>(Tq) * B * e->in0);
    dout.alloc(static_cast<size_t>(B) * e->O);
    // the shared-memory-resident kernels (seqstack.cuh k_seq_fwd_fast / k_seq_bwd_fast) when a
    // layer's weights, the (h, c) rings and the step tiles fit; else the stepwise kernels that
    // keep every activation in a per-4-row scratch (k_seq_forward / k_seq_backward)
    int dmax = 1;
    for (int l = 0; l < e->L; ++l) dmax = std::max(dmax, sl.dil[l]);
    const size_t G = 4 * static_cast<size_t>(e->H);
    const size_t fast_smem = r * ((static_cast<size_t>(sl.in_max) + e->H + 1) * G + 2 * static_cast<size_t>(sl.in_max) * kSeqFR +
                                  2 * static_cast<size_t>(dmax) * e->H * kSeqFR + kSeqFR * G);
    const size_t bwd_smem = r * ((static_cast<size_t>(sl.in_max) + e->H) * G + kSeqFR * G +
                                 2 * static_cast<size_t>(dmax) * e->H * kSeqFR +
                                 (static_cast<size_t>(sl.in_max) + e->H) * kSeqFR);
    const bool naive_env = std::getenv("ESRNN_SEQ_NAIVE") != nullptr;
    const bool fast_fwd = fast_smem <= static_cast<size_t>(g_smem_optin) && kSeqSplit * ((G + 31) / 32 * 32) <= 1024 &&
                          !naive_env;
    const bool fast_bwd = fast_fwd && sizeof(Real) == 4 && bwd_smem <= static_cast<size_t>(g_smem_optin) &&
                          (static_cast<size_t>(sl.in_max) + e->H + 1) * G <= static_cast<size_t>(kSeqBwdAcc) * kSeqBwdThreads;
    const bool fast = out_bar ? fast_bwd : fast_fwd;
    const int nfast = (B + kSeqFR - 1) / kSeqFR;
    if (!fast) scratch.alloc(r * static_cast<size_t>(nblk) * SeqScratch<Real>::size(sl));
    DBuf<unsigned char> dcurbuf;
    if (fast) {
        if (out_bar) {
            scratch.alloc(r * static_cast<size_t>(nfast) * SeqSave<Real>::per_cta(sl));
            dcurbuf.alloc(r * static_cast<size_t>(nfast) * e->L * Tq * kSeqFR * e->H);
            CUDA_OK(cudaFuncSetAttribute(k_seq_fwd_fast<Real, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(fast_smem)));
            CUDA_OK(cudaFuncSetAttribute(k_seq_bwd_fast<Real>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(bwd_smem)));
        } else {
            scratch.alloc(r * static_cast<size_t>(nfast) * 3 * Tq * kSeqFR * e->H);
            CUDA_OK(cudaFuncSetAttribute(k_seq_fwd_fast<Real, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(fast_smem)));
        }
    }
    CUDA_OK(cudaEventRecord(e->ev0, e->stream));
    const int nt = kSeqSplit * static_cast<int>((std::max<size_t>(G, 32) + 31) / 32 * 32);
    if (fast && !out_bar) {
        k_seq_fwd_fast<Real, false><<<nfast, nt, fast_smem, e->stream>>>(
            sl, reinterpret_cast<const Real*>(w.p), reinterpret_cast<const Real*>(x.p), reinterpret_cast<Real*>(scratch.p),
            dout.p);
        e->launches += 1;
    } else if (fast) {
        k_seq_fwd_fast<Real, true><<<nfast, nt, fast_smem, e->stream>>>(
            sl, reinterpret_cast<const Real*>(w.p), reinterpret_cast<const Real*>(x.p), reinterpret_cast<Real*>(scratch.p),
            dout.p);
        ob.alloc(r * static_cast<size_t>(B) * e->O);
        upload_real(e, ob.p, out_bar, static_cast<size_t>(B) * e->O);
        wpart.alloc(r * static_cast<size_t>(nfast) * e->P);
        if (xbar) xb.alloc(r * static_cast<size_t>(Tq) * B * e->in0);
        k_seq_bwd_fast<Real><<<nfast, kSeqBwdThreads, bwd_smem, e->stream>>>(
            sl, reinterpret_cast<const Real*>(w.p), reinterpret_cast<const Real*>(x.p), reinterpret_cast<Real*>(scratch.p),
            reinterpret_cast<Real*>(dcurbuf.p), reinterpret_cast<const Real*>(ob.p), reinterpret_cast<Real*>(wpart.p),
            xbar ? reinterpret_cast<Real*>(xb.p) : nullptr);
        dwbar.alloc(e->P);
        k_seq_reduce<Real><<<static_cast<int>((e->P + 255) / 256), 256, 0, e->stream>>>(
            reinterpret_cast<const Real*>(wpart.p), nfast, e->P, dwbar.p);
        e->launches += 3;
    } else {
        k_seq_forward<Real><<<nblk, kSeqThreads, 0, e->stream>>>(sl, reinterpret_cast<const Real*>(w.p),
                                                                  reinterpret_cast<const Real*>(x.p),
                                                                  reinterpret_cast<Real*>(scratch.p), dout.p);
        e->launches += 1;
        if (out_bar) {
            ob.alloc(r * static_cast<size_t>(B) * e->O);
            upload_real(e, ob.p, out_bar, static_cast<size_t>(B) * e->O);
            wpart.alloc(r * static_cast<size_t>(nblk) * e->P);
            if (xbar) xb.alloc(r * static_cast<size_t>(Tq) * B * e->in0);
            k_seq_backward<Real><<<nblk, kSeqThreads, 0, e->stream>>>(
                sl, reinterpret_cast<const Real*>(w.p), reinterpret_cast<const Real*>(x.p),
                reinterpret_cast<Real*>(scratch.p), reinterpret_cast<const Real*>(ob.p), reinterpret_cast<Real*>(wpart.p),
                xbar ? reinterpret_cast<Real*>(xb.p) : nullptr);
            dwbar.alloc(e->P);
            k_seq_reduce<Real><<<static_cast<int>((e->P + 255) / 256), 256, 0, e->stream>>>(
                reinterpret_cast<const Real*>(wpart.p), nblk, e->P, dwbar.p);
            e->launches += 2;
        }
    }
    CUDA_OK(cudaEventRecord(e->ev1, e->stream));
    CUDA_OK(cudaGetLastError());
    CUDA_OK(cudaStreamSynchronize(e->stream));
    float ms = 0.f;
    CUDA_OK(cudaEventElapsedTime(&ms, e->ev0, e->ev1));
    e->last_ms = ms;
    if (out) CUDA_OK(cudaMemcpy(out, dout.p, sizeof(double) * B * e->O, cudaMemcpyDeviceToHost));
    if (out_bar && wbar) CUDA_OK(cudaMemcpy(wbar, dwbar.p, sizeof(double) * e->P, cudaMemcpyDeviceToHost));
    if (out_bar && xbar) download_real(e, xb.p, static_cast<size_t>(Tq) * B * e->in0, xbar);
}

template <typename Real>
void hw_state_impl(Eng* e, int64_t row, int64_t t_len, double* levels, double* seas) {
    const int S = e->S;
    const int lr = static_cast<int>(row - e->row0);
    if (lr < 0 || lr >= e->N) raise(ESRNN_SHAPE_ERROR, "hw_state: row %lld not owned", static_cast<long long>(row));
    if (t_len < S || t_len > e->LEN)
        raise(ESRNN_INSUFFICIENT_LENGTH, "hybrid_primer: series length %lld shorter than season length %d",
              static_cast<long long>(t_len), S);
    const size_t r = sizeof(Real);
    if (e->dump_lv.n < r * e->LEN) {
        e->dump_lv.alloc(r * e->LEN);
        e->dump_se.alloc(r * (e->LEN + S));
    }
    StateDev<Real> st = e->state<Real>();
    // the dump row's thread writes its full state; X == nullptr skips the window build
    launch_forecast_scan<Real>(e, static_cast<int>(t_len), nullptr, nullptr, nullptr,
                               reinterpret_cast<Real*>(e->dump_lv.p), reinterpret_cast<Real*>(e->dump_se.p),
                               static_cast<int>(lr), nullptr);
    e->launches += 1;
    CUDA_OK(cudaGetLastError());
    CUDA_OK(cudaStreamSynchronize(e->stream));
    throw_device_error(e);
    download_real(e, e->dump_lv.p, t_len, levels);
    download_real(e, e->dump_se.p, t_len + S, seas);
}

}  // namespace

// ======================================================================= C-ABI
extern "C" {

const char* esrnn_version(void) { return "esrnn-b200 0.1 (sm_100a CUDA engine)"; }
int32_t esrnn_abi_version(void) { return ESRNN_ABI_VERSION; }
const char* esrnn_last_error(const esrnn_trainer* t) { return t ? t->err.c_str() : g_create_err.c_str(); }

esrnn_status esrnn_trainer_create(const esrnn_profile* profile, const esrnn_train_config* cfg, int64_t n_series,
                                  int32_t length, const double* values, const int32_t* category,
                                  const esrnn_dist* dist, esrnn_trainer** out) {
    *out = nullptr;
    std::unique_ptr<Eng> e(new Eng());
    using clk = std::chrono::steady_clock;
    static const bool dbg_host = std::getenv("ESRNN_DEBUG_HOST") != nullptr;
    clk::time_point c[8];
    int nc = 0;
    c[nc++] = clk::now();
    esrnn_status st = guarded(g_create_err, [&] {
        validate_config(*profile, *cfg);
        if (n_series <= 0) raise(ESRNN_CONTRACT_ERROR, "trainer: no series");
        const int O = profile->horizon, S = profile->seasonality_length, I = profile->input_window;
        if (length < 2 * O + 1)
            raise(ESRNN_INSUFFICIENT_LENGTH, "split: need at least %d values, got %d", 2 * O + 1, length);
        const int T = length - 2 * O;
        if (T < I + O) raise(ESRNN_INSUFFICIENT_LENGTH, "trainer: train segment of %d cannot hold an input window plus horizon", T);
        if (T < S) raise(ESRNN_INSUFFICIENT_LENGTH, "trainer: train segment shorter than one season");
        e->prof = *profile;
        e->cfg = *cfg;
        e->fp64 = cfg->precision == ESRNN_FP64;
        e->rsz = e->fp64 ? sizeof(double) : sizeof(float);
        e->N_global = static_cast<int>(n_series);
        const bool force = dist && (dist->flags & ESRNN_DIST_FORCE_COLLECTIVE) != 0;
        if (dist && (dist->world_size > 1 || force)) {
            e->rank = dist->rank;
            e->world = dist->world_size;
            if (e->world < 1 || e->rank < 0 || e->rank >= e->world) raise(ESRNN_CONFIG_ERROR, "dist: rank out of range");
            if (dist->group && dist->group->W != e->world)
                raise(ESRNN_CONFIG_ERROR, "dist: group of %d ranks, world_size %d", dist->group->W, e->world);
        }
        // contiguous row blocks
        e->row0 = static_cast<int>((static_cast<int64_t>(e->rank) * n_series) / e->world);
        const int row1 = static_cast<int>((static_cast<int64_t>(e->rank + 1) * n_series) / e->world);
        e->N = row1 - e->row0;
        e->LEN = length;
        e->T = T;
        e->S = S;
        e->I = I;
        e->O = O;
        e->H = profile->hidden_size;
        e->in0 = I + ESRNN_NUM_CATEGORIES;
        e->L = 0;
        for (int b = 0; b < profile->n_blocks; ++b) e->L += profile->block_len[b];
        // network.hpp:89-116 init order on the trainer RNG (identical on every rank).  The
        // first epoch's shuffle is the RNG's next consumer, so a helper thread draws the
        // weights' raw numbers (one block), hands them to this thread for conversion, then
        // shuffles and plans epoch 1 -- started first, so it overlaps the layout, device and
        // NCCL setup below; the weights are uploaded once converted.
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            raise(ESRNN_CUDA_ERROR, "no CUDA device visible: the B200 engine has no CPU fallback");
        if (cfg->device < 0 || cfg->device >= ndev) raise(ESRNN_CUDA_ERROR, "device %d out of range", cfg->device);
        CUDA_OK(cudaSetDevice(cfg->device));  // pinned blocks below come from this device's context
        e->rng = HostRng(cfg->seed);
        e->cur_plan = plan_pool_get();
        e->next_plan = plan_pool_get();
        Eng* ep = e.get();
        // draw order: per layer W_in (in x 4H) then W_rec (H x 4H), then the head (H x H)
        // and the adapter (H x O); biases are constants (forget chunk 1.0)
        {
            const int64_t H = e->H;
            int64_t n_draw = (e->in0 + H) * 4 * H + static_cast<int64_t>(e->L - 1) * 2 * H * 4 * H + H * H + H * e->O;
            e->w_draws = static_cast<size_t>(n_draw);
            e->w_raw.reserve(e->w_draws);
        }
        auto weights_drawn = std::make_shared<std::promise<void>>();
        std::future<void> weights_ready = weights_drawn->get_future();
        if (std::max(0, T - e->O - e->I + 1) > 0) {
            ep->plan_done = async_runner().submit([ep, weights_drawn] {
                cudaSetDevice(ep->cfg.device);  // the plan's pinned upload block
                ep->rng.gen.fill(ep->w_raw.p, ep->w_draws);
                weights_drawn->set_value();
                try {
                    build_epoch_plan(ep, ep->next_plan);
                } catch (...) {
                    ep->next_plan.ready = false;  // rebuilt (from a fresh shuffle) by train_epoch
                }
            });
        } else {
            ep->rng.gen.fill(ep->w_raw.p, ep->w_draws);
            weights_drawn->set_value();
        }
        c[nc++] = clk::now();
        build_layout(e.get());
        e->w_host.assign(e->P, 0.0);
        auto convert_weights = [ep] {
            const int H = ep->H;
            const double bound = 1.0 / std::sqrt(static_cast<double>(H));
            const uint64_t* r = ep->w_raw.p;
            // Rng::uniform(lo, hi) on each raw draw, in draw order
            auto u = [&](int64_t off, int64_t n) {
                double* w = ep->w_host.data() + off;
                for (int64_t i = 0; i < n; ++i)
                    w[i] = -bound + (bound - -bound) * (static_cast<double>(r[i] >> 11) * 0x1.0p-53);
                r += n;
            };
            for (int l = 0; l < ep->L; ++l) {
                u(ep->off_win[l], static_cast<int64_t>(ep->layer_in[l]) * 4 * H);
                u(ep->off_wrec[l], static_cast<int64_t>(H) * 4 * H);
                for (int c2 = H; c2 < 2 * H; ++c2) ep->w_host[ep->off_bias[l] + c2] = 1.0;
            }
            u(ep->off_nlw, static_cast<int64_t>(H) * H);
            u(ep->off_outw, static_cast<int64_t>(H) * ep->O);
            if (r != ep->w_raw.p + ep->w_draws) raise(ESRNN_ERROR, "weight init: draw count mismatch");
            ep->w_raw.release();
        };

        CUDA_OK(cudaDeviceGetAttribute(&g_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, cfg->device));
        CUDA_OK(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, cfg->device));
        CUDA_OK(cudaDeviceGetAttribute(&g_smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, cfg->device));
        stream_get(e->stream, e->ev0, e->ev1);
        c[nc++] = clk::now();
        if (e->world > 1 || force) {
            if (dist->group) {
                std::lock_guard<std::mutex> lk(dist->group->mu);
                if (dist->group->joined.empty()) dist->group->joined.assign(dist->group->W, 0);
                if (dist->group->joined[e->rank])
                    raise(ESRNN_CONFIG_ERROR, "group: rank %d already joined (a group serves one set of trainers)", e->rank);
                dist->group->joined[e->rank] = 1;
                e->group = dist->group;
                ++e->group->refs;
                e->sharded = true;
            } else {
                // an id of 128 x 0xEE is the local-partials test mode: the shard runs its data
                // path but skips the collective, so a test can sum per-rank partials itself
                bool local_only = true;
                for (int i = 0; i < 128; ++i) local_only = local_only && dist->nccl_unique_id[i] == 0xEE;
                if (!local_only) {
                    ncclUniqueId id;
                    static_assert(sizeof(id.internal) == 128, "nccl id size");
                    std::memcpy(id.internal, dist->nccl_unique_id, 128);
                    NCCL_OK(ncclCommInitRank(&e->comm, e->world, id, e->rank));
                    e->sharded = true;
                }
            }
        }

        c[nc++] = clk::now();
        e->bc_tab = bc_table(e->cfg.device);
        if (e->fp64) {
            alloc_state<double>(e.get());
            upload_values<double>(e.get(), values, category);
        } else {
            alloc_state<float>(e.get());
            upload_values<float>(e.get(), values, category);
        }
        if (e->group) e->group->ensure_device(cfg->device, 32 + static_cast<long long>(e->rsz) * e->lay.P_pad);
        weights_ready.wait();
        convert_weights();
        c[nc++] = clk::now();
        upload_theta(e.get(), &e->stage_theta);
        ensure_capacity(e.get(), cfg->batch_size);
        CUDA_OK(cudaStreamSynchronize(e->stream));
        e->stage_raw.free();
        e->stage_pin.release();
        e->stage_theta.release();
        e->stage_cat.release();
        c[nc++] = clk::now();
        if (dbg_host) {
            std::fprintf(stderr, "[esrnn host] create:");
            for (int i = 1; i < nc; ++i)
                std::fprintf(stderr, " %.0f", std::chrono::duration<double, std::micro>(c[i] - c[i - 1]).count());
            std::fprintf(stderr, " us (plan hand-off, layout+device+stream, nccl, alloc+values+weights, theta+capacity+sync)\n");
        }
    });
    if (st == ESRNN_OK) *out = e.release();
    return st;
}

void esrnn_trainer_destroy(esrnn_trainer* t) {
    if (!t) return;
    cudaSetDevice(t->cfg.device);
    delete t;
}

esrnn_status esrnn_trainer_shard(const esrnn_trainer* t, int64_t* b, int64_t* e) {
    *b = t->row0;
    *e = t->row0 + t->N;
    return ESRNN_OK;
}

esrnn_status esrnn_trainer_param_count(const esrnn_trainer* t, int32_t* n_arrays, int64_t* n_values) {
    *n_arrays = 3 * t->L + 4;
    *n_values = t->P;
    return ESRNN_OK;
}

esrnn_status esrnn_trainer_param_info(const esrnn_trainer* t, int32_t idx, esrnn_param_info* o) {
    std::memset(o, 0, sizeof *o);
    const int H = t->H;
    if (idx < 0 || idx >= 3 * t->L + 4) return ESRNN_SHAPE_ERROR;
    if (idx < 3 * t->L) {
        const int l = idx / 3, k = idx % 3;
        if (k == 0) { std::snprintf(o->name, 32, "lstm%d.w_input", l); o->rows = t->layer_in[l]; o->cols = 4 * H; o->offset = t->off_win[l]; }
        if (k == 1) { std::snprintf(o->name, 32, "lstm%d.w_recur", l); o->rows = H; o->cols = 4 * H; o->offset = t->off_wrec[l]; }
        if (k == 2) { std::snprintf(o->name, 32, "lstm%d.bias", l); o->rows = 1; o->cols = 4 * H; o->offset = t->off_bias[l]; }
        return ESRNN_OK;
    }
    switch (idx - 3 * t->L) {
        case 0: std::snprintf(o->name, 32, "head.nl_w"); o->rows = H; o->cols = H; o->offset = t->off_nlw; break;
        case 1: std::snprintf(o->name, 32, "head.nl_b"); o->rows = 1; o->cols = H; o->offset = t->off_nlb; break;
        case 2: std::snprintf(o->name, 32, "head.out_w"); o->rows = H; o->cols = t->O; o->offset = t->off_outw; break;
        default: std::snprintf(o->name, 32, "head.out_b"); o->rows = 1; o->cols = t->O; o->offset = t->off_outb; break;
    }
    return ESRNN_OK;
}

esrnn_status esrnn_trainer_get_weights(esrnn_trainer* t, double* flat, int64_t count) {
    return guarded(t->err, [&] {
        if (count != t->P) raise(ESRNN_SHAPE_ERROR, "get_weights: count %lld != %lld", (long long)count, (long long)t->P);
        CUDA_OK(cudaSetDevice(t->cfg.device));
        sync_weights_from_device(t);
        std::memcpy(flat, t->w_host.data(), sizeof(double) * t->P);
    });
}

esrnn_status esrnn_trainer_set_weights(esrnn_trainer* t, const double* flat, int64_t count) {
    return guarded(t->err, [&] {
        if (count != t->P) raise(ESRNN_CHECKPOINT_ERROR, "checkpoint network shapes incompatible with configuration");
        CUDA_OK(cudaSetDevice(t->cfg.device));
        std::memcpy(t->w_host.data(), flat, sizeof(double) * t->P);
        upload_theta(t);
    });
}

static void ps_io(esrnn_trainer* t, int64_t r0, int64_t n, double* a, double* g, double* s, bool get) {
    const int S = t->S, N = t->N;
    const int64_t lr0 = r0 - t->row0;
    if (n < 0 || lr0 < 0 || lr0 + n > N) raise(ESRNN_SHAPE_ERROR, "per_series: rows [%lld, %lld) not owned by this rank", (long long)r0, (long long)(r0 + n));
    if (n == 0) return;
    CUDA_OK(cudaSetDevice(t->cfg.device));
    std::vector<double> buf(n);
    for (int j = 0; j < 2 + S; ++j) {
        unsigned char* dev = t->ps.p + t->rsz * (static_cast<size_t>(j) * N + lr0);
        double* dst = j == 0 ? a : (j == 1 ? g : nullptr);
        if (get) {
            download_real(t, dev, n, buf.data());
            for (int64_t i = 0; i < n; ++i) {
                if (j < 2) { if (dst) dst[i] = buf[i]; }
                else if (s) s[i * S + (j - 2)] = buf[i];
            }
        } else {
            const double* src = j == 0 ? a : (j == 1 ? g : nullptr);
            if (j < 2 && !src) continue;
            if (j >= 2 && !s) continue;
            for (int64_t i = 0; i < n; ++i) buf[i] = j < 2 ? src[i] : s[i * S + (j - 2)];
            upload_real(t, dev, buf.data(), n);
        }
    }
}

esrnn_status esrnn_trainer_get_per_series(esrnn_trainer* t, int64_t r0, int64_t n, double* a, double* g, double* s) {
    return guarded(t->err, [&] { ps_io(t, r0, n, a, g, s, true); });
}

esrnn_status esrnn_trainer_set_per_series(esrnn_trainer* t, int64_t r0, int64_t n, const double* a, const double* g,
                                          const double* s) {
    return guarded(t->err, [&] {
        ps_io(t, r0, n, const_cast<double*>(a), const_cast<double*>(g), const_cast<double*>(s), false);
    });
}

// ---- exact-resume training state (B200 extension; checkpoint.hpp:37-46 saves neither) ----
esrnn_status esrnn_trainer_get_train_state(esrnn_trainer* t, double* adam_m, double* adam_v, int64_t n_values,
                                           int64_t row_begin, int64_t n, double* ps_m, double* ps_v,
                                           int64_t* ps_steps, int64_t* net_step, char* rng_text, int64_t rng_cap) {
    return guarded(t->err, [&] {
        CUDA_OK(cudaSetDevice(t->cfg.device));
        if (adam_m || adam_v) {
            if (n_values != t->P) raise(ESRNN_CHECKPOINT_ERROR, "train state: %lld network values, expected %lld", (long long)n_values, (long long)t->P);
            const size_t np = static_cast<size_t>(t->lay.P_pad);
            std::vector<double> c(np);
            for (int which = 0; which < 2; ++which) {
                double* dst = which ? adam_v : adam_m;
                if (!dst) continue;
                download_real(t, (which ? t->vW : t->mW).p, np, c.data());
                std::fill(dst, dst + t->P, 0.0);  // structurally dead entries: m = v = 0 (zero gradients)
                for (size_t i = 0; i < np; ++i)
                    if (t->live_flat[i] >= 0) dst[t->live_flat[i]] = c[i];
            }
        }
        const int S = t->S, N = t->N;
        const int64_t lr0 = row_begin - t->row0;
        if (n < 0 || lr0 < 0 || lr0 + n > N) raise(ESRNN_SHAPE_ERROR, "train state: rows not owned by this rank");
        if (n > 0 && (ps_m || ps_v || ps_steps)) {
            std::vector<double> buf(n);
            for (int which = 0; which < 2; ++which) {
                double* dst = which ? ps_v : ps_m;
                if (!dst) continue;
                for (int j = 0; j < 2 + S; ++j) {
                    download_real(t, (which ? t->ps_v : t->ps_m).p + t->rsz * (static_cast<size_t>(j) * N + lr0), n, buf.data());
                    for (int64_t i = 0; i < n; ++i) dst[i * (2 + S) + j] = buf[i];
                }
            }
            if (ps_steps) {
                std::vector<int> st(n);
                CUDA_OK(cudaMemcpy(st.data(), t->ps_steps.p + lr0, sizeof(int) * n, cudaMemcpyDeviceToHost));
                for (int64_t i = 0; i < n; ++i) ps_steps[i] = st[i];
            }
        }
        if (net_step) {
            long long v = 0;
            CUDA_OK(cudaMemcpy(&v, t->net_step.p, sizeof v, cudaMemcpyDeviceToHost));
            *net_step = v;
        }
        if (rng_text) {
            // the trainer RNG before the next epoch's shuffle (the engine plans epochs ahead)
            t->join_plan();
            std::ostringstream os;
            os << (t->next_plan.ready ? t->next_plan.rng_before : t->rng.gen).to_std();
            const std::string txt = os.str();
            if (static_cast<int64_t>(txt.size()) + 1 > rng_cap) raise(ESRNN_SHAPE_ERROR, "train state: rng buffer too small (%zu)", txt.size() + 1);
            std::memcpy(rng_text, txt.c_str(), txt.size() + 1);
        }
    });
}

esrnn_status esrnn_trainer_set_train_state(esrnn_trainer* t, const double* adam_m, const double* adam_v,
                                           int64_t n_values, int64_t row_begin, int64_t n, const double* ps_m,
                                           const double* ps_v, const int64_t* ps_steps, int64_t net_step,
                                           const char* rng_text) {
    return guarded(t->err, [&] {
        CUDA_OK(cudaSetDevice(t->cfg.device));
        if (adam_m || adam_v) {
            if (n_values != t->P) raise(ESRNN_CHECKPOINT_ERROR, "train state: %lld network values, expected %lld", (long long)n_values, (long long)t->P);
            const size_t np = static_cast<size_t>(t->lay.P_pad);
            std::vector<double> c(np);
            for (int which = 0; which < 2; ++which) {
                const double* src = which ? adam_v : adam_m;
                if (!src) continue;
                for (size_t i = 0; i < np; ++i) c[i] = t->live_flat[i] >= 0 ? src[t->live_flat[i]] : 0.0;
                upload_real(t, (which ? t->vW : t->mW).p, c.data(), np);
            }
        }
        const int S = t->S, N = t->N;
        const int64_t lr0 = row_begin - t->row0;
        if (n < 0 || lr0 < 0 || lr0 + n > N) raise(ESRNN_SHAPE_ERROR, "train state: rows not owned by this rank");
        if (n > 0) {
            std::vector<double> buf(n);
            for (int which = 0; which < 2; ++which) {
                const double* src = which ? ps_v : ps_m;
                if (!src) continue;
                for (int j = 0; j < 2 + S; ++j) {
                    for (int64_t i = 0; i < n; ++i) buf[i] = src[i * (2 + S) + j];
                    upload_real(t, (which ? t->ps_v : t->ps_m).p + t->rsz * (static_cast<size_t>(j) * N + lr0), buf.data(), n);
                }
            }
            if (ps_steps) {
                std::vector<int> st(n);
                for (int64_t i = 0; i < n; ++i) st[i] = static_cast<int>(ps_steps[i]);
                CUDA_OK(cudaMemcpy(t->ps_steps.p + lr0, st.data(), sizeof(int) * n, cudaMemcpyHostToDevice));
            }
        }
        if (net_step < 0) raise(ESRNN_CHECKPOINT_ERROR, "train state: negative Adam step");
        const long long v = net_step;
        CUDA_OK(cudaMemcpy(t->net_step.p, &v, sizeof v, cudaMemcpyHostToDevice));
        if (rng_text) {
            std::istringstream is(rng_text);
            std::mt19937_64 g;
            is >> g;
            if (is.fail()) raise(ESRNN_CHECKPOINT_ERROR, "train state: malformed rng state");
            t->join_plan();
            t->rng.gen = Mt64::from_std(g);
            t->next_plan.ready = false;  // re-planned from the restored RNG at the next epoch
        }
    });
}

esrnn_status esrnn_trainer_train_epoch(esrnn_trainer* t, double* mean_loss) {
    return guarded(t->err, [&] {
        CUDA_OK(cudaSetDevice(t->cfg.device));
        const double l = t->fp64 ? train_epoch_impl<double>(t) : train_epoch_impl<float>(t);
        *mean_loss = l;
    });
}

esrnn_status esrnn_trainer_run_batch(esrnn_trainer* t, int32_t B, const int32_t* rows, const int32_t* anchors,
                                     const double* mask, int32_t flags, double* loss, double* mask_count,
                                     double* inputs, double* targets, double* seas, double* levels,
                                     double* net_grads, int32_t* n_slots, int32_t* slot_rows, double* ps_grads) {
    return guarded(t->err, [&] {
        CUDA_OK(cudaSetDevice(t->cfg.device));
        if (t->fp64)
            run_batch_impl<double>(t, B, rows, anchors, mask, flags, loss, mask_count, inputs, targets, seas, levels,
                                   net_grads, n_slots, slot_rows, ps_grads);
        else
            run_batch_impl<float>(t, B, rows, anchors, mask, flags, loss, mask_count, inputs, targets, seas, levels,
                                  net_grads, n_slots, slot_rows, ps_grads);
    });
}

esrnn_status esrnn_trainer_forecast(esrnn_trainer* t, int64_t drop_tail, double* out) {
    return guarded(t->err, [&] {
        CUDA_OK(cudaSetDevice(t->cfg.device));
        if (t->fp64) forecast_impl<double>(t, drop_tail, out, 0, ScoreOut{});
        else forecast_impl<float>(t, drop_tail, out, 0, ScoreOut{});
    });
}

esrnn_status esrnn_trainer_validate(esrnn_trainer* t, double* forecasts, double* smape, double* mean) {
    return guarded(t->err, [&] {
        CUDA_OK(cudaSetDevice(t->cfg.device));
        const int64_t dt = 2 * static_cast<int64_t>(t->O);
        ScoreOut so;
        so.smape = smape;
        so.mean = mean;
        if (t->fp64) forecast_impl<double>(t, dt, forecasts, 1, so);
        else forecast_impl<float>(t, dt, forecasts, 1, so);
    });
}

esrnn_status esrnn_trainer_evaluate(esrnn_trainer* t, int32_t against_test, double* forecasts, double* smape,
                                    double* mase, double* naive_smape, double* naive_mase, double* totals) {
    return guarded(t->err, [&] {
        CUDA_OK(cudaSetDevice(t->cfg.device));
        const int64_t dt = (against_test ? 1 : 2) * static_cast<int64_t>(t->O);
        ScoreOut so;
        so.smape = smape;
        so.mase = mase;
        so.naive_smape = naive_smape;
        so.naive_mase = naive_mase;
        so.totals = totals;
        if (t->fp64) forecast_impl<double>(t, dt, forecasts, 2, so);
        else forecast_impl<float>(t, dt, forecasts, 2, so);
    });
}

esrnn_status esrnn_trainer_forward_stack(esrnn_trainer* t, int32_t seq_len, int32_t B, const double* inputs,
                                         double* out, const double* out_bar, double* weights_bar, double* inputs_bar) {
    return guarded(t->err, [&] {
        CUDA_OK(cudaSetDevice(t->cfg.device));
        if (t->fp64) forward_stack_impl<double>(t, seq_len, B, inputs, out, out_bar, weights_bar, inputs_bar);
        else forward_stack_impl<float>(t, seq_len, B, inputs, out, out_bar, weights_bar, inputs_bar);
    });
}

esrnn_status esrnn_trainer_hw_state(esrnn_trainer* t, int64_t row, int64_t t_len, double* levels, double* seas) {
    return guarded(t->err, [&] {
        CUDA_OK(cudaSetDevice(t->cfg.device));
        if (t->fp64) hw_state_impl<double>(t, row, t_len, levels, seas);
        else hw_state_impl<float>(t, row, t_len, levels, seas);
    });
}

esrnn_status esrnn_trainer_last_epoch_windows(const esrnn_trainer* t, int32_t* rows, int32_t* anchors, int64_t n) {
    if (!t->have_last || n != t->cur_plan.n_windows) return ESRNN_SHAPE_ERROR;
    const uint64_t* w = t->cur_plan.wbuf.data();
    for (int64_t i = 0; i < n; ++i) {
        rows[i] = static_cast<int32_t>(w[i] >> 32);
        anchors[i] = static_cast<int32_t>(static_cast<uint32_t>(w[i]));
    }
    return ESRNN_OK;
}

esrnn_status esrnn_trainer_last_device_ms(const esrnn_trainer* t, double* ms) {
    *ms = t->last_ms;
    return ESRNN_OK;
}

esrnn_status esrnn_trainer_kernel_launches(const esrnn_trainer* t, int64_t* n) {
    *n = t->launches;
    return ESRNN_OK;
}

esrnn_status esrnn_trainer_profile_kernels(esrnn_trainer* t, int32_t enable) {
    t->profiling = enable == 1;
    t->span_mode = enable == 2;
    for (int i = 0; i < ESRNN_KERNEL_CLASSES; ++i) {
        t->prof_ms[i] = 0.0;
        t->prof_n[i] = 0;
    }
    return ESRNN_OK;
}

esrnn_status esrnn_trainer_kernel_times(esrnn_trainer* t, double* total_ms, int64_t* launches) {
    for (int i = 0; i < ESRNN_KERNEL_CLASSES; ++i) {
        if (total_ms) total_ms[i] = t->prof_ms[i];
        if (launches) launches[i] = t->prof_n[i];
    }
    return ESRNN_OK;
}

esrnn_status esrnn_release_cached_memory(void) {
    std::string err;
    return guarded(err, [&] {
        graph_cache().clear();
        BlockCache& c = block_cache();
        std::lock_guard<std::mutex> g(c.mu);
        int dev0 = current_device();
        for (auto& kv : c.dev) {
            cudaSetDevice(kv.first.first);
            for (void* p : kv.second) cudaFree(p);
        }
        for (auto& kv : c.streams) {
            cudaSetDevice(kv.first);
            for (auto& t : kv.second) {
                cudaEventDestroy(static_cast<cudaEvent_t>(t[1]));
                cudaEventDestroy(static_cast<cudaEvent_t>(t[2]));
                cudaStreamDestroy(static_cast<cudaStream_t>(t[0]));
            }
        }
        cudaSetDevice(dev0);
        for (auto& kv : c.host)
            for (void* p : kv.second) cudaFreeHost(p);
        c.dev.clear();
        c.host.clear();
        c.streams.clear();
    });
}

esrnn_status esrnn_group_create(int32_t world_size, esrnn_group** out) {
    *out = nullptr;
    return guarded(g_create_err, [&] {
        if (world_size < 1) raise(ESRNN_CONFIG_ERROR, "group: world_size must be >= 1");
        esrnn_group* g = new esrnn_group();
        g->W = world_size;
        g->deposit.resize(world_size);
        *out = g;
    });
}

void esrnn_group_destroy(esrnn_group* g) {
    if (!g) return;
    bool del = false;
    {
        std::lock_guard<std::mutex> lk(g->mu);
        g->orphaned = true;
        del = g->refs == 0;
    }
    if (del) delete g;
}

esrnn_status esrnn_trainer_gather_per_series(esrnn_trainer* t, double* a, double* g, double* s) {
    return guarded(t->err, [&] {
        CUDA_OK(cudaSetDevice(t->cfg.device));
        const int S = t->S, np = 2 + S;
        // this rank's rows as [row][alpha, gamma, seas...], padded to the largest shard
        const int64_t maxn = (static_cast<int64_t>(t->N_global) + t->world - 1) / t->world + 1;
        std::vector<double> a0(t->N), g0(t->N), s0(static_cast<size_t>(t->N) * S);
        ps_io(t, t->row0, t->N, a0.data(), g0.data(), s0.data(), true);
        std::vector<double> mine(static_cast<size_t>(maxn) * np, 0.0);
        for (int i = 0; i < t->N; ++i) {
            mine[static_cast<size_t>(i) * np] = a0[i];
            mine[static_cast<size_t>(i) * np + 1] = g0[i];
            for (int j = 0; j < S; ++j) mine[static_cast<size_t>(i) * np + 2 + j] = s0[static_cast<size_t>(i) * S + j];
        }
        const std::vector<double> all = t->sharded ? allgather_host(t, mine) : mine;
        const int W = t->sharded ? t->world : 1;
        for (int r = 0; r < W; ++r) {
            const int64_t b = t->sharded ? (static_cast<int64_t>(r) * t->N_global) / t->world : t->row0;
            const int64_t e = t->sharded ? (static_cast<int64_t>(r + 1) * t->N_global) / t->world : t->row0 + t->N;
            const double* src = all.data() + static_cast<size_t>(r) * maxn * np;
            for (int64_t i = 0; i < e - b; ++i) {
                if (a) a[b + i] = src[i * np];
                if (g) g[b + i] = src[i * np + 1];
                if (s)
                    for (int j = 0; j < S; ++j) s[(b + i) * S + j] = src[i * np + 2 + j];
            }
        }
    });
}

esrnn_status esrnn_nccl_unique_id(uint8_t out[128]) {
    return guarded(g_create_err, [&] {
        ncclUniqueId id;
        NCCL_OK(ncclGetUniqueId(&id));
        std::memcpy(out, id.internal, 128);
    });
}

}  // extern "C"
