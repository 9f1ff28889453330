// Forecast-side Holt-Winters scan (the training scan runs in K2's prologue, tile.cuh).
//
//   K6 k_forecast_scan  forecast scan over values[0:t_ins) + window build (holt_winters.hpp:66-97,
//                       deseasonalize_normalize :153-166, HWState::seasonal_at :55-59); with
//                       `score`, also the series' MASE scale and the seasonal-naive scores
//                       (metrics.hpp:33-59, commands.hpp:285-308) from the staged column
//
// One thread per series.  The whole observation column is first staged into shared
// memory with every load in flight at once, the last S seasonalities live in a
// shared-memory ring, so the recurrence waits only on its own FMA chain
// (l_t = a*y/s_t + (1-a)*l_{t-1}; the division feeding s_{t+S} has S steps of slack).
#pragma once
#include "common.cuh"

namespace esrnn_dev {

constexpr int kScanThreads = 64;

// Stage y[0:n) of this thread's series (stride N in global) into ys[t*bd] (shared).
// All n element copies are issued back to back as cp.async (LDGSTS) and waited once.
template <typename Real>
__device__ __forceinline__ void stage_column(Real* ys, const Real* __restrict__ y, int n, int N, int bd) {
#pragma unroll 8
    for (int t = 0; t < n; ++t) cp_async_elem(ys + t * bd, y + (size_t)t * N);
    cp_async_wait_all();
}

// ------------------------------------------------------------------------------ K6
// smem: ys [t_ins][bd] | ring [S][bd] | win [I][bd]
// SC > 0: the season length as a compile-time constant (1, 4, 12): the S live
// seasonalities sit in registers and the recurrence is unrolled by S, so each step is its
// FMA chain with the error checks folded into a select (flagged after the loop, at the
// first failing t, as the reference throws there); SC = 0: any S, ring in shared memory.
template <typename Real, int SC = 0>
__global__ void __launch_bounds__(kScanThreads) k_forecast_scan(StateDev<Real> st, NetLayout lay, int t_ins, Real* X,
                                                                Real* FL, Real* FS, Real* dump_lv, Real* dump_se,
                                                                int dump_row, double* score) {
    using M = Math<Real>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int S = SC > 0 ? SC : lay.S, I = lay.I, O = lay.O, in0 = lay.in0, N = st.N;
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= N) return;
    const int bd = blockDim.x, tid = threadIdx.x;
    Real* ys = reinterpret_cast<Real*>(smem_raw) + tid;
    Real* ring = reinterpret_cast<Real*>(smem_raw) + t_ins * bd + tid;
    Real* win = ring + S * bd;
    for (int j = 0; j < S; ++j) cp_async_elem(ring + j * bd, st.ps + (size_t)(2 + j) * N + row);
    const Real a_raw = st.ps[row], g_raw = st.ps[N + row];
    stage_column(ys, st.vals + row, t_ins, N, bd);
    {
        int bad = INT_MAX;  // first non-positive observation (a select per t, no exit branch)
#pragma unroll 8
        for (int t = t_ins - 1; t >= 0; --t) bad = (ys[t * bd] > Real(0)) ? bad : t;
        if (bad != INT_MAX) {
            flag_error(st.err, kErrObs, bad);
            return;
        }
    }
    if (score != nullptr) {
        // mase(): in-sample seasonal-naive MAE over y[0:t_ins) (metrics.hpp:40-44); the
        // seasonal-naive forecast y[t_ins-S+(o mod S)] (metrics.hpp:52-59) scored with
        // smape() (:17-28) and mase() against the held-out block y[t_ins:t_ins+O)
        double den = 0.0;
        for (int t = S; t < t_ins; ++t)
            den += fabs(static_cast<double>(ys[t * bd]) - static_cast<double>(ys[(t - S) * bd]));
        den /= static_cast<double>(t_ins - S);
        double acc = 0.0, mae = 0.0;
        for (int o = 0; o < O; ++o) {
            const double f = static_cast<double>(ys[(t_ins - S + o % S) * bd]);
            const double a = static_cast<double>(st.vals[(size_t)(t_ins + o) * N + row]);
            const double d = fabs(a) + fabs(f);
            if (d > 0.0) acc += fabs(a - f) / d;
            mae += fabs(a - f);
        }
        score[row] = den;
        score[N + row] = 200.0 * acc / static_cast<double>(O);
        score[2 * N + row] = den == 0.0 ? NAN : (mae / static_cast<double>(O)) / den;
    }
    const bool dump = row == dump_row;
    const Real alpha = M::logistic_ps(a_raw);
    const Real gamma = M::logistic_ps(g_raw);
    const Real oma = Real(1) - alpha, omg = Real(1) - gamma;
    Real lp = 0;
    for (int j = 0; j < S; ++j) {
        const Real s0 = M::exp_ps(ring[j * bd]);
        ring[j * bd] = s0;
        if (dump) dump_se[j] = s0;
        lp += ys[j * bd];
    }
    lp = lp / Real(S);
    // seasonality index u is produced at step u-S; the window needs u in [t_ins-I, t_ins)
    for (int u = t_ins - I; u < S && u < t_ins; ++u)
        if (u >= 0) win[(u - (t_ins - I)) * bd] = ring[u * bd];
    if constexpr (SC > 0) {
        Real rg[SC];
#pragma unroll
        for (int q = 0; q < SC; ++q) rg[q] = ring[q * bd];
        int bad = INT_MAX;
        for (int t0 = 0; t0 < t_ins; t0 += SC) {
#pragma unroll
            for (int q = 0; q < SC; ++q) {
                const int t = t0 + q;
                if (t < t_ins) {  // warp-uniform
                    const Real yt = ys[t * bd];
                    const Real s_t = rg[q];
                    const Real l = alpha * fdiv(yt, s_t) + oma * lp;
                    bad = (bad == INT_MAX && !(l > Real(0) && isfinite(l))) ? t : bad;
                    const Real sn = gamma * fdiv(yt, lp) + omg * s_t;
                    rg[q] = sn;
                    const int uu = t + S;
                    if (uu >= t_ins - I && uu < t_ins) win[(uu - (t_ins - I)) * bd] = sn;
                    if (dump) {
                        dump_lv[t] = l;
                        dump_se[uu] = sn;
                    }
                    lp = l;
                }
            }
        }
        if (bad != INT_MAX) {
            flag_error(st.err, kErrFcLevel, bad);
            return;
        }
        // slot q holds the seasonality of the index u = q (mod S) in [t_ins, t_ins + S)
#pragma unroll
        for (int q = 0; q < SC; ++q) ring[q * bd] = rg[q];
    } else {
        int j = 0;
        for (int t = 0; t < t_ins; ++t) {
            const Real yt = ys[t * bd];
            const Real s_t = ring[j * bd];
            const Real l = alpha * fdiv(yt, s_t) + oma * lp;
            if (!(l > Real(0)) || !isfinite(l)) {
                flag_error(st.err, kErrFcLevel, t);
                return;
            }
            const Real sn = gamma * fdiv(yt, lp) + omg * s_t;
            ring[j * bd] = sn;
            const int uu = t + S;
            if (uu >= t_ins - I && uu < t_ins) win[(uu - (t_ins - I)) * bd] = sn;
            if (dump) {
                dump_lv[t] = l;
                dump_se[uu] = sn;
            }
            lp = l;
            j = (j + 1 == S) ? 0 : j + 1;
        }
    }
    if (X == nullptr) return;
    const Real level = lp;
    for (int c = 0; c < I; ++c) {
        const Real sv = win[c * bd];
        if (!(sv > Real(0))) {
            flag_error(st.err, kErrSeas, t_ins);
            return;
        }
        X[(size_t)row * in0 + c] = fdiv(ys[(t_ins - I + c) * bd], level * sv);
    }
    for (int c = 0; c < 6; ++c) X[(size_t)row * in0 + I + c] = (st.cat[row] == c) ? Real(1) : Real(0);
    FL[row] = level;
    // seasonal_at(t_ins + o): indices [t_ins, t_ins+S) sit in ring slot (index mod S)
    for (int o = 0; o < O; ++o) {
        int idx = t_ins + o;
        while (idx >= t_ins + S) idx -= S;
        FS[(size_t)row * O + o] = ring[(idx % S) * bd];
    }
}

// ------------------------------------------------------------------------------ K6, S fixed
// k_forecast_scan for the M4 season lengths (SC = 1, 4, 12), restructured for bandwidth:
//  * every global input is requested up front (observation column, seasonality raws, alpha,
//    gamma, category), then one wait;
//  * the recurrence runs in two loops: steps whose new seasonality is not in the input window
//    (no window stores, no checks beyond the level select), then the last steps that produce
//    the window's seasonalities; the hw_state dump is a separate instantiation (DUMP);
//  * the outputs (window row X, anchor level, the horizon's seasonalities) are staged in shared
//    memory and written by the whole block: the block's rows are contiguous in X / FS / FL,
//    so every store is coalesced (a thread's own row stores touch 32 rows per instruction).
// smem: ys [t_ins][bd] | ring [S][bd] | win [I][bd] | ox [bd][in0] | ofs [bd][O] | ofl [bd]
template <typename Real, int SC, bool DUMP>
__global__ void __launch_bounds__(kScanThreads) k_forecast_scan_sc(StateDev<Real> st, NetLayout lay, int t_ins, Real* X,
                                                                   Real* FL, Real* FS, Real* dump_lv, Real* dump_se,
                                                                   int dump_row, double* score) {
    using M = Math<Real>;
    constexpr int S = SC;
    constexpr Real kMax = sizeof(Real) == 4 ? Real(FLT_MAX) : Real(DBL_MAX);
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int I = lay.I, O = lay.O, in0 = lay.in0, N = st.N;
    const int bd = blockDim.x, tid = threadIdx.x;
    const int row0 = blockIdx.x * bd, nrow = min(bd, N - row0);
    const int row = row0 + tid;
    const bool live = tid < nrow;
    Real* ys = reinterpret_cast<Real*>(smem_raw) + tid;
    Real* ring = reinterpret_cast<Real*>(smem_raw) + t_ins * bd + tid;
    Real* win = ring + S * bd;
    Real* ox = reinterpret_cast<Real*>(smem_raw) + (t_ins + S + I) * bd;  // [bd][in0]
    Real* ofs = ox + bd * in0;                                            // [bd][O]
    Real* ofl = ofs + bd * O;                                             // [bd]
    Real a_raw = 0, g_raw = 0;
    int cat = 5;
    if (live) {
#pragma unroll
        for (int j = 0; j < S; ++j) cp_async_elem(ring + j * bd, st.ps + (size_t)(2 + j) * N + row);
#pragma unroll 8
        for (int t = 0; t < t_ins; ++t) cp_async_elem(ys + t * bd, st.vals + (size_t)t * N + row);
        a_raw = st.ps[row];
        g_raw = st.ps[N + row];
        cat = st.cat[row];
    }
    cp_async_wait_all();
    bool ok = live;
    if (live) {
        int bad = INT_MAX;  // first non-positive observation
#pragma unroll 8
        for (int t = t_ins - 1; t >= 0; --t) bad = (ys[t * bd] > Real(0)) ? bad : t;
        if (bad != INT_MAX) {
            flag_error(st.err, kErrObs, bad);
            ok = false;
        }
    }
    if (ok && score != nullptr) {
        // mase() denominator, seasonal-naive sMAPE / MASE (metrics.hpp:17-59)
        double den = 0.0;
        for (int t = S; t < t_ins; ++t)
            den += fabs(static_cast<double>(ys[t * bd]) - static_cast<double>(ys[(t - S) * bd]));
        den /= static_cast<double>(t_ins - S);
        double acc = 0.0, mae = 0.0;
        for (int o = 0; o < O; ++o) {
            const double f = static_cast<double>(ys[(t_ins - S + o % S) * bd]);
            const double a = static_cast<double>(st.vals[(size_t)(t_ins + o) * N + row]);
            const double d = fabs(a) + fabs(f);
            if (d > 0.0) acc += fabs(a - f) / d;
            mae += fabs(a - f);
        }
        score[row] = den;
        score[N + row] = 200.0 * acc / static_cast<double>(O);
        score[2 * N + row] = den == 0.0 ? NAN : (mae / static_cast<double>(O)) / den;
    }
    Real lp = 0;
    if (ok) {
        const Real alpha = M::logistic_ps(a_raw);
        const Real gamma = M::logistic_ps(g_raw);
        const Real oma = Real(1) - alpha, omg = Real(1) - gamma;
        Real rg[SC];
#pragma unroll
        for (int j = 0; j < S; ++j) {
            rg[j] = M::exp_ps(ring[j * bd]);
            if (DUMP && row == dump_row) dump_se[j] = rg[j];
            lp += ys[j * bd];
        }
        lp = lp / Real(S);
        const int w0 = t_ins - I;  // first window index; seasonality u is produced at step u - S
        for (int u = max(w0, 0); u < S && u < t_ins; ++u) win[(u - w0) * bd] = rg[u];
        int bad = INT_MAX;
        auto step = [&](int t, Real& sq, bool tail) {
            const Real yt = ys[t * bd];
            const Real l = alpha * fdiv(yt, sq) + oma * lp;
            bad = (bad == INT_MAX && !(l > Real(0) && l <= kMax)) ? t : bad;
            sq = gamma * fdiv(yt, lp) + omg * sq;
            if (tail) {
                const int uu = t + S;
                if (uu >= w0 && uu < t_ins) win[(uu - w0) * bd] = sq;
            }
            if (DUMP && row == dump_row) {
                dump_lv[t] = l;
                dump_se[t + S] = sq;
            }
            lp = l;
        };
        // steps t < w0 - S produce indices below the window: no stores
        const int t_free = max(0, min(t_ins, w0 - S));
        int t0 = 0;
        for (; t0 + SC <= t_free; t0 += SC) {
#pragma unroll
            for (int q = 0; q < SC; ++q) step(t0 + q, rg[q], false);
        }
        for (; t0 < t_ins; t0 += SC) {
#pragma unroll
            for (int q = 0; q < SC; ++q)
                if (t0 + q < t_ins) step(t0 + q, rg[q], true);  // warp-uniform
        }
        if (bad != INT_MAX) {
            flag_error(st.err, kErrFcLevel, bad);
            ok = false;
        }
        // slot q holds the seasonality of index u = q (mod S) in [t_ins, t_ins + S)
        if (ok && X != nullptr) {
            const Real level = lp;
            for (int c = 0; c < I; ++c) {
                const Real sv = win[c * bd];
                if (!(sv > Real(0))) {
                    flag_error(st.err, kErrSeas, t_ins);
                    ok = false;
                    break;
                }
                ox[tid * in0 + c] = fdiv(ys[(t_ins - I + c) * bd], level * sv);
            }
            for (int c = 0; c < 6; ++c) ox[tid * in0 + I + c] = (cat == c) ? Real(1) : Real(0);
            ofl[tid] = level;
            for (int o = 0; o < O; ++o) {  // seasonal_at(t_ins + o): ring slot (t_ins + o) mod S
                const int slot = (t_ins + o) % S;
                Real v = rg[0];
#pragma unroll
                for (int q = 1; q < SC; ++q) v = slot == q ? rg[q] : v;
                ofs[tid * O + o] = v;
            }
        }
    }
    if (X == nullptr) return;  // (uniform) hw_state: nothing staged
    __syncthreads();
    // coalesced block stores of the contiguous output rows
    for (int e = tid; e < nrow * in0; e += bd) X[(size_t)row0 * in0 + e] = ox[e];
    for (int e = tid; e < nrow * O; e += bd) FS[(size_t)row0 * O + e] = ofs[e];
    for (int e = tid; e < nrow; e += bd) FL[row0 + e] = ofl[e];
}

}  // namespace esrnn_dev
