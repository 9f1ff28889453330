// sm_100a kernels of the ES-RNN training / forecasting step.
//
// One training step (reference: Trainer::step = build_graph + Tape::backward +
// apply_updates, trainer.hpp:484-655) is five launches on one stream, captured once per
// trainer into a CUDA graph covering the whole epoch:
//
//   K1 k_scan_fwd      slot-parallel Holt-Winters level/seasonality scan   (holt_winters.hpp:236-283)
//   K2 k_stack<TRAIN>  row-tile-parallel: window gather/normalise (trainer.hpp:524-566),
//                      LSTM stack fwd at sequence length 1 (network.hpp:148-210), masked
//                      pinball (autodiff.hpp:370-395) and its adjoint (:611-628), the whole
//                      stack adjoint, per-tile weight-gradient partials, per-window ES
//                      adjoint contributions
//   K4 k_es_bwd        slot-parallel: gathers its windows' contributions in batch order
//                      (Gather adjoint, autodiff.hpp:603-610) then the reverse HW scan
//   K3 k_net_reduce    parameter-parallel fixed-order reduction of the tile partials,
//                      squared norms, last-CTA finalisation of clip scale / bias
//                      corrections / loss (trainer.hpp:603-620)
//   K5 k_adam          parameter- and slot-parallel Adam (trainer.hpp:617-655)
//
// Every reduction has a fixed order (tile order, slot-window CSR order, CTA order), so a
// run is bit-reproducible on a given GPU count; no float atomics anywhere.
//
// Layout in HBM: values time-major y[t][N] (coalesced across series), per-series
// parameters / Adam moments SoA [(2+S)][N], shared parameters in a compact "live" layout
// that drops the structurally-dead forget-gate columns and recurrent matrices (their
// gradients are exactly zero at sequence length 1), scan state
// [t][slot].
#pragma once
#include <cstdint>

#include "devmath.cuh"

namespace esrnn_dev {

constexpr int kMaxLayers = 16;

// Compact live layout of the shared parameters and the network shape.
struct NetLayout {
    int L, nb, H, O, I, S, in0, T;
    int layer_in[kMaxLayers];
    int res_src[kMaxLayers];     // >=0: layer output index added as residual after this layer (-2: x)
    int block_first[kMaxLayers]; // 1 if layer is the first of a block b>0 (adjoint joins the residual)
    int block_last[kMaxLayers];  // 1 if layer is the last of a block b>0 (residual added here)
    long long cw[kMaxLayers], cb[kMaxLayers];
    long long c_nlw, c_nlb, c_outw, c_outb, P_live;
};

// Per-epoch (or single-batch) plan: windows in global batch order, filtered to the
// rows this rank owns, with per-step slot lists and per-slot window CSR.
struct PlanDev {
    const int* w_row;         // local row of each window
    const int* w_anchor;
    const int* w_slot;        // slot within its step
    const int* step_win_off;  // [steps+1]
    const int* step_slot_off; // [steps+1]
    const int* slot_row;      // local row of each slot
    const int* slot_win_off;  // [total_slots+1] into slot_win
    const int* slot_win;      // window index relative to its step's first window
    const double* step_M;     // global mask count per step
    const unsigned char* mask;// [window][O] or nullptr (all ones)
};

template <typename Real>
struct StateDev {
    const Real* vals;       // [LEN][N] time-major, local rows
    const signed char* cat; // [N]
    int N, LEN, kcap;
    Real* ps;               // [(2+S)][N]: alpha_raw, gamma_raw, seas_raw[S]
    Real* ps_m;
    Real* ps_v;
    int* ps_steps;
    Real* theta;            // [P_live]
    Real* mW;
    Real* vW;
    // scratch
    Real* lv;               // [T][kcap]
    Real* se;               // [T+S][kcap]
    Real* lbar;             // [T][kcap]
    Real* sbar;             // [T+S][kcap]
    Real* cI;               // [Bcap][I]   ES adjoint contributions per window
    Real* cO;               // [Bcap][O]
    Real* cl;               // [Bcap]
    Real* part;             // [tiles][P_live]
    double* loss_part;      // [tiles]
    Real* gbuf;             // [P_live + 2]  (comm buffer: grads | ps sq-norm | loss sum)
    Real* psg;              // [kcap][2+S]
    double* es_sq_part;     // [es blocks]
    double* red_sq_part;    // [reduce blocks]
    unsigned int* done_ctr; // [2]
    double* scal;           // [4] scale, bc1, bc2, loss
    long long* net_step;
    double* loss_hist;      // [steps]
    int* err;               // [2] code, min t
    // optional dumps (run_batch): WindowBatch matrices, step-local window order
    Real* d_inputs;
    Real* d_targets;
    Real* d_seas;
    Real* d_levels;
    double tau, lr_net, lr_ps, clip;
    int has_clip, attach;
};

enum ErrCode { kErrNone = 0, kErrTrainLevel = 1, kErrObs = 2, kErrFcLevel = 3, kErrSeas = 4 };

__device__ __forceinline__ void flag_error(int* err, int code, int t) {
    atomicMin(err + 1, t);
    atomicCAS(err, 0, code);
}

template <typename T>
__device__ __forceinline__ T block_sum(T v, T* red) {
    // fixed-order block reduction (warp shuffles then warp 0), deterministic
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[wid] = v;
    __syncthreads();
    T r = 0;
    if (threadIdx.x == 0)
        for (int w = 0; w < nw; ++w) r += red[w];
    __syncthreads();
    return r;  // valid in thread 0
}

// ------------------------------------------------------------------------------ K1
// hybrid_primer_tape forward (holt_winters.hpp:245-277): one thread per slot; the last
// S seasonalities live in a shared-memory ring so the recurrence never waits on L2.
template <typename Real>
__global__ void k_scan_fwd(StateDev<Real> st, PlanDev pl, NetLayout lay, int s) {
    using M = Math<Real>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Real* ring = reinterpret_cast<Real*>(smem_raw);
    const int k0 = pl.step_slot_off[s];
    const int k = pl.step_slot_off[s + 1] - k0;
    const int slot = blockIdx.x * blockDim.x + threadIdx.x;
    if (slot >= k) return;
    const int bd = blockDim.x, tid = threadIdx.x;
    const int N = st.N, S = lay.S, T = lay.T, kc = st.kcap;
    const int row = pl.slot_row[k0 + slot];
    const Real alpha = M::logistic_ps(st.ps[row]);
    const Real gamma = M::logistic_ps(st.ps[N + row]);
    const Real oma = Real(1) - alpha, omg = Real(1) - gamma;
    Real lp = 0;
    for (int j = 0; j < S; ++j) {
        const Real s0 = M::exp_ps(st.ps[(2 + j) * N + row]);
        ring[j * bd + tid] = s0;
        st.se[j * kc + slot] = s0;
        lp += st.vals[j * N + row];
    }
    lp = lp / Real(S);
    int bad = -1;
    int j = 0;
#pragma unroll 4
    for (int t = 0; t < T; ++t) {
        const Real yt = st.vals[t * N + row];
        const Real s_t = ring[j * bd + tid];
        const Real l = alpha * (yt / s_t) + oma * lp;
        if (!(l > Real(0)) || !isfinite(l)) bad = bad < 0 ? t : bad;
        const Real sn = gamma * (yt / lp) + omg * s_t;
        ring[j * bd + tid] = sn;
        st.se[(t + S) * kc + slot] = sn;
        st.lv[t * kc + slot] = l;
        lp = l;
        j = (j + 1 == S) ? 0 : j + 1;
    }
    if (bad >= 0) flag_error(st.err, kErrTrainLevel, bad);
}

// ------------------------------------------------------------------------------ K2
enum StackMode { kTrain = 0, kLossOnly = 1, kForecast = 2 };

struct ForecastArgs {
    const float* dummy;
    int t_ins;
    int validate;
    const void* X;       // [N][in0] Real
    const void* lvl;     // [N] Real
    const void* sout;    // [N][O] Real
    double* out;         // [N][O]
    double* smape;       // [N]
};

// Shared-memory carve-up of one row tile (all in Real units).
struct TileSmem {
    int xin, sin, sout, lvl, tgt, msk, act, gates, z, pred, pbar, pre, hbar, resid, ubar, wsm, total;
    int ldw, max_in;
    __host__ __device__ static TileSmem make(const NetLayout& lay, int R) {
        TileSmem t;
        const int H = lay.H, O = lay.O, I = lay.I, in0 = lay.in0, L = lay.L;
        const int G = 3 * H;
        t.max_in = in0 > H ? in0 : H;
        t.ldw = (G > H ? G : H) + 1;
        int o = 0;
        t.xin = o; o += R * in0;
        t.sin = o; o += R * I;
        t.sout = o; o += R * O;
        t.lvl = o; o += R;
        t.tgt = o; o += R * O;
        t.msk = o; o += R * O;
        t.act = o; o += L * R * H;
        t.gates = o; o += 4 * L * R * H;
        t.z = o; o += R * H;
        t.pred = o; o += R * O;
        t.pbar = o; o += R * O;
        t.pre = o; o += R * G;
        t.hbar = o; o += R * H;
        t.resid = o; o += R * H;
        t.ubar = o; o += R * t.max_in;
        o = (o + 3) & ~3;
        t.wsm = o; o += t.max_in * t.ldw;
        t.total = o;
        return t;
    }
};

template <typename Real>
__device__ __forceinline__ void stage_matrix(Real* dst, int ld, const Real* src, int rows, int cols) {
    for (int e = threadIdx.x; e < rows * cols; e += blockDim.x) {
        const int r = e / cols, c = e - r * cols;
        dst[r * ld + c] = src[e];
    }
}

// Row tile of R windows (kTrain / kLossOnly) or R series (kForecast).
template <typename Real, int R, int MODE>
__global__ void __launch_bounds__(256) k_stack(StateDev<Real> st, PlanDev pl, NetLayout lay, int s,
                                               ForecastArgs fa) {
    using M = Math<Real>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Real* sm = reinterpret_cast<Real*>(smem_raw);
    __shared__ double red[32];
    const TileSmem ts = TileSmem::make(lay, R);
    const int H = lay.H, O = lay.O, I = lay.I, in0 = lay.in0, L = lay.L, G = 3 * H, S = lay.S;
    const int tid = threadIdx.x, NT = blockDim.x;
    const int tile = blockIdx.x;
    const Real* th = st.theta;

    Real* xin = sm + ts.xin;
    Real* s_in = sm + ts.sin;
    Real* s_out = sm + ts.sout;
    Real* lvl = sm + ts.lvl;
    Real* tgt = sm + ts.tgt;
    Real* msk = sm + ts.msk;
    Real* act = sm + ts.act;
    Real* gates = sm + ts.gates;
    Real* z = sm + ts.z;
    Real* pred = sm + ts.pred;
    Real* pbar = sm + ts.pbar;
    Real* pre = sm + ts.pre;
    Real* hbar = sm + ts.hbar;
    Real* resid = sm + ts.resid;
    Real* ubar = sm + ts.ubar;
    Real* wsm = sm + ts.wsm;
    const int ldw = ts.ldw;

    int nrows, w0 = 0;
    if (MODE == kForecast) {
        nrows = min(R, st.N - tile * R);
    } else {
        w0 = pl.step_win_off[s];
        const int Bl = pl.step_win_off[s + 1] - w0;
        nrows = min(R, Bl - tile * R);
    }
    if (nrows <= 0) return;

    // ---- prologue: window gather + normalisation (trainer.hpp:532-566) -------------
    if (MODE == kForecast) {
        const Real* X = reinterpret_cast<const Real*>(fa.X);
        const Real* FL = reinterpret_cast<const Real*>(fa.lvl);
        const Real* FS = reinterpret_cast<const Real*>(fa.sout);
        for (int e = tid; e < R * in0; e += NT) {
            const int r = e / in0, c = e - r * in0;
            xin[e] = r < nrows ? X[(size_t)(tile * R + r) * in0 + c] : Real(0);
        }
        for (int e = tid; e < R * O; e += NT) {
            const int r = e / O;
            s_out[e] = r < nrows ? FS[(size_t)(tile * R) * O + e] : Real(0);
        }
        for (int r = tid; r < R; r += NT) lvl[r] = r < nrows ? FL[tile * R + r] : Real(0);
    } else {
        for (int e = tid; e < R * (I + O + 1); e += NT) {
            const int r = e / (I + O + 1), c = e - r * (I + O + 1);
            const int wb = w0 + tile * R + r;
            if (r >= nrows) {
                if (c < I) { xin[r * in0 + c] = 0; s_in[r * I + c] = 1; }
                else if (c < I + O) { tgt[r * O + c - I] = 0; s_out[r * O + c - I] = 1; msk[r * O + c - I] = 0; }
                else lvl[r] = 1;
                continue;
            }
            const int row = pl.w_row[wb], a = pl.w_anchor[wb], slot = pl.w_slot[wb];
            const Real l = st.lv[a * st.kcap + slot];
            if (c < I) {
                const int idx = a - I + 1 + c;
                const Real sv = st.se[idx * st.kcap + slot];
                xin[r * in0 + c] = st.vals[(size_t)idx * st.N + row] / (sv * l);
                s_in[r * I + c] = sv;
            } else if (c < I + O) {
                const int j = c - I, idx = a + 1 + j;
                const Real sv = st.se[idx * st.kcap + slot];
                tgt[r * O + j] = st.vals[(size_t)idx * st.N + row] / (sv * l);
                s_out[r * O + j] = sv;
                msk[r * O + j] = (pl.mask == nullptr || pl.mask[(size_t)wb * O + j] != 0) ? Real(1) : Real(0);
            } else {
                lvl[r] = l;
            }
        }
        for (int e = tid; e < R * 6; e += NT) {
            const int r = e / 6, c = e - r * 6;
            Real v = 0;
            if (r < nrows) v = (st.cat[pl.w_row[w0 + tile * R + r]] == c) ? Real(1) : Real(0);
            xin[r * in0 + I + c] = v;
        }
    }
    __syncthreads();
    if (MODE != kForecast && st.d_inputs != nullptr) {
        const int base = tile * R;
        for (int e = tid; e < nrows * in0; e += NT) st.d_inputs[(size_t)base * in0 + e] = xin[e];
        for (int e = tid; e < nrows * O; e += NT) {
            st.d_targets[(size_t)base * O + e] = tgt[e];
            st.d_seas[(size_t)base * O + e] = s_out[e];
        }
        for (int r = tid; r < nrows; r += NT) st.d_levels[base + r] = lvl[r];
    }

    // ---- forward through the stack (network.hpp:148-210, sequence length 1) --------
    for (int l = 0; l < L; ++l) {
        const int in = lay.layer_in[l];
        const Real* u = l == 0 ? xin : act + (l - 1) * R * H;
        stage_matrix(wsm, ldw, th + lay.cw[l], in, G);
        __syncthreads();
        for (int q = tid; q < G; q += NT) {
            Real acc[R];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = 0;
            for (int k = 0; k < in; ++k) {
                const Real w = wsm[k * ldw + q];
#pragma unroll
                for (int r = 0; r < R; ++r) acc[r] += u[r * in + k] * w;
            }
            const Real b = th[lay.cb[l] + q];
#pragma unroll
            for (int r = 0; r < R; ++r) pre[r * G + q] = acc[r] + b;
        }
        __syncthreads();
        Real* gi = gates + (4 * l + 0) * R * H;
        Real* gg = gates + (4 * l + 1) * R * H;
        Real* go = gates + (4 * l + 2) * R * H;
        Real* gt = gates + (4 * l + 3) * R * H;
        Real* out = act + l * R * H;
        const Real* radd = lay.block_last[l] ? (lay.res_src[l] >= 0 ? act + lay.res_src[l] * R * H : xin) : nullptr;
        for (int e = tid; e < R * H; e += NT) {
            const int r = e / H, hh = e - r * H;
            const Real i = M::logistic(pre[r * G + hh]);
            const Real g = M::tanh(pre[r * G + H + hh]);
            const Real o = M::logistic(pre[r * G + 2 * H + hh]);
            const Real c = i * g;
            const Real tc = M::tanh(c);
            Real h = o * tc;
            if (radd) h = h + radd[e];
            gi[e] = i;
            gg[e] = g;
            go[e] = o;
            gt[e] = tc;
            out[e] = h;
        }
        __syncthreads();
    }
    // head (network.hpp:207-209)
    const Real* cur = act + (L - 1) * R * H;
    stage_matrix(wsm, ldw, th + lay.c_nlw, H, H);
    __syncthreads();
    for (int j = tid; j < H; j += NT) {
        Real acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = 0;
        for (int k = 0; k < H; ++k) {
            const Real w = wsm[k * ldw + j];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] += cur[r * H + k] * w;
        }
        const Real b = th[lay.c_nlb + j];
#pragma unroll
        for (int r = 0; r < R; ++r) z[r * H + j] = M::tanh(acc[r] + b);
    }
    __syncthreads();
    double lsum = 0.0;
    const Real* ow = th + lay.c_outw;
    for (int e = tid; e < R * O; e += NT) {
        const int r = e / O, o = e - r * O;
        Real acc = 0;
        for (int k = 0; k < H; ++k) acc += z[r * H + k] * ow[k * O + o];
        const Real p = acc + th[lay.c_outb + o];
        pred[e] = p;
        if (MODE == kForecast) {
            if (r < nrows) {
                const int row = tile * R + r;
                const double f = static_cast<double>(p * lvl[r] * s_out[e]);
                fa.out[(size_t)row * O + o] = f;
            }
        } else {
            // masked pinball (autodiff.hpp:384-392) and its adjoint (:620-626)
            Real pb = 0;
            if (msk[e] != Real(0)) {
                const Real d = tgt[e] - p;
                lsum += (d >= Real(0)) ? static_cast<double>(st.tau) * d : (static_cast<double>(st.tau) - 1.0) * d;
                const Real gscale = static_cast<Real>(1.0 / pl.step_M[s]);
                pb = gscale * ((tgt[e] >= p) ? -static_cast<Real>(st.tau) : Real(1) - static_cast<Real>(st.tau));
            }
            pbar[e] = pb;
        }
    }
    if (MODE == kForecast) {
        if (fa.validate) {
            __syncthreads();
            // sMAPE against the validation block (metrics.hpp:17-28)
            for (int r = tid; r < nrows; r += NT) {
                const int row = tile * R + r;
                double acc = 0.0;
                for (int o = 0; o < O; ++o) {
                    const double a = static_cast<double>(st.vals[(size_t)(lay.T + o) * st.N + row]);
                    const double f = fa.out[(size_t)row * O + o];
                    const double den = fabs(a) + fabs(f);
                    if (den > 0.0) acc += fabs(a - f) / den;
                }
                fa.smape[row] = 200.0 * acc / static_cast<double>(O);
            }
        }
        return;
    }
    const double ltot = block_sum(lsum, red);
    if (tid == 0) st.loss_part[tile] = ltot;
    if (MODE == kLossOnly) return;
    __syncthreads();

    // ---- backward: head ------------------------------------------------------------
    Real* part = st.part + (size_t)tile * lay.P_live;
    for (int e = tid; e < (H + 1) * O; e += NT) {
        Real acc = 0;
        if (e < H * O) {
            const int k = e / O, o = e - k * O;
#pragma unroll
            for (int r = 0; r < R; ++r) acc += z[r * H + k] * pbar[r * O + o];
            part[lay.c_outw + e] = acc;
        } else {
            const int o = e - H * O;
#pragma unroll
            for (int r = 0; r < R; ++r) acc += pbar[r * O + o];
            part[lay.c_outb + o] = acc;
        }
    }
    Real* zb = ubar;  // reuse: z adjoint through tanh
    for (int e = tid; e < R * H; e += NT) {
        const int r = e / H, k = e - r * H;
        Real acc = 0;
        for (int o = 0; o < O; ++o) acc += pbar[r * O + o] * ow[k * O + o];
        const Real zz = z[e];
        zb[e] = acc * (Real(1) - zz * zz);
    }
    __syncthreads();
    for (int e = tid; e < (H + 1) * H; e += NT) {
        Real acc = 0;
        if (e < H * H) {
            const int k = e / H, j = e - k * H;
#pragma unroll
            for (int r = 0; r < R; ++r) acc += cur[r * H + k] * zb[r * H + j];
            part[lay.c_nlw + e] = acc;
        } else {
            const int j = e - H * H;
#pragma unroll
            for (int r = 0; r < R; ++r) acc += zb[r * H + j];
            part[lay.c_nlb + j] = acc;
        }
    }
    for (int e = tid; e < R * H; e += NT) {
        const int r = e / H, k = e - r * H;
        Real acc = 0;
        for (int j = 0; j < H; ++j) acc += zb[r * H + j] * wsm[k * ldw + j];
        hbar[e] = acc;
    }
    __syncthreads();

    // ---- backward: layers (reverse) ------------------------------------------------
    for (int l = L - 1; l >= 0; --l) {
        const int in = lay.layer_in[l];
        const Real* u = l == 0 ? xin : act + (l - 1) * R * H;
        if (lay.block_last[l])
            for (int e = tid; e < R * H; e += NT) resid[e] = hbar[e];
        stage_matrix(wsm, ldw, th + lay.cw[l], in, G);
        const Real* gi = gates + (4 * l + 0) * R * H;
        const Real* gg = gates + (4 * l + 1) * R * H;
        const Real* go = gates + (4 * l + 2) * R * H;
        const Real* gt = gates + (4 * l + 3) * R * H;
        for (int e = tid; e < R * H; e += NT) {
            const int r = e / H, hh = e - r * H;
            const Real hb = hbar[e];
            const Real i = gi[e], g = gg[e], o = go[e], tc = gt[e];
            const Real ob = hb * tc;
            const Real cb = (hb * o) * (Real(1) - tc * tc);
            const Real ib = cb * g, gb = cb * i;
            pre[r * G + hh] = ib * i * (Real(1) - i);
            pre[r * G + H + hh] = gb * (Real(1) - g * g);
            pre[r * G + 2 * H + hh] = ob * o * (Real(1) - o);
        }
        __syncthreads();
        for (int q = tid; q < G; q += NT) {
            Real pr[R];
            Real accb = 0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                pr[r] = pre[r * G + q];
                accb += pr[r];
            }
            part[lay.cb[l] + q] = accb;
            for (int k = 0; k < in; ++k) {
                Real acc = 0;
#pragma unroll
                for (int r = 0; r < R; ++r) acc += u[r * in + k] * pr[r];
                part[lay.cw[l] + (long long)k * G + q] = acc;
            }
        }
        for (int e = tid; e < R * in; e += NT) {
            const int r = e / in, k = e - r * in;
            Real acc = 0;
            for (int q = 0; q < G; ++q) acc += pre[r * G + q] * wsm[k * ldw + q];
            ubar[e] = acc;
        }
        __syncthreads();
        if (l > 0) {
            for (int e = tid; e < R * H; e += NT) hbar[e] = lay.block_first[l] ? ubar[e] + resid[e] : ubar[e];
            __syncthreads();
        }
    }

    // ---- ES adjoint contributions per window (Div / Mul / BroadcastCol adjoints) ----
    if (st.attach) {
        for (int r = tid; r < nrows; r += NT) {
            const int wl = tile * R + r;  // step-local window index
            const Real lv = lvl[r];
            Real acc_o = 0;
            for (int j = 0; j < O; ++j) {
                const Real tb = -pbar[r * O + j];
                const Real den = s_out[r * O + j] * lv;
                const Real denb = -(tb * tgt[r * O + j] / den);
                st.cO[(size_t)wl * O + j] = denb * lv;
                acc_o += denb * s_out[r * O + j];
            }
            Real acc_i = 0;
            for (int j = 0; j < I; ++j) {
                const Real den = s_in[r * I + j] * lv;
                const Real denb = -(ubar[r * in0 + j] * xin[r * in0 + j] / den);
                st.cI[(size_t)wl * I + j] = denb * lv;
                acc_i += denb * s_in[r * I + j];
            }
            st.cl[wl] = acc_o + acc_i;
        }
    }
    (void)S;
}

// ------------------------------------------------------------------------------ K4
// Window-adjoint gather (in batch order per slot) + reverse HW scan.
template <typename Real>
__global__ void k_es_bwd(StateDev<Real> st, PlanDev pl, NetLayout lay, int s) {
    using M = Math<Real>;
    __shared__ double red[32];
    const int k0 = pl.step_slot_off[s];
    const int k = pl.step_slot_off[s + 1] - k0;
    const int slot = blockIdx.x * blockDim.x + threadIdx.x;
    double sq = 0.0;
    if (slot < k && st.attach) {
        const int N = st.N, S = lay.S, T = lay.T, I = lay.I, O = lay.O, kc = st.kcap;
        const int row = pl.slot_row[k0 + slot];
        Real* lb = st.lbar + slot;
        Real* sb = st.sbar + slot;
        for (int t = 0; t < T; ++t) lb[t * kc] = 0;
        for (int t = 0; t < T + S; ++t) sb[t * kc] = 0;
        const int w0 = pl.step_win_off[s];
        for (int w = pl.slot_win_off[k0 + slot]; w < pl.slot_win_off[k0 + slot + 1]; ++w) {
            const int b = pl.slot_win[w];
            const int a = pl.w_anchor[w0 + b];
            lb[a * kc] += st.cl[b];
            for (int j = 0; j < O; ++j) sb[(a + 1 + j) * kc] += st.cO[(size_t)b * O + j];
            for (int j = 0; j < I; ++j) sb[(a - I + 1 + j) * kc] += st.cI[(size_t)b * I + j];
        }
        const Real alpha = M::logistic_ps(st.ps[row]);
        const Real gamma = M::logistic_ps(st.ps[N + row]);
        Real l0 = 0;
        for (int j = 0; j < S; ++j) l0 += st.vals[j * N + row];
        l0 = l0 / Real(S);
        Real abar = 0, gbar = 0, omab = 0, omgb = 0;
        Real lbn = lb[(T - 1) * kc];  // running adjoint of l[t]
        for (int t = T - 1; t >= 0; --t) {
            const Real yt = st.vals[t * N + row];
            const Real lp = t > 0 ? st.lv[(t - 1) * kc + slot] : l0;
            const Real s_t = st.se[t * kc + slot];
            const Real Sb = sb[(t + S) * kc];
            Real sbt = sb[t * kc];
            // s_{t+S} = gamma*(y/lp) + (1-gamma)*s_t
            omgb += Sb * s_t;
            sbt += Sb * (Real(1) - gamma);
            const Real d2 = yt / lp;
            gbar += Sb * d2;
            const Real d2b = Sb * gamma;
            Real lpb = t > 0 ? lb[(t - 1) * kc] : Real(0);
            if (t > 0) lpb -= d2b * d2 / lp;
            // l_t = alpha*(y/s_t) + (1-alpha)*lp
            const Real Lb = lbn;
            omab += Lb * lp;
            if (t > 0) lpb += Lb * (Real(1) - alpha);
            const Real d1 = yt / s_t;
            abar += Lb * d1;
            sbt -= (Lb * alpha) * d1 / s_t;
            sb[t * kc] = sbt;
            lbn = lpb;
        }
        abar -= omab;
        gbar -= omgb;
        Real* o = st.psg + (size_t)slot * (2 + S);
        const Real ga = abar * alpha * (Real(1) - alpha);
        const Real gg = gbar * gamma * (Real(1) - gamma);
        o[0] = ga;
        o[1] = gg;
        sq += static_cast<double>(ga) * ga + static_cast<double>(gg) * gg;
        for (int j = 0; j < S; ++j) {
            const Real sj = M::exp_ps(st.ps[(2 + j) * N + row]);
            const Real g = sb[j * kc] * sj;
            o[2 + j] = g;
            sq += static_cast<double>(g) * g;
        }
    }
    const double tot = block_sum(sq, red);
    if (threadIdx.x == 0) st.es_sq_part[blockIdx.x] = tot;
}

// ------------------------------------------------------------------------------ K3
// Finalisation shared by the single-GPU fused path and the post-all-reduce kernel:
// clip scale (trainer.hpp:603-615), global Adam step and bias corrections (:617-620),
// step loss (masked mean, autodiff.hpp:392).
template <typename Real>
__device__ void finalize_scalars(StateDev<Real>& st, const PlanDev& pl, int s, double sq, double loss_sum) {
    double scale = 1.0;
    if (st.has_clip) {
        const double norm = sqrt(sq);
        if (norm > st.clip) scale = st.clip / norm;
    }
    st.scal[0] = scale;
    st.scal[3] = loss_sum / pl.step_M[s];
    st.loss_hist[s] = loss_sum / pl.step_M[s];
    if (st.err[0] == 0) {
        const long long step = ++(*st.net_step);
        st.scal[1] = 1.0 - pow(0.9, static_cast<double>(step));
        st.scal[2] = 1.0 - pow(0.999, static_cast<double>(step));
    }
}

template <typename Real, int R>
__global__ void k_net_reduce(StateDev<Real> st, PlanDev pl, NetLayout lay, int s, int n_es_blocks,
                             int finalize) {
    __shared__ double red[32];
    __shared__ bool last;
    const int w0 = pl.step_win_off[s];
    const int Bl = pl.step_win_off[s + 1] - w0;
    const int nt = (Bl + R - 1) / R;
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    double sq = 0.0;
    if (q < lay.P_live) {
        Real g = 0;
        for (int t = 0; t < nt; ++t) g += st.part[(size_t)t * lay.P_live + q];
        st.gbuf[q] = g;
        sq = static_cast<double>(g) * g;
    }
    const double tot = block_sum(sq, red);
    if (threadIdx.x == 0) {
        st.red_sq_part[blockIdx.x] = tot;
        __threadfence();
        const unsigned ticket = atomicAdd(st.done_ctr, 1u);
        last = (ticket == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (threadIdx.x == 0) {
        double es = 0.0;
        if (st.attach)
            for (int b = 0; b < n_es_blocks; ++b) es += st.es_sq_part[b];
        double ls = 0.0;
        for (int t = 0; t < nt; ++t) ls += st.loss_part[t];
        st.gbuf[lay.P_live] = static_cast<Real>(es);
        st.gbuf[lay.P_live + 1] = static_cast<Real>(ls);
        if (finalize) {
            double all = 0.0;
            for (unsigned b = 0; b < gridDim.x; ++b) all += st.red_sq_part[b];
            finalize_scalars(st, pl, s, all + es, ls);
        }
        *st.done_ctr = 0;
    }
}

// After the NCCL all-reduce of gbuf (sharded mode): global squared norm + scalars.
template <typename Real>
__global__ void k_finalize(StateDev<Real> st, PlanDev pl, NetLayout lay, int s) {
    __shared__ double red[32];
    __shared__ bool last;
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    double sq = 0.0;
    if (q < lay.P_live) {
        const double g = st.gbuf[q];
        sq = g * g;
    }
    const double tot = block_sum(sq, red);
    if (threadIdx.x == 0) {
        st.red_sq_part[blockIdx.x] = tot;
        __threadfence();
        last = atomicAdd(st.done_ctr + 1, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    __threadfence();
    double all = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) all += st.red_sq_part[b];
    const double es = st.attach ? static_cast<double>(st.gbuf[lay.P_live]) : 0.0;
    finalize_scalars(st, pl, s, all + es, static_cast<double>(st.gbuf[lay.P_live + 1]));
    st.done_ctr[1] = 0;
}

// ------------------------------------------------------------------------------ K5
template <typename Real>
__global__ void k_adam(StateDev<Real> st, PlanDev pl, NetLayout lay, int s) {
    if (st.err[0] != 0) return;  // the reference throws before apply_updates
    const double scale = st.scal[0], bc1 = st.scal[1], bc2 = st.scal[2];
    const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q < lay.P_live) {
        const double g = static_cast<double>(st.gbuf[q]) * scale;
        const double m = b1 * static_cast<double>(st.mW[q]) + (1.0 - b1) * g;
        const double v = b2 * static_cast<double>(st.vW[q]) + (1.0 - b2) * g * g;
        st.mW[q] = static_cast<Real>(m);
        st.vW[q] = static_cast<Real>(v);
        st.theta[q] = static_cast<Real>(static_cast<double>(st.theta[q]) - st.lr_net * (m / bc1) / (sqrt(v / bc2) + eps));
        return;
    }
    if (!st.attach) return;
    const int k0 = pl.step_slot_off[s];
    const int k = pl.step_slot_off[s + 1] - k0;
    const long long slot = q - lay.P_live;
    if (slot >= k) return;
    const int N = st.N, S = lay.S;
    const int row = pl.slot_row[k0 + slot];
    const int steps = ++st.ps_steps[row];
    const double sc1 = 1.0 - pow(b1, static_cast<double>(steps));
    const double sc2 = 1.0 - pow(b2, static_cast<double>(steps));
    const Real* g = st.psg + (size_t)slot * (2 + S);
    for (int j = 0; j < 2 + S; ++j) {
        const size_t e = (size_t)j * N + row;
        const double gg = static_cast<double>(g[j]) * scale;
        const double m = b1 * static_cast<double>(st.ps_m[e]) + (1.0 - b1) * gg;
        const double v = b2 * static_cast<double>(st.ps_v[e]) + (1.0 - b2) * gg * gg;
        st.ps_m[e] = static_cast<Real>(m);
        st.ps_v[e] = static_cast<Real>(v);
        st.ps[e] = static_cast<Real>(static_cast<double>(st.ps[e]) - st.lr_ps * (m / sc1) / (sqrt(v / sc2) + eps));
    }
}

// ------------------------------------------------------------------------------ K6
// Forecast scan (holt_winters.hpp:66-97 + deseasonalize_normalize :153-166 +
// HWState::seasonal_at :55-59): one thread per series over values[0:t_ins).
template <typename Real>
__global__ void k_forecast_scan(StateDev<Real> st, NetLayout lay, int t_ins, Real* X, Real* FL, Real* FS,
                                Real* dump_lv, Real* dump_se, int dump_row) {
    using M = Math<Real>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int S = lay.S, I = lay.I, O = lay.O, in0 = lay.in0, N = st.N;
    // ring of the last S seasonalities plus the I window seasonalities needed at the end
    Real* ring = reinterpret_cast<Real*>(smem_raw);
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= N) return;
    const int bd = blockDim.x, tid = threadIdx.x;
    for (int t = 0; t < t_ins; ++t)
        if (!(st.vals[t * N + row] > Real(0))) {
            flag_error(st.err, kErrObs, t);
            return;
        }
    const bool dump = row == dump_row;
    const Real alpha = M::logistic_ps(st.ps[row]);
    const Real gamma = M::logistic_ps(st.ps[N + row]);
    const Real oma = Real(1) - alpha, omg = Real(1) - gamma;
    Real lp = 0;
    for (int j = 0; j < S; ++j) {
        const Real s0 = M::exp_ps(st.ps[(2 + j) * N + row]);
        ring[j * bd + tid] = s0;
        if (dump) dump_se[j] = s0;
        lp += st.vals[j * N + row];
    }
    lp = lp / Real(S);
    // seasonality index u is produced at step u-S; window inputs need u in [t_ins-I, t_ins)
    Real* win = ring + S * bd;  // [I][bd]
    for (int u = t_ins - I; u < S && u < t_ins; ++u)
        if (u >= 0) win[(u - (t_ins - I)) * bd + tid] = ring[u * bd + tid];
    int j = 0;
    for (int t = 0; t < t_ins; ++t) {
        const Real yt = st.vals[t * N + row];
        const Real s_t = ring[j * bd + tid];
        const Real l = alpha * (yt / s_t) + oma * lp;
        if (!(l > Real(0)) || !isfinite(l)) {
            flag_error(st.err, kErrFcLevel, t);
            return;
        }
        const Real sn = gamma * (yt / lp) + omg * s_t;
        ring[j * bd + tid] = sn;
        const int u = t + S;
        if (u >= t_ins - I && u < t_ins) win[(u - (t_ins - I)) * bd + tid] = sn;
        if (dump) {
            dump_lv[t] = l;
            dump_se[u] = sn;
        }
        lp = l;
        j = (j + 1 == S) ? 0 : j + 1;
    }
    if (X == nullptr) return;
    const Real level = lp;
    for (int c = 0; c < I; ++c) {
        const Real sv = win[c * bd + tid];
        if (!(sv > Real(0))) {
            flag_error(st.err, kErrSeas, t_ins);
            return;
        }
        X[(size_t)row * in0 + c] = st.vals[(t_ins - I + c) * N + row] / (level * sv);
    }
    for (int c = 0; c < 6; ++c) X[(size_t)row * in0 + I + c] = (st.cat[row] == c) ? Real(1) : Real(0);
    FL[row] = level;
    // seasonal_at(t_ins + o): indices [t_ins, t_ins+S) are the ring (slot (t_ins+o) mod S)
    for (int o = 0; o < O; ++o) {
        int idx = t_ins + o;
        while (idx >= t_ins + S) idx -= S;
        FS[(size_t)row * O + o] = ring[(idx % S) * bd + tid];
    }
}

}  // namespace esrnn_dev
