// sm_100a kernels of the ES-RNN training / forecasting step.
//
// One training step (reference: Trainer::step = build_graph + Tape::backward +
// apply_updates, trainer.hpp:484-655) is four launches on one stream, captured once per
// trainer into a CUDA graph covering the whole epoch:
//
//   K1 k_scan_fwd      slot-parallel Holt-Winters level/seasonality scan   (holt_winters.hpp:236-283)
//   K2 k_stack<TRAIN>  row-tile-parallel: window gather/normalise (trainer.hpp:524-566),
//                      LSTM stack fwd at sequence length 1 (network.hpp:148-210), masked
//                      pinball (autodiff.hpp:370-395) and its adjoint (:611-628), the whole
//                      stack adjoint, per-tile weight-gradient partials and per-window ES
//                      adjoint contributions.  Weights arrive in shared memory by one TMA
//                      bulk copy (cp.async.bulk + mbarrier) that overlaps the window gather.
//   K3 k_grad_finish   blocks [0, es_blocks): per-slot gather of its windows' contributions
//                      in batch order (Gather adjoint, autodiff.hpp:603-610) + reverse HW
//                      scan; remaining blocks: fixed-order reduction of the tile partials;
//                      the last CTA finalises clip scale / bias corrections / loss
//                      (trainer.hpp:603-620)
//   K4 k_adam          parameter- and slot-parallel Adam (trainer.hpp:617-655)
//
// Every reduction has a fixed order (tile groups, slot-window CSR order, CTA order), so a
// run is bit-reproducible on a given GPU count; no float atomics anywhere.
//
// Layout in HBM: values time-major y[t][N] (coalesced across series), per-series
// parameters / Adam moments SoA [(2+S)][N], shared parameters in a compact "live" layout
// that drops the structurally-dead forget-gate columns and recurrent matrices (their
// gradients are exactly zero at sequence length 1), scan state [t][slot].
#pragma once
#include <cstdint>

#include "devmath.cuh"

namespace esrnn_dev {

constexpr int kMaxLayers = 16;

// Compact live layout of the shared parameters and the network shape.  Every segment
// offset is a multiple of 4 elements (16-byte aligned for fp32) so rows can be moved
// with vector loads and TMA bulk copies.
struct NetLayout {
    int L, nb, H, O, I, S, in0, T;
    int ldx, ldh;                // padded row strides (multiples of 4) of x and hidden activations
    int layer_in[kMaxLayers];
    int res_src[kMaxLayers];     // >=0: layer output added as residual after this layer
    int block_first[kMaxLayers]; // 1 if layer is the first of a block b>0 (adjoint joins the residual)
    int block_last[kMaxLayers];  // 1 if layer is the last of a block b>0 (residual added here)
    long long cw[kMaxLayers], cb[kMaxLayers];
    long long c_nlw, c_nlb, c_outw, c_outb, P_live, P_pad;
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
    Real* theta;            // [P_pad]
    Real* mW;
    Real* vW;
    // scratch
    Real* lv;               // [T][kcap]
    Real* se;               // [T+S][kcap]
    Real* cI;               // [Bcap][I]   ES adjoint contributions per window
    Real* cO;               // [Bcap][O]
    Real* cl;               // [Bcap]
    Real* part;             // [tiles][P_pad]
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

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ------------------------------------------------------------------ TMA bulk copy
__device__ __forceinline__ unsigned smem_addr(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
    unsigned ok = 0;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(ok)
            : "r"(smem_addr(bar)), "r"(phase)
            : "memory");
    } while (!ok);
}

// 4-wide shared-memory vector (16 B for fp32, 2 x 16 B for fp64)
template <typename Real>
struct V4 {
    Real x, y, z, w;
};
template <typename Real>
__device__ __forceinline__ V4<Real> lds4(const Real* p) {
    if constexpr (sizeof(Real) == 4) {
        const float4 v = *reinterpret_cast<const float4*>(p);
        return {v.x, v.y, v.z, v.w};
    } else {
        const double2 a = *reinterpret_cast<const double2*>(p);
        const double2 b = *reinterpret_cast<const double2*>(p + 2);
        return {a.x, a.y, b.x, b.y};
    }
}

// ------------------------------------------------------------------------------ K1
// hybrid_primer_tape forward (holt_winters.hpp:245-277): one thread per slot; the last
// S seasonalities live in a shared-memory ring and the observations are prefetched 8
// steps ahead, so the recurrence only waits on its own FMA chain.
template <typename Real>
__global__ void __launch_bounds__(128) k_scan_fwd(StateDev<Real> st, PlanDev pl, NetLayout lay, int s) {
    using M = Math<Real>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Real* ring = reinterpret_cast<Real*>(smem_raw);
    const int k0 = pl.step_slot_off[s];
    const int k = pl.step_slot_off[s + 1] - k0;
    const int slot = blockIdx.x * blockDim.x + threadIdx.x;
    if (slot >= k) return;
    const int bd = blockDim.x, tid = threadIdx.x;
    const int N = st.N, S = lay.S, T = lay.T, kc = st.kcap;
    const int row = pl.slot_row[k0 + slot];
    const Real* __restrict__ y = st.vals + row;
    Real* __restrict__ se = st.se + slot;
    Real* __restrict__ lv = st.lv + slot;
    const Real alpha = M::logistic_ps(st.ps[row]);
    const Real gamma = M::logistic_ps(st.ps[N + row]);
    const Real oma = Real(1) - alpha, omg = Real(1) - gamma;
    Real lp = 0;
    for (int j = 0; j < S; ++j) {
        const Real s0 = M::exp_ps(st.ps[(2 + j) * N + row]);
        ring[j * bd + tid] = s0;
        se[j * kc] = s0;
        lp += __ldg(y + (size_t)j * N);
    }
    lp = lp / Real(S);
    int bad = -1;
    int j = 0;
    constexpr int CH = 8;
    for (int t0 = 0; t0 < T; t0 += CH) {
        Real yb[CH];
#pragma unroll
        for (int u = 0; u < CH; ++u) yb[u] = (t0 + u < T) ? __ldg(y + (size_t)(t0 + u) * N) : Real(1);
#pragma unroll
        for (int u = 0; u < CH; ++u) {
            const int t = t0 + u;
            if (t < T) {
                const Real yt = yb[u];
                const Real s_t = ring[j * bd + tid];
                const Real l = alpha * (yt / s_t) + oma * lp;
                if (!(l > Real(0)) || !isfinite(l)) bad = bad < 0 ? t : bad;
                const Real sn = gamma * (yt / lp) + omg * s_t;
                ring[j * bd + tid] = sn;
                se[(t + S) * kc] = sn;
                lv[t * kc] = l;
                lp = l;
                j = (j + 1 == S) ? 0 : j + 1;
            }
        }
    }
    if (bad >= 0) flag_error(st.err, kErrTrainLevel, bad);
}

// ------------------------------------------------------------------------------ K2
enum StackMode { kTrain = 0, kLossOnly = 1, kForecast = 2 };

struct ForecastArgs {
    int t_ins;
    int validate;
    const void* X;       // [N][in0] Real
    const void* lvl;     // [N] Real
    const void* sout;    // [N][O] Real
    double* out;         // [N][O]
    double* smape;       // [N]
};

// Shared-memory carve-up of one row tile (all in Real units).  `w` holds either the
// whole compact weight vector (resident mode) or one staged layer.
struct TileSmem {
    int w, xin, sin, sout, lvl, tgt, msk, act, gates, z, pred, pbar, pre, hbar, resid, ubar, total;
    int wsize;
    __host__ __device__ static int r4(int x) { return (x + 3) & ~3; }
    __host__ __device__ static TileSmem make(const NetLayout& lay, int R, bool resident) {
        TileSmem t;
        const int H = lay.H, O = lay.O, I = lay.I, L = lay.L, G = 3 * H;
        const int max_in = lay.in0 > H ? lay.in0 : H;
        int o = 0;
        const int head = static_cast<int>(lay.P_pad - lay.c_nlw);
        const int stage = max_in * (G > H ? G : H);
        t.wsize = resident ? static_cast<int>(lay.P_pad) : r4(stage > head ? stage : head);
        t.w = o; o += t.wsize;
        t.xin = o; o += r4(R * lay.ldx);
        t.sin = o; o += r4(R * I);
        t.sout = o; o += r4(R * O);
        t.lvl = o; o += r4(R);
        t.tgt = o; o += r4(R * O);
        t.msk = o; o += r4(R * O);
        t.act = o; o += r4(L * R * lay.ldh);
        t.gates = o; o += r4(4 * L * R * H);
        t.z = o; o += r4(R * lay.ldh);
        t.pred = o; o += r4(R * O);
        t.pbar = o; o += r4(R * O);
        t.pre = o; o += r4(R * G);
        t.hbar = o; o += r4(R * lay.ldh);
        t.resid = o; o += r4(R * lay.ldh);
        t.ubar = o; o += r4(R * (lay.ldx > lay.ldh ? lay.ldx : lay.ldh));
        t.total = o;
        return t;
    }
};

// Vectorised global->shared copy of one contiguous segment (non-resident mode).
template <typename Real>
__device__ __forceinline__ void stage_segment(Real* __restrict__ dst, const Real* __restrict__ src, int n) {
    for (int e = threadIdx.x * 4; e < n; e += blockDim.x * 4) {
        if (e + 4 <= n) {
            if constexpr (sizeof(Real) == 4) {
                *reinterpret_cast<float4*>(dst + e) = __ldg(reinterpret_cast<const float4*>(src + e));
            } else {
                *reinterpret_cast<double2*>(dst + e) = __ldg(reinterpret_cast<const double2*>(src + e));
                *reinterpret_cast<double2*>(dst + e + 2) = __ldg(reinterpret_cast<const double2*>(src + e + 2));
            }
        } else {
            for (int i = e; i < n; ++i) dst[i] = src[i];
        }
    }
}

// y[r] = sum_k u[r][k] * W[k][q] for the R rows, u rows padded to ldu (multiple of 4).
template <typename Real, int R>
__device__ __forceinline__ void rows_dot_col(Real (&acc)[R], const Real* __restrict__ u, int ldu,
                                             const Real* __restrict__ W, int ldw, int in, int q) {
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0;
    int k = 0;
    for (; k + 4 <= in; k += 4) {
        const Real w0 = W[(k + 0) * ldw + q], w1 = W[(k + 1) * ldw + q];
        const Real w2 = W[(k + 2) * ldw + q], w3 = W[(k + 3) * ldw + q];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const V4<Real> x = lds4(u + r * ldu + k);
            acc[r] += x.x * w0;
            acc[r] += x.y * w1;
            acc[r] += x.z * w2;
            acc[r] += x.w * w3;
        }
    }
    for (; k < in; ++k) {
        const Real w = W[k * ldw + q];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] += u[r * ldu + k] * w;
    }
}

// out[r][k] = sum_q a[r][q] * W[k][q] for k in [0, nk): one warp per k, lanes over q,
// butterfly (warp-shuffle) reduction of the R row sums.
template <typename Real, int R>
__device__ __forceinline__ void rows_dot_rowT(Real* __restrict__ out, int ldo, const Real* __restrict__ a, int lda,
                                              const Real* __restrict__ W, int ldw, int nk, int nq) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int k = wid; k < nk; k += nw) {
        Real acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = 0;
        for (int q = lane; q < nq; q += 32) {
            const Real w = W[k * ldw + q];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] += a[r * lda + q] * w;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = warp_sum(acc[r]);
        if (lane < R) {
            Real v = acc[0];
#pragma unroll
            for (int r = 1; r < R; ++r)
                if (lane == r) v = acc[r];
            out[lane * ldo + k] = v;
        }
    }
}

// Row tile of R windows (kTrain / kLossOnly) or R series (kForecast).
template <typename Real, int R, int MODE, bool RESIDENT>
__global__ void __launch_bounds__(256) k_stack(StateDev<Real> st, PlanDev pl, NetLayout lay, int s,
                                               ForecastArgs fa) {
    using M = Math<Real>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Real* sm = reinterpret_cast<Real*>(smem_raw);
    __shared__ double red[32];
    __shared__ __align__(8) uint64_t wbar;
    const TileSmem ts = TileSmem::make(lay, R, RESIDENT);
    const int H = lay.H, O = lay.O, I = lay.I, in0 = lay.in0, L = lay.L, G = 3 * H;
    const int ldx = lay.ldx, ldh = lay.ldh;
    const int tid = threadIdx.x, NT = blockDim.x;
    const int tile = blockIdx.x;
    const Real* __restrict__ th = st.theta;

    Real* wsm = sm + ts.w;
    Real* xin = sm + ts.xin;
    Real* s_in = sm + ts.sin;
    Real* s_out = sm + ts.sout;
    Real* lvl = sm + ts.lvl;
    Real* tgt = sm + ts.tgt;
    Real* msk = sm + ts.msk;
    Real* act = sm + ts.act;
    Real* gates = sm + ts.gates;
    Real* z = sm + ts.z;
    Real* pbar = sm + ts.pbar;
    Real* pre = sm + ts.pre;
    Real* hbar = sm + ts.hbar;
    Real* resid = sm + ts.resid;
    Real* ubar = sm + ts.ubar;

    int nrows, w0 = 0;
    if (MODE == kForecast) {
        nrows = min(R, st.N - tile * R);
    } else {
        w0 = pl.step_win_off[s];
        const int Bl = pl.step_win_off[s + 1] - w0;
        nrows = min(R, Bl - tile * R);
    }
    if (nrows <= 0) return;

    // ---- weights: one TMA bulk copy of the compact parameter vector (resident mode) ---
    if (RESIDENT) {
        if (tid == 0) {
            mbar_init(&wbar, 1);
            const unsigned total = static_cast<unsigned>(lay.P_pad * sizeof(Real));
            mbar_expect_tx(&wbar, total);
            constexpr unsigned kChunk = 32768;
            for (unsigned off = 0; off < total; off += kChunk) {
                const unsigned n = total - off < kChunk ? total - off : kChunk;
                bulk_g2s(reinterpret_cast<unsigned char*>(wsm) + off,
                         reinterpret_cast<const unsigned char*>(th) + off, n, &wbar);
            }
        }
    }

    // ---- prologue: window gather + normalisation (trainer.hpp:532-566) -------------
    if (MODE == kForecast) {
        const Real* X = reinterpret_cast<const Real*>(fa.X);
        const Real* FL = reinterpret_cast<const Real*>(fa.lvl);
        const Real* FS = reinterpret_cast<const Real*>(fa.sout);
        for (int e = tid; e < R * in0; e += NT) {
            const int r = e / in0, c = e - r * in0;
            xin[r * ldx + c] = r < nrows ? X[(size_t)(tile * R + r) * in0 + c] : Real(0);
        }
        for (int e = tid; e < R * O; e += NT) {
            const int r = e / O;
            s_out[e] = r < nrows ? FS[(size_t)(tile * R) * O + e] : Real(0);
        }
        for (int r = tid; r < R; r += NT) lvl[r] = r < nrows ? FL[tile * R + r] : Real(0);
    } else {
        const int per = I + O + 1;
        for (int e = tid; e < R * per; e += NT) {
            const int r = e / per, c = e - r * per;
            const int wb = w0 + tile * R + r;
            if (r >= nrows) {
                if (c < I) { xin[r * ldx + c] = 0; s_in[r * I + c] = 1; }
                else if (c < I + O) { tgt[r * O + c - I] = 0; s_out[r * O + c - I] = 1; msk[r * O + c - I] = 0; }
                else lvl[r] = 1;
                continue;
            }
            const int row = pl.w_row[wb], a = pl.w_anchor[wb], slot = pl.w_slot[wb];
            const Real l = st.lv[a * st.kcap + slot];
            if (c < I) {
                const int idx = a - I + 1 + c;
                const Real sv = st.se[idx * st.kcap + slot];
                xin[r * ldx + c] = st.vals[(size_t)idx * st.N + row] / (sv * l);
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
            xin[r * ldx + I + c] = v;
        }
    }
    // zero the row padding so 4-wide loads past `in` only ever see zeros
    for (int e = tid; e < R * (ldx - in0); e += NT) {
        const int r = e / (ldx - in0), c = e - r * (ldx - in0);
        xin[r * ldx + in0 + c] = 0;
    }
    for (int e = tid; e < L * R * (ldh - H); e += NT) {
        const int r = e / (ldh - H), c = e - r * (ldh - H);
        act[r * ldh + H + c] = 0;
    }
    __syncthreads();
    if (MODE != kForecast && st.d_inputs != nullptr) {
        const int base = tile * R;
        for (int e = tid; e < nrows * in0; e += NT) {
            const int r = e / in0, c = e - r * in0;
            st.d_inputs[(size_t)base * in0 + e] = xin[r * ldx + c];
        }
        for (int e = tid; e < nrows * O; e += NT) {
            st.d_targets[(size_t)base * O + e] = tgt[e];
            st.d_seas[(size_t)base * O + e] = s_out[e];
        }
        for (int r = tid; r < nrows; r += NT) st.d_levels[base + r] = lvl[r];
    }
    if (RESIDENT) mbar_wait(&wbar, 0);

    auto wl = [&](long long off) -> const Real* { return RESIDENT ? wsm + off : wsm; };

    // ---- forward through the stack (network.hpp:148-210, sequence length 1) --------
    for (int l = 0; l < L; ++l) {
        const int in = lay.layer_in[l];
        const Real* u = l == 0 ? xin : act + (l - 1) * R * ldh;
        const int ldu = l == 0 ? ldx : ldh;
        if (!RESIDENT) {
            __syncthreads();
            stage_segment(wsm, th + lay.cw[l], in * G);
            __syncthreads();
        }
        const Real* W = wl(lay.cw[l]);
        for (int q = tid; q < G; q += NT) {
            Real acc[R];
            rows_dot_col<Real, R>(acc, u, ldu, W, G, in, q);
            const Real b = th[lay.cb[l] + q];
#pragma unroll
            for (int r = 0; r < R; ++r) pre[r * G + q] = acc[r] + b;
        }
        __syncthreads();
        Real* gi = gates + (4 * l + 0) * R * H;
        Real* gg = gates + (4 * l + 1) * R * H;
        Real* go = gates + (4 * l + 2) * R * H;
        Real* gt = gates + (4 * l + 3) * R * H;
        Real* out = act + l * R * ldh;
        const Real* radd = lay.block_last[l] ? act + lay.res_src[l] * R * ldh : nullptr;
        for (int e = tid; e < R * H; e += NT) {
            const int r = e / H, hh = e - r * H;
            const Real i = M::logistic(pre[r * G + hh]);
            const Real g = M::tanh(pre[r * G + H + hh]);
            const Real o = M::logistic(pre[r * G + 2 * H + hh]);
            const Real c = i * g;
            const Real tc = M::tanh(c);
            Real h = o * tc;
            if (radd) h = h + radd[r * ldh + hh];
            gi[e] = i;
            gg[e] = g;
            go[e] = o;
            gt[e] = tc;
            out[r * ldh + hh] = h;
        }
        __syncthreads();
    }
    // head (network.hpp:207-209)
    const Real* cur = act + (L - 1) * R * ldh;
    if (!RESIDENT) {
        stage_segment(wsm, th + lay.c_nlw, static_cast<int>(lay.P_pad - lay.c_nlw));  // nl_w | nl_b | out_w | out_b
        __syncthreads();
    }
    const long long hb0 = RESIDENT ? 0 : lay.c_nlw;  // staged head lives at wsm[c_* - c_nlw]
    const Real* nlw = RESIDENT ? wsm + lay.c_nlw : wsm;
    const Real* nlb = RESIDENT ? wsm + lay.c_nlb : wsm + (lay.c_nlb - hb0);
    const Real* ow = RESIDENT ? wsm + lay.c_outw : wsm + (lay.c_outw - hb0);
    const Real* obias = RESIDENT ? wsm + lay.c_outb : wsm + (lay.c_outb - hb0);
    for (int j = tid; j < H; j += NT) {
        Real acc[R];
        rows_dot_col<Real, R>(acc, cur, ldh, nlw, H, H, j);
        const Real b = nlb[j];
#pragma unroll
        for (int r = 0; r < R; ++r) z[r * ldh + j] = M::tanh(acc[r] + b);
    }
    for (int e = tid; e < R * (ldh - H); e += NT) {
        const int r = e / (ldh - H), c = e - r * (ldh - H);
        z[r * ldh + H + c] = 0;
    }
    __syncthreads();
    double lsum = 0.0;
    for (int e = tid; e < R * O; e += NT) {
        const int r = e / O, o = e - r * O;
        Real acc = 0;
        for (int k = 0; k < H; ++k) acc += z[r * ldh + k] * ow[k * O + o];
        const Real p = acc + obias[o];
        if (MODE == kForecast) {
            if (r < nrows) {
                const int row = tile * R + r;
                fa.out[(size_t)row * O + o] = static_cast<double>(p * lvl[r] * s_out[e]);
            }
        } else {
            // masked pinball (autodiff.hpp:384-392) and its adjoint (:620-626)
            Real pb = 0;
            if (msk[e] != Real(0)) {
                const Real d = tgt[e] - p;
                lsum += (d >= Real(0)) ? st.tau * static_cast<double>(d) : (st.tau - 1.0) * static_cast<double>(d);
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

    // ---- backward: head ------------------------------------------------------------
    Real* __restrict__ part = st.part + (size_t)tile * lay.P_pad;
    for (int e = tid; e < (H + 1) * O; e += NT) {
        Real acc = 0;
        if (e < H * O) {
            const int k = e / O, o = e - k * O;
#pragma unroll
            for (int r = 0; r < R; ++r) acc += z[r * ldh + k] * pbar[r * O + o];
            part[lay.c_outw + e] = acc;
        } else {
            const int o = e - H * O;
#pragma unroll
            for (int r = 0; r < R; ++r) acc += pbar[r * O + o];
            part[lay.c_outb + o] = acc;
        }
    }
    Real* zb = ubar;  // z adjoint through tanh, rows padded to ldh
    for (int e = tid; e < R * ldh; e += NT) {
        const int r = e / ldh, k = e - r * ldh;
        Real v = 0;
        if (k < H) {
            Real acc = 0;
            for (int o = 0; o < O; ++o) acc += pbar[r * O + o] * ow[k * O + o];
            const Real zz = z[r * ldh + k];
            v = acc * (Real(1) - zz * zz);
        }
        zb[e] = v;
    }
    __syncthreads();
    // nl_w / nl_b partials: thread per column j, rows k
    for (int j = tid; j < H; j += NT) {
        Real zc[R];
        Real accb = 0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            zc[r] = zb[r * ldh + j];
            accb += zc[r];
        }
        part[lay.c_nlb + j] = accb;
        for (int k = 0; k < H; ++k) {
            Real acc = 0;
#pragma unroll
            for (int r = 0; r < R; ++r) acc += cur[r * ldh + k] * zc[r];
            part[lay.c_nlw + (long long)k * H + j] = acc;
        }
    }
    rows_dot_rowT<Real, R>(hbar, ldh, zb, ldh, nlw, H, H, H);
    __syncthreads();

    // ---- backward: layers (reverse) ------------------------------------------------
    for (int l = L - 1; l >= 0; --l) {
        const int in = lay.layer_in[l];
        const Real* u = l == 0 ? xin : act + (l - 1) * R * ldh;
        const int ldu = l == 0 ? ldx : ldh;
        if (lay.block_last[l])
            for (int e = tid; e < R * ldh; e += NT) resid[e] = hbar[e];
        if (!RESIDENT) stage_segment(wsm, th + lay.cw[l], in * G);
        const Real* W = wl(lay.cw[l]);
        const Real* gi = gates + (4 * l + 0) * R * H;
        const Real* gg = gates + (4 * l + 1) * R * H;
        const Real* go = gates + (4 * l + 2) * R * H;
        const Real* gt = gates + (4 * l + 3) * R * H;
        for (int e = tid; e < R * H; e += NT) {
            const int r = e / H, hh = e - r * H;
            const Real hb = hbar[r * ldh + hh];
            const Real i = gi[e], g = gg[e], o = go[e], tc = gt[e];
            const Real ob = hb * tc;
            const Real cb = (hb * o) * (Real(1) - tc * tc);
            const Real ib = cb * g, gb = cb * i;
            pre[r * G + hh] = ib * i * (Real(1) - i);
            pre[r * G + H + hh] = gb * (Real(1) - g * g);
            pre[r * G + 2 * H + hh] = ob * o * (Real(1) - o);
        }
        __syncthreads();
        // W / b partials: thread per gate column q, 4 input rows per step
        for (int q = tid; q < G; q += NT) {
            Real pr[R];
            Real accb = 0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                pr[r] = pre[r * G + q];
                accb += pr[r];
            }
            part[lay.cb[l] + q] = accb;
            int k = 0;
            for (; k + 4 <= in; k += 4) {
                Real a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const V4<Real> x = lds4(u + r * ldu + k);
                    a0 += x.x * pr[r];
                    a1 += x.y * pr[r];
                    a2 += x.z * pr[r];
                    a3 += x.w * pr[r];
                }
                part[lay.cw[l] + (long long)(k + 0) * G + q] = a0;
                part[lay.cw[l] + (long long)(k + 1) * G + q] = a1;
                part[lay.cw[l] + (long long)(k + 2) * G + q] = a2;
                part[lay.cw[l] + (long long)(k + 3) * G + q] = a3;
            }
            for (; k < in; ++k) {
                Real acc = 0;
#pragma unroll
                for (int r = 0; r < R; ++r) acc += u[r * ldu + k] * pr[r];
                part[lay.cw[l] + (long long)k * G + q] = acc;
            }
        }
        // input adjoint: u_bar = pre_bar . W^T (warp-shuffle reductions over gate columns)
        rows_dot_rowT<Real, R>(ubar, l == 0 ? ldx : ldh, pre, G, W, G, in, G);
        __syncthreads();
        if (l > 0) {
            for (int e = tid; e < R * ldh; e += NT) hbar[e] = lay.block_first[l] ? ubar[e] + resid[e] : ubar[e];
            __syncthreads();
        }
    }

    // ---- ES adjoint contributions per window (Div / Mul / BroadcastCol adjoints) ----
    if (st.attach) {
        for (int r = tid; r < nrows; r += NT) {
            const int wl_ = tile * R + r;  // step-local window index
            const Real lv = lvl[r];
            Real acc_o = 0;
            for (int j = 0; j < O; ++j) {
                const Real tb = -pbar[r * O + j];
                const Real den = s_out[r * O + j] * lv;
                const Real denb = -(tb * tgt[r * O + j] / den);
                st.cO[(size_t)wl_ * O + j] = denb * lv;
                acc_o += denb * s_out[r * O + j];
            }
            Real acc_i = 0;
            for (int j = 0; j < I; ++j) {
                const Real den = s_in[r * I + j] * lv;
                const Real denb = -(ubar[r * ldx + j] * xin[r * ldx + j] / den);
                st.cI[(size_t)wl_ * I + j] = denb * lv;
                acc_i += denb * s_in[r * I + j];
            }
            st.cl[wl_] = acc_o + acc_i;
        }
    }
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

constexpr int kGroups = 4;      // tile groups per reduce block
constexpr int kRedChunks = 4;   // 32-parameter chunks per reduce block
constexpr int kFinishThreads = 128;

// ES backward (blocks [0, es_blocks)) and the fixed-order reduction of the tile
// partials (blocks [es_blocks, gridDim)); the last CTA to finish finalises.
template <typename Real, int R>
__global__ void __launch_bounds__(kFinishThreads) k_grad_finish(StateDev<Real> st, PlanDev pl, NetLayout lay, int s,
                                                                int es_blocks, int finalize) {
    using M = Math<Real>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ double red[32];
    __shared__ Real gsum[kGroups][32];
    __shared__ bool last;
    const int tid = threadIdx.x;
    double sq = 0.0;
    if (static_cast<int>(blockIdx.x) < es_blocks) {
        // ---------------- per-slot window-adjoint gather + reverse HW scan ---------------
        const int k0 = pl.step_slot_off[s];
        const int k = pl.step_slot_off[s + 1] - k0;
        const int slot = blockIdx.x * blockDim.x + tid;
        if (slot < k && st.attach) {
            const int N = st.N, S = lay.S, T = lay.T, I = lay.I, O = lay.O, kc = st.kcap, bd = blockDim.x;
            Real* lb = reinterpret_cast<Real*>(smem_raw) + tid;  // [T][bd]
            Real* sb = lb + T * bd;                               // [T+S][bd]
            const int row = pl.slot_row[k0 + slot];
            for (int t = 0; t < T; ++t) lb[t * bd] = 0;
            for (int t = 0; t < T + S; ++t) sb[t * bd] = 0;
            const int w0 = pl.step_win_off[s];
            for (int w = pl.slot_win_off[k0 + slot]; w < pl.slot_win_off[k0 + slot + 1]; ++w) {
                const int b = pl.slot_win[w];
                const int a = pl.w_anchor[w0 + b];
                lb[a * bd] += st.cl[b];
                for (int j = 0; j < O; ++j) sb[(a + 1 + j) * bd] += st.cO[(size_t)b * O + j];
                for (int j = 0; j < I; ++j) sb[(a - I + 1 + j) * bd] += st.cI[(size_t)b * I + j];
            }
            const Real* __restrict__ y = st.vals + row;
            const Real* __restrict__ lvp = st.lv + slot;
            const Real* __restrict__ sep = st.se + slot;
            const Real alpha = M::logistic_ps(st.ps[row]);
            const Real gamma = M::logistic_ps(st.ps[N + row]);
            Real l0 = 0;
            for (int j = 0; j < S; ++j) l0 += __ldg(y + (size_t)j * N);
            l0 = l0 / Real(S);
            Real abar = 0, gbar = 0, omab = 0, omgb = 0;
            Real lbn = lb[(T - 1) * bd];  // running adjoint of l[t]
            constexpr int CH = 8;
            for (int tc = T - 1; tc >= 0; tc -= CH) {
                Real yb[CH], lpb_[CH], sb_[CH];
#pragma unroll
                for (int u = 0; u < CH; ++u) {
                    const int t = tc - u;
                    yb[u] = t >= 0 ? __ldg(y + (size_t)t * N) : Real(1);
                    lpb_[u] = t > 0 ? lvp[(t - 1) * kc] : Real(1);
                    sb_[u] = t >= 0 ? sep[t * kc] : Real(1);
                }
#pragma unroll
                for (int u = 0; u < CH; ++u) {
                    const int t = tc - u;
                    if (t >= 0) {
                        const Real yt = yb[u];
                        const Real lp = t > 0 ? lpb_[u] : l0;
                        const Real s_t = sb_[u];
                        const Real Sb = sb[(t + S) * bd];
                        Real sbt = sb[t * bd];
                        // s_{t+S} = gamma*(y/lp) + (1-gamma)*s_t
                        omgb += Sb * s_t;
                        sbt += Sb * (Real(1) - gamma);
                        const Real d2 = yt / lp;
                        gbar += Sb * d2;
                        const Real d2b = Sb * gamma;
                        Real lpb = t > 0 ? lb[(t - 1) * bd] : Real(0);
                        if (t > 0) lpb -= d2b * d2 / lp;
                        // l_t = alpha*(y/s_t) + (1-alpha)*lp
                        const Real Lb = lbn;
                        omab += Lb * lp;
                        if (t > 0) lpb += Lb * (Real(1) - alpha);
                        const Real d1 = yt / s_t;
                        abar += Lb * d1;
                        sbt -= (Lb * alpha) * d1 / s_t;
                        sb[t * bd] = sbt;
                        lbn = lpb;
                    }
                }
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
                const Real g = sb[j * bd] * sj;
                o[2 + j] = g;
                sq += static_cast<double>(g) * g;
            }
        }
        const double tot = block_sum(sq, red);
        if (tid == 0) st.es_sq_part[blockIdx.x] = tot;
    } else {
        // ------- tile-partial reduction: kRedChunks x 32 params, kGroups tile groups -------
        const int rb = blockIdx.x - es_blocks;
        const int w0 = pl.step_win_off[s];
        const int Bl = pl.step_win_off[s + 1] - w0;
        const int nt = (Bl + R - 1) / R;
        const int lane = tid & 31, grp = tid >> 5;
        for (int ch = 0; ch < kRedChunks; ++ch) {
            const long long q = ((long long)rb * kRedChunks + ch) * 32 + lane;
            Real g = 0;
            if (q < lay.P_pad) {
                const Real* __restrict__ p = st.part + q;
                int t = grp;
                Real a0 = 0, a1 = 0, a2 = 0, a3 = 0;
                for (; t + 3 * kGroups < nt; t += 4 * kGroups) {
                    a0 += p[(size_t)(t)*lay.P_pad];
                    a1 += p[(size_t)(t + kGroups) * lay.P_pad];
                    a2 += p[(size_t)(t + 2 * kGroups) * lay.P_pad];
                    a3 += p[(size_t)(t + 3 * kGroups) * lay.P_pad];
                }
                for (; t < nt; t += kGroups) a0 += p[(size_t)t * lay.P_pad];
                g = (a0 + a1) + (a2 + a3);
            }
            gsum[grp][lane] = g;
            __syncthreads();
            if (grp == 0) {
                Real tot = gsum[0][lane];
#pragma unroll
                for (int gi = 1; gi < kGroups; ++gi) tot += gsum[gi][lane];
                if (q < lay.P_pad) {
                    st.gbuf[q] = tot;
                    sq += static_cast<double>(tot) * tot;
                }
            }
            __syncthreads();
        }
        const double tot = block_sum(sq, red);
        if (tid == 0) st.red_sq_part[rb] = tot;
    }
    // ---------------- last CTA finalises ------------------------------------------------
    if (tid == 0) {
        __threadfence();
        const unsigned ticket = atomicAdd(st.done_ctr, 1u);
        last = (ticket == gridDim.x - 1);
    }
    __syncthreads();
    if (!last || tid != 0) return;
    __threadfence();
    const int nrb = gridDim.x - es_blocks;
    const int w0 = pl.step_win_off[s];
    const int nt = (pl.step_win_off[s + 1] - w0 + R - 1) / R;
    double es = 0.0;
    if (st.attach)
        for (int b = 0; b < es_blocks; ++b) es += *reinterpret_cast<volatile double*>(st.es_sq_part + b);
    double ls = 0.0;
    for (int t = 0; t < nt; ++t) ls += st.loss_part[t];
    st.gbuf[lay.P_pad] = static_cast<Real>(es);
    st.gbuf[lay.P_pad + 1] = static_cast<Real>(ls);
    if (finalize) {
        double all = 0.0;
        for (int b = 0; b < nrb; ++b) all += *reinterpret_cast<volatile double*>(st.red_sq_part + b);
        finalize_scalars(st, pl, s, all + es, ls);
    }
    *st.done_ctr = 0;
}

// After the NCCL all-reduce of gbuf (sharded mode): global squared norm + scalars.
template <typename Real>
__global__ void k_finalize(StateDev<Real> st, PlanDev pl, NetLayout lay, int s) {
    __shared__ double red[32];
    __shared__ bool last;
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    double sq = 0.0;
    if (q < lay.P_pad) {
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
    for (unsigned b = 0; b < gridDim.x; ++b) all += *reinterpret_cast<volatile double*>(st.red_sq_part + b);
    const double es = st.attach ? static_cast<double>(st.gbuf[lay.P_pad]) : 0.0;
    finalize_scalars(st, pl, s, all + es, static_cast<double>(st.gbuf[lay.P_pad + 1]));
    st.done_ctr[1] = 0;
}

// ------------------------------------------------------------------------------ K4
template <typename Real>
__global__ void k_adam(StateDev<Real> st, PlanDev pl, NetLayout lay, int s) {
    if (st.err[0] != 0) return;  // the reference throws before apply_updates
    const double scale = st.scal[0], bc1 = st.scal[1], bc2 = st.scal[2];
    const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q < lay.P_pad) {
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
    const long long slot = q - lay.P_pad;
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
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int S = lay.S, I = lay.I, O = lay.O, in0 = lay.in0, N = st.N;
    // ring of the last S seasonalities plus the I window seasonalities needed at the end
    Real* ring = reinterpret_cast<Real*>(smem_raw);
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= N) return;
    const int bd = blockDim.x, tid = threadIdx.x;
    const Real* __restrict__ y = st.vals + row;
    for (int t = 0; t < t_ins; ++t)
        if (!(__ldg(y + (size_t)t * N) > Real(0))) {
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
        lp += __ldg(y + (size_t)j * N);
    }
    lp = lp / Real(S);
    // seasonality index u is produced at step u-S; window inputs need u in [t_ins-I, t_ins)
    Real* win = ring + S * bd;  // [I][bd]
    for (int u = t_ins - I; u < S && u < t_ins; ++u)
        if (u >= 0) win[(u - (t_ins - I)) * bd + tid] = ring[u * bd + tid];
    int j = 0;
    constexpr int CH = 8;
    for (int t0 = 0; t0 < t_ins; t0 += CH) {
        Real yb[CH];
#pragma unroll
        for (int u = 0; u < CH; ++u) yb[u] = (t0 + u < t_ins) ? __ldg(y + (size_t)(t0 + u) * N) : Real(1);
#pragma unroll
        for (int u = 0; u < CH; ++u) {
            const int t = t0 + u;
            if (t < t_ins) {
                const Real yt = yb[u];
                const Real s_t = ring[j * bd + tid];
                const Real l = alpha * (yt / s_t) + oma * lp;
                if (!(l > Real(0)) || !isfinite(l)) {
                    flag_error(st.err, kErrFcLevel, t);
                    return;
                }
                const Real sn = gamma * (yt / lp) + omg * s_t;
                ring[j * bd + tid] = sn;
                const int uu = t + S;
                if (uu >= t_ins - I && uu < t_ins) win[(uu - (t_ins - I)) * bd + tid] = sn;
                if (dump) {
                    dump_lv[t] = l;
                    dump_se[uu] = sn;
                }
                lp = l;
                j = (j + 1 == S) ? 0 : j + 1;
            }
        }
    }
    if (X == nullptr) return;
    const Real level = lp;
    for (int c = 0; c < I; ++c) {
        const Real sv = win[c * bd + tid];
        if (!(sv > Real(0))) {
            flag_error(st.err, kErrSeas, t_ins);
            return;
        }
        X[(size_t)row * in0 + c] = __ldg(y + (size_t)(t_ins - I + c) * N) / (level * sv);
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
