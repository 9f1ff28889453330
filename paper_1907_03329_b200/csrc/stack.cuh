// K2: the row-tile kernel — window gather/normalise, LSTM stack forward/backward at
// sequence length 1, masked pinball and its adjoint, per-tile weight-gradient partials
// and per-window ES adjoint contributions.
//
// Reference: build_graph (trainer.hpp:524-591), forward_stack / lstm_cell
// (network.hpp:148-210), ad::pinball (autodiff.hpp:370-395, adjoint :611-628) and the
// MatMul / Logistic / Tanh / Mul / Add / Div / Gather adjoints of Tape::backward
// (autodiff.hpp:428-610).
//
// A CTA owns R windows.  Weights: in resident mode the whole compact vector arrives in
// shared memory by one TMA bulk copy (cp.async.bulk + mbarrier) overlapped with the window
// gather; otherwise (fp64 nets that do not fit) one layer is staged at a time.
//
// The tile is a chain of barrier-separated phases, so the phase count is the latency:
//   forward   one phase per layer: thread (row pair, hidden unit) accumulates the three
//             live gate pre-activations (i, g, o) over the input and applies the cell
//             nonlinearities in registers (no separate gate phase);
//   backward  per layer: [combine input-adjoint partials + residual + gate adjoints] and
//             [input adjoint u_bar = pre_bar . W^T over q groups]; the weight-gradient
//             partials (not on the dependency chain) are produced afterwards for every
//             layer and the head in one barrier-free tail, coalesced over k.
// Thread mappings use power-of-two strides (shift/mask, no runtime integer division)
// and the product helpers are out-of-line so the kernel body stays i-cache resident.
#pragma once
#include "common.cuh"

namespace esrnn_dev {

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

constexpr int kRowsPerThread = 2;  // forward: 2 rows x 1 hidden unit (3 gates) per thread

template <int R>
__host__ __device__ inline int stack_threads_for_r(const NetLayout& lay) {
    const int nt = (R / kRowsPerThread) << log2_ceil(lay.H);
    return nt < 64 ? 64 : (nt > 512 ? 512 : nt);
}

// Shared-memory carve-up of one row tile (Real units; every offset a multiple of 4).
struct TileSmem {
    int w, xin, sin, sout, lvl, tgt, msk, act, gates, z, zb, pred, pbar, preb, hbar, resid, ubar, upart, total;
    int wsize;
    __host__ __device__ static int r4(int x) { return (x + 3) & ~3; }
    __host__ __device__ static long long stage_size(const NetLayout& lay) {
        long long m = lay.P_pad - lay.c_nlw;  // head segment
        for (int l = 0; l < lay.L; ++l) {
            const long long seg = lay.cb[l] - lay.cw[l] + 3 * lay.H;  // W^T_l and its bias
            m = seg > m ? seg : m;
        }
        return m;
    }
    __host__ __device__ static TileSmem make(const NetLayout& lay, int R, int NT, bool resident) {
        TileSmem t;
        const int H = lay.H, I = lay.I, L = lay.L;
        int o = 0;
        t.wsize = resident ? static_cast<int>(lay.P_pad) : r4(static_cast<int>(stage_size(lay)));
        t.w = o; o += t.wsize;
        t.xin = o; o += r4(R * lay.ldx);
        t.sin = o; o += r4(R * I);
        t.sout = o; o += r4(R * lay.ldo);
        t.lvl = o; o += r4(R);
        t.tgt = o; o += r4(R * lay.ldo);
        t.msk = o; o += r4(R * lay.ldo);
        t.act = o; o += r4(L * R * lay.ldh);
        t.gates = o; o += r4(4 * L * R * H);
        t.z = o; o += r4(R * lay.ldh);
        t.zb = o; o += r4(R * lay.ldh);
        t.pred = o; o += r4(R * lay.ldo);
        t.pbar = o; o += r4(R * lay.ldo);
        t.preb = o; o += r4(L * R * lay.ldg);
        t.hbar = o; o += r4(R * lay.ldh);
        t.resid = o; o += r4(R * lay.ldh);
        t.ubar = o; o += r4(R * (lay.ldx > lay.ldh ? lay.ldx : lay.ldh));
        t.upart = o; o += r4(R * NT);
        t.total = o;
        return t;
    }
};

// Iterate (r, c) over an R x W block: c = tid & (2^lw - 1), rows r = tid >> lw (+ stride).
template <typename F>
__device__ __forceinline__ void for_rc(int R, int W, F&& f) {
    const int lw = log2_ceil(W);
    const int nrg = blockDim.x >> lw;
    if (nrg > 0) {
        const int c = threadIdx.x & ((1 << lw) - 1), rg = threadIdx.x >> lw;
        if (c < W && rg < nrg)
            for (int r = rg; r < R; r += nrg) f(r, c);
    } else {
        for (int r = 0; r < R; ++r)
            for (int c = threadIdx.x; c < W; c += blockDim.x) f(r, c);
    }
}

// Vectorised global->shared copy of one contiguous segment (non-resident mode).
template <typename Real>
__device__ __forceinline__ void stage_segment(Real* __restrict__ dst, const Real* __restrict__ src, long long n) {
    for (long long e = threadIdx.x * 4LL; e < n; e += blockDim.x * 4LL) {
        if (e + 4 <= n) {
            if constexpr (sizeof(Real) == 4) {
                *reinterpret_cast<float4*>(dst + e) = __ldg(reinterpret_cast<const float4*>(src + e));
            } else {
                *reinterpret_cast<double2*>(dst + e) = __ldg(reinterpret_cast<const double2*>(src + e));
                *reinterpret_cast<double2*>(dst + e + 2) = __ldg(reinterpret_cast<const double2*>(src + e + 2));
            }
        } else {
            for (long long i = e; i < n; ++i) dst[i] = src[i];
        }
    }
}

// One LSTM layer at sequence length 1 (lstm_cell, network.hpp:148-163), fused:
// pre = u . W_in + b for the live gates of hidden unit hh, then i, g, o, c = i*g,
// h = o*tanh(c) (+ residual).  Thread (row group, hh), RPT rows each.
template <typename Real, int R, int RPT>
__device__ __noinline__ void fwd_layer(Real* __restrict__ gates, Real* __restrict__ out, const Real* __restrict__ radd,
                                       const Real* __restrict__ u, int ldu, const Real* __restrict__ WT, int ldk,
                                       const Real* __restrict__ bias, int in, int H, int ldh) {
    using M = Math<Real>;
    const int lh = log2_ceil(H);
    constexpr int NG = R / RPT;
    for (int idx = threadIdx.x; idx < (NG << lh); idx += blockDim.x) {
        const int hh = idx & ((1 << lh) - 1), rg = idx >> lh;
        if (hh >= H) continue;
        const Real* wi = WT + hh * ldk;
        const Real* wg = WT + (H + hh) * ldk;
        const Real* wo = WT + (2 * H + hh) * ldk;
        const Real* ub = u + rg * RPT * ldu;
        Real ai[RPT], ag[RPT], ao[RPT];
#pragma unroll
        for (int j = 0; j < RPT; ++j) ai[j] = ag[j] = ao[j] = 0;
        int k = 0;
#pragma unroll 1
        for (; k + 4 <= in; k += 4) {
            Real vi[4], vg[4], vo[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                vi[c] = wi[k + c];
                vg[c] = wg[k + c];
                vo[c] = wo[k + c];
            }
#pragma unroll
            for (int j = 0; j < RPT; ++j) {
                const V4<Real> x = lds4(ub + j * ldu + k);
                const Real xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    ai[j] += xs[c] * vi[c];
                    ag[j] += xs[c] * vg[c];
                    ao[j] += xs[c] * vo[c];
                }
            }
        }
#pragma unroll 1
        for (; k < in; ++k) {
            const Real a = wi[k], b = wg[k], c = wo[k];
#pragma unroll
            for (int j = 0; j < RPT; ++j) {
                const Real x = ub[j * ldu + k];
                ai[j] += x * a;
                ag[j] += x * b;
                ao[j] += x * c;
            }
        }
        const Real bi = bias[hh], bg = bias[H + hh], bo = bias[2 * H + hh];
        const int RH = R * H;
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            const int r = rg * RPT + j;
            const Real i = M::logistic(ai[j] + bi);
            const Real g = M::tanh(ag[j] + bg);
            const Real o = M::logistic(ao[j] + bo);
            const Real c = i * g;
            const Real tc = M::tanh(c);
            Real h = o * tc;
            if (radd) h = h + radd[r * ldh + hh];
            const int e = r * H + hh;
            gates[e] = i;
            gates[RH + e] = g;
            gates[2 * RH + e] = o;
            gates[3 * RH + e] = tc;
            out[r * ldh + hh] = h;
        }
    }
}

// out[r][q] = act(sum_k u[r][k] * WT[q][k] + bias[q]) for the head (q < G).
template <typename Real, int R, int RPT>
__device__ __noinline__ void gemm_fwd(Real* __restrict__ out, int ldo, const Real* __restrict__ u, int ldu,
                                      const Real* __restrict__ WT, int ldk, const Real* __restrict__ bias, int in, int G,
                                      bool tanh_act) {
    using M = Math<Real>;
    const int lg = log2_ceil(G);
    constexpr int NG = R / RPT;
    for (int idx = threadIdx.x; idx < (NG << lg); idx += blockDim.x) {
        const int q = idx & ((1 << lg) - 1), rg = idx >> lg;
        if (q >= G) continue;
        const Real* w = WT + q * ldk;
        const Real* ub = u + rg * RPT * ldu;
        Real acc[RPT];
#pragma unroll
        for (int j = 0; j < RPT; ++j) acc[j] = 0;
        int k = 0;
#pragma unroll 1
        for (; k + 4 <= in; k += 4) {
            const Real w0 = w[k], w1 = w[k + 1], w2 = w[k + 2], w3 = w[k + 3];
#pragma unroll
            for (int j = 0; j < RPT; ++j) {
                const V4<Real> x = lds4(ub + j * ldu + k);
                acc[j] += x.x * w0;
                acc[j] += x.y * w1;
                acc[j] += x.z * w2;
                acc[j] += x.w * w3;
            }
        }
#pragma unroll 1
        for (; k < in; ++k) {
            const Real wk = w[k];
#pragma unroll
            for (int j = 0; j < RPT; ++j) acc[j] += ub[j * ldu + k] * wk;
        }
        const Real b = bias[q];
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            const Real v = acc[j] + b;
            out[(rg * RPT + j) * ldo + q] = tanh_act ? M::tanh(v) : v;
        }
    }
}

// q groups for the adjoint products: thread (group, k) with lanes over k.
__device__ __forceinline__ void q_groups(int in, int G, int& li, int& QG, int& qs) {
    li = log2_ceil(in);
    QG = static_cast<int>(blockDim.x) >> li;
    QG = QG < 1 ? 1 : QG;
    qs = (G + QG - 1) / QG;
    qs = (qs + 3) & ~3;
    QG = (G + qs - 1) / qs;
}

// Input adjoint partials: upart[g][r][k] = sum_{q in group g} a[r][q] * WT[q][k].
// Returns the number of groups (QG) the caller sums in a fixed order.
template <typename Real, int R>
__device__ __noinline__ int gemm_adj(Real* __restrict__ upart, const Real* __restrict__ a, int lda,
                                     const Real* __restrict__ WT, int ldk, int in, int G) {
    int li, QG, qs;
    q_groups(in, G, li, QG, qs);
    for (int idx = threadIdx.x; idx < (QG << li); idx += blockDim.x) {
        const int k = idx & ((1 << li) - 1), g = idx >> li;
        if (k >= in) continue;
        const int q0 = g * qs, q1 = min(G, q0 + qs);
        Real au[R];
#pragma unroll
        for (int r = 0; r < R; ++r) au[r] = 0;
        int q = q0;
#pragma unroll 1
        for (; q + 4 <= q1; q += 4) {
            const Real w0 = WT[(q + 0) * ldk + k], w1 = WT[(q + 1) * ldk + k];
            const Real w2 = WT[(q + 2) * ldk + k], w3 = WT[(q + 3) * ldk + k];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const V4<Real> x = lds4(a + r * lda + q);
                au[r] += x.x * w0;
                au[r] += x.y * w1;
                au[r] += x.z * w2;
                au[r] += x.w * w3;
            }
        }
#pragma unroll 1
        for (; q < q1; ++q) {
            const Real w = WT[q * ldk + k];
#pragma unroll
            for (int r = 0; r < R; ++r) au[r] += a[r * lda + q] * w;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) upart[(g * R + r) * in + k] = au[r];
    }
    return QG;
}

// Weight-gradient partials of one matrix, part_w[q*ldk + k] = sum_r u[r][k] * a[r][q]
// (rows summed in order), plus the bias partial part_b[q] = sum_r a[r][q].  Reads only
// shared memory that is final by now and writes disjoint global ranges: consecutive calls
// need no barrier.
template <typename Real, int R>
__device__ __noinline__ void gemm_wgrad(Real* __restrict__ part_w, Real* __restrict__ part_b, const Real* __restrict__ u,
                                        int ldu, const Real* __restrict__ a, int lda, int ldk, int in, int G) {
    int li, QG, qs;
    q_groups(in, G, li, QG, qs);
    for (int idx = threadIdx.x; idx < (QG << li); idx += blockDim.x) {
        const int k = idx & ((1 << li) - 1), g = idx >> li;
        if (k >= in) continue;
        const int q0 = g * qs, q1 = min(G, q0 + qs);
        Real uk[R];
#pragma unroll
        for (int r = 0; r < R; ++r) uk[r] = u[r * ldu + k];
        int q = q0;
#pragma unroll 1
        for (; q + 4 <= q1; q += 4) {
            Real g0 = 0, g1 = 0, g2 = 0, g3 = 0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const V4<Real> x = lds4(a + r * lda + q);
                g0 += uk[r] * x.x;
                g1 += uk[r] * x.y;
                g2 += uk[r] * x.z;
                g3 += uk[r] * x.w;
            }
            part_w[(q + 0) * ldk + k] = g0;
            part_w[(q + 1) * ldk + k] = g1;
            part_w[(q + 2) * ldk + k] = g2;
            part_w[(q + 3) * ldk + k] = g3;
        }
#pragma unroll 1
        for (; q < q1; ++q) {
            Real g0 = 0;
#pragma unroll
            for (int r = 0; r < R; ++r) g0 += uk[r] * a[r * lda + q];
            part_w[q * ldk + k] = g0;
        }
    }
    for (int q = threadIdx.x; q < G; q += blockDim.x) {
        Real acc = 0;
#pragma unroll
        for (int r = 0; r < R; ++r) acc += a[r * lda + q];
        part_b[q] = acc;
    }
}

// Row tile of R windows (kTrain / kLossOnly) or R series (kForecast).
template <typename Real, int R, int MODE, bool RESIDENT>
__global__ void __launch_bounds__(512) k_stack(StateDev<Real> st, PlanDev pl, NetLayout lay_p, int s, ForecastArgs fa) {
    using M = Math<Real>;
    constexpr int RPT = kRowsPerThread;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Real* sm = reinterpret_cast<Real*>(smem_raw);
    __shared__ double red[32];
    __shared__ __align__(8) uint64_t wbar;
    // the layout is read with dynamic layer indices in every phase: one shared copy
    __shared__ NetLayout lay_s;
    if (threadIdx.x == 0) lay_s = lay_p;
    __syncthreads();
    const NetLayout& lay = lay_s;
    const int tid = threadIdx.x, NT = blockDim.x;
    const TileSmem ts = TileSmem::make(lay, R, NT, RESIDENT);
    const int H = lay.H, O = lay.O, I = lay.I, in0 = lay.in0, L = lay.L, G = 3 * H;
    const int ldx = lay.ldx, ldh = lay.ldh, ldg = lay.ldg, ldo = lay.ldo, ldkh = lay.ldkh;
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
    Real* zb = sm + ts.zb;
    Real* pred = sm + ts.pred;
    Real* pbar = sm + ts.pbar;
    Real* preb = sm + ts.preb;
    Real* resid = sm + ts.resid;
    Real* ubar = sm + ts.ubar;
    Real* upart = sm + ts.upart;

    int nrows, w0 = 0;
    if (MODE == kForecast) {
        nrows = min(R, st.N - tile * R);
    } else {
        w0 = pl.step_win_off[s];
        const int Bl = pl.step_win_off[s + 1] - w0;
        nrows = min(R, Bl - tile * R);
    }
    if (nrows <= 0) return;
    int _dbg = 0;
    if (MODE == kTrain) DBG_GT(st, 2);
    DBG_CLK(st, 0);

    // ---- weights: TMA bulk copy of the compact parameter vector (resident mode) ----
    if (RESIDENT && tid == 0) {
        mbar_init(&wbar, 1);
        const unsigned total = static_cast<unsigned>(lay.P_pad * sizeof(Real));
        mbar_expect_tx(&wbar, total);
        constexpr unsigned kChunk = 32768;
        for (unsigned off = 0; off < total; off += kChunk) {
            const unsigned n = total - off < kChunk ? total - off : kChunk;
            bulk_g2s(reinterpret_cast<unsigned char*>(wsm) + off, reinterpret_cast<const unsigned char*>(th) + off, n,
                     &wbar);
        }
    }

    // ---- prologue: window gather + normalisation (trainer.hpp:532-566) -------------
    if (MODE == kForecast) {
        const Real* X = reinterpret_cast<const Real*>(fa.X);
        const Real* FL = reinterpret_cast<const Real*>(fa.lvl);
        const Real* FS = reinterpret_cast<const Real*>(fa.sout);
        for_rc(R, ldx, [&](int r, int c) {
            xin[r * ldx + c] = (r < nrows && c < in0) ? X[(size_t)(tile * R + r) * in0 + c] : Real(0);
        });
        for_rc(R, O, [&](int r, int o) { s_out[r * ldo + o] = r < nrows ? FS[(size_t)(tile * R + r) * O + o] : Real(0); });
        for (int r = tid; r < R; r += NT) lvl[r] = r < nrows ? FL[tile * R + r] : Real(0);
    } else {
        // column c < I: input window; c < I+O: target window; c == I+O: level; the rest: one-hot
        for_rc(R, I + O + 1 + (ldx - I), [&](int r, int c) {
            const int wb = w0 + tile * R + r;
            if (r >= nrows) {
                if (c < I) {
                    xin[r * ldx + c] = 0;
                    s_in[r * I + c] = 1;
                } else if (c < I + O) {
                    tgt[r * ldo + c - I] = 0;
                    s_out[r * ldo + c - I] = 1;
                    msk[r * ldo + c - I] = 0;
                } else if (c == I + O) {
                    lvl[r] = 1;
                } else {
                    xin[r * ldx + (c - O - 1)] = 0;
                }
                return;
            }
            const int row = pl.w_row[wb];
            if (c > I + O) {
                const int cc = c - O - 1;  // x column in [I, ldx)
                xin[r * ldx + cc] = (cc < in0 && st.cat[row] == cc - I) ? Real(1) : Real(0);
                return;
            }
            const int a = pl.w_anchor[wb], slot = pl.w_slot[wb];
            const Real l = st.lv[a * st.kcap + slot];
            if (c < I) {
                const int idx = a - I + 1 + c;
                const Real sv = st.se[idx * st.kcap + slot];
                xin[r * ldx + c] = fdiv(st.vrm[(size_t)row * st.ldv + idx], sv * l);
                s_in[r * I + c] = sv;
            } else if (c < I + O) {
                const int j = c - I, idx = a + 1 + j;
                const Real sv = st.se[idx * st.kcap + slot];
                tgt[r * ldo + j] = fdiv(st.vrm[(size_t)row * st.ldv + idx], sv * l);
                s_out[r * ldo + j] = sv;
                msk[r * ldo + j] = (pl.mask == nullptr || pl.mask[(size_t)wb * O + j] != 0) ? Real(1) : Real(0);
            } else {
                lvl[r] = l;
            }
        });
    }
    __syncthreads();
    DBG_CLK(st, 1);
    if (MODE != kForecast && st.d_inputs != nullptr) {
        const int base = tile * R;
        for_rc(nrows, in0, [&](int r, int c) { st.d_inputs[(size_t)(base + r) * in0 + c] = xin[r * ldx + c]; });
        for_rc(nrows, O, [&](int r, int o) {
            st.d_targets[(size_t)(base + r) * O + o] = tgt[r * ldo + o];
            st.d_seas[(size_t)(base + r) * O + o] = s_out[r * ldo + o];
        });
        for (int r = tid; r < nrows; r += NT) st.d_levels[base + r] = lvl[r];
    }
    if (RESIDENT) mbar_wait(&wbar, 0);

    // ---- forward through the stack (network.hpp:148-210, sequence length 1) --------
    for (int l = 0; l < L; ++l) {
        const Real* u = l == 0 ? xin : act + (l - 1) * R * ldh;
        if (!RESIDENT) {
            stage_segment(wsm, th + lay.cw[l], lay.cb[l] - lay.cw[l] + G);
            __syncthreads();
        }
        const Real* WT = RESIDENT ? wsm + lay.cw[l] : wsm;
        const Real* bias = RESIDENT ? wsm + lay.cb[l] : wsm + (lay.cb[l] - lay.cw[l]);
        const Real* radd = lay.block_last[l] ? act + lay.res_src[l] * R * ldh : nullptr;
        fwd_layer<Real, R, RPT>(gates + 4 * l * R * H, act + l * R * ldh, radd, u, l == 0 ? ldx : ldh, WT, lay.ldk[l],
                                bias, lay.layer_in[l], H, ldh);
        __syncthreads();
        DBG_CLK(st, 2);
    }
    // head (network.hpp:207-209)
    const Real* cur = act + (L - 1) * R * ldh;
    if (!RESIDENT) {
        stage_segment(wsm, th + lay.c_nlw, lay.P_pad - lay.c_nlw);
        __syncthreads();
    }
    const long long hb0 = RESIDENT ? 0 : lay.c_nlw;
    const Real* nlwT = wsm + (lay.c_nlw - hb0);
    const Real* nlb = wsm + (lay.c_nlb - hb0);
    const Real* owT = wsm + (lay.c_outw - hb0);
    const Real* obias = wsm + (lay.c_outb - hb0);
    gemm_fwd<Real, R, RPT>(z, ldh, cur, ldh, nlwT, ldkh, nlb, H, H, true);
    __syncthreads();
    gemm_fwd<Real, R, RPT>(pred, ldo, z, ldh, owT, ldkh, obias, H, O, false);
    __syncthreads();
    DBG_CLK(st, 3);
    if (MODE == kForecast) {
        for_rc(nrows, O, [&](int r, int o) {
            fa.out[(size_t)(tile * R + r) * O + o] = static_cast<double>(pred[r * ldo + o] * lvl[r] * s_out[r * ldo + o]);
        });
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
    // masked pinball (autodiff.hpp:384-392) and its adjoint (:620-626)
    double lsum = 0.0;
    const Real gscale = static_cast<Real>(1.0 / pl.step_M[s]);
    const Real tau = static_cast<Real>(st.tau);
    for_rc(R, ldo, [&](int r, int o) {
        const int e = r * ldo + o;
        Real pb = 0;
        if (o < O && msk[e] != Real(0)) {
            const Real p = pred[e], t = tgt[e];
            const Real d = t - p;
            lsum += (d >= Real(0)) ? st.tau * static_cast<double>(d) : (st.tau - 1.0) * static_cast<double>(d);
            pb = gscale * ((t >= p) ? -tau : Real(1) - tau);
        }
        pbar[e] = pb;
    });
    const double ltot = block_sum(lsum, red);  // its barriers also publish pbar
    if (tid == 0) st.loss_part[tile] = ltot;
    if (MODE == kLossOnly) return;
    DBG_CLK(st, 4);

    // ---- backward: the dependency chain (input adjoints only) -----------------------
    int QG = gemm_adj<Real, R>(upart, pbar, ldo, owT, ldkh, H, O);
    __syncthreads();
    for_rc(R, H, [&](int r, int k) {  // z adjoint through tanh
        Real acc = 0;
        for (int g = 0; g < QG; ++g) acc += upart[(g * R + r) * H + k];
        const Real zz = z[r * ldh + k];
        zb[r * ldh + k] = acc * (Real(1) - zz * zz);
    });
    __syncthreads();
    QG = gemm_adj<Real, R>(upart, zb, ldh, nlwT, ldkh, H, H);
    __syncthreads();
    DBG_CLK(st, 5);
    for (int l = L - 1; l >= 0; --l) {
        // h_bar of layer l = input adjoint of the layer above (+ the block residual adjoint
        // when layer l+1 opens a block b>0); the gate adjoints follow in the same phase
        const bool add_res = (l + 1 < L) && lay.block_first[l + 1];
        const bool save_res = lay.block_last[l] != 0;
        const Real* gl = gates + 4 * l * R * H;
        Real* pb = preb + l * R * ldg;
        const int QGc = QG;
        for_rc(R, H, [&](int r, int hh) {
            Real hb = 0;
            for (int g = 0; g < QGc; ++g) hb += upart[(g * R + r) * H + hh];
            if (add_res) hb = hb + resid[r * ldh + hh];
            if (save_res) resid[r * ldh + hh] = hb;
            const int e = r * H + hh, RH = R * H;
            const Real i = gl[e], g = gl[RH + e], o = gl[2 * RH + e], tc = gl[3 * RH + e];
            const Real ob = hb * tc;
            const Real cb = (hb * o) * (Real(1) - tc * tc);
            const Real ib = cb * g, gb = cb * i;
            pb[r * ldg + hh] = ib * i * (Real(1) - i);
            pb[r * ldg + H + hh] = gb * (Real(1) - g * g);
            pb[r * ldg + 2 * H + hh] = ob * o * (Real(1) - o);
        });
        if (!RESIDENT) stage_segment(wsm, th + lay.cw[l], lay.cb[l] - lay.cw[l]);
        __syncthreads();
        const Real* WT = RESIDENT ? wsm + lay.cw[l] : wsm;
        QG = gemm_adj<Real, R>(upart, pb, ldg, WT, lay.ldk[l], lay.layer_in[l], G);
        __syncthreads();
        DBG_CLK(st, 6);
    }
    // x_bar (layer 0's input adjoint) for the ES contributions
    for_rc(R, in0, [&](int r, int k) {
        Real acc = 0;
        for (int g = 0; g < QG; ++g) acc += upart[(g * R + r) * in0 + k];
        ubar[r * ldx + k] = acc;
    });

    // ---- weight-gradient partials: every matrix of the tile, no barriers in between ----
    Real* __restrict__ part = st.part + (size_t)tile * lay.P_pad;
    gemm_wgrad<Real, R>(part + lay.c_outw, part + lay.c_outb, z, ldh, pbar, ldo, ldkh, H, O);
    gemm_wgrad<Real, R>(part + lay.c_nlw, part + lay.c_nlb, cur, ldh, zb, ldh, ldkh, H, H);
    for (int l = L - 1; l >= 0; --l)
        gemm_wgrad<Real, R>(part + lay.cw[l], part + lay.cb[l], l == 0 ? xin : act + (l - 1) * R * ldh,
                            l == 0 ? ldx : ldh, preb + l * R * ldg, ldg, lay.ldk[l], lay.layer_in[l], G);
    __syncthreads();
    DBG_CLK(st, 7);

    // ---- ES adjoint contributions per window (Div / Mul / BroadcastCol adjoints) ----
    // written in slot-major CSR order so each slot's windows are contiguous for K3;
    // row = [inputs (s index a-I+1..a) | targets (a+1..a+O) | level a | anchor a]
    if (st.attach) {
        for (int r = tid; r < nrows; r += NT) {
            Real* __restrict__ cr = st.contrib + (size_t)pl.w_csr[w0 + tile * R + r] * st.cwp;
            cr[I + O + 1] = static_cast<Real>(pl.w_anchor[w0 + tile * R + r]);  // exact (< 2^24)
            const Real lv = lvl[r];
            Real acc_o = 0;
            for (int j = 0; j < O; ++j) {
                const Real tb = -pbar[r * ldo + j];
                const Real den = s_out[r * ldo + j] * lv;
                const Real denb = -fdiv(tb * tgt[r * ldo + j], den);
                cr[I + j] = denb * lv;
                acc_o += denb * s_out[r * ldo + j];
            }
            Real acc_i = 0;
            for (int j = 0; j < I; ++j) {
                const Real den = s_in[r * I + j] * lv;
                const Real denb = -fdiv(ubar[r * ldx + j] * xin[r * ldx + j], den);
                cr[j] = denb * lv;
                acc_i += denb * s_in[r * I + j];
            }
            cr[O + I] = acc_o + acc_i;
        }
    }
    if (MODE == kTrain) DBG_GT(st, 3);
}

}  // namespace esrnn_dev
