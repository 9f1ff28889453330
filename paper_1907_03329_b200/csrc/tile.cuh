// K2 k_tile: the row-tile kernel — window gather/normalise, LSTM stack forward/backward at
// sequence length 1, masked pinball and its adjoint, per-window ES adjoint contributions.
// The weight gradients are NOT formed here: the tile writes each window's layer inputs and
// gate adjoints to the step's row store, and K3 contracts them over the whole batch
// (finish.cuh, k_grad_finish GEMM blocks).
//
// Reference: build_graph (trainer.hpp:524-591), forward_stack / lstm_cell
// (network.hpp:148-210), ad::pinball (autodiff.hpp:370-395, adjoint :611-628) and the
// MatMul / Logistic / Tanh / Mul / Add / Div / Gather adjoints of Tape::backward
// (autodiff.hpp:428-610).
//
// A CTA owns R = 8 windows.  Every activation-like array lives in shared memory
// feature-major, [feature][kLdr] with the 8 rows contiguous, so one feature's 8 rows are two
// 16-byte loads that a warp broadcasts.  The products are warp reduce-scatters:
//
//   forward  (outputs = hidden units)  lane = (ks = lane>>2, c = lane&3): unit c of the warp,
//            inputs k = ks (mod 8); 8 row accumulators per gate; three xor-shuffle levels
//            (16, 8, 4) fold the 8 k-slices and leave lane ks owning row r = ks, so the cell
//            nonlinearities run right after the product, no extra phase;
//   backward (outputs = input features) lane = (qs = lane>>2, c = lane&3): feature c of the
//            warp's 4, gate rows q = qs (mod 8); the same three shuffle levels leave lane qs
//            owning row r = qs, and the lane immediately forms the gate adjoints of the layer
//            below.
//
// W^T rows have stride ldk = 8 * odd (NetLayout), which makes both access patterns
// bank-conflict free.  One barrier per layer forward and one per layer backward.
#pragma once
#include "common.cuh"

// k_tile<kLossOnly> returns after the loss; its backward half is statically unreachable
#pragma nv_diag_suppress 128

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
    double* mase;        // [N] or nullptr (evaluate)
    const double* score; // [N] MASE scale from k_forecast_scan (evaluate)
};

constexpr int kR = 8;  // windows per tile = the reduce-scatter fan-in

// row-set stride: 8 rows + padding so the 8 k-slices' 16-byte loads hit distinct bank groups
template <typename Real>
__host__ __device__ constexpr int ldr() {
    return sizeof(Real) == 4 ? 12 : 10;
}

__host__ __device__ inline int tile_threads(const NetLayout& lay) {
    int w = (lay.H + 3) / 4;                                        // forward: 4 units per warp
    const int wb = ((lay.in0 > lay.H ? lay.in0 : lay.H) + 3) / 4;  // backward: 4 features per warp
    w = w > wb ? w : wb;
    w = w < 4 ? 4 : (w > 16 ? 16 : w);
    return 32 * w;
}

// Shared-memory carve-up of one tile (Real units, offsets multiples of 4).
struct TileSmem {
    int w, wsize, xt, ht, gt, zt, pt, pbt, zbt, prt0, prt1, rest, ubt, sin, sout, lvl, tgt, msk, ys, lvr, ser, psm, total;
    int tp, ldl, lds;  // staged-row stride, level / seasonality row strides of the tile's scans
    __host__ __device__ static int r4(int x) { return (x + 3) & ~3; }
    __host__ __device__ static long long stage_size(const NetLayout& lay) {
        long long m = lay.P_pad - lay.c_nlw;  // head segment
        for (int l = 0; l < lay.L; ++l) {
            const long long seg = lay.cb[l] - lay.cw[l] + 3 * lay.H;  // W^T_l and its bias
            m = seg > m ? seg : m;
        }
        return m;
    }
    template <typename Real>
    __host__ __device__ static TileSmem make(const NetLayout& lay, bool resident) {
        TileSmem t;
        constexpr int LD = ldr<Real>();
        const int H = lay.H, L = lay.L, O = lay.O;
        int o = 0;
        t.wsize = resident ? static_cast<int>(lay.P_pad) : r4(static_cast<int>(stage_size(lay)));
        t.w = o; o += t.wsize;
        t.xt = o; o += r4(lay.in0 * LD);
        t.ht = o; o += r4(L * H * LD);
        t.gt = o; o += r4(4 * L * H * kR);
        t.zt = o; o += r4(H * LD);
        t.pt = o; o += r4(O * LD);
        t.pbt = o; o += r4(O * LD);
        t.zbt = o; o += r4(H * LD);
        t.prt0 = o; o += r4(3 * H * LD);
        t.prt1 = o; o += r4(3 * H * LD);
        t.rest = o; o += r4(H * LD);
        t.ubt = o; o += r4(lay.in0 * LD);
        t.sin = o; o += r4(kR * lay.I);
        t.sout = o; o += r4(kR * lay.ldo);
        t.lvl = o; o += r4(kR);
        t.tgt = o; o += r4(kR * lay.ldo);
        t.msk = o; o += r4(kR * lay.ldo);
        // Holt-Winters scans of the tile's rows: observations [R][tp], levels [R][T],
        // seasonalities [R][T+S]
        t.tp = row_pad<Real>(lay.T);
        t.ldl = r4(lay.T);
        t.lds = r4(lay.T + lay.S);
        t.ys = o; o += kR * t.tp;
        t.lvr = o; o += kR * t.ldl;
        t.ser = o; o += kR * t.lds;
        t.psm = o; o += r4(kR * (2 + lay.S));
        t.total = o;
        return t;
    }
};

// acc[r] += x[r] * w over the 8 rows; fp32 pairs rows into Blackwell's paired FMA (FFMA2,
// two independent round-to-nearest FMAs: bit-identical to the scalar form)
template <typename Real>
__device__ __forceinline__ void fma_rows(Real (&acc)[kR], const Real (&x)[kR], Real w) {
    if constexpr (sizeof(Real) == 4) {
#pragma unroll
        for (int r = 0; r < kR; r += 2)
            asm("{ .reg .b64 a, x, w;\n\t"
                "mov.b64 a, {%0, %1};\n\t"
                "mov.b64 x, {%2, %3};\n\t"
                "mov.b64 w, {%4, %4};\n\t"
                "fma.rn.f32x2 a, x, w, a;\n\t"
                "mov.b64 {%0, %1}, a; }"
                : "+f"(acc[r]), "+f"(acc[r + 1])
                : "f"(x[r]), "f"(x[r + 1]), "f"(w));
    } else {
#pragma unroll
        for (int r = 0; r < kR; ++r) acc[r] += x[r] * w;
    }
}

// Offsets of the two 4-row halves a lane loads first / second: lanes with bit 4 set load the
// halves swapped (reduce_scatter8's first level then needs no selects)
__device__ __forceinline__ int row_half0(int lane) { return (lane & 16) ? 4 : 0; }

template <typename Real>
__device__ __forceinline__ void ld_rows(Real (&x)[kR], const Real* p0, const Real* p1) {
    const V4<Real> a = lds4(p0), b = lds4(p1);
    x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
    x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
}


// Reduce-scatter of per-lane partial sums over the warp's 8 slices (lane bits 4, 3, 2):
// afterwards lane keeps in out[u] the full sum of row lane>>2.  acc[u][j] holds row j, except
// that lanes with bit 4 set hold row j ^ 4 (their row halves are loaded swapped, see
// row_halves), so the first level exchanges acc[j + 4] for acc[j] without selects.
template <typename Real, int U>
__device__ __forceinline__ void reduce_scatter8(Real (&out)[U], Real (&acc)[U][kR], int lane) {
    const bool b1 = lane & 8, b0 = lane & 4;
    Real a4[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < 4; ++j) a4[u][j] = acc[u][j] + __shfl_xor_sync(0xffffffffu, acc[u][j + 4], 16);
    Real a2[U][2];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const Real send = b1 ? a4[u][j] : a4[u][j + 2];
            const Real keep = b1 ? a4[u][j + 2] : a4[u][j];
            a2[u][j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
        }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const Real send = b0 ? a2[u][0] : a2[u][1];
        const Real keep = b0 ? a2[u][1] : a2[u][0];
        out[u] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
}

// Forward-type product for the lane's U output units (W^T rows wrow[u]): returns in out[u]
// the full sum over k < K for row r = lane>>2.  All 32 lanes must call (shuffles).
template <typename Real, int U>
__device__ __forceinline__ void fwd_prod(Real (&out)[U], const Real* __restrict__ XT, const Real* const (&wrow)[U],
                                         int K) {
    constexpr int LD = ldr<Real>();
    const int lane = threadIdx.x & 31, ks = lane >> 2;
    Real acc[U][kR];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
        for (int r = 0; r < kR; ++r) acc[u][r] = 0;
    const Real* X0 = XT + row_half0(lane);
    const Real* X1 = XT + (4 - row_half0(lane));
#pragma unroll 2
    for (int k = ks; k < K; k += 8) {
        Real x[kR];
        ld_rows(x, X0 + k * LD, X1 + k * LD);
#pragma unroll
        for (int u = 0; u < U; ++u) fma_rows<Real>(acc[u], x, wrow[u][k]);
    }
    reduce_scatter8<Real, U>(out, acc, lane);
}

// Backward-type product for one input feature k per lane quad (column wcol = WT + k):
// returns the full sum over q < Q of AT[q][r] * WT[q*ldk + k] for row r = lane>>2.  Eight
// q-slices per warp (lane bits 4, 3, 2) and the forward's reduce-scatter, so a warp covers 4
// features and a layer's input adjoint spreads over all warps.  All 32 lanes must call.
template <typename Real>
__device__ __forceinline__ Real bwd_prod(const Real* __restrict__ AT, const Real* __restrict__ wcol, int ldk, int Q) {
    constexpr int LD = ldr<Real>();
    const int lane = threadIdx.x & 31, qs = lane >> 2;
    Real acc[1][kR];
#pragma unroll
    for (int r = 0; r < kR; ++r) acc[0][r] = 0;
    const Real* A0 = AT + row_half0(lane);
    const Real* A1 = AT + (4 - row_half0(lane));
#pragma unroll 2
    for (int q = qs; q < Q; q += 8) {
        Real a[kR];
        ld_rows(a, A0 + q * LD, A1 + q * LD);
        fma_rows<Real>(acc[0], a, wcol[q * ldk]);
    }
    Real out[1];
    reduce_scatter8<Real, 1>(out, acc, lane);
    return out[0];
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

// Gate adjoints of one cell (Mul / Tanh / Logistic adjoints of lstm_cell): from h_bar and the
// saved i, g, o, tanh(c) to the pre-activation adjoints of the live gates.
template <typename Real>
__device__ __forceinline__ void cell_adjoint(Real hb, Real i, Real g, Real o, Real tc, Real& pi, Real& pg, Real& po) {
    const Real ob = hb * tc;
    const Real cb = (hb * o) * (Real(1) - tc * tc);
    const Real ib = cb * g, gb = cb * i;
    pi = ib * i * (Real(1) - i);
    pg = gb * (Real(1) - g * g);
    po = ob * o * (Real(1) - o);
}

// Row tile of R windows (kTrain / kLossOnly) or R series (kForecast).
// Training scan of one series over its train segment (hybrid_primer_tape,
// holt_winters.hpp:236-283): l_{-1} = mean(y[0:S]); l_t = a*y_t/s_t + (1-a)*l_{t-1};
// s_{t+S} = g*y_t/l_{t-1} + (1-g)*s_t.  ys: the staged row; lv[t], se[t] out (shared).
// SC > 0: the last S seasonalities live in a register ring; SC == 0: se[] is the ring.
// Returns the first step with a non-positive / non-finite level, INT_MAX if none.
// CHECK = false: no level check in the serial loop (K3 reruns the scan K2 already checked;
// returns INT_MAX).
template <typename Real, int SC, bool CHECK = true>
__device__ __forceinline__ int hw_scan_row(const Real* __restrict__ ys, const Real* __restrict__ pr, int T, int S,
                                           Real* __restrict__ lv, Real* __restrict__ se) {
    using M = Math<Real>;
    const Real alpha = M::logistic_ps(pr[0]);
    const Real gamma = M::logistic_ps(pr[1]);
    const Real oma = Real(1) - alpha, omg = Real(1) - gamma;
    constexpr Real kMax = sizeof(Real) == 4 ? Real(FLT_MAX) : Real(DBL_MAX);
    Real lp = 0;
    int bad = INT_MAX;
    if constexpr (SC > 0) {
        Real rg[SC], yv[SC];
#pragma unroll
        for (int j = 0; j < SC; ++j) {
            rg[j] = M::exp_ps(pr[2 + j]);
            se[j] = rg[j];
            yv[j] = ys[j];
            lp += yv[j];
        }
        lp = lp / Real(SC);
        // l depends on l_{t-1} through one FMA; the reciprocals feed steps S later
        auto step = [&](int t, Real& sj, Real yt) {
            const Real l = alpha * (yt * rcp_of(sj)) + oma * lp;
            if constexpr (CHECK) {
                const bool ok = (l > Real(0)) & (l <= kMax);
                bad = min(bad, ok ? INT_MAX : t);
            }
            sj = gamma * (yt * rcp_of(lp)) + omg * sj;
            se[t + SC] = sj;
            lv[t] = l;
            lp = l;
        };
        // groups of SC steps, the next group's observations loaded before this group's
        // stores (shared-memory loads cannot move past possibly-aliasing stores)
        int t0 = 0;
        for (; t0 + SC <= T; t0 += SC) {
            Real yn[SC];
#pragma unroll
            for (int j = 0; j < SC; ++j) yn[j] = t0 + SC + j < T ? ys[t0 + SC + j] : Real(0);
#pragma unroll
            for (int j = 0; j < SC; ++j) step(t0 + j, rg[j], yv[j]);
#pragma unroll
            for (int j = 0; j < SC; ++j) yv[j] = yn[j];
        }
#pragma unroll
        for (int j = 0; j < SC; ++j)
            if (t0 + j < T) step(t0 + j, rg[j], yv[j]);
    } else {
        for (int j = 0; j < S; ++j) {
            se[j] = M::exp_ps(pr[2 + j]);
            lp += ys[j];
        }
        lp = lp / Real(S);
#pragma unroll 4
        for (int t = 0; t < T; ++t) {
            const Real yt = ys[t];
            const Real s_t = se[t];
            const Real l = alpha * fdiv(yt, s_t) + oma * lp;
            if constexpr (CHECK) {
                const bool ok = (l > Real(0)) & (l <= kMax);
                bad = min(bad, ok ? INT_MAX : t);
            }
            se[t + S] = gamma * fdiv(yt, lp) + omg * s_t;
            lv[t] = l;
            lp = l;
        }
    }
    return bad;
}

// RESIDENT: all weights in shared memory, one CTA per SM; staged fp32 tiles (weights one
// layer at a time) fit two CTAs per SM, so their register budget is capped accordingly.
// NG = 2 (fp32, resident): two tiles per CTA, one group of warps each, sharing ONE resident copy
// of the weights (one TMA copy per CTA); each group synchronises on its own named barrier.
// Two Quarterly tiles fit one SM this way (77 KB of weights + 2 x 56 KB) where two CTAs of one
// tile each (2 x 133 KB) do not, so multi-wave steps run two tiles per SM without the staged
// variant's per-layer weight copies.
template <typename Real, int MODE, bool RESIDENT, int SC, int NG = 1>
__global__ void __launch_bounds__(NG == 2 ? 768 : ((RESIDENT || sizeof(Real) == 8) ? 512 : 384),
                                  (NG == 2 || RESIDENT || sizeof(Real) == 8) ? 1 : 2)
    k_tile(StateDev<Real> st, PlanDev pl, NetLayout lay_p, int s, ForecastArgs fa) {
    using M = Math<Real>;
    constexpr int R = kR, LD = ldr<Real>();
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ double red_all[NG][32];
    __shared__ __align__(8) uint64_t wbar;
    __shared__ NetLayout lay_s;  // read with dynamic layer indices in every phase
    if (threadIdx.x == 0) {
        lay_s = lay_p;
        if (NG > 1 && RESIDENT) mbar_init(&wbar, 1);  // before any group can wait on it
    }
    __syncthreads();
    const NetLayout& lay = lay_s;
    const int NT = static_cast<int>(blockDim.x) / NG, grp = static_cast<int>(threadIdx.x) / NT;
    const int tid = static_cast<int>(threadIdx.x) - grp * NT, lane = tid & 31, warp = tid >> 5, NW = NT >> 5;
    double* red = red_all[grp];
    // the group's barrier (named barrier 1 + grp over its NT threads); the whole CTA for NG = 1
    auto gsync = [&]() {
        if constexpr (NG == 1) {
            __syncthreads();
        } else {
            asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(NT) : "memory");
        }
    };
    const TileSmem ts = TileSmem::make<Real>(lay, RESIDENT);
    const int H = lay.H, O = lay.O, I = lay.I, in0 = lay.in0, L = lay.L, G = 3 * H;
    const int ldo = lay.ldo, ldkh = lay.ldkh;
    const int tile = static_cast<int>(blockIdx.x) * NG + grp;
    const Real* __restrict__ th = st.theta;
    Real* smw = reinterpret_cast<Real*>(smem_raw);
    Real* sm = smw + grp * (ts.total - ts.wsize);  // this group's tile region (offsets past the weights)

    Real* wsm = smw + ts.w;
    Real* XT = sm + ts.xt;
    Real* HT = sm + ts.ht;
    Real* GT = sm + ts.gt;
    Real* ZT = sm + ts.zt;
    Real* PT = sm + ts.pt;
    Real* PBT = sm + ts.pbt;
    Real* ZBT = sm + ts.zbt;
    Real* RES = sm + ts.rest;
    Real* UBT = sm + ts.ubt;
    Real* s_in = sm + ts.sin;
    Real* s_out = sm + ts.sout;
    Real* lvl = sm + ts.lvl;
    Real* tgt = sm + ts.tgt;
    Real* msk = sm + ts.msk;

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
    if (MODE == kTrain) DBG_SPAN_MIN(st, s, 0);
    if (MODE == kTrain) DBG_TILE(st, s, tile, 0);
    DBG_CLK(st, 0);
    // row store of this tile's windows (K3 operands): [b][rs_ld], b = step-local window
    Real* __restrict__ rs = (MODE == kTrain) ? st.rowstore + (size_t)(tile * R) * lay.rs_ld : nullptr;
    // the tile's windows' plan entries (epoch constants), one load per thread, all in flight:
    // series row, anchor, publishing slot (-1 unless the window is its slot's first), CSR
    // position, category
    __shared__ int w_info_all[NG][5][kR];
    auto& w_info = w_info_all[grp];
    if (MODE != kForecast) {
        if (tid < 4 * R) {
            const int q = tid / R, r = tid - q * R;
            int v = 0;
            if (r < nrows) {
                const int wb = w0 + tile * R + r;
                if (q == 0) v = pl.w_row[wb];
                else if (q == 1) v = pl.w_anchor[wb];
                else if (q == 2) v = (MODE == kTrain && pl.w_first[wb] != 0) ? pl.w_slot[wb] : -1;
                else v = MODE == kTrain ? pl.w_csr[wb] : 0;
            }
            w_info[q][r] = v;
        }
        gsync();
        if (tid < nrows) w_info[4][tid] = st.cat[w_info[0][tid]];
    }
    const int* w_rowv = w_info[0];
    const int* w_ancv = w_info[1];
    // the step's global mask count (epoch constant): loaded now, used by the pinball adjoint
    const double step_m = MODE == kForecast ? 1.0 : pl.step_M[s];

    // ---- weights: TMA bulk copy of the compact parameter vector (resident mode), issued
    // once the previous step's Adam has completed (after pdl_wait) ----
    auto weights_tma = [&]() {
        if (!(RESIDENT && tid == 0 && grp == 0)) return;
        if (NG == 1) mbar_init(&wbar, 1);
        const unsigned total = static_cast<unsigned>(lay.P_pad * sizeof(Real));
        mbar_expect_tx(&wbar, total);
        constexpr unsigned kChunk = 32768;
        for (unsigned off = 0; off < total; off += kChunk) {
            const unsigned n = total - off < kChunk ? total - off : kChunk;
            bulk_g2s(reinterpret_cast<unsigned char*>(wsm) + off, reinterpret_cast<const unsigned char*>(th) + off, n,
                     &wbar);
        }
    };

    // ---- prologue: Holt-Winters scan of each window's series (K1 fused here) ---------
    Real* LVR = sm + ts.lvr;
    Real* SER = sm + ts.ser;
    Real* YS = sm + ts.ys;
    if (MODE != kForecast) {
        Real* PSM = sm + ts.psm;
        const int T = lay.T, S = lay.S, np = 2 + S;
        constexpr int e16 = 16 / static_cast<int>(sizeof(Real));
        const int nch = (T + e16 - 1) / e16;
        // observation rows (constant for the epoch: staged before the dependency wait, so
        // the copies overlap the previous kernel's tail under programmatic dependent
        // launch), then the per-series parameters the previous step's Adam wrote
        for (int e = tid; e < nrows * nch; e += NT) {
            const int r = e / nch, c = e - r * nch;
            cp_async16(YS + r * ts.tp + c * e16, st.vrm + (size_t)w_rowv[r] * st.ldv + c * e16);
        }
        pdl_wait();
        // dependents (K3) may launch once every tile has passed its wait: the previous
        // step's K4 has then completed, so K3's pre-wait prologue may read the per-series
        // parameters it wrote (K3 still waits for this grid's completion before the rest).
        // kTrain triggers after the forward pass instead (below), so K3's pre-wait work
        // shares the SMs with the backward half only
        if (MODE != kTrain || st.tile_trigger_early) pdl_trigger();
        if (MODE == kTrain) {
            DBG_SPAN_MIN(st, s, 1);
            DBG_SPAN_MIN(st, s - 1, 9);
            SPAN_BEGIN(st, s, kSpanTile);
            DBG_TILE(st, s, tile, 1);
        }
        weights_tma();
        for (int e = tid; e < nrows * np; e += NT) {
            const int r = e / np, c = e - r * np;
            cp_async_elem(PSM + r * np + c, st.ps + (size_t)c * st.N + w_rowv[r]);
        }
        cp_async_wait_all();
        gsync();
        DBG_CLK(st, 0);
        // the tile holding a slot's first window (batch order) publishes the slot's states
        const int* pub_slot = w_info[2];
        if (tid < nrows) {
            const int bad = hw_scan_row<Real, SC>(YS + tid * ts.tp, PSM + tid * np, T, S, LVR + tid * ts.ldl,
                                                  SER + tid * ts.lds);
            if (bad != INT_MAX) flag_error(st.err, kErrTrainLevel, bad);
        }
        DBG_CLK(st, 0);
        gsync();
        // published states for K3's fp64 reverse scan: lv [T][kcap], se [T+S][kcap] (fp32:
        // K3's ES blocks rerun this scan themselves before their dependency wait,
        // finish.cuh es_block_fp32)
        if (MODE == kTrain && sizeof(Real) == 8) {
            for (int r = warp; r < nrows; r += NW) {  // a warp per window row, lanes over t
                const int slot = pub_slot[r];
                if (slot < 0) continue;
                for (int t = lane; t < T; t += 32) st.lv[(size_t)t * st.kcap + slot] = LVR[r * ts.ldl + t];
                for (int t = lane; t < T + S; t += 32) st.se[(size_t)t * st.kcap + slot] = SER[r * ts.lds + t];
            }
        }
    }
    DBG_CLK(st, 0);
    // ---- window gather + normalisation (trainer.hpp:532-566) --------------------------
    if (MODE == kForecast) {
        pdl_wait();
        pdl_trigger();
        weights_tma();
        const Real* X = reinterpret_cast<const Real*>(fa.X);
        const Real* FL = reinterpret_cast<const Real*>(fa.lvl);
        const Real* FS = reinterpret_cast<const Real*>(fa.sout);
        for (int e = tid; e < in0 * R; e += NT) {
            const int c = e >> 3, r = e & 7;
            XT[c * LD + r] = r < nrows ? X[(size_t)(tile * R + r) * in0 + c] : Real(0);
        }
        for (int e = tid; e < O * R; e += NT) {
            const int o = e >> 3, r = e & 7;
            s_out[r * ldo + o] = r < nrows ? FS[(size_t)(tile * R + r) * O + o] : Real(0);
        }
        for (int r = tid; r < R; r += NT) lvl[r] = r < nrows ? FL[tile * R + r] : Real(0);
    } else {
        // column c < I: input window; c < I+O: target window; c == I+O: level; the rest: one-hot
        const int ncol = I + O + 1 + (in0 - I);
        for (int e = tid; e < ncol * R; e += NT) {
            const int c = e >> 3, r = e & 7;
            const int wb = w0 + tile * R + r;
            if (r >= nrows) {
                if (c < I) {
                    XT[c * LD + r] = 0;
                    s_in[r * I + c] = 1;
                } else if (c < I + O) {
                    tgt[r * ldo + c - I] = 0;
                    s_out[r * ldo + c - I] = 1;
                    msk[r * ldo + c - I] = 0;
                } else if (c == I + O) {
                    lvl[r] = 1;
                } else {
                    XT[(c - O - 1) * LD + r] = 0;
                }
                continue;
            }
            if (c > I + O) {
                const int cc = c - O - 1;  // x column in [I, in0)
                const Real v = (w_info[4][r] == cc - I) ? Real(1) : Real(0);
                XT[cc * LD + r] = v;
                if (rs) rs[r * lay.rs_ld + lay.rs_x + cc] = v;
                continue;
            }
            const int a = w_ancv[r];
            const Real l = LVR[r * ts.ldl + a];
            if (c < I) {
                const int idx = a - I + 1 + c;
                const Real sv = SER[r * ts.lds + idx];
                const Real v = fdiv(YS[r * ts.tp + idx], sv * l);
                XT[c * LD + r] = v;
                if (rs) rs[r * lay.rs_ld + lay.rs_x + c] = v;
                s_in[r * I + c] = sv;
            } else if (c < I + O) {
                const int j = c - I, idx = a + 1 + j;
                const Real sv = SER[r * ts.lds + idx];
                tgt[r * ldo + j] = fdiv(YS[r * ts.tp + idx], sv * l);
                s_out[r * ldo + j] = sv;
                msk[r * ldo + j] = (pl.mask == nullptr || pl.mask[(size_t)wb * O + j] != 0) ? Real(1) : Real(0);
            } else {
                lvl[r] = l;
            }
        }
    }
    gsync();
    DBG_CLK(st, 1);
    if (MODE != kForecast && st.d_inputs != nullptr) {
        const int base = tile * R;
        for (int e = tid; e < nrows * in0; e += NT) {
            const int r = e / in0, c = e - r * in0;
            st.d_inputs[(size_t)(base + r) * in0 + c] = XT[c * LD + r];
        }
        for (int e = tid; e < nrows * O; e += NT) {
            const int r = e / O, o = e - r * O;
            st.d_targets[(size_t)(base + r) * O + o] = tgt[r * ldo + o];
            st.d_seas[(size_t)(base + r) * O + o] = s_out[r * ldo + o];
        }
        for (int r = tid; r < nrows; r += NT) st.d_levels[base + r] = lvl[r];
    }
    if (RESIDENT) mbar_wait(&wbar, 0);

    // ---- forward through the stack (network.hpp:148-210, sequence length 1) --------
    const int rf = lane >> 2;  // the row a forward lane owns after the reduce-scatter
    for (int l = 0; l < L; ++l) {
        const Real* U = l == 0 ? XT : HT + (l - 1) * H * LD;
        if (!RESIDENT) {
            stage_segment(wsm, th + lay.cw[l], lay.cb[l] - lay.cw[l] + G);
            gsync();
        }
        const Real* WT = RESIDENT ? wsm + lay.cw[l] : wsm;
        const Real* bias = RESIDENT ? wsm + lay.cb[l] : wsm + (lay.cb[l] - lay.cw[l]);
        const int ldk = lay.ldk[l], K = lay.layer_in[l];
        const Real* radd = lay.block_last[l] ? HT + lay.res_src[l] * H * LD : nullptr;
        Real* out = HT + l * H * LD;
        Real* gl = GT + 4 * l * H * R;
        for (int h0 = warp * 4; h0 < H; h0 += NW * 4) {  // warp-uniform
            const int hh = h0 + (lane & 3);
            const int hc = hh < H ? hh : H - 1;
            const Real* wr[3] = {WT + hc * ldk, WT + (H + hc) * ldk, WT + (2 * H + hc) * ldk};
            Real pre[3];
            fwd_prod<Real, 3>(pre, U, wr, K);
            if (hh < H) {
                const Real i = M::logistic(pre[0] + bias[hc]);
                const Real g = M::tanh(pre[1] + bias[H + hc]);
                const Real o = M::logistic(pre[2] + bias[2 * H + hc]);
                const Real c = i * g;
                const Real tc = M::tanh(c);
                Real h = o * tc;
                if (radd) h = h + radd[hh * LD + rf];
                out[hh * LD + rf] = h;
                const int e = hh * R + rf;
                gl[e] = i;
                gl[H * R + e] = g;
                gl[2 * H * R + e] = o;
                gl[3 * H * R + e] = tc;
                if (rs && rf < nrows) rs[rf * lay.rs_ld + lay.rs_h[l] + hh] = h;
            }
        }
        gsync();
        DBG_CLK(st, 2);
    }
    if (MODE == kTrain && !st.tile_trigger_early) pdl_trigger();
    // head (network.hpp:207-209): z = tanh(h nl_w + nl_b); pred = z out_w + out_b
    const Real* cur = HT + (L - 1) * H * LD;
    if (!RESIDENT) {
        stage_segment(wsm, th + lay.c_nlw, lay.P_pad - lay.c_nlw);
        gsync();
    }
    const long long hb0 = RESIDENT ? 0 : lay.c_nlw;
    const Real* nlwT = wsm + (lay.c_nlw - hb0);
    const Real* nlb = wsm + (lay.c_nlb - hb0);
    const Real* owT = wsm + (lay.c_outw - hb0);
    const Real* obias = wsm + (lay.c_outb - hb0);
    for (int h0 = warp * 4; h0 < H; h0 += NW * 4) {
        const int hh = h0 + (lane & 3);
        const int hc = hh < H ? hh : H - 1;
        const Real* wr[1] = {nlwT + hc * ldkh};
        Real v[1];
        fwd_prod<Real, 1>(v, cur, wr, H);
        if (hh < H) {
            const Real z = M::tanh(v[0] + nlb[hc]);
            ZT[hh * LD + rf] = z;
            if (rs && rf < nrows) rs[rf * lay.rs_ld + lay.rs_z + hh] = z;
        }
    }
    gsync();
    // adapter output, fused with the masked pinball (autodiff.hpp:384-392) and its adjoint
    // (:620-626): the lane owning (output oo, row rf) forms its loss term and pred_bar
    double lsum = 0.0;
    const Real gscale = static_cast<Real>(1.0 / step_m);
    const Real tau = static_cast<Real>(st.tau);
    for (int o0 = warp * 4; o0 < O; o0 += NW * 4) {
        const int oo = o0 + (lane & 3);
        const int oc = oo < O ? oo : O - 1;
        const Real* wr[1] = {owT + oc * ldkh};
        Real v[1];
        fwd_prod<Real, 1>(v, ZT, wr, H);
        if (oo < O) {
            const Real p = v[0] + obias[oc];
            PT[oo * LD + rf] = p;
            if (MODE != kForecast) {
                Real pb = 0;
                if (msk[rf * ldo + oo] != Real(0)) {
                    const Real t = tgt[rf * ldo + oo];
                    const Real d = t - p;
                    lsum += (d >= Real(0)) ? st.tau * static_cast<double>(d) : (st.tau - 1.0) * static_cast<double>(d);
                    pb = gscale * ((t >= p) ? -tau : Real(1) - tau);
                }
                PBT[oo * LD + rf] = pb;
                if (rs && rf < nrows) rs[rf * lay.rs_ld + lay.rs_pb + oo] = pb;
            }
        }
    }
    if (MODE != kForecast) {
        // fixed-order block sum (warp shuffles, then warps in order); the barrier below also
        // publishes PT and PBT
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) lsum += __shfl_down_sync(0xffffffffu, lsum, o);
        if (lane == 0) red[warp] = lsum;
    }
    gsync();
    DBG_CLK(st, 3);
    if (MODE == kForecast) {
        for (int e = tid; e < nrows * O; e += NT) {
            const int r = e / O, o = e - r * O;
            fa.out[(size_t)(tile * R + r) * O + o] = static_cast<double>(PT[o * LD + r] * lvl[r] * s_out[r * ldo + o]);
        }
        if (fa.validate) {
            gsync();
            // sMAPE (metrics.hpp:17-28) and MASE (:33-49) against the held-out block
            // y[t_ins : t_ins+O) (validate: the validation block; evaluate: the test block)
            for (int r = tid; r < nrows; r += NT) {
                const int row = tile * R + r;
                double acc = 0.0, mae = 0.0;
                for (int o = 0; o < O; ++o) {
                    const double a = static_cast<double>(st.vals[(size_t)(fa.t_ins + o) * st.N + row]);
                    const double f = fa.out[(size_t)row * O + o];
                    const double den = fabs(a) + fabs(f);
                    if (den > 0.0) acc += fabs(a - f) / den;
                    mae += fabs(a - f);
                }
                fa.smape[row] = 200.0 * acc / static_cast<double>(O);
                if (fa.mase) {
                    const double d = fa.score[row];
                    fa.mase[row] = d == 0.0 ? NAN : (mae / static_cast<double>(O)) / d;
                }
            }
        }
        return;
    }
    // the tile's loss partial (fixed warp order): kLossOnly now; kTrain at the end, by the last
    // warp (idle in the final per-window phase), off warp 0's backward critical path
    auto loss_partial = [&]() {
        double ltot = 0.0;
        for (int w = 0; w < NW; ++w) ltot += red[w];
        st.loss_part[tile] = ltot;
    };
    if (MODE == kLossOnly) {
        if (tid == 0) loss_partial();
        return;
    }
    DBG_CLK(st, 4);

    // ---- backward: input adjoints, each fused with the epilogue of the layer below ----
    // backward lanes: feature k0 + (lane & 3) of the warp's 4, row rf = lane >> 2
    // z_bar = pbar . out_w^T, then through tanh
    for (int k0 = warp * 4; k0 < H; k0 += NW * 4) {
        const int k = k0 + (lane & 3);
        const int kc = k < H ? k : H - 1;
        const Real v = bwd_prod<Real>(PBT, owT + kc, ldkh, O);
        if (k < H) {
            const int r = rf;
            const Real zz = ZT[k * LD + r];
            const Real zb = v * (Real(1) - zz * zz);
            ZBT[k * LD + r] = zb;
            if (rs && r < nrows) rs[r * lay.rs_ld + lay.rs_zb + k] = zb;
        }
    }
    gsync();
    DBG_CLK(st, 5);
    // h_bar of layer l comes from the product of the layer above (or the head); the lane that
    // owns (row, unit) forms the gate adjoints of layer l right away
    const Real* AT = ZBT;
    const Real* WA = nlwT;
    int lda = ldkh, QA = H;
    for (int l = L - 1; l >= -1; --l) {
        // product: input adjoint of the consumer of layer l's output (head for l = L-1)
        const int Kout = l >= 0 ? H : in0;
        const bool add_res = l >= 0 && (l + 1 < L) && lay.block_first[l + 1];
        const bool save_res = l >= 0 && lay.block_last[l] != 0;
        Real* PR = sm + ((l & 1) ? ts.prt1 : ts.prt0);
        const Real* gl = GT + 4 * (l >= 0 ? l : 0) * H * R;
        for (int k0 = warp * 4; k0 < Kout; k0 += NW * 4) {
            const int k = k0 + (lane & 3);
            const int kc = k < Kout ? k : Kout - 1;
            const Real v = bwd_prod<Real>(AT, WA + kc, lda, QA);
            if (k < Kout) {
                const int r = rf;
                if (l < 0) {
                    UBT[k * LD + r] = v;  // x_bar: the ES contributions read it
                } else {
                    Real hb = v;
                    if (add_res) hb = hb + RES[k * LD + r];
                    if (save_res) RES[k * LD + r] = hb;
                    const int e = k * R + r;
                    Real pi, pg, po;
                    cell_adjoint(hb, gl[e], gl[H * R + e], gl[2 * H * R + e], gl[3 * H * R + e], pi, pg, po);
                    PR[k * LD + r] = pi;
                    PR[(H + k) * LD + r] = pg;
                    PR[(2 * H + k) * LD + r] = po;
                    if (rs && r < nrows) {
                        Real* d = rs + r * lay.rs_ld + lay.rs_pr[l];
                        d[k] = pi;
                        d[H + k] = pg;
                        d[2 * H + k] = po;
                    }
                }
            }
        }
        if (l < 0) break;
        // next product: layer l's input adjoint through W^T_l
        if (!RESIDENT) {
            gsync();
            stage_segment(wsm, th + lay.cw[l], lay.cb[l] - lay.cw[l]);
        }
        gsync();
        DBG_CLK(st, 6);
        AT = PR;
        WA = RESIDENT ? wsm + lay.cw[l] : wsm;
        lda = lay.ldk[l];
        QA = G;
    }
    gsync();
    DBG_CLK(st, 7);

    // ---- ES adjoint contributions per window (Div / Mul / BroadcastCol adjoints) ----
    // written in slot-major CSR order so each slot's windows are contiguous for K3;
    // row = [inputs (s index a-I+1..a) | targets (a+1..a+O) | level a | anchor a].
    // Stored as LOG adjoints: a normalised entry z = y / (s l) (input x or target t) with
    // adjoint zb gives e = -zb * z, so dL/ds = e / s and dL/dl = (sum of e) / l.  A window's
    // seasonality and level adjoints
    // cancel almost exactly downstream (x is invariant under s -> c s, l -> l / c), so K3
    // divides the per-slot sums by its own double forward states once, instead of this
    // kernel dividing each term by its fp32 states (whose rounding the cancellation would
    // amplify ~1e4x for S = 1).  Formed in double in both precisions.
    if (st.attach) {
        // one warp per window, lanes over its I + O normalised entries; fixed-order warp sum
        const int nio = I + O;
        for (int r = warp; r < nrows; r += NW) {
            double* __restrict__ cr = st.contrib + (size_t)w_info[3][r] * st.cwp;
            double acc = 0;
            for (int j = lane; j < nio; j += 32) {
                double v;
                if (j < I) {
                    v = static_cast<double>(UBT[j * LD + r]) * static_cast<double>(XT[j * LD + r]);
                } else {
                    const int o = j - I;
                    v = -(static_cast<double>(PBT[o * LD + r]) * static_cast<double>(tgt[r * ldo + o]));
                }
                cr[j] = -v;
                acc -= v;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) {
                cr[nio] = acc;
                cr[nio + 1] = static_cast<double>(w_ancv[r]);
            }
        }
    }
    if (MODE == kTrain && warp == NW - 1 && lane == 0) loss_partial();
    if (MODE == kTrain) DBG_GT(st, 3);
    if (MODE == kTrain) DBG_SPAN_MAX(st, s, 2);
    if (MODE == kTrain) SPAN_END(st, s, kSpanTile);
    if (MODE == kTrain) DBG_TILE(st, s, tile, 2);
}

}  // namespace esrnn_dev
