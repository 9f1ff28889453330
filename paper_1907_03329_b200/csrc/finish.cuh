// K3 k_grad_finish: per-slot ES backward + the weight-gradient contraction over the step's
//                   windows (row store written by K2), last CTA finalises the step scalars
//                   (single GPU).
// K3' k_finalize:   post-all-reduce finalisation (sharded mode).
// K4 k_adam:        Adam over the compact shared vector and the step's per-series slots.
//
// Reference: Gather adjoint (autodiff.hpp:603-610), the HW recursion adjoint through the
// tape (holt_winters.hpp:266-277, Logistic :483, Exp :501), apply_updates
// (trainer.hpp:602-655).
#pragma once
#include "common.cuh"
#include "tile.cuh"
#include "umma.cuh"

namespace esrnn_dev {

constexpr int kFinishThreads = 256;
constexpr int kEsSlotsPerBlock = 32;  // fp64 ES blocks: warp 0 owns 32 slots; all warps stage the windows
constexpr int kEsSlots32 = 16;        // fp32 ES blocks (es_block_fp32): at most 16 slots; the launch picks
                                      // 8 or 16 (engine.cu es_slots_fp32)
constexpr int kEsChunk = 64;          // contribution rows staged per round (64: K3 fits four blocks per SM at Monthly)
constexpr int kGq = 16, kGk = 8;      // K3 GEMM output block (gate rows x input features)
constexpr int kGChunk = 256;          // row-store rows staged per round
constexpr int kWq = 32, kWr = 64;      // q-strip GEMM: G rows per block, row-store rows per chunk
constexpr int kWkMax = 64;             // q-strip GEMM: K (+ padding) at most (else the 16 x 8 tiles)
constexpr int kGBuf = 3;              // staging ring depth, maximum (ring - 1 chunks in flight; the
                                      // launch picks 3 or 2, engine.cu finish_ring)
// fp32 mode with S = 1: K3's ES blocks recompute the forward states in double (see there)
template <typename Real, int SC>
constexpr bool kEsRecompute = sizeof(Real) == 4 && SC == 1;

// clip scale (trainer.hpp:603-615), global Adam step and bias corrections (:617-620),
// step loss (masked mean, autodiff.hpp:392).  err_any: some rank's error word is set (the
// reference throws before apply_updates): Adam's step does not advance anywhere.
template <typename Real>
__device__ void finalize_scalars(StateDev<Real>& st, const PlanDev& pl, int s, double sq, double loss_sum,
                                 bool advance, bool err_any) {
    double scale = 1.0;
    if (st.has_clip) {
        const double norm = sqrt(sq);
        if (norm > st.clip) scale = st.clip / norm;
    }
    st.scal[0] = scale;
    st.scal[3] = loss_sum / pl.step_M[s];
    st.loss_hist[s] = loss_sum / pl.step_M[s];
    if (err_any) st.err[2] = 1;
    if (advance && !err_any) {  // only a step that applies updates advances Adam's t
        const long long step = ++(*st.net_step);
        st.scal[1] = bias_c1(st, step);
        st.scal[2] = bias_c2(st, step);
    }
}

// ---------------------------------------------------------------------------------------
// K3 weight-gradient block on the tensor cores (fp32 mode, large steps; umma.cuh): block
// gbp = (tile, part).  Tiles enumerate the matrices' 128-row slices (layer W_in^T [3H][in],
// nl_w^T, out_w^T); part p contracts the step's rows [p*span, (p+1)*span) into a 128 x 64
// partial (columns: the K inputs, then the bias column) in st.upart.  The last part to finish
// a tile (ticket) sums the parts in part order -- fixed order, no float atomics -- and writes
// the tile's gradients and bias gradients into gbuf and its squared norm into red_sq_part.
__device__ __forceinline__ void dw_umma_block(StateDev<float>& st, const PlanDev& pl, const NetLayout& lay, int s,
                                              int gbp, int parts, unsigned char* smem_raw, double* red) {
    const int tile = gbp / parts, part = gbp - tile * parts;
    int m = 0, t0 = 0;
    for (; m < lay.nmat; ++m) {
        const int nt = (lay.mats[m].Q + kUM - 1) / kUM;
        if (tile < t0 + nt) break;
        t0 += nt;
    }
    const MatDesc md = lay.mats[m];
    const int mt = tile - t0;
    const int Mv = min(kUM, md.Q - mt * kUM), Kv = md.K;
    const int wb0 = pl.step_win_off[s];
    const int Bstep = pl.step_win_off[s + 1] - wb0;
    const int span = ((Bstep + parts - 1) / parts + kUK - 1) / kUK * kUK;
    const int r0 = min(Bstep, part * span), nrows = min(Bstep, r0 + span) - r0;
    float* mine = st.upart + (size_t)(tile * parts + part) * kUM * kUN;
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    umma_partial_dw(sm, st.rowstore + md.a_off + mt * kUM, st.rowstore + md.u_off, lay.rs_ld, r0, nrows, Kv, mine);
    __shared__ bool last_part;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last_part = atomicAdd(st.gtile_ctr + tile, 1u) == static_cast<unsigned>(parts - 1);
    __syncthreads();
    if (!last_part) return;
    __threadfence();
    if (threadIdx.x == 0) st.gtile_ctr[tile] = 0;
    double sq = 0.0;
    for (int e = threadIdx.x; e < Mv * (Kv + 1); e += blockDim.x) {
        const int q = e / (Kv + 1), k = e - q * (Kv + 1);
        float g = 0.f;
        for (int p = 0; p < parts; ++p) g += __ldcg(st.upart + (size_t)(tile * parts + p) * kUM * kUN + q * kUN + k);
        const int qq = mt * kUM + q;
        if (k < Kv) st.gbuf[md.cw + (long long)qq * md.ldk + k] = g;
        else st.gbuf[md.cb + qq] = g;
        sq += static_cast<double>(g) * g;
    }
    const double tot = block_sum(sq, red);
    if (threadIdx.x == 0) {
        st.red_sq_part[tile] = tot;
        if (tile == 0)  // the FFMA path's tile count is what the finalisers sum over
            for (int i = st.umma_tiles; i < st.red_tiles; ++i) st.red_sq_part[i] = 0.0;
    }
}

// ---------------------------------------------------------------------------------------
// K3 ES block, fp32 mode: per-slot window-adjoint gather + reverse Holt-Winters adjoint for
// kEsSlots32 slots.  Everything that does not depend on K2's output runs BEFORE the
// dependency wait, overlapping K2 (whose tiles release this grid once they pass their own
// wait): the observation rows, the forward scan of the slots (the tile's own hw_scan_row,
// so the states equal K2's bit for bit; double for S = 1, see kEsRecompute), the optional
// level-variability penalty, and the recursion's per-step coefficients.  After the wait:
// the window log adjoints (thread per (slot, index), CSR order), their scaling by the
// reciprocal states, the serial reverse recursion (one thread per slot: loads + 6 DFMA per
// step, one DFMA on the dependency chain) and the per-series gradient outputs.
// Returns the thread's squared-gradient and penalty partials.
template <typename Real, int SC>
__device__ __forceinline__ void es_block_fp32(StateDev<Real>& st, const PlanDev& pl, const NetLayout& lay, int s,
                                              unsigned char* smem_raw, double& sq, double& pen, int bid, int bd) {
    const int tid = threadIdx.x;
    auto clk = [&](int i) {
        if (st.dbg_clk && bid == 0 && tid == 0) st.dbg_clk[32 + i] = clock64();
    };
    const int k0 = pl.step_slot_off[s];
    const int k = pl.step_slot_off[s + 1] - k0;
    const int sl0 = bid * bd, sl1 = min(k, sl0 + bd);
    if (!(sl0 < sl1 && st.attach)) {  // uniform per block
        pdl_wait();
        SPAN_BEGIN(st, s, kSpanFinish);
        return;
    }
    using CR = std::conditional_t<kEsRecompute<Real, SC>, double, float>;
    using MD = Math<double>;
    const int N = st.N, S = SC > 0 ? SC : lay.S, T = lay.T, I = lay.I, O = lay.O;
    const int tp = row_pad<Real>(T), cwp = st.cwp, nsl = sl1 - sl0, np = 2 + S;
    const int ldl = T | 1, lds = (T + S) | 1;
    double* LB = reinterpret_cast<double*>(smem_raw);  // [bd][ldl] level (log) adjoints
    double* SB = LB + bd * ldl;                        // [bd][lds] seasonality (log) adjoints
    CR* K1 = reinterpret_cast<CR*>(SB + bd * lds);     // 6 x [T][bd] recursion coefficients
    CR* K2 = K1 + T * bd;
    CR* CA = K2 + T * bd;
    CR* CG = CA + T * bd;
    CR* RS = CG + T * bd;
    CR* RI = RS + T * bd;
    double* E0 = reinterpret_cast<double*>(RI + T * bd);  // [bd][S] exp(init seasonality raw)
    unsigned char* X = reinterpret_cast<unsigned char*>(E0 + bd * S);  // scratch (engine.cu finish_smem)
    Real* YS = reinterpret_cast<Real*>(X);           // pre-wait: [bd][tp] observation rows
    CR* LVr = reinterpret_cast<CR*>(YS + bd * tp);   //           [bd][ldl] forward levels
    CR* SEr = LVr + bd * ldl;                        //           [bd][lds] forward seasonalities
    Real* PRM = reinterpret_cast<Real*>(SEr + bd * lds);  //      [bd][2+S] raw parameters
    double* cbuf = reinterpret_cast<double*>(X);     // post-wait: [kEsChunk][cwp] contribution rows
    __shared__ int woff[kEsSlots32 + 1];
    __shared__ double coef[3][kEsSlots32];  // alpha, gamma, l[-1] (double)
    const int slot = sl0 + tid;
    const bool mine = tid < nsl;
    clk(1);
    // ---- pre-wait: plan entries, observation rows, zeroed adjoints ----
    constexpr int e16 = 16 / static_cast<int>(sizeof(Real));
    const int nch = tp / e16;
    for (int e = tid; e < nsl * nch; e += kFinishThreads) {
        const int sl = e / nch, ch = e - sl * nch;
        const int row = pl.slot_row[k0 + sl0 + sl];
        cp_async16(YS + sl * tp + ch * e16, st.vrm + (size_t)row * st.ldv + ch * e16);
    }
    if (tid <= nsl) woff[tid] = pl.slot_win_off[k0 + sl0 + tid];
    for (int e = tid; e < bd * (ldl + lds); e += kFinishThreads) LB[e] = 0.0;  // LB and SB are contiguous
    const int lrow = mine ? pl.slot_row[k0 + slot] : 0;
    // per-series parameters: the previous step's K4 output, complete before K2 passed its
    // wait and released this grid; read at L2
    Real* pr = PRM + tid * np;
    if (mine)
        for (int j = 0; j < np; ++j) pr[j] = __ldcg(st.ps + (size_t)j * N + lrow);
    cp_async_wait_all();
    __syncthreads();
    clk(2);
    // ---- pre-wait: forward states of the block's slots ----
    if (mine) {
        const Real* ys = YS + tid * tp;
        double l0;
        if constexpr (kEsRecompute<Real, SC>) {
            // S = 1: double states (the reference's arithmetic)
            const double al = MD::logistic(static_cast<double>(pr[0])), ga = MD::logistic(static_cast<double>(pr[1]));
            CR* lv = LVr + tid * ldl;
            CR* se = SEr + tid * lds;
            for (int j = 0; j < S; ++j) se[j] = MD::exp(static_cast<double>(pr[2 + j]));
            l0 = 0.0;
            for (int j = 0; j < S; ++j) l0 += static_cast<double>(ys[j]);
            l0 /= S;
            double lp = l0;
            for (int t = 0; t < T; ++t) {
                const double yt = static_cast<double>(ys[t]), s_t = se[t];
                const double l = al * (yt / s_t) + (1.0 - al) * lp;
                se[t + S] = ga * (yt / lp) + (1.0 - ga) * s_t;
                lv[t] = l;
                lp = l;
            }
        } else {
            // the tile's own scan: states identical to the ones K2 normalised the windows with
            hw_scan_row<Real, SC, false>(ys, pr, T, S, LVr + tid * ldl, SEr + tid * lds);  // K2 flags bad levels
            Real l0r = 0;
            for (int j = 0; j < S; ++j) l0r += ys[j];
            l0 = static_cast<double>(l0r / Real(S));
        }
        for (int j = 0; j < S; ++j) E0[tid * S + j] = MD::exp(static_cast<double>(pr[2 + j]));
        coef[0][tid] = MD::logistic(static_cast<double>(pr[0]));
        coef[1][tid] = MD::logistic(static_cast<double>(pr[1]));
        coef[2][tid] = l0;
        if (st.lvp > 0.0 && T >= 3) {
            // opt-in level-variability penalty (oracle/esrnn_oracle.c lvp_series): with
            // u_t = log l_t and e_t = u_t - 2 u_{t-1} + u_{t-2}, this slot adds c * mean_t e_t^2,
            // c = lambda * O * (its windows) / M; its adjoint enters the LOG level adjoints
            const CR* lv = LVr + tid * ldl;
            double* lb = LB + tid * ldl;
            const int nw = pl.slot_win_off[k0 + slot + 1] - pl.slot_win_off[k0 + slot];
            const double cs = st.lvp * O * nw, c = cs / pl.step_M[s], inv = 1.0 / (T - 2);
            double um2 = ::log(static_cast<double>(lv[0])), um1 = ::log(static_cast<double>(lv[1])), acc = 0.0;
            for (int t = 2; t < T; ++t) {
                const double u = ::log(static_cast<double>(lv[t]));
                const double e = u - 2.0 * um1 + um2;
                acc += e * e;
                const double q = c * 2.0 * inv * e;
                lb[t] += q;
                lb[t - 1] -= 2.0 * q;
                lb[t - 2] += q;
                um2 = um1;
                um1 = u;
            }
            pen = cs * acc * inv;  // x M: the loss-sum units of loss_part
        }
    }
    __syncthreads();
    clk(3);
    // ---- pre-wait: the recursion's coefficients, [t][bd] (l' = l[t-1], l[-1] = mean y[0:S])
    //   K1 = alpha y / s^2, K2 = gamma y / l'^2, CA = y / s - l', CG = y / l' - s, RS = 1/s, RI = 1/l
    // double for S = 1, else the correctly rounded fp32 reciprocals of the fp32 states
    const int bsh = bd == 16 ? 4 : 3;  // bd is 8 or 16
    for (int e = tid; e < T * bd; e += kFinishThreads) {
        const int t = e >> bsh, sl = e - (t << bsh);
        if (sl >= nsl) continue;
        const double y = static_cast<double>(YS[sl * tp + t]);
        const CR lvc = LVr[sl * ldl + t], svc = SEr[sl * lds + t];
        const CR lpc = t > 0 ? LVr[sl * ldl + t - 1] : static_cast<CR>(coef[2][sl]);
        double rs, rl, ri;
        if constexpr (kEsRecompute<Real, SC>) {
            rs = 1.0 / svc, rl = 1.0 / lpc, ri = 1.0 / lvc;
        } else {
            rs = __frcp_rn(svc), rl = __frcp_rn(lpc), ri = __frcp_rn(lvc);
        }
        const double lpv = t > 0 ? static_cast<double>(lpc) : coef[2][sl];
        const double yrs = y * rs, yrl = y * rl;
        K1[e] = static_cast<CR>(coef[0][sl] * yrs * rs);
        K2[e] = static_cast<CR>(coef[1][sl] * yrl * rl);
        CA[e] = static_cast<CR>(yrs - lpv);
        CG[e] = static_cast<CR>(yrl - static_cast<double>(svc));
        RS[e] = static_cast<CR>(rs);
        RI[e] = static_cast<CR>(ri);
    }
    __syncthreads();  // the scratch region becomes the contribution staging buffer
    clk(4);
    pdl_wait();
    DBG_SPAN_MIN(st, s, 4);
    SPAN_BEGIN(st, s, kSpanFinish);
    DBG_K3(st, s, bid, 0);
    clk(5);
    // ---- window log adjoints (tile.cuh), chunks of kEsChunk contribution rows; a warp per
    // slot, lanes over the index u: seasonality u gets entry u - (a - I + 1) of each window
    // whose [a - I + 1, a + O] covers u, level u the level entry of each window anchored at
    // u.  The last chunk also turns the log adjoints into adjoints (x 1/s, x 1/l) in the same
    // pass ((sum + chunk) * r: the operations of a separate scaling pass, one barrier fewer) ----
    const int nio = I + O;
    const int cb0 = pl.slot_win_off[k0];
    const int blo = woff[0], bhi = woff[nsl];
    const int lane = tid & 31, wq = tid >> 5;
    constexpr int kW = kFinishThreads / 32;
    for (int clo = blo; clo < bhi; clo += kEsChunk) {
        const int chi = min(bhi, clo + kEsChunk);
        const bool lastc = chi == bhi;
        const double* src = st.contrib + (size_t)(clo - cb0) * cwp;
        const int nel = (chi - clo) * cwp;
        for (int i = tid * 2; i < nel; i += kFinishThreads * 2) cp_async16(cbuf + i, src + i);
        cp_async_wait_all();
        __syncthreads();
        if (clo == blo) clk(10);  // first chunk landed (dbg_clk[42])
        for (int sl = wq; sl < nsl; sl += kW) {  // warp-uniform
            const int wl = max(woff[sl], clo), wh = min(woff[sl + 1], chi);
            if (wl >= wh && !lastc) continue;
            double* sbr = SB + sl * lds;
            double* lbr = LB + sl * ldl;
            for (int u = lane; u < T; u += 32) {
                if (wl < wh) {
                    double as = 0.0, al = 0.0;
                    for (int w = wl; w < wh; ++w) {
                        const double* c = cbuf + (w - clo) * cwp;
                        const int a = static_cast<int>(c[nio + 1]);
                        const int j = u - (a - I + 1);
                        if (j >= 0 && j < nio) as += c[j];
                        if (u == a) al += c[nio];
                    }
                    sbr[u] += as;
                    lbr[u] += al;
                }
                if (lastc) {
                    lbr[u] *= static_cast<double>(RI[u * bd + sl]);
                    sbr[u] *= static_cast<double>(RS[u * bd + sl]);
                }
            }
        }
        __syncthreads();
    }
    clk(6);
    if (blo == bhi) {  // no windows (cannot happen for a slot in the step; kept total)
        for (int sl = wq; sl < nsl; sl += kW)
            for (int t = lane; t < T; t += 32) {
                LB[sl * ldl + t] *= static_cast<double>(RI[t * bd + sl]);
                SB[sl * lds + t] *= static_cast<double>(RS[t * bd + sl]);
            }
        __syncthreads();
    }
    clk(7);
    if (!mine) return;
    // ---- reverse recursion (holt_winters.hpp:266-277 adjoints), Sb = final adjoint of s[t+S]:
    //   s_t: sb[t] + Sb (1-gamma) - Lb K1_t,   Lb_{t-1} = lb[t-1] + Lb (1-alpha) - Sb K2_t,
    //   (abar - omab) += Lb CA_t,   (gbar - omgb) += Sb CG_t
    const double alpha = coef[0][tid], gamma = coef[1][tid];
    const double oma = 1.0 - alpha, omg = 1.0 - gamma;
    double* lb = LB + tid * ldl;
    double* sb = SB + tid * lds;
    double asum = 0.0, gsum = 0.0;
    double lbn = lb[T - 1];
    auto step = [&](int t, double Sb, auto first) -> double {
        constexpr bool kFirst = decltype(first)::value;
        const double Lb = lbn;
        const int e = t * bd + tid;
        const double sbt = (sb[t] + Sb * omg) - Lb * static_cast<double>(K1[e]);
        if constexpr (!kFirst) lbn = (lb[t - 1] - Sb * static_cast<double>(K2[e])) + Lb * oma;
        asum += Lb * static_cast<double>(CA[e]);
        gsum += Sb * static_cast<double>(CG[e]);
        return sbt;
    };
    using Mid = std::integral_constant<bool, false>;
    using First = std::integral_constant<bool, true>;
    double sfin[SC > 0 ? SC : 1];
    if constexpr (SC > 0) {
        double rg[SC];
#pragma unroll
        for (int j = 0; j < SC; ++j) rg[j] = 0;  // s[T..T+S) receive no adjoint
        int base = ((T - 1) / SC) * SC;
        if (base > 0) {
#pragma unroll
            for (int jj = SC - 1; jj >= 0; --jj)
                if (base + jj < T) rg[jj] = step(base + jj, rg[jj], Mid{});
            for (base -= SC; base > 0; base -= SC) {
#pragma unroll
                for (int jj = SC - 1; jj >= 0; --jj) rg[jj] = step(base + jj, rg[jj], Mid{});
            }
        }
#pragma unroll
        for (int jj = SC - 1; jj >= 1; --jj)
            if (jj < T) rg[jj] = step(jj, rg[jj], Mid{});
        rg[0] = step(0, rg[0], First{});
#pragma unroll
        for (int j = 0; j < SC; ++j) sfin[j] = rg[j];
    } else {
        for (int t = T - 1; t >= 1; --t) sb[t] = step(t, sb[t + S], Mid{});
        sb[0] = step(0, sb[S], First{});
    }
    clk(8);
    // ---- per-series gradients: chain rule through the squashes (Logistic :483, Exp :501) ----
    Real* o = st.psg + (size_t)slot * np;
    const Real ga = static_cast<Real>(asum * alpha * oma);
    const Real gg = static_cast<Real>(gsum * gamma * omg);
    o[0] = ga;
    o[1] = gg;
    sq += static_cast<double>(ga) * ga + static_cast<double>(gg) * gg;
    auto out = [&](int j, double fin) {  // (pr[] was in the scratch region: E0 holds exp(raw))
        const Real g = static_cast<Real>(fin * E0[tid * S + j]);
        o[2 + j] = g;
        sq += static_cast<double>(g) * g;
    };
    if constexpr (SC > 0) {
#pragma unroll
        for (int j = 0; j < SC; ++j) out(j, sfin[j]);
    } else {
        for (int j = 0; j < S; ++j) out(j, sb[j]);
    }
    clk(9);
}

// ---------------------------------------------------------------------------------------
// K3 weight gradients by q-strips (fp32): block gbp = (strip, part), strip = kWq rows q of one
// matrix's G = A^T U over ALL its K columns, part = a contiguous range of the step's rows.
// Each row-store row is read once per strip (the 16 x 8 tiles read A K/8 times and U Q/16
// times: 15.7 MB of L2 reads per cfg1 step, 57 MB at cfg3), chunks of kWr rows by two TMA
// tensor copies.  Thread t owns G[4 qq .. 4 qq + 3][2 kk, 2 kk + 1] (qq = t % 8, kk = t / 8)
// and the bias sums of its 4 rows (kk == 0), summing its part's rows in order; parts are
// combined in part order by the last part to arrive (ticket) -- fixed order, no atomics on
// values.  Returns this thread's squared-gradient contribution (writer block only).
__device__ __forceinline__ double dw_wide_block(StateDev<float>& st, const PlanDev& pl, const NetLayout& lay, int s,
                                               int gbp, int gsplit, unsigned char* smem_raw, int nring,
                                               bool& writer) {
    const int tid = threadIdx.x;
    writer = true;
    const int gb = gbp / gsplit, part = gbp - gb * gsplit;
    int m = 0;
    while (m + 1 < lay.nmat && gb >= lay.mat_wblk0[m + 1]) ++m;
    const MatDesc md = lay.mats[m];
    const int q0 = (gb - lay.mat_wblk0[m]) * kWq;
    const bool uin0 = md.K == lay.layer_in[0] && m == 0;
    const int kp = uin0 ? lay.wkp_in0 : lay.wkp_h;  // U box columns
    const int wb0 = pl.step_win_off[s];
    const int Bstep = pl.step_win_off[s + 1] - wb0;
    const int span = ((Bstep + gsplit - 1) / gsplit + kWr - 1) / kWr * kWr;
    const int r0 = min(Bstep, part * span);
    const int Bl = min(Bstep, r0 + span) - r0;
    const int nch = (Bl + kWr - 1) / kWr;
    const int kmax = max(lay.wkp_in0, lay.wkp_h);
    float* As = reinterpret_cast<float*>(smem_raw);  // [nring][kWr][kWq]
    float* Us = As + nring * kWr * kWq;              // [nring][kWr][kp] (buffer stride kmax)
    __shared__ __align__(8) uint64_t wbar[kGBuf];
    __shared__ bool wlast;
    if (tid == 0)
        for (int b = 0; b < nring; ++b) mbar_init(&wbar[b], 1);
    __syncthreads();
    const unsigned char* tmb = static_cast<const unsigned char*>(st.tm_rs);
    const void* tmA = tmb + 2 * 128;
    const void* tmU = tmb + (uin0 ? 3 : 4) * 128;
    auto stage = [&](int c) {
        if (tid != 0 || c >= nch) return;
        const int buf = c % nring;
        fence_proxy_async_smem();
        mbar_expect_tx(&wbar[buf], static_cast<unsigned>(sizeof(float) * kWr * (kWq + kp)));
        tma2d_g2s(As + buf * kWr * kWq, tmA, md.a_off + q0, r0 + c * kWr, &wbar[buf]);
        tma2d_g2s(Us + buf * kWr * kmax, tmU, md.u_off, r0 + c * kWr, &wbar[buf]);
    };
    const int qq = tid & 7, kk = tid >> 3;
    const bool act = 2 * kk < kp;  // compute threads (kk == 0 also forms the bias sums)
    float acc[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}}, bacc[4] = {0, 0, 0, 0};
    for (int c = 0; c < nring - 1; ++c) stage(c);
    for (int c = 0; c < nch; ++c) {
        stage(c + nring - 1);
        mbar_wait(&wbar[c % nring], static_cast<unsigned>((c / nring) & 1));
        const int nb = min(kWr, Bl - c * kWr);
        const float* Ab = As + (c % nring) * kWr * kWq + 4 * qq;
        const float* Ub = Us + (c % nring) * kWr * kmax + 2 * kk;
        if (act) {
#pragma unroll 4
            for (int b = 0; b < nb; ++b) {
                const float4 a = *reinterpret_cast<const float4*>(Ab + b * kWq);
                const float2 u = *reinterpret_cast<const float2*>(Ub + b * kp);
                // paired FMAs (FFMA2): bit-identical to the scalar form
                asm("{ .reg .b64 p0, p1, p2, p3, u, a0, a1, a2, a3;\n\t"
                    "mov.b64 u, {%8, %9};\n\t"
                    "mov.b64 a0, {%10, %10};\n\t"
                    "mov.b64 a1, {%11, %11};\n\t"
                    "mov.b64 a2, {%12, %12};\n\t"
                    "mov.b64 a3, {%13, %13};\n\t"
                    "mov.b64 p0, {%0, %1};\n\t"
                    "mov.b64 p1, {%2, %3};\n\t"
                    "mov.b64 p2, {%4, %5};\n\t"
                    "mov.b64 p3, {%6, %7};\n\t"
                    "fma.rn.f32x2 p0, a0, u, p0;\n\t"
                    "fma.rn.f32x2 p1, a1, u, p1;\n\t"
                    "fma.rn.f32x2 p2, a2, u, p2;\n\t"
                    "fma.rn.f32x2 p3, a3, u, p3;\n\t"
                    "mov.b64 {%0, %1}, p0;\n\t"
                    "mov.b64 {%2, %3}, p1;\n\t"
                    "mov.b64 {%4, %5}, p2;\n\t"
                    "mov.b64 {%6, %7}, p3; }"
                    : "+f"(acc[0][0]), "+f"(acc[0][1]), "+f"(acc[1][0]), "+f"(acc[1][1]), "+f"(acc[2][0]),
                      "+f"(acc[2][1]), "+f"(acc[3][0]), "+f"(acc[3][1])
                    : "f"(u.x), "f"(u.y), "f"(a.x), "f"(a.y), "f"(a.z), "f"(a.w));
                if (kk == 0) {
                    bacc[0] += a.x;
                    bacc[1] += a.y;
                    bacc[2] += a.z;
                    bacc[3] += a.w;
                }
            }
        }
        __syncthreads();  // buffer c % nring is restaged next round
    }
    // this part's strip: [kWq][kWkMax + 1] (column kWkMax: bias), parts combined in order
    constexpr int ld = kWkMax + 1;
    double sq = 0.0;
    auto emit = [&](int i, int j, float g) {  // G[q0 + 4 qq + i][2 kk + j] (j == 2: bias)
        const int q = q0 + 4 * qq + i;
        if (q >= md.Q) return;
        if (j < 2) {
            const int k = 2 * kk + j;
            if (k >= md.K) return;
            st.gbuf[md.cw + (long long)q * md.ldk + k] = g;
        } else {
            st.gbuf[md.cb + q] = g;
        }
        sq += static_cast<double>(g) * g;
    };
    if (gsplit == 1) {
        if (act)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                emit(i, 0, acc[i][0]);
                emit(i, 1, acc[i][1]);
                if (kk == 0) emit(i, 2, bacc[i]);
            }
        return sq;
    }
    float* mine = st.gpart + ((size_t)gb * gsplit + part) * kWq * ld;
    if (act)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            mine[(4 * qq + i) * ld + 2 * kk] = acc[i][0];
            mine[(4 * qq + i) * ld + 2 * kk + 1] = acc[i][1];
            if (kk == 0) mine[(4 * qq + i) * ld + kWkMax] = bacc[i];
        }
    __threadfence();
    __syncthreads();
    if (tid == 0) wlast = atomicAdd(st.gtile_ctr + gb, 1u) == static_cast<unsigned>(gsplit - 1);
    __syncthreads();
    writer = wlast;
    if (!wlast) return 0.0;
    __threadfence();
    if (tid == 0) st.gtile_ctr[gb] = 0;
    if (act) {
        const float* base = st.gpart + (size_t)gb * gsplit * kWq * ld;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                if (j == 2 && kk != 0) continue;
                const int col = j < 2 ? 2 * kk + j : kWkMax;
                float g = 0.f;
                for (int p = 0; p < gsplit; ++p) g += __ldcg(base + (size_t)p * kWq * ld + (4 * qq + i) * ld + col);
                emit(i, j, g);
            }
    }
    return sq;
}

// UMMA: the tensor-core weight-gradient instantiation (large fp32 steps); the small-step
// kernel is compiled without that code (it changes the ES path's register allocation)
template <typename Real, int SC, bool UMMA>
__global__ void __launch_bounds__(kFinishThreads) k_grad_finish(StateDev<Real> st, PlanDev pl, NetLayout lay, int s,
                                                                int es_blocks, int finalize, int gsplit,
                                                                int umma_parts_arg, int nring, int es_bd) {
    const int umma_parts = UMMA ? umma_parts_arg : 0;
    using M = Math<Real>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ double red[32];
    __shared__ bool last;
    pdl_trigger();
    const int tid = threadIdx.x;
    double sq = 0.0;
    double pen = 0.0;  // level-variability penalty of this thread's slot (pinball-sum units)
    // ESRNN_DEBUG_CLOCKS: ES block 0 stamps at [32, 40), reduce block 0 at [48, 56)
    const int dbg_base = blockIdx.x == 0 ? 32 : (static_cast<int>(blockIdx.x) == es_blocks ? 48 : -1);
    int fdbg = 0;
    auto FCLK = [&]() {
        if (st.dbg_clk && dbg_base >= 0 && tid == 0) st.dbg_clk[dbg_base + fdbg] = clock64();
        ++fdbg;
    };
    FCLK();
    DBG_GT(st, 4);
    DBG_SPAN_MIN(st, s, 3);
    // large (tensor-core) steps: the dW blocks take the low block indices, so the long
    // contraction starts first and the many short ES blocks fill in around it; otherwise the
    // ES blocks come first (they pre-compute on the SMs K2 leaves free)
    const int ngemm = umma_parts > 0 ? static_cast<int>(gridDim.x) - es_blocks : 0;
    const int bid = umma_parts > 0 ? (static_cast<int>(blockIdx.x) < ngemm ? es_blocks + static_cast<int>(blockIdx.x)
                                                                           : static_cast<int>(blockIdx.x) - ngemm)
                                   : static_cast<int>(blockIdx.x);
    if (bid < es_blocks && sizeof(Real) == 4) {
        if constexpr (sizeof(Real) == 4) es_block_fp32<Real, SC>(st, pl, lay, s, smem_raw, sq, pen, bid, es_bd);
        const double tot = block_sum(sq, red);
        if (tid == 0) st.es_sq_part[bid] = tot;
        if (st.lvp > 0.0) {
            const double pt = block_sum(pen, red);
            if (tid == 0) st.es_pen_part[bid] = pt;
        }
    } else if (bid < es_blocks) {
        if constexpr (sizeof(Real) == 8) {  // (fp32 ES blocks: es_block_fp32 above)
            // ---------------- per-slot window-adjoint gather + reverse HW scan ---------------
            const int k0 = pl.step_slot_off[s];
            const int k = pl.step_slot_off[s + 1] - k0;
            const int sl0 = blockIdx.x * kEsSlotsPerBlock;
            const int sl1 = min(k, sl0 + kEsSlotsPerBlock);
            if (sl0 < sl1 && st.attach) {  // uniform per block
                const int N = st.N, S = SC > 0 ? SC : lay.S, T = lay.T, I = lay.I, O = lay.O, kc = st.kcap;
                const int bd = kEsSlotsPerBlock, tp = row_pad<Real>(T), cwp = st.cwp;
                const int slot = sl0 + tid;
                const bool mine = tid < bd && slot < sl1;
                const int lane = tid & 31;                                         // slot lane (bd == 32)
                // window adjoints row-major per slot (odd strides: the per-slot reverse scan reads
                // them conflict-free; the per-window warp scatter writes consecutive words)
                // The ES adjoint runs in double in both precisions (see the K2 contributions): the
                // level and seasonality paths of a window's adjoint cancel almost exactly, so their
                // accumulation and the reverse recursion must not round on their own
                const int ldl = T | 1, lds = (T + S) | 1;
                double* LB = reinterpret_cast<double*>(smem_raw);                  // [bd][ldl] level adjoint
                double* SB = LB + bd * ldl;                                        // [bd][lds] seasonality adjoint
                Real* LV = reinterpret_cast<Real*>(SB + bd * lds);                 // [T][bd]   forward levels
                Real* SE = LV + T * bd;                                            // [T][bd]   forward seasonalities
                Real* YS = reinterpret_cast<Real*>(SE + T * bd);                   // [bd][tp]  observation rows
                double* cbuf = reinterpret_cast<double*>(YS + bd * tp);            // [kEsChunk][cwp]
                double* lb = LB + tid * ldl;
                double* sb = SB + tid * lds;
                Real* lvs = LV + tid;
                Real* ses = SE + tid;
                Real* ys = YS + tid * tp;
                FCLK();
                // ---- stage the forward state with the whole block (every copy in flight at once) ----
                const bool lane_ok = sl0 + lane < sl1;
                const int lrow = lane_ok ? pl.slot_row[k0 + sl0 + lane] : 0;
                constexpr int e16 = 16 / static_cast<int>(sizeof(Real));
                constexpr int d16 = 2;  // doubles per 16-byte copy
                // observation rows are epoch constants: staged before the dependency wait
                if (lane_ok)
                    for (int ch = tid >> 5; ch * e16 < tp; ch += kFinishThreads / 32)
                        cp_async16(YS + lane * tp + ch * e16, st.vrm + (size_t)lrow * st.ldv + ch * e16);
                Real a_raw = 0, g_raw = 0;
                Real s0[SC > 0 ? SC : 1];  // exp(seas_raw) for the output's chain rule, loaded up front
                double l0 = 0;             // l[-1] = mean(y[0:S]) (holt_winters.hpp:247-250)
                pdl_wait();
                DBG_SPAN_MIN(st, s, 4);
                SPAN_BEGIN(st, s, kSpanFinish);
                {
                    if (mine) {
                        a_raw = st.ps[lrow];
                        g_raw = st.ps[N + lrow];
                        if constexpr (SC > 0) {
#pragma unroll
                            for (int j = 0; j < SC; ++j) s0[j] = st.ps[(size_t)(2 + j) * N + lrow];
                        }
                    }
                    // forward levels / seasonalities of the block's slots from K2's scan: whole
                    // 16-byte pieces of the [t][kcap] rows (kcap and sl0 are multiples of
                    // kEsSlotsPerBlock)
                    for (int e = tid; e < 2 * T * (bd / e16); e += kFinishThreads) {
                        const int half = e / (T * (bd / e16)), r = e - half * T * (bd / e16);
                        const int t = r / (bd / e16), ch = r - t * (bd / e16);
                        cp_async16((half ? SE : LV) + t * bd + ch * e16, (half ? st.se : st.lv) + (size_t)t * kc + sl0 + ch * e16);
                    }
                }
                // ---- window adjoints: this block's windows are one contiguous range of the
                // CSR-ordered contribution table, staged in chunks of kEsChunk rows; then one warp
                // per slot adds the slot's windows in CSR order, lanes over the window's
                // contiguous run of seasonality indices [a-I+1, a+O] ----
                const int cb0 = pl.slot_win_off[k0];
                const int blo = pl.slot_win_off[k0 + sl0], bhi = pl.slot_win_off[k0 + sl1];
                const int nio = I + O;
                const int wq = tid >> 5;
                for (int sl = wq; sl < bd; sl += kFinishThreads / 32) {
                    for (int t = lane; t < lds; t += 32) SB[sl * lds + t] = 0;
                    for (int t = lane; t < ldl; t += 32) LB[sl * ldl + t] = 0;
                }
                FCLK();
                for (int clo = blo; clo < bhi; clo += kEsChunk) {
                    const int chi = min(bhi, clo + kEsChunk);
                    const double* src = st.contrib + (size_t)(clo - cb0) * cwp;
                    const int nel = (chi - clo) * cwp;
                    for (int i = tid * d16; i < nel; i += kFinishThreads * d16) cp_async16(cbuf + i, src + i);
                    cp_async_wait_all();
                    __syncthreads();
                    FCLK();
                    for (int sl = wq; sl0 + sl < sl1 && sl < bd; sl += kFinishThreads / 32) {
                        const int w_lo = max(pl.slot_win_off[k0 + sl0 + sl], clo);
                        const int w_hi = min(pl.slot_win_off[k0 + sl0 + sl + 1], chi);
                        double* sbr = SB + sl * lds;
                        for (int w = w_lo; w < w_hi; ++w) {
                            const double* c = cbuf + (w - clo) * cwp;
                            const int a = static_cast<int>(c[nio + 1]);
                            for (int j = lane; j < nio; j += 32) sbr[a - I + 1 + j] += c[j];
                            if (lane == 0) LB[sl * ldl + a] += c[nio];
                            __syncwarp();
                        }
                    }
                    __syncthreads();
                }
                if (blo == bhi) {  // no windows (cannot happen for a slot in the step; kept total)
                    cp_async_wait_all();
                    __syncthreads();
                }
                // ---- per-slot prologue (scanning threads): alpha, gamma, l[-1], the penalty ----
                using MD = Math<double>;
                const double alpha = mine ? MD::logistic(static_cast<double>(a_raw)) : 0.0;
                const double gamma = mine ? MD::logistic(static_cast<double>(g_raw)) : 0.0;
                const double oma = 1.0 - alpha, omg = 1.0 - gamma;
                if (mine) {
                    cp_async_wait_all();
                    FCLK();
                    {
                        Real l0r = 0;
                        for (int j = 0; j < S; ++j) l0r += ys[j];
                        l0 = static_cast<double>(l0r / Real(S));
                    }
                    if (st.lvp > 0.0 && T >= 3) {
                        // opt-in level-variability penalty (oracle/esrnn_oracle.c lvp_series): with
                        // u_t = log l_t and e_t = u_t - 2 u_{t-1} + u_{t-2}, this slot adds
                        // c * mean_t e_t^2, c = lambda * O * (its windows) / M; its adjoint enters the
                        // LOG level adjoints directly (d/du_t; divided by l_t below)
                        const int nw = pl.slot_win_off[k0 + slot + 1] - pl.slot_win_off[k0 + slot];
                        const double cs = st.lvp * O * nw, c = cs / pl.step_M[s], inv = 1.0 / (T - 2);
                        double um2 = ::log(static_cast<double>(lvs[0])), um1 = ::log(static_cast<double>(lvs[bd])), acc = 0.0;
                        for (int t = 2; t < T; ++t) {
                            const double u = ::log(static_cast<double>(lvs[t * bd]));
                            const double e = u - 2.0 * um1 + um2;
                            acc += e * e;
                            const double q = c * 2.0 * inv * e;
                            lb[t] += q;
                            lb[t - 1] -= 2.0 * q;
                            lb[t - 2] += q;
                            um2 = um1;
                            um1 = u;
                        }
                        pen = cs * acc * inv;  // x M: the loss-sum units of loss_part
                    }
                }
                FCLK();
                if (mine) {
                    const int row = lrow;
                    double abar = 0, gbar = 0, omab = 0, omgb = 0;
                    double sfin[SC > 0 ? SC : 1];
                    using Mid = std::integral_constant<bool, false>;
                    using First = std::integral_constant<bool, true>;
                    // fp64: the reference's arithmetic (IEEE divisions), linearised at K2's states
                    double lbn = lb[T - 1] / lvs[(T - 1) * bd];  // running adjoint of l[t]
                    // one reverse step (t > 0 unless FIRST): Sb = final adjoint of s[t+S],
                    // returns the final adjoint of s[t]
                    auto step = [&](int t, double Sb, auto first) -> double {
                        constexpr bool kFirst = decltype(first)::value;
                        const double yt = ys[t];
                        const double lp = kFirst ? l0 : lvs[(t - 1) * bd];
                        const double s_t = ses[t * bd];
                        double sbt = sb[t] / s_t;
                        // s_{t+S} = gamma*(y/lp) + (1-gamma)*s_t
                        omgb += Sb * s_t;
                        sbt += Sb * omg;
                        const double d2 = yt / lp;
                        gbar += Sb * d2;
                        // l_t = alpha*(y/s_t) + (1-alpha)*lp
                        const double Lb = lbn;
                        omab += Lb * lp;
                        const double d1 = yt / s_t;
                        abar += Lb * d1;
                        sbt -= ((Lb * alpha) * d1) / s_t;
                        if constexpr (!kFirst) {
                            const double d2b = Sb * gamma;
                            lbn = lb[t - 1] / lp - (d2b * d2) / lp + Lb * oma;
                        }
                        return sbt;
                    };
                    if constexpr (SC > 0) {
                        // register ring: rg[j] holds the final adjoint of the latest s index = j
                        // (mod S); full groups of SC steps are branch-free so steps interleave
                        double rg[SC];
#pragma unroll
                        for (int j = 0; j < SC; ++j) rg[j] = 0;  // s[T..T+S) receive no adjoint
                        int base = ((T - 1) / SC) * SC;
                        if (base > 0) {
#pragma unroll
                            for (int jj = SC - 1; jj >= 0; --jj)
                                if (base + jj < T) rg[jj] = step(base + jj, rg[jj], Mid{});
                            for (base -= SC; base > 0; base -= SC) {
#pragma unroll
                                for (int jj = SC - 1; jj >= 0; --jj) rg[jj] = step(base + jj, rg[jj], Mid{});
                            }
                        }
#pragma unroll
                        for (int jj = SC - 1; jj >= 1; --jj)
                            if (jj < T) rg[jj] = step(jj, rg[jj], Mid{});
                        rg[0] = step(0, rg[0], First{});
#pragma unroll
                        for (int j = 0; j < SC; ++j) sfin[j] = rg[j];
                    } else {
#pragma unroll 4
                        for (int t = T - 1; t >= 1; --t) sb[t] = step(t, sb[t + S], Mid{});
                        sb[0] = step(0, sb[S], First{});
                    }
                    FCLK();
                    abar -= omab;
                    gbar -= omgb;
                    Real* o = st.psg + (size_t)slot * (2 + S);
                    const Real ga = static_cast<Real>(abar * alpha * oma);
                    const Real gg = static_cast<Real>(gbar * gamma * omg);
                    o[0] = ga;
                    o[1] = gg;
                    sq += static_cast<double>(ga) * ga + static_cast<double>(gg) * gg;
                    if constexpr (SC > 0) {
#pragma unroll
                        for (int j = 0; j < SC; ++j) {
                            const Real g = static_cast<Real>(sfin[j] * MD::exp(static_cast<double>(s0[j])));
                            o[2 + j] = g;
                            sq += static_cast<double>(g) * g;
                        }
                    } else {
                        for (int j = 0; j < S; ++j) {
                            const Real g = static_cast<Real>(sb[j] * MD::exp(static_cast<double>(st.ps[(2 + j) * N + row])));
                            o[2 + j] = g;
                            sq += static_cast<double>(g) * g;
                        }
                    }
                }
            } else {
                pdl_wait();
                SPAN_BEGIN(st, s, kSpanFinish);
            }
            const double tot = block_sum(sq, red);
            if (tid == 0) st.es_sq_part[blockIdx.x] = tot;
            if (st.lvp > 0.0) {
                const double pt = block_sum(pen, red);
                if (tid == 0) st.es_pen_part[blockIdx.x] = pt;
            }
        }
    } else if (UMMA && sizeof(Real) == 4) {
        pdl_wait();
        SPAN_BEGIN(st, s, kSpanFinish);
        if constexpr (UMMA && sizeof(Real) == 4) dw_umma_block(st, pl, lay, s, bid - es_blocks, umma_parts, smem_raw, red);
    } else if (sizeof(Real) == 4 && st.gemm_wide) {
        pdl_wait();
        SPAN_BEGIN(st, s, kSpanFinish);
        DBG_K3(st, s, bid, 0);
        if constexpr (sizeof(Real) == 4) {
            const int gbp = bid - es_blocks;
            bool writer = true;
            sq = dw_wide_block(st, pl, lay, s, gbp, gsplit, smem_raw, nring, writer);
            const double tot = block_sum(sq, red);
            if (tid == 0 && writer) st.red_sq_part[gbp / gsplit] = tot;
        }
    } else {
        pdl_wait();
        SPAN_BEGIN(st, s, kSpanFinish);
        DBG_K3(st, s, bid, 0);
        FCLK();
        // ------- weight gradients: G[q][k] = sum_b A[b][q] U[b][k] over the step's windows ----
        // block -> (matrix, 16 q x 8 k output block, row part); warp w sums rows b = w (mod 8)
        // of its part in order, warps are combined in order, and for large steps (gsplit > 1
        // row parts) the last-arriving part adds the parts' tiles in part order: a fixed
        // summation order, no float atomics
        const int gbp = blockIdx.x - es_blocks;
        const int gb = gbp / gsplit, part = gbp - gb * gsplit;
        int m = 0;
        while (m + 1 < lay.nmat && gb >= lay.mat_blk0[m + 1]) ++m;
        const MatDesc md = lay.mats[m];
        const int local = gb - lay.mat_blk0[m];
        const int nkb = (md.K + kGk - 1) / kGk;
        const int q0 = (local / nkb) * kGq, k0 = (local % nkb) * kGk;
        const int wb0 = pl.step_win_off[s];
        const int Bstep = pl.step_win_off[s + 1] - wb0;
        // this part's rows [r0, r0 + Bl) of the step's row store (chunk-aligned split)
        const int span = ((Bstep + gsplit - 1) / gsplit + kGChunk - 1) / kGChunk * kGChunk;
        const int r0 = min(Bstep, part * span);
        const int Bl = min(Bstep, r0 + span) - r0;
        const int lane = tid & 31, warp = tid >> 5;
        const int qp = lane >> 2, kp = lane & 3;
        Real* As = reinterpret_cast<Real*>(smem_raw);       // [nring][kGChunk][kGq]
        Real* Us = As + nring * kGChunk * kGq;               // [nring][kGChunk][kGk]
        Real* Rd = Us + nring * kGChunk * kGk;               // [8 warps][32 lanes][6]
        // chunk staging by TMA: two 2-D tensor copies per chunk (the A and U column boxes of
        // kGChunk rows), completion on the buffer's mbarrier.  (16-byte cp.async of the
        // scattered row segments kept the SM's load pipeline busy ~1.5k cycles per chunk and
        // stalled the co-resident ES blocks' shared-memory traffic behind it.)  Rows past the
        // step's end are staged but never summed; rows past the allocation read as zeros.
        __shared__ __align__(8) uint64_t gbar[kGBuf];
        if (tid == 0) {
#pragma unroll
            for (int b = 0; b < kGBuf; ++b)
                if (b < nring) mbar_init(&gbar[b], 1);
        }
        __syncthreads();
        const int nch = (Bl + kGChunk - 1) / kGChunk;
        const void* tmA = st.tm_rs;
        const void* tmU = static_cast<const unsigned char*>(st.tm_rs) + 128;
        auto stage = [&](int c) {
            if (tid != 0 || c >= nch) return;
            const int buf = c % nring;
            fence_proxy_async_smem();  // the buffer's previous generic reads before the async writes
            mbar_expect_tx(&gbar[buf], static_cast<unsigned>(sizeof(Real) * kGChunk * (kGq + kGk)));
            tma2d_g2s(As + buf * kGChunk * kGq, tmA, md.a_off + q0, r0 + c * kGChunk, &gbar[buf]);
            tma2d_g2s(Us + buf * kGChunk * kGk, tmU, md.u_off + k0, r0 + c * kGChunk, &gbar[buf]);
        };
        Real acc[2][2] = {{0, 0}, {0, 0}}, bacc[2] = {0, 0};
        // nring - 1 chunks in flight ahead of the one being summed
        for (int c = 0; c < nring - 1; ++c) stage(c);
        for (int c = 0; c < nch; ++c) {
            stage(c + nring - 1);
            mbar_wait(&gbar[c % nring], static_cast<unsigned>((c / nring) & 1));
            if (c == 0) FCLK();
            const int nb = min(kGChunk, Bl - c * kGChunk);
            const Real* Ab = As + (c % nring) * kGChunk * kGq + 2 * qp;
            const Real* Ub = Us + (c % nring) * kGChunk * kGk + 2 * kp;
#pragma unroll 8
            for (int b = warp; b < nb; b += kFinishThreads / 32) {
                Real a0, a1, u0, u1;
                if constexpr (sizeof(Real) == 4) {  // 8-byte pairs (2*qp, 2*kp are even)
                    const float2 a = *reinterpret_cast<const float2*>(Ab + b * kGq);
                    const float2 u = *reinterpret_cast<const float2*>(Ub + b * kGk);
                    a0 = a.x, a1 = a.y, u0 = u.x, u1 = u.y;
                } else {
                    const double2 a = *reinterpret_cast<const double2*>(Ab + b * kGq);
                    const double2 u = *reinterpret_cast<const double2*>(Ub + b * kGk);
                    a0 = a.x, a1 = a.y, u0 = u.x, u1 = u.y;
                }
                if constexpr (sizeof(Real) == 4) {
                    // paired FMAs / adds (FFMA2, FADD2): bit-identical to the scalar form
                    asm("{ .reg .b64 p, q, u, a0, a1, b;\n\t"
                        "mov.b64 u, {%6, %7};\n\t"
                        "mov.b64 a0, {%8, %8};\n\t"
                        "mov.b64 a1, {%9, %9};\n\t"
                        "mov.b64 p, {%0, %1};\n\t"
                        "mov.b64 q, {%2, %3};\n\t"
                        "mov.b64 b, {%4, %5};\n\t"
                        "fma.rn.f32x2 p, a0, u, p;\n\t"
                        "fma.rn.f32x2 q, a1, u, q;\n\t"
                        "mov.b64 u, {%8, %9};\n\t"
                        "add.rn.f32x2 b, b, u;\n\t"
                        "mov.b64 {%0, %1}, p;\n\t"
                        "mov.b64 {%2, %3}, q;\n\t"
                        "mov.b64 {%4, %5}, b; }"
                        : "+f"(acc[0][0]), "+f"(acc[0][1]), "+f"(acc[1][0]), "+f"(acc[1][1]), "+f"(bacc[0]),
                          "+f"(bacc[1])
                        : "f"(u0), "f"(u1), "f"(a0), "f"(a1));
                } else {
                    acc[0][0] += a0 * u0;
                    acc[0][1] += a0 * u1;
                    acc[1][0] += a1 * u0;
                    acc[1][1] += a1 * u1;
                    bacc[0] += a0;
                    bacc[1] += a1;
                }
            }
            __syncthreads();  // buffer c % nring is restaged next round
        }
        FCLK();
        Real* rd = Rd + (warp * 32 + lane) * 6;
        rd[0] = acc[0][0];
        rd[1] = acc[0][1];
        rd[2] = acc[1][0];
        rd[3] = acc[1][1];
        rd[4] = bacc[0];
        rd[5] = bacc[1];
        __syncthreads();
        __shared__ bool last_part;
        Real t[6];
        if (warp == 0) {
#pragma unroll
            for (int j = 0; j < 6; ++j) t[j] = Rd[lane * 6 + j];
            for (int w = 1; w < kFinishThreads / 32; ++w)
#pragma unroll
                for (int j = 0; j < 6; ++j) t[j] += Rd[(w * 32 + lane) * 6 + j];
            if (gsplit > 1) {
                // publish this part's tile; the last part to arrive combines them
                Real* mine = st.gpart + ((size_t)part * st.red_tiles + gb) * 32 * 6 + lane * 6;
#pragma unroll
                for (int j = 0; j < 6; ++j) mine[j] = t[j];
                __threadfence();
                __syncwarp();
                if (lane == 0) last_part = atomicAdd(st.gtile_ctr + gb, 1u) == static_cast<unsigned>(gsplit - 1);
                __syncwarp();
            }
        }
        if (gsplit > 1) __syncthreads();  // last_part (block-uniform branch)
        const bool writer = gsplit == 1 || last_part;  // else another part writes this tile
        if (warp == 0 && writer) {
            if (gsplit > 1) {
                __threadfence();
                if (lane == 0) st.gtile_ctr[gb] = 0;
#pragma unroll
                for (int j = 0; j < 6; ++j) {
                    Real a = 0;
                    for (int p = 0; p < gsplit; ++p)
                        a += __ldcg(st.gpart + ((size_t)p * st.red_tiles + gb) * 32 * 6 + lane * 6 + j);
                    t[j] = a;
                }
            }
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int q = q0 + 2 * qp + i;
                if (q >= md.Q) continue;
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int k = k0 + 2 * kp + j;
                    if (k >= md.K) continue;
                    const Real g = t[2 * i + j];
                    st.gbuf[md.cw + (long long)q * md.ldk + k] = g;
                    sq += static_cast<double>(g) * g;
                }
                if (k0 == 0 && kp == 0) {
                    const Real g = t[4 + i];
                    st.gbuf[md.cb + q] = g;
                    sq += static_cast<double>(g) * g;
                }
            }
        }
        const double tot = block_sum(sq, red);
        if (tid == 0 && writer) st.red_sq_part[gb] = tot;
    }
    FCLK();
    DBG_K3(st, s, bid, 1);
    DBG_SPAN_MAX(st, s, 5);
    if (bid < es_blocks) DBG_SPAN_MAX(st, s, 10);
    else DBG_SPAN_MAX(st, s, 11);
    SPAN_END(st, s, kSpanFinish);
    if (finalize & 4) {
        // single GPU, updating step: K4 derives the step scalars from the partials itself
        // (no last-CTA ticket on this kernel's tail); only a step that applies updates
        // advances Adam's t (trainer.hpp:617) -- every block has passed pdl_wait, so the
        // tile's error word is final
        if (blockIdx.x == 0 && tid == 0 && st.err[0] == 0) ++(*st.net_step);
        return;
    }
    // ---------------- last CTA finalises ------------------------------------------------
    if (tid == 0) {
        __threadfence();
        const unsigned ticket = atomicAdd(st.done_ctr, 1u);
        last = (ticket == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (tid == 0 && st.dbg_clk) st.dbg_clk[85] = gtimer();
    // all threads sum the per-block parts (strided, then a fixed tree): L2 loads in flight at once
    const int nrb = st.red_tiles;
    const int w0 = pl.step_win_off[s];
    const int nt = (pl.step_win_off[s + 1] - w0 + kR - 1) / kR;
    double es = 0.0, ls = 0.0, all = 0.0;
    if (st.attach)
        for (int b = tid; b < es_blocks; b += kFinishThreads) es += __ldcg(st.es_sq_part + b);
    for (int t = tid; t < nt; t += kFinishThreads) ls += __ldcg(st.loss_part + t);
    if (st.lvp > 0.0)  // the penalty joins the loss sum (its partials are in the same units)
        for (int b = tid; b < es_blocks; b += kFinishThreads) ls += __ldcg(st.es_pen_part + b);
    for (int b = tid; b < nrb; b += kFinishThreads) all += __ldcg(st.red_sq_part + b);
    es = block_sum(es, red);
    ls = block_sum(ls, red);
    all = block_sum(all, red);
    if (tid != 0) return;
    st.gtail[0] = es;
    st.gtail[1] = ls;
    st.gtail[2] = st.err[0] != 0 ? 1.0 : 0.0;
    st.gtail[3] = 0.0;
    if (finalize & 1) finalize_scalars(st, pl, s, all + es, ls, (finalize & 2) != 0, st.err[0] != 0);
    *st.done_ctr = 0;
    DBG_SPAN_MAX(st, s, 6);
    SPAN_END(st, s, kSpanFinish);
}

// After the NCCL all-reduce of gbuf and gtail (sharded mode): global squared norm + scalars.
template <typename Real>
__global__ void __launch_bounds__(256) k_finalize(StateDev<Real> st, PlanDev pl, NetLayout lay, int s, int advance) {
    __shared__ double red[32];
    __shared__ bool last;
    SPAN_BEGIN(st, s, kSpanReduce);
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
    SPAN_END(st, s, kSpanReduce);
    if (!last) return;
    __threadfence();
    double all = 0.0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) all += __ldcg(st.red_sq_part + b);
    all = block_sum(all, red);
    if (threadIdx.x != 0) return;
    const double es = st.attach ? st.gtail[0] : 0.0;
    finalize_scalars(st, pl, s, all + es, st.gtail[1], advance != 0, st.gtail[2] != 0.0);
    st.done_ctr[1] = 0;
    SPAN_END(st, s, kSpanReduce);
}

// ------------------------------------------------------------------------------ K4
__device__ __forceinline__ void adam_update(double& theta, double& m, double& v, double g, double lr, double c1,
                                            double c2) {
    // trainer.hpp:626-630 / :642-647
    m = 0.9 * m + (1.0 - 0.9) * g;
    v = 0.999 * v + (1.0 - 0.999) * g * g;
    theta -= lr * (m / c1) / (sqrt(v / c2) + 1e-8);
}

// es_blocks >= 0 (single GPU): every block first derives the step scalars -- clip scale
// (trainer.hpp:603-615), bias corrections at the step K3 advanced (:617-620), step loss --
// from K3's per-block partials with the same loads, order and tree as the last-CTA
// finalisation, so all blocks hold bit-identical values and K3 needs no serial tail;
// block 0 publishes them.  es_blocks < 0 (sharded): k_finalize / k_group_reduce already
// wrote st.scal from the reduced buffers.
template <typename Real>
__global__ void __launch_bounds__(256) k_adam(StateDev<Real> st, PlanDev pl, NetLayout lay, int s, int es_blocks,
                                              int red_blocks, int net_blocks) {
    __shared__ double red[96];
    __shared__ double sc[3];
    pdl_trigger();
    const int tid = threadIdx.x;
    // this thread's Adam operands first: m, v and the parameter (no kernel of this step writes
    // them before this one) before the dependency wait -- under programmatic dependent launch
    // (ESRNN_K4_PDL) their latency overlaps K3's tail -- then the gradient after it; their L2
    // latency overlaps the scalar reduction below.  Network blocks: one live parameter; per-series blocks (trainer.hpp:636-650):
    // one (slot, parameter), a slot's 2+S threads in one block so its step counter is read
    // before it is advanced.
    const bool net = static_cast<int>(blockIdx.x) < net_blocks;
    const int N = st.N, np = 2 + lay.S;
    const long long q = (long long)blockIdx.x * blockDim.x + tid;
    bool mine = false;
    int row = 0, steps = 0, j = 0, slot = 0;
    size_t e = 0;
    Real g0 = 0, m0 = 0, v0 = 0, t0 = 0;
    double c1 = 1.0, c2 = 1.0;
    if (net) {
        mine = q < lay.P_pad;
        if (mine) m0 = st.mW[q], v0 = st.vW[q], t0 = st.theta[q];
    } else if (st.attach) {
        const int spb = static_cast<int>(blockDim.x) / np;
        const int k0 = pl.step_slot_off[s];
        const int k = pl.step_slot_off[s + 1] - k0;
        const int ls = tid / np;
        j = tid - ls * np;
        slot = (static_cast<int>(blockIdx.x) - net_blocks) * spb + ls;
        mine = ls < spb && slot < k;
        if (mine) {
            row = pl.slot_row[k0 + slot];
            steps = st.ps_steps[row] + 1;
            e = (size_t)j * N + row;
            m0 = st.ps_m[e], v0 = st.ps_v[e], t0 = st.ps[e];
            c1 = bias_c1(st, steps);
            c2 = bias_c2(st, steps);
        }
    }
    pdl_wait();
    DBG_GT(st, 6);
    DBG_SPAN_MIN(st, s, 7);
    SPAN_BEGIN(st, s, kSpanAdam);
    if (mine) g0 = net ? st.gbuf[q] : st.psg[(size_t)slot * np + j];
    if (es_blocks >= 0) {
        // single GPU: the step scalars from K3's partials -- clip scale (trainer.hpp:603-615),
        // bias corrections at the step K3 advanced (:617-620), step loss -- with the same
        // loads, order and tree as the last-CTA finalisation, so every block holds identical
        // values; block 0 publishes them
        const int w0 = pl.step_win_off[s];
        const int nt = (pl.step_win_off[s + 1] - w0 + kR - 1) / kR;
        double es = 0.0, ls = 0.0, all = 0.0;
        if (st.attach)
            for (int b = tid; b < es_blocks; b += blockDim.x) es += __ldcg(st.es_sq_part + b);
        for (int t = tid; t < nt; t += blockDim.x) ls += __ldcg(st.loss_part + t);
        if (st.lvp > 0.0)
            for (int b = tid; b < es_blocks; b += blockDim.x) ls += __ldcg(st.es_pen_part + b);
        for (int b = tid; b < red_blocks; b += blockDim.x) all += __ldcg(st.red_sq_part + b);
        block_sum3(es, ls, all, red);
        if (tid == 0) {
            double scale = 1.0;
            if (st.has_clip) {
                const double norm = sqrt(all + es);
                if (norm > st.clip) scale = st.clip / norm;
            }
            const long long step = *st.net_step;
            sc[0] = scale;
            sc[1] = bias_c1(st, step);
            sc[2] = bias_c2(st, step);
            if (blockIdx.x == 0) {
                st.gtail[0] = es;
                st.gtail[1] = ls;
                st.scal[0] = scale;
                st.scal[3] = ls / pl.step_M[s];
                st.loss_hist[s] = ls / pl.step_M[s];
                if (st.err[0] == 0) {
                    st.scal[1] = sc[1];
                    st.scal[2] = sc[2];
                }
            }
        }
    } else if (tid == 0) {  // sharded: k_finalize already wrote them
        sc[0] = st.scal[0];
        sc[1] = st.scal[1];
        sc[2] = st.scal[2];
    }
    __syncthreads();
    // the reference throws before apply_updates; sharded: err[2] is any rank's error
    if (!mine || st.err[0] != 0 || st.err[2] != 0) {
        SPAN_END(st, s, kSpanAdam);
        return;
    }
    double th = t0, m = m0, v = v0;
    if (net) {
        adam_update(th, m, v, static_cast<double>(g0) * sc[0], st.lr_net, sc[1], sc[2]);
        st.mW[q] = static_cast<Real>(m);
        st.vW[q] = static_cast<Real>(v);
        st.theta[q] = static_cast<Real>(th);
    } else {
        if (j == 0) st.ps_steps[row] = steps;
        adam_update(th, m, v, static_cast<double>(g0) * sc[0], st.lr_ps, c1, c2);
        st.ps_m[e] = static_cast<Real>(m);
        st.ps_v[e] = static_cast<Real>(v);
        st.ps[e] = static_cast<Real>(th);
    }
    DBG_SPAN_MAX(st, s, 8);
    SPAN_END(st, s, kSpanAdam);
}

}  // namespace esrnn_dev
