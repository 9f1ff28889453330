// The general dilated LSTM stack over an input sequence:
// forward_stack (network.hpp:190-210, plain mirror :268-287) with full LSTM cells -- forget
// gates, recurrent matrices, (h, c) read from step t - d (lstm_cell :148-163,
// dilated_lstm_layer :167-184) -- and the reverse-mode adjoints the reference's tape forms for
// it (Tape::backward, autodiff.hpp:397-631).  The training hot path runs the stack at sequence
// length 1 (tile.cuh); this is the rest of the forward_stack API, for callers that pass
// multi-step sequences (test_network.cpp:94-181, :235-267; acceptance.cpp:183-217).
//
// A CTA owns kSeqRows batch rows for the whole sequence: layer by layer, step by step (the
// recurrence is serial in t), threads over (row, gate output) for the products and over
// (row, unit) for the cell.  Saved activations live in a per-CTA global scratch (L2
// resident at these sizes).  Weight gradients are per-CTA partials, reduced in CTA order by
// k_seq_reduce: deterministic, no float atomics.
#pragma once
#include "common.cuh"

namespace esrnn_dev {

constexpr int kSeqRows = 4;
constexpr int kSeqThreads = 256;

// Offsets of the flat for_each_param weight vector (network.hpp:62-74) and the stack shape.
struct SeqLayout {
    int L, H, O, in0, T, B, in_max;
    int layer_in[kMaxLayers], dil[kMaxLayers];
    int res_src[kMaxLayers];    // >= 0: this layer's output gets layer res_src's output added (block b>0 skip)
    long long w_in[kMaxLayers], w_rec[kMaxLayers], bias[kMaxLayers];
    long long nl_w, nl_b, out_w, out_b, P;
};

// Per-CTA scratch (Real units), see seq_scratch_size
template <typename Real>
struct SeqScratch {
    Real *gates, *cst, *hraw, *cur, *dcur, *dhr, *dcr, *dpre, *din, *z, *dzp;
    __host__ __device__ static long long size(const SeqLayout& s) {
        const long long LT = static_cast<long long>(s.L) * s.T * kSeqRows;
        const long long TR = static_cast<long long>(s.T) * kSeqRows;
        return LT * (4LL * s.H) + 4 * LT * s.H + 2 * TR * s.H + TR * 4LL * s.H + TR * s.in_max + 2LL * kSeqRows * s.H;
    }
    __device__ static SeqScratch at(Real* base, const SeqLayout& s) {
        const long long LT = static_cast<long long>(s.L) * s.T * kSeqRows;
        const long long TR = static_cast<long long>(s.T) * kSeqRows;
        SeqScratch c;
        Real* p = base + static_cast<long long>(blockIdx.x) * size(s);
        c.gates = p; p += LT * 4 * s.H;   // [L][T][r][4H] i f g o
        c.cst = p; p += LT * s.H;         // [L][T][r][H] cell state
        c.hraw = p; p += LT * s.H;        // [L][T][r][H] cell output (the recurrent state)
        c.cur = p; p += LT * s.H;         // [L][T][r][H] layer output (+ block skip)
        c.dcur = p; p += LT * s.H;        // [L][T][r][H] adjoint of cur
        c.dhr = p; p += TR * s.H;         // [T][r][H] recurrent adjoint of h
        c.dcr = p; p += TR * s.H;         // [T][r][H] recurrent adjoint of c
        c.dpre = p; p += TR * 4 * s.H;    // [T][r][4H] pre-activation adjoints of one layer
        c.din = p; p += TR * s.in_max;    // [T][r][in] input adjoint of one layer
        c.z = p; p += kSeqRows * s.H;     // [r][H] head activations
        c.dzp = p;                        // [r][H] head pre-activation adjoints
        return c;
    }
};

__device__ __forceinline__ long long sidx(const SeqLayout& s, int l, int t, int r) {
    return (static_cast<long long>(l) * s.T + t) * kSeqRows + r;
}

// Layer input row (row r, step t) of layer l: the sequence for layer 0, else the previous
// layer's output.
template <typename Real>
__device__ __forceinline__ const Real* seq_in(const SeqLayout& s, const SeqScratch<Real>& c, const Real* X, int l,
                                              int t, int r, int b0) {
    return l == 0 ? X + (static_cast<long long>(t) * s.B + b0 + r) * s.in0 : c.cur + sidx(s, l - 1, t, r) * s.H;
}

template <typename Real>
__global__ void __launch_bounds__(kSeqThreads) k_seq_forward(SeqLayout s, const Real* __restrict__ W,
                                                              const Real* __restrict__ X, Real* scratch, double* out) {
    using M = Math<Real>;
    const int b0 = blockIdx.x * kSeqRows, nr = min(kSeqRows, s.B - b0);
    const int tid = threadIdx.x, NT = blockDim.x, H = s.H, G = 4 * H;
    const SeqScratch<Real> c = SeqScratch<Real>::at(scratch, s);
    for (int l = 0; l < s.L; ++l) {
        const int K = s.layer_in[l], d = s.dil[l];
        const Real* Wi = W + s.w_in[l];
        const Real* Wr = W + s.w_rec[l];
        const Real* bi = W + s.bias[l];
        for (int t = 0; t < s.T; ++t) {
            // pre = x W_in (+ h_{t-d} W_rec) + b (lstm_cell, network.hpp:152-154), then the gates
            for (int e = tid; e < nr * G; e += NT) {
                const int r = e / G, j = e - r * G;
                const Real* x = seq_in(s, c, X, l, t, r, b0);
                Real acc = 0;
                for (int k = 0; k < K; ++k) acc += x[k] * Wi[static_cast<long long>(k) * G + j];
                if (t >= d) {
                    const Real* hp = c.hraw + sidx(s, l, t - d, r) * H;
                    Real a2 = 0;
                    for (int k = 0; k < H; ++k) a2 += hp[k] * Wr[static_cast<long long>(k) * G + j];
                    acc += a2;
                }
                acc += bi[j];
                c.gates[sidx(s, l, t, r) * G + j] = (j >= 2 * H && j < 3 * H) ? M::tanh(acc) : M::logistic(acc);
            }
            __syncthreads();
            // c = f c_{t-d} + i g, h = o tanh(c); block skip added after the block's last layer
            for (int e = tid; e < nr * H; e += NT) {
                const int r = e / H, j = e - r * H;
                const Real* gt = c.gates + sidx(s, l, t, r) * G;
                const Real i = gt[j], f = gt[H + j], g = gt[2 * H + j], o = gt[3 * H + j];
                const Real cv = (t >= d ? f * c.cst[sidx(s, l, t - d, r) * H + j] : Real(0)) + i * g;
                const Real h = o * M::tanh(cv);
                c.cst[sidx(s, l, t, r) * H + j] = cv;
                c.hraw[sidx(s, l, t, r) * H + j] = h;
                c.cur[sidx(s, l, t, r) * H + j] =
                    s.res_src[l] >= 0 ? h + c.cur[sidx(s, s.res_src[l], t, r) * H + j] : h;
            }
            __syncthreads();
        }
    }
    // head on the last step (network.hpp:207-209)
    for (int e = tid; e < nr * H; e += NT) {
        const int r = e / H, j = e - r * H;
        const Real* last = c.cur + sidx(s, s.L - 1, s.T - 1, r) * H;
        Real acc = 0;
        for (int k = 0; k < H; ++k) acc += last[k] * W[s.nl_w + static_cast<long long>(k) * H + j];
        c.z[r * H + j] = M::tanh(acc + W[s.nl_b + j]);
    }
    __syncthreads();
    for (int e = tid; e < nr * s.O; e += NT) {
        const int r = e / s.O, o = e - r * s.O;
        Real acc = 0;
        for (int k = 0; k < H; ++k) acc += c.z[r * H + k] * W[s.out_w + static_cast<long long>(k) * s.O + o];
        out[static_cast<long long>(b0 + r) * s.O + o] = static_cast<double>(acc + W[s.out_b + o]);
    }
}

// Reverse sweep of the same graph for the adjoint out_bar [B][O]: per-CTA weight-gradient
// partials wpart [gridDim][P] (for_each_param order) and input adjoints xbar [T][B][in0].
template <typename Real>
__global__ void __launch_bounds__(kSeqThreads) k_seq_backward(SeqLayout s, const Real* __restrict__ W,
                                                               const Real* __restrict__ X, Real* scratch,
                                                               const Real* __restrict__ obar, Real* wpart, Real* xbar) {
    const int b0 = blockIdx.x * kSeqRows, nr = min(kSeqRows, s.B - b0);
    const int tid = threadIdx.x, NT = blockDim.x, H = s.H, G = 4 * H, O = s.O;
    const SeqScratch<Real> c = SeqScratch<Real>::at(scratch, s);
    Real* wp = wpart + static_cast<long long>(blockIdx.x) * s.P;
    for (long long e = tid; e < s.P; e += NT) wp[e] = 0;
    for (long long e = tid; e < static_cast<long long>(s.L) * s.T * kSeqRows * H; e += NT) c.dcur[e] = 0;
    __syncthreads();
    // head: out = z out_w + out_b, z = tanh(last nl_w + nl_b)
    const Real* ob = obar + static_cast<long long>(b0) * O;
    for (int e = tid; e < H * O + O; e += NT) {
        Real acc = 0;
        if (e < H * O) {
            const int k = e / O, o = e - k * O;
            for (int r = 0; r < nr; ++r) acc += c.z[r * H + k] * ob[r * O + o];
            wp[s.out_w + e] = acc;
        } else {
            for (int r = 0; r < nr; ++r) acc += ob[r * O + (e - H * O)];
            wp[s.out_b + (e - H * O)] = acc;
        }
    }
    for (int e = tid; e < nr * H; e += NT) {
        const int r = e / H, k = e - r * H;
        Real acc = 0;
        for (int o = 0; o < O; ++o) acc += ob[r * O + o] * W[s.out_w + static_cast<long long>(k) * O + o];
        const Real z = c.z[r * H + k];
        c.dzp[r * H + k] = acc * (Real(1) - z * z);
    }
    __syncthreads();
    for (int e = tid; e < H * H + H; e += NT) {
        Real acc = 0;
        if (e < H * H) {
            const int k = e / H, j = e - k * H;
            for (int r = 0; r < nr; ++r) acc += c.cur[sidx(s, s.L - 1, s.T - 1, r) * H + k] * c.dzp[r * H + j];
            wp[s.nl_w + e] = acc;
        } else {
            for (int r = 0; r < nr; ++r) acc += c.dzp[r * H + (e - H * H)];
            wp[s.nl_b + (e - H * H)] = acc;
        }
    }
    for (int e = tid; e < nr * H; e += NT) {
        const int r = e / H, k = e - r * H;
        Real acc = 0;
        for (int j = 0; j < H; ++j) acc += c.dzp[r * H + j] * W[s.nl_w + static_cast<long long>(k) * H + j];
        c.dcur[sidx(s, s.L - 1, s.T - 1, r) * H + k] = acc;
    }
    __syncthreads();
    for (int l = s.L - 1; l >= 0; --l) {
        const int K = s.layer_in[l], d = s.dil[l];
        const Real* Wi = W + s.w_in[l];
        const Real* Wr = W + s.w_rec[l];
        // block skip: its source receives the layer output's adjoint too
        if (s.res_src[l] >= 0)
            for (int e = tid; e < s.T * nr * H; e += NT) {
                const int t = e / (nr * H), rj = e - t * nr * H, r = rj / H, j = rj - r * H;
                c.dcur[sidx(s, s.res_src[l], t, r) * H + j] += c.dcur[sidx(s, l, t, r) * H + j];
            }
        for (int e = tid; e < 2 * s.T * kSeqRows * H; e += NT) c.dhr[e] = 0;  // dhr and dcr are contiguous
        __syncthreads();
        for (int t = s.T - 1; t >= 0; --t) {
            // cell adjoints (Mul / Tanh / Logistic / Add adjoints of lstm_cell)
            for (int e = tid; e < nr * H; e += NT) {
                const int r = e / H, j = e - r * H;
                const long long q = sidx(s, l, t, r);
                const Real* gt = c.gates + q * G;
                const Real i = gt[j], f = gt[H + j], g = gt[2 * H + j], o = gt[3 * H + j];
                const Real tc = Math<Real>::tanh(c.cst[q * H + j]);
                const long long rt = (static_cast<long long>(t) * kSeqRows + r) * H + j;
                const Real dh = c.dcur[q * H + j] + c.dhr[rt];
                const Real dc = c.dcr[rt] + dh * o * (Real(1) - tc * tc);
                Real df = 0;
                if (t >= d) {
                    df = dc * c.cst[sidx(s, l, t - d, r) * H + j];
                    c.dcr[(static_cast<long long>(t - d) * kSeqRows + r) * H + j] += dc * f;
                }
                Real* dp = c.dpre + (static_cast<long long>(t) * kSeqRows + r) * G;
                dp[j] = dc * g * i * (Real(1) - i);
                dp[H + j] = df * f * (Real(1) - f);
                dp[2 * H + j] = dc * i * (Real(1) - g * g);
                dp[3 * H + j] = dh * tc * o * (Real(1) - o);
            }
            __syncthreads();
            // input adjoint of step t and the recurrent adjoint of h_{t-d}
            const int kmax = K > H ? K : H;
            for (int e = tid; e < nr * kmax; e += NT) {
                const int r = e / kmax, k = e - r * kmax;
                const Real* dp = c.dpre + (static_cast<long long>(t) * kSeqRows + r) * G;
                if (k < K) {
                    Real acc = 0;
                    for (int j = 0; j < G; ++j) acc += dp[j] * Wi[static_cast<long long>(k) * G + j];
                    c.din[(static_cast<long long>(t) * kSeqRows + r) * s.in_max + k] = acc;
                }
                if (t >= d && k < H) {
                    Real acc = 0;
                    for (int j = 0; j < G; ++j) acc += dp[j] * Wr[static_cast<long long>(k) * G + j];
                    c.dhr[(static_cast<long long>(t - d) * kSeqRows + r) * H + k] += acc;
                }
            }
            __syncthreads();
        }
        // this layer's weight gradients: x^T dpre, h_{t-d}^T dpre, 1^T dpre (reverse-step order)
        for (long long e = tid; e < static_cast<long long>(K + H + 1) * G; e += NT) {
            const int k = static_cast<int>(e / G), j = static_cast<int>(e - static_cast<long long>(k) * G);
            Real acc = 0;
            for (int t = s.T - 1; t >= 0; --t)
                for (int r = 0; r < nr; ++r) {
                    const Real a = c.dpre[(static_cast<long long>(t) * kSeqRows + r) * G + j];
                    if (k < K) acc += seq_in(s, c, X, l, t, r, b0)[k] * a;
                    else if (k < K + H) {
                        if (t >= d) acc += c.hraw[sidx(s, l, t - d, r) * H + (k - K)] * a;
                    } else {
                        acc += a;
                    }
                }
            if (k < K) wp[s.w_in[l] + static_cast<long long>(k) * G + j] = acc;
            else if (k < K + H) wp[s.w_rec[l] + static_cast<long long>(k - K) * G + j] = acc;
            else wp[s.bias[l] + j] = acc;
        }
        // the input adjoint goes to the previous layer's output or to the sequence
        for (int e = tid; e < s.T * nr * K; e += NT) {
            const int t = e / (nr * K), rk = e - t * nr * K, r = rk / K, k = rk - r * K;
            const Real v = c.din[(static_cast<long long>(t) * kSeqRows + r) * s.in_max + k];
            if (l > 0) c.dcur[sidx(s, l - 1, t, r) * H + k] += v;
            else if (xbar) xbar[(static_cast<long long>(t) * s.B + b0 + r) * s.in0 + k] = v;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------
// Inference forward_stack at speed: k_seq_fwd_fast.  A CTA owns kSeqFR batch rows for the
// whole sequence; per layer its input (W_in), recurrent (W_rec) and bias weights sit in
// shared memory, and each step is two barrier-separated phases:
//   gates: kSeqSplit threads per gate column (4H <= 256) each accumulate the column for a
//          quarter of the kSeqFR rows in registers -- x_t W_in over the staged layer input, then h_{t-d}
//          W_rec from the recurrent ring -- one shared-memory weight load feeds kSeqFR/2
//          FMAs, the row values are broadcast reads ([k][row] layout, 16-byte vectors)
//   cell:  thread per (row, unit): c = f c_{t-d} + i g, h = o tanh(c) into the (h, c) rings
//          (depth d: slot t mod d holds step t), the layer output to the CTA's private
//          sequence buffer (L2 resident) with the block skip added, and the next step's
//          input staged.
// Same summation order as k_seq_forward (x W_in, + h W_rec, + bias).  Used when no adjoint
// is requested and the layer weights fit in shared memory (host: seq_fast_smem).
constexpr int kSeqFR = 16;
constexpr int kSeqSplit = 4;  // threads per gate column in the gate phase

// Saved activations of the fast path for its adjoint (k_seq_bwd_fast), per CTA of kSeqFR rows:
// gates [L][T][R][4H] (post-activation i f g o), c / h (the cell state and the recurrent
// output) / cur (the layer output incl. the block skip) [L][T][R][H]
template <typename Real>
struct SeqSave {
    Real *gates, *cst, *hraw, *cur;
    __host__ __device__ static long long per_cta(const SeqLayout& s) {
        return static_cast<long long>(s.L) * s.T * kSeqFR * (4LL * s.H + 3LL * s.H);
    }
    __device__ static SeqSave at(Real* base, const SeqLayout& s) {
        const long long LTR = static_cast<long long>(s.L) * s.T * kSeqFR;
        SeqSave v;
        Real* p = base + static_cast<long long>(blockIdx.x) * per_cta(s);
        v.gates = p, p += LTR * 4 * s.H;
        v.cst = p, p += LTR * s.H;
        v.hraw = p, p += LTR * s.H;
        v.cur = p;
        return v;
    }
};

// SAVE: also keep every step's activations (SeqSave in seqbuf) for the adjoint kernel
template <typename Real, bool SAVE>
__global__ void __launch_bounds__(1024) k_seq_fwd_fast(SeqLayout s, const Real* __restrict__ W,
                                                       const Real* __restrict__ X, Real* __restrict__ seqbuf,
                                                       double* out) {
    using M = Math<Real>;
    constexpr int R = kSeqFR;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int b0 = blockIdx.x * R, nr = min(R, s.B - b0);
    const int tid = threadIdx.x, NT = blockDim.x, H = s.H, G = 4 * H, T = s.T;
    int dmax = 1;
    for (int l = 0; l < s.L; ++l) dmax = max(dmax, s.dil[l]);
    // shared layout: weights [in_max + H + 1][G] | xs [2][in_max][R] | hring, cring [dmax][H][R] | gates [R][G]
    Real* Ws = reinterpret_cast<Real*>(smem_raw);
    Real* xs = Ws + static_cast<size_t>(s.in_max + H + 1) * G;
    Real* hr = xs + 2 * static_cast<size_t>(s.in_max) * R;
    Real* cr = hr + static_cast<size_t>(dmax) * H * R;
    Real* gs = cr + static_cast<size_t>(dmax) * H * R;
    // per-CTA sequence buffers: two layer outputs in flight + the current block's input
    // (SAVE: every layer's output kept, the block input read in place)
    const size_t TRH = static_cast<size_t>(T) * R * H;
    SeqSave<Real> sv{};
    if constexpr (SAVE) sv = SeqSave<Real>::at(seqbuf, s);
    Real* cur0 = SAVE ? sv.cur : seqbuf + static_cast<size_t>(blockIdx.x) * 3 * TRH;  // layer outputs
    Real* bin = SAVE ? nullptr : cur0 + 2 * TRH;
    for (int l = 0; l < s.L; ++l) {
        const int K = s.layer_in[l], d = s.dil[l];
        const Real* Xin = l == 0 ? nullptr : cur0 + (SAVE ? (l - 1) : ((l - 1) & 1)) * TRH;
        Real* Y = cur0 + (SAVE ? l : (l & 1)) * TRH;
        if constexpr (SAVE) bin = s.res_src[l] >= 0 ? cur0 + s.res_src[l] * TRH : nullptr;
        __syncthreads();  // previous layer done with the weights / its output complete
        const Real* Wi = W + s.w_in[l];
        const Real* Wr = W + s.w_rec[l];
        const Real* Bi = W + s.bias[l];
        for (int e = tid; e < K * G; e += NT) Ws[e] = Wi[e];
        for (int e = tid; e < H * G; e += NT) Ws[K * G + e] = Wr[e];
        for (int e = tid; e < G; e += NT) Ws[(K + H) * G + e] = Bi[e];
        for (int e = tid; e < 2 * d * H * R; e += NT) hr[e] = Real(0);  // h and c rings are contiguous
        // x_t as [k][row] in buffer t & 1, copied asynchronously one step ahead (rows past
        // the batch stay zero: the buffers are cleared per layer)
        auto stage_x = [&](int t) {
            Real* dst = xs + static_cast<size_t>(t & 1) * s.in_max * R;
            for (int e = tid; e < K * nr; e += NT) {
                const int k = e / nr, r = e - k * nr;
                const Real* src = l == 0 ? X + (static_cast<size_t>(t) * s.B + b0 + r) * s.in0 + k
                                         : Xin + (static_cast<size_t>(t) * R + r) * H + k;
                cp_async_elem(dst + k * R + r, src);
            }
            cp_async_commit();
        };
        for (int e = tid; e < 2 * s.in_max * R; e += NT) xs[e] = Real(0);
        __syncthreads();
        stage_x(0);
        cp_async_wait_all();
        __syncthreads();
        for (int t = 0; t < T; ++t) {
            const Real* xcur = xs + static_cast<size_t>(t & 1) * s.in_max * R;
            if (t + 1 < T) stage_x(t + 1);  // lands during this step's two phases
            // ---- gates ----
            // kSeqSplit threads per gate column, each over R / kSeqSplit rows: more warps to
            // hide the shared-memory latency of the k loops (one CTA per SM holds the weights)
            const int Gp = (G + 31) & ~31;
            const int col = tid % Gp, half = tid / Gp;
            if (col < G && half < kSeqSplit) {
                constexpr int RH = R / kSeqSplit;
                Real acc[RH], a2[RH];
#pragma unroll
                for (int r = 0; r < RH; ++r) acc[r] = 0, a2[r] = 0;
                const Real* wcol = Ws + col;
                const Real* xh = xcur + half * RH;
#pragma unroll 4
                for (int k = 0; k < K; ++k) {  // unrolled: the next k's loads issue under these FMAs
                    const Real w = wcol[k * G];
                    const Real* xk = xh + k * R;
#pragma unroll
                    for (int r = 0; r < RH; ++r) acc[r] += xk[r] * w;
                }
                if (t >= d) {
                    const Real* hp = hr + static_cast<size_t>((t - d) % d) * H * R + half * RH;
                    const Real* wrc = Ws + K * G + col;
#pragma unroll 4
                    for (int k = 0; k < H; ++k) {
                        const Real w = wrc[k * G];
                        const Real* hk = hp + k * R;
#pragma unroll
                        for (int r = 0; r < RH; ++r) a2[r] += hk[r] * w;
                    }
                }
                const Real b = Ws[(K + H) * G + col];
                const bool is_g = col >= 2 * H && col < 3 * H;
#pragma unroll
                for (int r = 0; r < RH; ++r) {
                    const Real v = (t >= d ? acc[r] + a2[r] : acc[r]) + b;
                    const Real a = is_g ? M::tanh(v) : M::logistic(v);
                    gs[(half * RH + r) * G + col] = a;
                    if constexpr (SAVE)
                        if (half * RH + r < nr) sv.gates[((static_cast<size_t>(l) * T + t) * R + half * RH + r) * G + col] = a;
                }
            }
            __syncthreads();
            // ---- cell, outputs, next input ----
            const int slot = t % d;
            for (int e = tid; e < nr * H; e += NT) {
                const int r = e / H, j = e - r * H;
                const Real* gt = gs + r * G;
                const Real i = gt[j], f = gt[H + j], g = gt[2 * H + j], o = gt[3 * H + j];
                Real* cpos = cr + (static_cast<size_t>(slot) * H + j) * R + r;  // also c_{t-d} (same slot)
                const Real cv = (t >= d ? f * *cpos : Real(0)) + i * g;
                const Real h = o * M::tanh(cv);
                *cpos = cv;
                hr[(static_cast<size_t>(slot) * H + j) * R + r] = h;
                const size_t q = (static_cast<size_t>(t) * R + r) * H + j;
                if constexpr (SAVE) {
                    sv.cst[l * TRH + q] = cv;
                    sv.hraw[l * TRH + q] = h;
                }
                if (s.res_src[l] >= 0) Y[q] = h + bin[q];
                else Y[q] = h;
            }
            cp_async_wait_all();
            __syncthreads();
        }
        // the block skip of a later layer m adds the output of layer res_src[m] (the previous
        // block's last layer, i.e. the block input): keep it when this layer is that source
        if constexpr (!SAVE) {
            bool is_src = false;
            for (int m = l + 1; m < s.L; ++m) is_src |= s.res_src[m] == l;
            if (is_src)
                for (size_t e = tid; e < static_cast<size_t>(T) * R * H; e += NT) bin[e] = Y[e];
        }
    }
    __syncthreads();
    // head on the last step (network.hpp:207-209)
    const Real* last = cur0 + (SAVE ? s.L - 1 : ((s.L - 1) & 1)) * TRH + static_cast<size_t>(T - 1) * R * H;
    Real* z = gs;  // [R][H]
    for (int e = tid; e < nr * H; e += NT) {
        const int r = e / H, j = e - r * H;
        Real acc = 0;
        for (int k = 0; k < H; ++k) acc += last[r * H + k] * W[s.nl_w + static_cast<long long>(k) * H + j];
        z[r * H + j] = M::tanh(acc + W[s.nl_b + j]);
    }
    __syncthreads();
    for (int e = tid; e < nr * s.O; e += NT) {
        const int r = e / s.O, o = e - r * s.O;
        Real acc = 0;
        for (int k = 0; k < H; ++k) acc += z[r * H + k] * W[s.out_w + static_cast<long long>(k) * s.O + o];
        out[static_cast<long long>(b0 + r) * s.O + o] = static_cast<double>(acc + W[s.out_b + o]);
    }
}

// ---------------------------------------------------------------------------------------
// Adjoint of the fast forward (k_seq_fwd_fast<SAVE>): k_seq_bwd_fast, a CTA per kSeqFR rows,
// the reverse sweep of k_seq_backward's graph with a layer's W_in / W_rec in shared memory.
// Per step (reverse): cell adjoints (thread per (row, unit)) into the pre-activation adjoints
// dpre [R][4H] and the (h, c) recurrent-adjoint rings; then, per thread, the input and
// recurrent adjoints (thread per (input feature, row quarter): a dot over 4H with the
// feature's weight row) and its share of the weight gradients, accumulated in registers over
// the layer's steps (thread-owned (feature, gate column) entries; reverse-step, row-ascending
// order as k_seq_backward).  dcur [L][T][R][H] (the adjoint of every layer output) lives in a
// CTA-private global buffer; per-CTA weight-gradient partials are reduced by k_seq_reduce.
constexpr int kSeqBwdThreads = 1024;
constexpr int kSeqBwdAcc = 24;  // weight-gradient entries per thread ((in_max + H + 1) * 4H <= 24 * 1024)

template <typename Real>
__global__ void __launch_bounds__(kSeqBwdThreads) k_seq_bwd_fast(SeqLayout s, const Real* __restrict__ W,
                                                                  const Real* __restrict__ X, Real* __restrict__ seqbuf,
                                                                  Real* __restrict__ dcurbuf,
                                                                  const Real* __restrict__ obar, Real* __restrict__ wpart,
                                                                  Real* __restrict__ xbar) {
    using M = Math<Real>;
    constexpr int R = kSeqFR;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int b0 = blockIdx.x * R, nr = min(R, s.B - b0);
    const int tid = threadIdx.x, NT = blockDim.x, H = s.H, G = 4 * H, T = s.T, O = s.O;
    int dmax = 1;
    for (int l = 0; l < s.L; ++l) dmax = max(dmax, s.dil[l]);
    // shared: Wi [in_max][G] | Wr [H][G] | dpre [R][G] | dh, dc rings [dmax][H][R] | xs, hs [in_max][R], [H][R]
    Real* Wi = reinterpret_cast<Real*>(smem_raw);
    Real* Wr = Wi + static_cast<size_t>(s.in_max) * G;
    Real* dp = Wr + static_cast<size_t>(H) * G;
    Real* dhr = dp + static_cast<size_t>(R) * G;
    Real* dcr = dhr + static_cast<size_t>(dmax) * H * R;
    Real* xs = dcr + static_cast<size_t>(dmax) * H * R;
    Real* hs = xs + static_cast<size_t>(s.in_max) * R;
    const SeqSave<Real> sv = SeqSave<Real>::at(seqbuf, s);
    const size_t TRH = static_cast<size_t>(T) * R * H;
    Real* dcur = dcurbuf + static_cast<size_t>(blockIdx.x) * s.L * TRH;
    Real* wp = wpart + static_cast<long long>(blockIdx.x) * s.P;
    for (size_t e = tid; e < static_cast<size_t>(s.L) * TRH; e += NT) dcur[e] = Real(0);
    // ---- head: out = z out_w + out_b, z = tanh(last nl_w + nl_b) (z recomputed) ----
    const Real* last = sv.cur + static_cast<size_t>(s.L - 1) * TRH + static_cast<size_t>(T - 1) * R * H;
    Real* z = dp;            // [R][H]
    Real* dzp = dp + R * H;  // [R][H]
    for (int e = tid; e < nr * H; e += NT) {
        const int r = e / H, j = e - r * H;
        Real acc = 0;
        for (int k = 0; k < H; ++k) acc += last[r * H + k] * W[s.nl_w + static_cast<long long>(k) * H + j];
        z[r * H + j] = M::tanh(acc + W[s.nl_b + j]);
    }
    __syncthreads();
    const Real* ob = obar + static_cast<long long>(b0) * O;
    for (int e = tid; e < H * O + O; e += NT) {
        Real acc = 0;
        if (e < H * O) {
            const int k = e / O, o = e - k * O;
            for (int r = 0; r < nr; ++r) acc += z[r * H + k] * ob[r * O + o];
            wp[s.out_w + e] = acc;
        } else {
            for (int r = 0; r < nr; ++r) acc += ob[r * O + (e - H * O)];
            wp[s.out_b + (e - H * O)] = acc;
        }
    }
    for (int e = tid; e < nr * H; e += NT) {
        const int r = e / H, k = e - r * H;
        Real acc = 0;
        for (int o = 0; o < O; ++o) acc += ob[r * O + o] * W[s.out_w + static_cast<long long>(k) * O + o];
        const Real zz = z[r * H + k];
        dzp[r * H + k] = acc * (Real(1) - zz * zz);
    }
    __syncthreads();
    for (int e = tid; e < H * H + H; e += NT) {
        Real acc = 0;
        if (e < H * H) {
            const int k = e / H, j = e - k * H;
            for (int r = 0; r < nr; ++r) acc += last[r * H + k] * dzp[r * H + j];
            wp[s.nl_w + e] = acc;
        } else {
            for (int r = 0; r < nr; ++r) acc += dzp[r * H + (e - H * H)];
            wp[s.nl_b + (e - H * H)] = acc;
        }
    }
    Real* dlast = dcur + static_cast<size_t>(s.L - 1) * TRH + static_cast<size_t>(T - 1) * R * H;
    for (int e = tid; e < nr * H; e += NT) {
        const int r = e / H, k = e - r * H;
        Real acc = 0;
        for (int j = 0; j < H; ++j) acc += dzp[r * H + j] * W[s.nl_w + static_cast<long long>(k) * H + j];
        dlast[r * H + k] = acc;
    }
    __syncthreads();
    // ---- layers in reverse ----
    for (int l = s.L - 1; l >= 0; --l) {
        const int K = s.layer_in[l], d = s.dil[l];
        Real* dcl = dcur + static_cast<size_t>(l) * TRH;
        // block skip: its source receives the layer output's adjoint too
        if (s.res_src[l] >= 0) {
            Real* dsrc = dcur + static_cast<size_t>(s.res_src[l]) * TRH;
            for (size_t e = tid; e < TRH; e += NT) dsrc[e] += dcl[e];
        }
        for (int e = tid; e < K * G; e += NT) Wi[e] = W[s.w_in[l] + e];
        for (int e = tid; e < H * G; e += NT) Wr[e] = W[s.w_rec[l] + e];
        for (int e = tid; e < 2 * d * H * R; e += NT) dhr[e] = Real(0);  // dh and dc rings are contiguous
        for (int e = tid; e < (s.in_max + H) * R; e += NT) xs[e] = Real(0);
        // weight-gradient accumulators: entry q = tid + i * NT of the layer's (K + H + 1) x G block
        // (rows: input features, recurrent features, bias)
        const int nq = (K + H + 1) * G;
        Real acc[kSeqBwdAcc];
#pragma unroll
        for (int i = 0; i < kSeqBwdAcc; ++i) acc[i] = 0;
        const Real* Xin = l == 0 ? nullptr : sv.cur + static_cast<size_t>(l - 1) * TRH;
        __syncthreads();
        for (int t = T - 1; t >= 0; --t) {
            const int slot = t % d;
            // ---- phase 1: cell adjoints (Mul / Tanh / Logistic / Add adjoints of lstm_cell) and
            // the step's layer input / recurrent input staged for the weight gradients ----
            for (int e = tid; e < nr * H; e += NT) {
                const int r = e / H, j = e - r * H;
                const size_t q = (static_cast<size_t>(l) * T + t) * R + r;
                const Real* gt = sv.gates + q * G;
                const Real i = gt[j], f = gt[H + j], g = gt[2 * H + j], o = gt[3 * H + j];
                const Real tc = M::tanh(sv.cst[q * H + j]);
                Real* dhp = dhr + (static_cast<size_t>(slot) * H + j) * R + r;
                Real* dcp = dcr + (static_cast<size_t>(slot) * H + j) * R + r;
                const Real dh = dcl[(static_cast<size_t>(t) * R + r) * H + j] + *dhp;
                const Real dc = *dcp + dh * o * (Real(1) - tc * tc);
                Real df = 0;
                if (t >= d) {
                    df = dc * sv.cst[(q - static_cast<size_t>(d) * R) * H + j];
                    *dcp = dc * f;  // the adjoint of c_{t-d} (read at step t - d, same slot)
                } else {
                    *dcp = Real(0);
                }
                Real* dr = dp + r * G;
                dr[j] = dc * g * i * (Real(1) - i);
                dr[H + j] = df * f * (Real(1) - f);
                dr[2 * H + j] = dc * i * (Real(1) - g * g);
                dr[3 * H + j] = dh * tc * o * (Real(1) - o);
            }
            for (int e = tid; e < K * nr; e += NT) {
                const int k = e / nr, r = e - k * nr;
                xs[k * R + r] = l == 0 ? X[(static_cast<size_t>(t) * s.B + b0 + r) * s.in0 + k]
                                       : Xin[(static_cast<size_t>(t) * R + r) * H + k];
            }
            for (int e = tid; e < H * nr; e += NT) {
                const int k = e / nr, r = e - k * nr;
                hs[k * R + r] = t >= d ? sv.hraw[(static_cast<size_t>(l) * T + t - d) * R * H + r * H + k] : Real(0);
            }
            __syncthreads();
            // ---- phase 2: input adjoint of step t, recurrent adjoint of h_{t-d}, weight grads ----
            const int kmax = K > H ? K : H;
            for (int e = tid; e < kmax * nr; e += NT) {
                const int k = e / nr, r = e - k * nr;
                const Real* dr = dp + r * G;
                if (k < K) {
                    Real a = 0;
                    const Real* wrow = Wi + k * G;
                    for (int j = 0; j < G; ++j) a += dr[j] * wrow[j];
                    if (l > 0) dcur[static_cast<size_t>(l - 1) * TRH + (static_cast<size_t>(t) * R + r) * H + k] += a;
                    else if (xbar) xbar[(static_cast<size_t>(t) * s.B + b0 + r) * s.in0 + k] = a;
                }
                if (k < H) {
                    Real a = 0;
                    if (t >= d) {
                        const Real* wrow = Wr + k * G;
                        for (int j = 0; j < G; ++j) a += dr[j] * wrow[j];
                    }
                    dhr[(static_cast<size_t>(slot) * H + k) * R + r] = a;  // for step t - d (same slot)
                }
            }
#pragma unroll
            for (int i = 0; i < kSeqBwdAcc; ++i) {
                const int q = tid + i * NT;
                if (q < nq) {
                    const int k = q / G, j = q - k * G;
                    Real a = acc[i];
                    if (k < K) {
                        for (int r = 0; r < nr; ++r) a += xs[k * R + r] * dp[r * G + j];
                    } else if (k < K + H) {
                        if (t >= d)
                            for (int r = 0; r < nr; ++r) a += hs[(k - K) * R + r] * dp[r * G + j];
                    } else {
                        for (int r = 0; r < nr; ++r) a += dp[r * G + j];
                    }
                    acc[i] = a;
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int i = 0; i < kSeqBwdAcc; ++i) {
            const int q = tid + i * NT;
            if (q < nq) {
                const int k = q / G, j = q - k * G;
                if (k < K) wp[s.w_in[l] + static_cast<long long>(k) * G + j] = acc[i];
                else if (k < K + H) wp[s.w_rec[l] + static_cast<long long>(k - K) * G + j] = acc[i];
                else wp[s.bias[l] + j] = acc[i];
            }
        }
        __syncthreads();
    }
}

// weights_bar[p] = sum over CTAs b (in order) of wpart[b][p]
template <typename Real>
__global__ void k_seq_reduce(const Real* __restrict__ wpart, int nblk, long long P, double* out) {
    const long long p = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= P) return;
    double acc = 0;
    for (int b = 0; b < nblk; ++b) acc += static_cast<double>(wpart[static_cast<long long>(b) * P + p]);
    out[p] = acc;
}

}  // namespace esrnn_dev
