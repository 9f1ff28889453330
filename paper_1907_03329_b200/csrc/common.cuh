// Shared device-side types and helpers of the ES-RNN B200 kernels.
//
// Layout in HBM: series values time-major y[t][N] (coalesced across series), per-series
// parameters and Adam moments SoA [(2+S)][N], scan state [t][slot], and the shared
// network parameters in a compact "live" vector that drops the structurally-dead
// forget-gate columns and recurrent matrices (their gradients are exactly zero at
// sequence length 1).  Every weight matrix is stored transposed, [out][in]
// with an odd row stride, so both the forward product (threads over outputs) and the
// input adjoint (threads over inputs) read shared memory without bank conflicts, and
// the whole vector moves into shared memory with one TMA bulk copy.
#pragma once
#include <cstdint>
#include <cfloat>
#include <climits>
#include <type_traits>

#include "devmath.cuh"

namespace esrnn_dev {

constexpr int kMaxLayers = 16;
constexpr int kMaxMats = kMaxLayers + 2;

// One weight matrix of the K3 gradient contraction G[q][k] = sum_b A[b][q] * U[b][k]
// (A, U: columns of the row store), written into W^T at cw (row stride ldk) and its bias
// gradient sum_b A[b][q] at cb.
struct MatDesc {
    int a_off, Q, u_off, K, ldk, pad_;
    long long cw, cb;
};

struct NetLayout {
    int L, nb, H, O, I, S, in0, T;
    int ldx, ldh, ldg, ldo;      // padded (multiple of 4) row strides: x, hidden, 3H gates, horizon
    int ldkh;                    // row stride of the transposed head matrices (8 * odd >= H)
    int layer_in[kMaxLayers];
    int ldk[kMaxLayers];         // row stride of layer l's transposed input matrix (8 * odd >= in_l)
    int res_src[kMaxLayers];     // >=0: layer output added as residual after this layer
    int block_first[kMaxLayers]; // 1 if layer is the first of a block b>0 (adjoint joins the residual)
    int block_last[kMaxLayers];  // 1 if layer is the last of a block b>0 (residual added here)
    long long cw[kMaxLayers], cb[kMaxLayers];  // WT_l [3H][ldk_l], bias_l [3H]
    long long c_nlw, c_nlb, c_outw, c_outb;     // nl_w^T [H][ldkh], nl_b [H], out_w^T [O][ldkh], out_b [O]
    long long P_live, P_pad;
    // per-window row store written by K2 for K3 (Real units, offsets multiples of 4):
    // x | h_0..h_{L-1} | z | pre_bar_0..pre_bar_{L-1} (i, g, o) | z_bar | pred_bar
    int rs_ld, rs_x, rs_z, rs_zb, rs_pb;
    int rs_h[kMaxLayers], rs_pr[kMaxLayers];
    int nmat;                      // L + 2 (layers, nl head, out head)
    int mat_blk0[kMaxMats + 1];    // prefix of K3 GEMM blocks per matrix
    int mat_wblk0[kMaxMats + 1];   // prefix of K3 q-strip blocks (kWq rows of G) per matrix
    int wkp_in0, wkp_h;            // q-strip U boxes: in0 / H rounded up to 4 columns
    MatDesc mats[kMaxMats];
};

// Per-epoch (or single-batch) plan: windows in global batch order, filtered to the
// rows this rank owns, with per-step slot lists and per-slot window CSR.
struct PlanDev {
    const int* w_row;         // local row of each window
    const int* w_anchor;
    const int* w_slot;        // slot within its step
    const int* w_first;       // 1 if the window is its slot's first in batch order
    const int* step_win_off;  // [steps+1]
    const int* step_slot_off; // [steps+1]
    const int* slot_row;      // local row of each slot
    const int* slot_win_off;  // [total_slots+1] into slot_win
    const int* slot_win;      // window index relative to its step's first window
    const int* w_csr;         // step-local CSR position of each window (slot-major order)
    const int* csr_anchor;    // anchor of each CSR entry
    const double* step_M;     // global mask count per step
    const unsigned char* mask;// [window][O] or nullptr (all ones)
};

template <typename Real>
struct StateDev {
    const Real* vals;       // [LEN][N] time-major, local rows (series-parallel readers)
    const Real* vrm;        // [N][ldv] row-major copy (slot-parallel readers: random rows)
    int ldv;
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
    double* contrib;        // [Bcap][cwp] ES adjoint contributions per window, in slot-major
                            // CSR order: [0,I) input seasonalities, [I,I+O) target
                            // seasonalities, [I+O] anchor level, [I+O+1] the anchor.
                            // fp64 in both precisions: the ES adjoint (these contributions
                            // and K3's reverse scan) runs in double, see finish.cuh
    int cwp;                // row stride of contrib (multiple of 4 >= I+O+2)
    Real* rowstore;         // [Bcap][rs_ld] per-window K3 operands (NetLayout rs_*)
    const void* tm_rs;      // two CUtensorMaps (global memory) over the row store for K3's GEMM
                            // staging: [0] box kGq x kGChunk (A columns), [1] kGk x kGChunk (U)
    double* loss_part;      // [tiles]
    Real* gbuf;             // [P_pad] shared-network gradients (the all-reduced buffer, sharded)
    double* gtail;          // [4] step partials reduced with gbuf: per-series sq-norm, loss sum,
                            // error flag (1 if this rank's error word is set), 0
    long long* coll_seq;    // in-process group collective: calls completed (collective.cuh)
    Real* psg;              // [kcap][2+S]
    double* es_sq_part;     // [es blocks]
    double* es_pen_part;    // [es blocks] level-variability penalty, in pinball-sum units (x M)
    double* red_sq_part;    // [weight-gradient tiles]
    Real* gpart;            // [gsplit][tiles][32 lanes][6]: row-part tile partials (large steps)
    unsigned* gtile_ctr;    // [tiles] arrival tickets of a tile's row parts
    int red_tiles;          // K3 weight-gradient output tiles
    int gemm_wide;          // 1: K3 weight gradients by q-strip blocks (finish.cuh dw_wide_block)
    int tile_trigger_early; // 1: K2 releases K3 right after its wait (ESRNN_TILE_TRIGGER_EARLY)
    float* upart;           // [umma tiles][parts][128][64] tensor-core dW partials (fp32, large steps)
    int umma_tiles;         // 128-row matrix slices of the tensor-core dW path
    unsigned int* done_ctr; // [2]
    double* scal;           // [4] scale, bc1, bc2, loss
    long long* net_step;
    double* loss_hist;      // [steps]
    const double* bc;       // [2 * bc_n] Adam bias corrections {1 - 0.9^t, 1 - 0.999^t} by step t,
                            // host std::pow like trainer.hpp:617-620 / :640-641
    long long bc_n;         // table length; both corrections are exactly 1.0 from t = bc_n on
    int* err;               // [4] code, min t, any-rank error (sharded: set from the reduced
                            // flag; Adam is skipped on every rank), 0
    // optional dumps (run_batch): WindowBatch matrices, step-local window order
    Real* d_inputs;
    Real* d_targets;
    Real* d_seas;
    Real* d_levels;
    double tau, lr_net, lr_ps, clip;
    double lvp;             // level-variability penalty weight (0: off, the reference's loss)
    int has_clip, attach;
    long long* dbg_clk;     // optional phase timestamps (ESRNN_DEBUG_CLOCKS), block 0 thread 0
    long long* spans;       // optional in-graph kernel spans [step][kSpanKinds][2]: earliest
                            // CTA start (after its dependency wait), latest CTA end, global
                            // timer ns (esrnn_trainer_profile_kernels(t, 2))
};

// span kinds (the ABI's kernel classes: tile 1, finish 2, adam 4, finalize/group 5)
enum SpanKind { kSpanTile = 0, kSpanFinish = 1, kSpanAdam = 2, kSpanReduce = 3, kSpanKinds = 4 };

// Adam bias corrections of step t (StateDev::bc; exactly 1.0 past the table)
template <typename Real>
__device__ __forceinline__ double bias_c1(const StateDev<Real>& st, long long t) {
    return t < st.bc_n ? st.bc[2 * t] : 1.0;
}
template <typename Real>
__device__ __forceinline__ double bias_c2(const StateDev<Real>& st, long long t) {
    return t < st.bc_n ? st.bc[2 * t + 1] : 1.0;
}

enum ErrCode { kErrNone = 0, kErrTrainLevel = 1, kErrObs = 2, kErrFcLevel = 3, kErrSeas = 4, kErrPeer = 5 };

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

// Three block sums at once, each in block_sum's fixed order (bit-identical results), with
// one barrier pair instead of three.  Valid in thread 0.
__device__ __forceinline__ void block_sum3(double& a, double& b, double& c, double* red /*[3 * 32]*/) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_down_sync(0xffffffffu, a, o);
        b += __shfl_down_sync(0xffffffffu, b, o);
        c += __shfl_down_sync(0xffffffffu, c, o);
    }
    if (lane == 0) red[wid] = a, red[32 + wid] = b, red[64 + wid] = c;
    __syncthreads();
    double ra = 0, rb = 0, rc = 0;
    if (threadIdx.x == 0)
        for (int w = 0; w < nw; ++w) ra += red[w], rb += red[32 + w], rc += red[64 + w];
    __syncthreads();
    a = ra, b = rb, c = rc;
}

// global-timer stamp (ns) into dbg_clk[80 + i], block 0 thread 0 (kernel start/end timeline)
__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define DBG_GT(st, i)                                                               \
    do {                                                                            \
        if ((st).dbg_clk && blockIdx.x == 0 && threadIdx.x == 0) (st).dbg_clk[80 + (i)] = gtimer(); \
    } while (0)

// step-5 kernel spans (ESRNN_DEBUG_CLOCKS): earliest / latest global-timer stamp over all
// blocks in dbg_clk[100 + i] (the host seeds min slots with LLONG_MAX, max slots with 0)
#define DBG_SPAN_MIN(st, step, i)                                                   \
    do {                                                                            \
        if ((st).dbg_clk && (step) == 5 && threadIdx.x == 0)                        \
            atomicMin(reinterpret_cast<long long*>((st).dbg_clk) + 100 + (i), gtimer()); \
    } while (0)
#define DBG_SPAN_MAX(st, step, i)                                                   \
    do {                                                                            \
        if ((st).dbg_clk && (step) == 5 && threadIdx.x == 0)                        \
            atomicMax(reinterpret_cast<long long*>((st).dbg_clk) + 100 + (i), gtimer()); \
    } while (0)

// in-graph kernel spans: one atomic per CTA at its start (after pdl_wait) and at its end
#define SPAN_BEGIN(st, step, kind)                                                              \
    do {                                                                                        \
        if ((st).spans && threadIdx.x == 0)                                                     \
            atomicMin((st).spans + ((long long)(step) * kSpanKinds + (kind)) * 2, gtimer());    \
    } while (0)
#define SPAN_END(st, step, kind)                                                                \
    do {                                                                                        \
        if ((st).spans && threadIdx.x == 0)                                                     \
            atomicMax((st).spans + ((long long)(step) * kSpanKinds + (kind)) * 2 + 1, gtimer()); \
    } while (0)

// step-5 per-tile spans of k_tile (entry, after the dependency wait, end): dbg_clk[128 + 3 tile + j]
constexpr int kDbgTiles = 8192;
#define DBG_TILE(st, step, tile, j)                                                 \
    do {                                                                            \
        if ((st).dbg_clk && (step) == 5 && threadIdx.x == 0 && (tile) < kDbgTiles)  \
            (st).dbg_clk[128 + 3 * (tile) + (j)] = gtimer();                        \
    } while (0)

// step-5 per-block spans of k_grad_finish (after the dependency wait, end): dbg_clk[128 + 3 kDbgTiles + 2 bid + j]
constexpr int kDbgK3 = 4096;
#define DBG_K3(st, step, bid, j)                                                    \
    do {                                                                            \
        if ((st).dbg_clk && (step) == 5 && threadIdx.x == 0 && (bid) < kDbgK3)      \
            (st).dbg_clk[128 + 3 * kDbgTiles + 2 * (bid) + (j)] = gtimer();         \
    } while (0)

#define DBG_CLK(st, i)                                                              \
    do {                                                                            \
        if ((st).dbg_clk && blockIdx.x == 0 && threadIdx.x == 0 && _dbg < 64) (st).dbg_clk[_dbg] = clock64(); \
        ++_dbg;                                                                     \
    } while (0)

// ------------------------------------------------------------------ programmatic dependent launch
// Kernels of a training step are launched with programmatic stream serialisation: each
// kernel lets its dependent launch as soon as every CTA has started (pdl_trigger) and
// waits for its predecessor grid's completion and memory (pdl_wait) before touching data
// the predecessor writes -- or data the predecessor reads that this kernel overwrites.
// Before the wait a kernel may only read epoch-constant data (observations, plan).  Both
// are no-ops for a kernel launched without the attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

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
// 2-D tensor copy global -> shared (TMA), box origin (x = column, y = row) in elements;
// the tensor map lives in global memory (64-byte aligned)
__device__ __forceinline__ void tma2d_g2s(void* dst, const void* tmap, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_addr(dst)),
        "l"(tmap), "r"(x), "r"(y), "r"(smem_addr(bar))
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

// 4-wide shared-memory vector (16 B for fp32, 2 x 16 B for fp64); p must be 4-aligned
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

template <typename Real>
__device__ __forceinline__ V4<Real> ldg4(const Real* p) {
    if constexpr (sizeof(Real) == 4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(p));
        return {v.x, v.y, v.z, v.w};
    } else {
        const double2 a = __ldg(reinterpret_cast<const double2*>(p));
        const double2 b = __ldg(reinterpret_cast<const double2*>(p + 2));
        return {a.x, a.y, b.x, b.y};
    }
}

// Asynchronous global->shared element copies (LDGSTS): every load of a scattered
// column is in flight at once without staging through registers.
template <typename Real>
__device__ __forceinline__ void cp_async_elem(Real* smem, const Real* gmem) {
    if constexpr (sizeof(Real) == 4)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(smem)), "l"(gmem) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(smem)), "l"(gmem) : "memory");
}

// Row stride (elements) for per-thread rows staged with 16-byte copies: a multiple of
// 16 bytes, and an odd number of 16-byte units so a warp's same-column reads spread over
// 8 bank groups.
template <typename Real>
__host__ __device__ __forceinline__ int row_pad(int n) {
    constexpr int e = 16 / static_cast<int>(sizeof(Real));
    int p = (n + e - 1) / e * e;
    if (((p / e) & 1) == 0) p += e;
    return p;
}

// Stage this thread's contiguous row src[0:n) (16-byte aligned) into dst[0:n) with
// 16-byte cp.async copies; caller waits with cp_async_wait_all().
template <typename Real>
__device__ __forceinline__ void stage_row_async(Real* dst, const Real* __restrict__ src, int n) {
    constexpr int e = 16 / static_cast<int>(sizeof(Real));
#pragma unroll 4
    for (int t = 0; t < n; t += e) cp_async16(dst + t, src + t);
}

__host__ __device__ __forceinline__ int log2_ceil(int w) {
    int l = 0;
    while ((1 << l) < w) ++l;
    return l;
}

// fp32 performance mode divides with the SFU reciprocal (MUFU.RCP, <= 1 ulp, flush-to-zero;
// the path's operands are positive levels/seasonalities of O(1e-3..1e6)); fp64 keeps IEEE
// division, as the reference does
__device__ __forceinline__ float rcp_fast(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
template <typename Real>
__device__ __forceinline__ Real fdiv(Real a, Real b) {
    if constexpr (sizeof(Real) == 4) return a * rcp_fast(b);
    else return a / b;
}
// a / b with a reciprocal the caller computed once (rb = rcp(b)); IEEE a / b in fp64
template <typename Real>
__device__ __forceinline__ Real rcp_of(Real b) {
    if constexpr (sizeof(Real) == 4) return rcp_fast(b);
    else return Real(1) / b;
}
template <typename Real>
__device__ __forceinline__ Real fdiv_r(Real a, Real b, Real rb) {
    if constexpr (sizeof(Real) == 4) return a * rb;
    else return a / b;
}

}  // namespace esrnn_dev
