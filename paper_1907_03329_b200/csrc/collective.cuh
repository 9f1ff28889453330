// In-process group collective: the step's shared-gradient all-reduce fused with the
// post-reduction finalisation (K3' of the sharded step), for W ranks that live in ONE
// process -- W trainers driven from W host threads, on one GPU or on several GPUs with
// peer access (NVLink / NVSwitch: the slots are plain device memory every rank can load).
//
// Reference: the sharded step of SURVEY §8(e) -- the reference itself is single-process
// (trainer.hpp:602-655 apply_updates over the whole batch); the decomposition is
// "partial sums of the global-M-scaled loss / gradients, summed over ranks" (tests/
// test_sharding.py proves it on the oracle).
//
// One launch per step per rank, G CTAs each:
//   1. copy this rank's gbuf (Real[P_pad]) and gtail (double[4]) into its slot of the
//      current parity (slots are double-buffered by call parity, so a rank that runs ahead
//      into call n+1 never overwrites data a slower rank still reads for call n: reaching
//      call n+2 needs every rank past call n+1's barrier, i.e. done reading call n);
//   2. the last CTA to finish its copy publishes done[rank] = seq (release, system scope);
//      every CTA waits until all W ranks published seq (acquire), with a timeout that raises
//      kErrPeer instead of hanging when a rank never arrives;
//   3. each CTA sums its chunk over the W slots IN RANK ORDER (the same bits on every rank)
//      into gbuf, with the squared norm of the summed gradients;
//   4. the last CTA (ticket) folds the CTA norm parts in order and the summed tail, and
//      finalises the step scalars (clip scale, Adam step / bias corrections, step loss,
//      any-rank error flag) exactly like k_finalize does after an NCCL all-reduce.
// Deterministic: fixed summation orders everywhere, no float atomics.
#pragma once
#include "finish.cuh"

namespace esrnn_dev {

struct GroupDev {
    unsigned char* slots;      // [2 parities][W ranks][stride bytes]: gtail (4 doubles) | gbuf (Real[P_pad])
    unsigned long long* done;  // [W] last call each rank published
    unsigned* ctr;             // [W][2] CTA arrival ticket (phase 1), finalise ticket (phase 4)
    long long stride;          // bytes per rank slot (multiple of 256)
    int W, rank;
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

constexpr long long kGroupTimeoutNs = 60LL * 1000 * 1000 * 1000;  // a rank that never arrives

template <typename Real>
__global__ void __launch_bounds__(256) k_group_reduce(StateDev<Real> st, PlanDev pl, NetLayout lay, int s, int advance,
                                                      GroupDev g) {
    __shared__ double red[32];
    __shared__ bool last;
    const int tid = threadIdx.x, G = gridDim.x, c = blockIdx.x;
    SPAN_BEGIN(st, s, kSpanReduce);
    const long long n = lay.P_pad;
    const unsigned long long seq = static_cast<unsigned long long>(*st.coll_seq) + 1;
    const int par = static_cast<int>(seq & 1);
    auto slot = [&](int r) { return g.slots + (static_cast<long long>(par) * g.W + r) * g.stride; };
    const long long chunk = ((n + G - 1) / G + 3) & ~3LL;
    const long long i0 = min(n, c * chunk), i1 = min(n, i0 + chunk);
    // 1. this rank's partials into its slot
    {
        double* tail = reinterpret_cast<double*>(slot(g.rank));
        Real* mine = reinterpret_cast<Real*>(tail + 4);
        for (long long i = i0 + tid; i < i1; i += blockDim.x) mine[i] = st.gbuf[i];
        if (c == 0 && tid < 4) tail[tid] = st.gtail[tid];
    }
    __threadfence_system();
    __syncthreads();
    // 2. publish (last CTA of this rank) and wait for every rank
    if (tid == 0) {
        const unsigned t = atomicAdd(g.ctr + 2 * g.rank, 1u);
        if (t == static_cast<unsigned>(G - 1)) {
            g.ctr[2 * g.rank] = 0;
            __threadfence_system();
            st_release_sys(g.done + g.rank, seq);
        }
    }
    if (tid < g.W) {
        const long long t0 = gtimer();
        while (ld_acquire_sys(g.done + tid) < seq) {
            if (gtimer() - t0 > kGroupTimeoutNs) {
                flag_error(st.err, kErrPeer, tid);
                break;
            }
            __nanosleep(64);
        }
    }
    __syncthreads();
    // 3. rank-ordered sums of this CTA's chunk; squared norm of the summed gradients
    double sq = 0.0;
    for (long long i = i0 + tid; i < i1; i += blockDim.x) {
        Real v = 0;
        for (int r = 0; r < g.W; ++r) v += __ldcg(reinterpret_cast<const Real*>(reinterpret_cast<const double*>(slot(r)) + 4) + i);
        st.gbuf[i] = v;
        sq += static_cast<double>(v) * v;
    }
    if (c == 0 && tid < 4) {
        double v = 0.0;
        for (int r = 0; r < g.W; ++r) v += __ldcg(reinterpret_cast<const double*>(slot(r)) + tid);
        st.gtail[tid] = v;
    }
    const double tot = block_sum(sq, red);
    // 4. last CTA finalises
    if (tid == 0) {
        st.red_sq_part[c] = tot;
        __threadfence();
        last = atomicAdd(g.ctr + 2 * g.rank + 1, 1u) == static_cast<unsigned>(G - 1);
    }
    __syncthreads();
    SPAN_END(st, s, kSpanReduce);
    if (!last) return;
    __threadfence();
    double all = 0.0;
    for (int b = tid; b < G; b += blockDim.x) all += __ldcg(st.red_sq_part + b);
    all = block_sum(all, red);
    if (tid != 0) return;
    g.ctr[2 * g.rank + 1] = 0;
    const double es = st.attach ? __ldcg(st.gtail + 0) : 0.0;
    const bool err_any = __ldcg(st.gtail + 2) != 0.0 || st.err[0] == kErrPeer;
    finalize_scalars(st, pl, s, all + es, __ldcg(st.gtail + 1), advance != 0, err_any);
    *st.coll_seq = static_cast<long long>(seq);
    SPAN_END(st, s, kSpanReduce);
}

}  // namespace esrnn_dev
