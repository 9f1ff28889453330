// tcgen05 (5th-generation tensor core) building blocks for K3's weight-gradient contraction
// on large steps ("tcgen05 3xTF32 dW GEMM for B >= ~8k, used only if it
// passes parity"):  D[m][n] = sum_b A[b][m] * U[b][n]  over a part of the step's windows,
// with A = the gate (or head) adjoints and U = the layer inputs of the row store, plus a
// ones column in U for the bias gradient.  3xTF32: every fp32 operand is split into a TF32
// high part and a TF32 remainder, and D accumulates hi*hi + hi*lo + lo*hi in fp32 in TMEM
// (relative error ~2^-21 per product, fp32-accumulated: inside the 1e-4 contract).
//
// Shared-memory operand layout: K-major, no swizzle ("interleaved" canonical layout,
// cute make_umma_desc<Major::K> INTERLEAVE: ((8,m),2):((1,SBO),LBO) in 16-byte units): a
// core matrix is 8 rows x 16 bytes (4 TF32 along K), contiguous 128 bytes; core (g, kg) of an
// R-row operand sits at byte (kg * R/8 + g) * 128, so SBO (next 8 rows) = 128 B and LBO (next
// 4 K elements) = R/8 * 128 B.  One MMA (K = 8) reads core columns kg = 2i, 2i+1.
#pragma once
#include <cstdint>

namespace esrnn_dev {

__device__ __forceinline__ uint32_t tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}

// TF32 high part and remainder of x (both as fp32 bit patterns with 13 zero low bits)
__device__ __forceinline__ void tf32_split(float x, uint32_t& hi, uint32_t& lo) {
    hi = tf32_rna(x);
    lo = tf32_rna(x - __uint_as_float(hi));
}

// shared-memory matrix descriptor (tcgen05 "version 1"), no swizzle
__device__ __forceinline__ uint64_t umma_smem_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
    d |= static_cast<uint64_t>(1) << 46;  // version 1 (Blackwell)
    // base offset 0, lbo mode 0, layout type 0 = SWIZZLE_NONE
    return d;
}

// instruction descriptor: kind::tf32, D fp32, A/B tf32 K-major, M x N
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int M, int N) {
    return (1u << 4)                                  // c_format F32
           | (2u << 7)                                // a_format TF32
           | (2u << 10)                               // b_format TF32
           | (0u << 15) | (0u << 16)                  // a, b K-major
           | (static_cast<uint32_t>(N >> 3) << 17)    // n_dim
           | (static_cast<uint32_t>(M >> 4) << 24);   // m_dim
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// arrive on an mbarrier once every previously issued tcgen05.mma of this thread completed
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {  // one full warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {  // one full warp
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 16 consecutive fp32 accumulator columns of this thread's TMEM lane (warp w reads lanes
// 32*(w%4) .. +31; taddr = base | (lane_base << 16) | column)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// ---------------------------------------------------------------------------------------
// One CTA's partial contraction over rows [r0, r0 + nrows):
//   D[m][n] = sum_b A(b, m) * U(b, n),  A(b, m) = a_src[b * ld + m],  U(b, n) = u_src[b * ld + n]
// for m < kUM, n < kUN, with U's column Kv replaced by ones (the bias gradient).  Rows of D at
// m >= Mv and columns n > Kv hold whatever the neighbouring row-store columns contribute and
// are discarded by the caller (a garbage operand row / column only reaches its own D row /
// column), so no operand masking is needed besides the ones column and the tail rows.
//
// Per chunk of kUK rows: 16-byte cp.async copies bring the rows in their natural layout
// (row b: kUM A values, then kUN U values) into a raw ring (coalesced, conflict-free, several
// chunks in flight); a transposing pass writes the K-major core-matrix planes (TF32 high part
// = the fp32 bits truncated as the tensor core reads them, remainder = x - high): thread
// (operand row r, 4-row group kq) gathers 4 rows of one column (lanes over r: conflict-free),
// and a quarter warp fills one core matrix's 128 contiguous bytes.
constexpr int kUmmaMinRows = 4096;  // steps from this many windows take the tensor-core path (measured: 4,096 -4%)
constexpr int kUM = 128;
constexpr int kUN = 64;      // TMEM columns (N tile): Kv + 1 <= 64
constexpr int kUK = 16;      // rows per stage
constexpr int kUStages = 2;  // operand stages (hi + lo planes)
constexpr int kURaw = 3;     // raw copy ring depth
constexpr int kUAbytes = kUM * kUK * 4;  // one plane of an A stage
constexpr int kUBbytes = kUN * kUK * 4;
constexpr int kUStageBytes = 2 * kUAbytes + 2 * kUBbytes;  // hi + lo planes of A and B
constexpr int kURawBytes = kUK * (kUM + kUN) * 4;           // one chunk, natural layout
constexpr int kUSmem = kUStages * kUStageBytes + kURaw * kURawBytes + 64;  // + barriers / TMEM address

// async copies of one chunk's rows into a raw slot [kUK][kUM + kUN] (rows >= nb zero-filled);
// with 256 threads each issues exactly kUK * 48 / 256 = 3 copies (compile-time unrolled)
constexpr int kUPieces = kUK * (kUM + kUN) / 4;
static_assert(kUPieces % 256 == 0, "copy pieces per thread");
__device__ __forceinline__ void umma_async_chunk(unsigned char* raw, const float* __restrict__ a_src,
                                                 const float* __restrict__ u_src, long long ld, int b0, int nb) {
    const uint32_t base = smem_addr(raw);
    constexpr int pq = (kUM + kUN) / 4;  // 16-byte pieces per row
    const int last = max(nb - 1, 0);
#pragma unroll
    for (int i = 0; i < kUPieces / 256; ++i) {
        const int w = threadIdx.x + i * 256;
        const int b = w / pq, q = w - b * pq;
        const bool isA = q < kUM / 4;
        const float* src = (isA ? a_src + q * 4 : u_src + (q - kUM / 4) * 4) + (long long)(b0 + min(b, last)) * ld;
        const int bytes = b < nb ? 16 : 0;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(base + static_cast<uint32_t>(w * 16)),
                     "l"(src), "r"(bytes)
                     : "memory");
    }
    cp_async_commit();
}

// raw chunk -> K-major TF32 hi / lo planes of a stage; B's column Kv becomes the ones column.
// Items (operand row r, 4-row group kq), lanes over r; with 256 threads and kUK = 16 each
// thread takes items tid, tid + 256 (A) and tid + 512 (B): roles fixed at compile time.
template <bool IS_A>
__device__ __forceinline__ void umma_transpose_item(uint32_t* hi, uint32_t* lo, const float* R, int wi, int Kv) {
    constexpr int nr = IS_A ? kUM : kUN, ldr = kUM + kUN;
    const int kq = wi / nr, r = wi - kq * nr;
    const int col = IS_A ? r : kUM + r;
    float x[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) x[j] = R[(kq * 4 + j) * ldr + col];
    if (!IS_A && r == Kv) x[0] = x[1] = x[2] = x[3] = 1.f;
    uint4 h, l;
    uint32_t* hh = reinterpret_cast<uint32_t*>(&h);
    uint32_t* ll = reinterpret_cast<uint32_t*>(&l);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        hh[j] = __float_as_uint(x[j]) & 0xFFFFE000u;
        ll[j] = __float_as_uint(x[j] - __uint_as_float(hh[j]));
    }
    const int off = ((kq * (nr / 8) + (r >> 3)) * 128 + (r & 7) * 16) >> 2;
    *reinterpret_cast<uint4*>(hi + off) = h;
    *reinterpret_cast<uint4*>(lo + off) = l;
}

static_assert(kUM * (kUK / 4) == 512 && kUN * (kUK / 4) == 256, "transpose item roles assume 256 threads");
__device__ __forceinline__ void umma_transpose_chunk(unsigned char* stage, const unsigned char* raw, int Kv) {
    const float* R = reinterpret_cast<const float*>(raw);
    uint32_t* Ahi = reinterpret_cast<uint32_t*>(stage);
    uint32_t* Alo = Ahi + kUM * kUK;
    uint32_t* Bhi = Alo + kUM * kUK;
    uint32_t* Blo = Bhi + kUN * kUK;
    const int tid = threadIdx.x;
    umma_transpose_item<true>(Ahi, Alo, R, tid, Kv);
    umma_transpose_item<true>(Ahi, Alo, R, tid + 256, Kv);
    umma_transpose_item<false>(Bhi, Blo, R, tid, Kv);
}

// issue the 3xTF32 MMAs of one stage (one thread): hi*hi + hi*lo + lo*hi; descriptors advanced
// by adding to the start-address field (16-byte units)
__device__ __forceinline__ void umma_issue_stage(unsigned char* stage, uint32_t tmem_d, bool first) {
    constexpr uint32_t a_lbo = (kUM / 8) * 128, b_lbo = (kUN / 8) * 128, sbo = 128;
    constexpr uint32_t idesc = umma_idesc_tf32(kUM, kUN);
    const uint32_t base = smem_addr(stage);
    const uint64_t dahi = umma_smem_desc(base, a_lbo, sbo);
    const uint64_t dalo = dahi + (kUAbytes >> 4);
    const uint64_t dbhi = umma_smem_desc(base + 2 * kUAbytes, b_lbo, sbo);
    const uint64_t dblo = dbhi + (kUBbytes >> 4);
#pragma unroll
    for (int k8 = 0; k8 < kUK / 8; ++k8) {
        const uint64_t ao = (2 * k8 * a_lbo) >> 4, bo = (2 * k8 * b_lbo) >> 4;
        const uint32_t acc0 = (first && k8 == 0) ? 0u : 1u;
        umma_tf32(tmem_d, dahi + ao, dbhi + bo, idesc, acc0);
        umma_tf32(tmem_d, dahi + ao, dblo + bo, idesc, 1u);
        umma_tf32(tmem_d, dalo + ao, dbhi + bo, idesc, 1u);
    }
}

// The whole partial contraction (all threads of the CTA call; blockDim.x a multiple of 128,
// warps 0..3 read the accumulator).  smem: kUSmem bytes (16-byte aligned).  out: kUM x kUN.
// Pipeline: kURaw - 1 chunks of copies in flight ahead of the one being transposed; an
// operand stage is rewritten only after its MMAs committed (one mbarrier per stage).
__device__ __forceinline__ void umma_partial_dw(unsigned char* smem, const float* __restrict__ a_src,
                                                const float* __restrict__ u_src, long long ld, int r0, int nrows,
                                                int Kv, float* __restrict__ out, long long* tprobe = nullptr) {
    const int tid = threadIdx.x, warp = tid >> 5;
    long long tt[6] = {0, 0, 0, 0, 0, 0};
    unsigned char* rawbase = smem + kUStages * kUStageBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(rawbase + kURaw * kURawBytes);  // [kUStages]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kUStages);
    if (warp == 0) tmem_alloc(tmem_slot, kUN);
    if (tid == 0)
        for (int s = 0; s < kUStages; ++s) mbar_init(bars + s, 1);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_d = *tmem_slot;
    const int nch = (nrows + kUK - 1) / kUK;
    uint32_t phase_bits = 0;  // bit s: parity of stage s's next commit wait
    // prologue: kURaw - 1 chunks in flight (empty groups keep the count uniform)
#pragma unroll
    for (int c = 0; c < kURaw - 1; ++c) {
        if (c < nch) umma_async_chunk(rawbase + c * kURawBytes, a_src, u_src, ld, r0 + c * kUK, min(kUK, nrows - c * kUK));
        else cp_async_commit();
    }
    for (int c = 0; c < nch; ++c) {
        const int s = c % kUStages;
        unsigned char* stage = smem + s * kUStageBytes;
        const int cn = c + kURaw - 1;  // refill the raw slot the previous chunk freed
        const long long t0 = tprobe ? clock64() : 0;
        if (cn < nch) umma_async_chunk(rawbase + (cn % kURaw) * kURawBytes, a_src, u_src, ld, r0 + cn * kUK,
                                       min(kUK, nrows - cn * kUK));
        else cp_async_commit();
        const long long t1 = tprobe ? clock64() : 0;
        cp_async_wait<kURaw - 1>();  // chunk c landed
        const long long t2 = tprobe ? clock64() : 0;
        if (c >= kUStages) {         // stage s's previous MMAs (chunk c - kUStages) are done
            mbar_wait(bars + s, (phase_bits >> s) & 1u);
            phase_bits ^= 1u << s;
        }
        __syncthreads();
        const long long t3 = tprobe ? clock64() : 0;
        umma_transpose_chunk(stage, rawbase + (c % kURaw) * kURawBytes, Kv);
        fence_proxy_async_smem();  // generic-proxy stores -> visible to the tensor core
        __syncthreads();
        const long long t4 = tprobe ? clock64() : 0;
        if (tid == 0) {
            tc_fence_after();
            umma_issue_stage(stage, tmem_d, c == 0);
            umma_commit(bars + s);
        }
        if (tprobe) {
            const long long t5 = clock64();
            tt[0] += t1 - t0, tt[1] += t2 - t1, tt[2] += t3 - t2, tt[3] += t4 - t3, tt[4] += t5 - t4;
        }
    }
    cp_async_wait<0>();
    // drain: the last stage's commit covers every earlier MMA
    if (nch > 0) {
        const int s = (nch - 1) % kUStages;
        mbar_wait(bars + s, (phase_bits >> s) & 1u);
    }
    tc_fence_after();
    if (warp < 4) {
        const int m = warp * 32 + (tid & 31);
#pragma unroll
        for (int c0 = 0; c0 < kUN; c0 += 16) {
            float v[16];
            tmem_ld16(tmem_d + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
#pragma unroll
            for (int i = 0; i < 16; ++i) out[m * kUN + c0 + i] = nch > 0 ? v[i] : 0.f;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem_d, kUN);
    if (tprobe && tid == 0)
        for (int i = 0; i < 5; ++i) tprobe[i] = tt[i];
}

}  // namespace esrnn_dev
