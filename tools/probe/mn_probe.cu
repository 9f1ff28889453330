// one tcgen05.mma kind::tf32 (M=128, N=64, K=8) with MN-major no-swizzle operands: which
// (LBO, SBO) assignment reproduces D = A^T-ish product?  A(m,k) at core (m/4, k/8)...
#include <cstdio>
#include <vector>
#include "common.cuh"
#include "umma.cuh"
using namespace esrnn_dev;
__host__ __device__ constexpr uint32_t idesc_mn(int M, int N, int amaj, int bmaj) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(amaj) << 15) | (uint32_t(bmaj) << 16) |
           (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
__global__ void k(const float* A, const float* B, float* D, int mode) {
    // A: [K=8][M=128] (A(m,k) = A[k*128+m]); B: [K=8][N=64]
    __shared__ __align__(1024) float sa[128 * 8];
    __shared__ __align__(1024) float sb[64 * 8];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x;
    // MN-major core layout: core(g = m/4) at g*128 bytes, inside: k row (k%8)*16 bytes + (m%4)*4
    for (int i = tid; i < 128 * 8; i += blockDim.x) { int m = i % 128, kk = i / 128; sa[(m / 4) * 32 + kk * 4 + (m % 4)] = A[kk * 128 + m]; }
    for (int i = tid; i < 64 * 8; i += blockDim.x) { int n = i % 64, kk = i / 64; sb[(n / 4) * 32 + kk * 4 + (n % 4)] = B[kk * 64 + n]; }
    if (tid < 32) tmem_alloc(&tslot, 64);
    if (tid == 0) mbar_init(&bar, 1);
    fence_proxy_async_smem();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t td = tslot;
    if (tid == 0) {
        uint32_t lbo, sbo;
        if (mode == 0) { sbo = 128; lbo = 128 * 32; }   // SBO = MN-group stride
        else { lbo = 128; sbo = 128 * 32; }             // swapped
        const uint64_t da = umma_smem_desc(smem_addr(sa), mode == 0 ? 128 * 32 : 128, mode == 0 ? 128 : 128 * 32);
        const uint64_t db = umma_smem_desc(smem_addr(sb), mode == 0 ? 128 * 16 : 128, mode == 0 ? 128 : 128 * 16);
        (void)lbo; (void)sbo;
        umma_tf32(td, da, db, idesc_mn(128, 64, 1, 1), 0u);
        umma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    if (tid < 128) {
        for (int c0 = 0; c0 < 64; c0 += 16) {
            float v[16];
            tmem_ld16(td + ((uint32_t)((tid / 32) * 32) << 16) + c0, v);
            for (int i = 0; i < 16; ++i) D[tid * 64 + c0 + i] = v[i];
        }
    }
    tc_fence_before(); __syncthreads();
    if (tid < 32) tmem_dealloc(td, 64);
}
int main() {
    std::vector<float> A(8 * 128), B(8 * 64), D(128 * 64);
    for (int i = 0; i < 8 * 128; ++i) A[i] = (i % 7) - 3;
    for (int i = 0; i < 8 * 64; ++i) B[i] = (i % 5) - 2;
    float *dA, *dB, *dD; cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice); cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 2; ++mode) {
        cudaMemset(dD, 0, D.size() * 4);
        k<<<1, 128>>>(dA, dB, dD, mode);
        printf("mode %d: %s ", mode, cudaGetErrorString(cudaDeviceSynchronize()));
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double maxerr = 0, maxref = 0;
        for (int m = 0; m < 128; ++m) for (int n = 0; n < 64; ++n) {
            double r = 0; for (int kk = 0; kk < 8; ++kk) r += A[kk * 128 + m] * B[kk * 64 + n];
            maxerr = fmax(maxerr, fabs(r - D[m * 64 + n])); maxref = fmax(maxref, fabs(r));
        }
        printf("max|ref| %g max|err| %g  D[0][0]=%g D[1][0]=%g D[0][1]=%g\n", maxref, maxerr, D[0], D[64], D[1]);
    }
}
