// Standalone check of csrc/umma.cuh (tcgen05 3xTF32 partial contraction) against a CPU
// double reference: build with nvcc -gencode arch=compute_100a,code=sm_100a, run on a B200.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "common.cuh"
#include "umma.cuh"

using namespace esrnn_dev;

__global__ void k_probe(const float* A, const float* U, long long ld, int r0, int nrows, int Mv, int Kv, float* out,
                        long long* tp) {
    extern __shared__ __align__(1024) unsigned char smem[];
    umma_partial_dw(smem, A, U, ld, r0, nrows, Kv, out, tp);
}

int main(int argc, char** argv) {
    const int B = argc > 1 ? atoi(argv[1]) : 1000, Mv = argc > 2 ? atoi(argv[2]) : 120, Kv = argc > 3 ? atoi(argv[3]) : 40;
    const long long ld = 256;
    std::vector<float> A(B * ld), U(B * ld);
    srand(1);
    for (auto& x : A) x = (rand() / (float)RAND_MAX - 0.5f) * 2.f;
    for (auto& x : U) x = (rand() / (float)RAND_MAX - 0.5f) * 2.f;
    float *dA, *dU, *dO;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dU, U.size() * 4); cudaMalloc(&dO, kUM * kUN * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dU, U.data(), U.size() * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, kUSmem);
    long long* tp; cudaMallocManaged(&tp, 64);
    k_probe<<<1, 256, kUSmem>>>(dA, dU, ld, 0, B, Mv, Kv, dO, tp);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    std::vector<float> O(kUM * kUN);
    cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0, maxerr_tf32 = 0;
    for (int m = 0; m < Mv; ++m)
        for (int n = 0; n <= Kv; ++n) {
            double ref = 0;
            for (int b = 0; b < B; ++b) {
                const double a = m < Mv ? A[b * ld + m] : 0.0;
                const double u = n < Kv ? U[b * ld + n] : (n == Kv ? 1.0 : 0.0);
                ref += a * u;
            }
            maxref = fmax(maxref, fabs(ref));
            maxerr = fmax(maxerr, fabs(ref - O[m * kUN + n]));
        }
    printf("B=%d M=%d K=%d  max|ref|=%.4g  max|err|=%.3g  tensor-scaled %.3g  D[0][0]=%g D[1][2]=%g\n", B, Mv, Kv,
           maxref, maxerr, maxerr / maxref, O[0], O[1 * kUN + 2]);
    // timing
    cudaEvent_t t0, t1; cudaEventCreate(&t0); cudaEventCreate(&t1);
    cudaEventRecord(t0);
    for (int i = 0; i < 20; ++i) k_probe<<<1, 256, kUSmem>>>(dA, dU, ld, 0, B, Mv, Kv, dO, nullptr);
    cudaEventRecord(t1); cudaEventSynchronize(t1);
    float ms; cudaEventElapsedTime(&ms, t0, t1);
    printf("avg %.2f us per CTA-partial of %d rows\n", ms * 1000 / 20, B);
    k_probe<<<1, 256, kUSmem>>>(dA, dU, ld, 0, B, Mv, Kv, dO, tp); cudaDeviceSynchronize();
    printf("thread0 cycles: issue-copies %lld  wait-copies %lld  mbar+sync %lld  transpose+sync %lld  mma-issue %lld\n", tp[0], tp[1], tp[2], tp[3], tp[4]);

    return maxerr / maxref < 1e-5 ? 0 : 1;
}
