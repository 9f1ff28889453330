#include <cstdio>
#include <vector>
#include "common.cuh"
#include "umma.cuh"
using namespace esrnn_dev;
__global__ void k(const float* A, const float* U, long long ld, int nb, int Kv, float* dump) {
    extern __shared__ __align__(1024) unsigned char smem[];
    umma_async_chunk(smem, A, U, ld, 0, nb);
    cp_async_wait<0>();
    __syncthreads();
    umma_remainders(smem, Kv);
    __syncthreads();
    const float* f = reinterpret_cast<const float*>(smem);
    for (int i = threadIdx.x; i < kUStageBytes / 4; i += blockDim.x) dump[i] = f[i];
}
int main() {
    const long long ld = 256; const int B = 64;
    std::vector<float> A(B * ld), U(B * ld);
    for (int b = 0; b < B; ++b) for (int c = 0; c < ld; ++c) { A[b * ld + c] = 1000 * b + c + 0.5f; U[b * ld + c] = -(1000 * b + c) - 0.25f; }
    float *dA, *dU, *dd; cudaMalloc(&dA, B*ld*4); cudaMalloc(&dU, B*ld*4); cudaMalloc(&dd, kUStageBytes);
    cudaMemcpy(dA, A.data(), B*ld*4, cudaMemcpyHostToDevice); cudaMemcpy(dU, U.data(), B*ld*4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kUSmem);
    k<<<1, 256, kUSmem>>>(dA, dU, ld, 32, 40, dd);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    std::vector<float> d(kUStageBytes / 4); cudaMemcpy(d.data(), dd, kUStageBytes, cudaMemcpyDeviceToHost);
    // A raw core (g=0,kg=0): 8 rows b x 4 m
    for (int i = 0; i < 12; ++i) printf("%g ", d[i]); printf(" | A raw first 12\n");
    for (int i = 32; i < 40; ++i) printf("%g ", d[i]); printf(" | A raw core 1\n");
    int bofs = 2 * kUAbytes / 4; for (int i = 0; i < 8; ++i) printf("%g ", d[bofs + i]); printf(" | B raw\n");
    int lofs = kUAbytes / 4; for (int i = 0; i < 4; ++i) printf("%g ", d[lofs + i]); printf(" | A lo\n");
}
