#include <cstdio>
#include "common.cuh"
#include "umma.cuh"
using namespace esrnn_dev;
__global__ void k_st(const float* A, const float* U, long long ld, int nrows, int Mv, int Kv, long long* t, int mode) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const int nch = (nrows + kUK - 1) / kUK;
    UChunk cur;
    long long tl = 0, tw = 0, ts = 0;
    for (int c = 0; c < nch; ++c) {
        long long a = clock64();
        umma_load_chunk(cur, A, U, ld, c * kUK, min(kUK, nrows - c * kUK));
        long long b = clock64();
        float acc = 0;
        for (int j = 0; j < 4; ++j) acc += cur.f[0][j].x + cur.f[0][j].w;
        asm volatile("" :: "f"(acc));
        long long d = clock64();
        if (mode) umma_store_chunk(smem + (c % 2) * kUStageBytes, cur, min(kUK, nrows - c * kUK), Mv, Kv);
        __syncthreads();
        long long e = clock64();
        tl += b - a; tw += d - b; ts += e - d;
    }
    if (threadIdx.x == 0) { t[0] = tl; t[1] = tw; t[2] = ts; }
}
int main() {
    float *dA, *dU; long long* t; int B = 1000; long long ld = 256;
    cudaMalloc(&dA, B * ld * 4 + 4096); cudaMalloc(&dU, B * ld * 4 + 4096); cudaMallocManaged(&t, 64);
    cudaMemset(dA, 0, B*ld*4); cudaMemset(dU, 0, B*ld*4);
    cudaFuncSetAttribute(k_st, cudaFuncAttributeMaxDynamicSharedMemorySize, kUSmem);
    for (int rep = 0; rep < 2; ++rep)
      for (int mode = 0; mode < 2; ++mode) {
        k_st<<<1, 256, kUSmem>>>(dA, dU, ld, B, 120, 40, t, mode); cudaDeviceSynchronize();
        printf("mode %d: load-issue %lld  load-wait %lld  store+sync %lld  (32 chunks) %s\n", mode, t[0], t[1], t[2], cudaGetErrorString(cudaGetLastError()));
      }
}
