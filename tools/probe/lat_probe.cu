// global-load latency as seen by a 256-thread CTA: 8 float4 loads per thread, L2-resident data
#include <cstdio>
__global__ void k(const float* a, long long ld, int nb, long long* t, float* sink) {
    const int tid = threadIdx.x;
    float acc = 0;
    long long tot = 0;
    for (int rep = 0; rep < 32; ++rep) {
        long long t0 = clock64();
        float4 f[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
            f[j] = __ldg(reinterpret_cast<const float4*>(a + (long long)((rep * 32 + (tid >> 5) * 4 + (j & 3)) % nb) * ld + (tid & 31) * 4 + (j >> 2) * 128));
#pragma unroll
        for (int j = 0; j < 8; ++j) acc += f[j].x + f[j].y + f[j].z + f[j].w;
        asm volatile("" :: "f"(acc));
        long long t1 = clock64();
        tot += t1 - t0;
    }
    if (tid == 0) t[0] = tot / 32;
    if (acc == 1234.f) sink[0] = acc;
}
int main() {
    float* a; float* s; long long* t;
    cudaMalloc(&a, 4096 * 256 * 4); cudaMalloc(&s, 4); cudaMallocManaged(&t, 8);
    cudaMemset(a, 0, 4096 * 256 * 4);
    for (int r = 0; r < 3; ++r) { k<<<1, 256>>>(a, 256, 1000, t, s); cudaDeviceSynchronize(); printf("avg per 8xLDG.128 round: %lld cycles\n", t[0]); }
    k<<<148, 256>>>(a, 256, 1000, t, s); cudaDeviceSynchronize(); printf("148 CTAs: %lld\n", t[0]);
}
