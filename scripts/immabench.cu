// IMMA (mma.sync m16n8k32 u8) throughput on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/immabench scripts/immabench.cu && /tmp/immabench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_imma(int *out, int iters, uint32_t seed) {
    uint32_t a[4], b[2];
    for (int i = 0; i < 4; i++) a[i] = seed * (threadIdx.x + i + 1);
    for (int i = 0; i < 2; i++) b[i] = seed ^ (threadIdx.x * 7 + i);
    int d[8][4] = {};
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int t = 0; t < 8; t++)
            asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+r"(d[t][0]), "+r"(d[t][1]), "+r"(d[t][2]), "+r"(d[t][3])
                         : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    int s = 0;
    for (int t = 0; t < 8; t++) s += d[t][0] + d[t][1] + d[t][2] + d[t][3];
    if (s == 0x12345) out[0] = s;
}

int main() {
    int *out;
    cudaMalloc(&out, 64);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 4096;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int warps : {4, 8, 16}) {
        k_imma<<<sms, 32 * warps>>>(out, 16, 3);
        cudaEventRecord(a);
        k_imma<<<sms * 4, 32 * warps>>>(out, iters, 3);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double ops = (double)sms * 4 * warps * iters * 8 * (16.0 * 8 * 32 * 2);
        printf("IMMA m16n8k32 u8, %d warps/CTA, 4 CTAs/SM: %.1f TOPS (%s)\n", warps, ops / (ms * 1e-3) / 1e12,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
