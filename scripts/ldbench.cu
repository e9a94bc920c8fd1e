// Load-path microbenchmark (B200): read bandwidth of the NTT access patterns.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ldbench scripts/ldbench.cu && /tmp/ldbench
// p1-like: CTA = 128 rows x 32 columns of 8 B (rows 2 KB apart), 256 threads, 16 loads each.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256, 4) k_ldg(const uint64_t *__restrict__ src, uint64_t *out) {
    const size_t limb = blockIdx.y;
    const int col = blockIdx.x * 32 + (threadIdx.x & 31), wq = threadIdx.x >> 5;
    const uint64_t *p = src + (limb << 15);
    uint64_t v[16];
#pragma unroll
    for (int x = 0; x < 16; x++) v[x] = __ldg(p + (size_t)(wq + 8 * x) * 256 + col);
    uint64_t s = 0;
#pragma unroll
    for (int x = 0; x < 16; x++) s += v[x];
    if (s == 0x1234567) out[0] = s;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(256, 4) k_bulk(const uint64_t *__restrict__ src, uint64_t *out) {
    __shared__ alignas(128) uint64_t sm[128 * 32];
    __shared__ alignas(8) uint64_t bar;
    const size_t limb = blockIdx.y;
    const uint64_t *p = src + (limb << 15) + blockIdx.x * 32;
    const int tid = threadIdx.x;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (tid == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(128 * 256));
    __syncthreads();
    if (tid < 128)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];" ::"r"(
                         smem_u32(sm + tid * 32)),
                     "l"(p + (size_t)tid * 256), "r"(smem_u32(&bar))
                     : "memory");
    uint32_t done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done)
                     : "r"(smem_u32(&bar)));
    uint64_t s = 0;
#pragma unroll
    for (int x = 0; x < 16; x++) s += sm[tid + 256 * x];
    if (s == 0x1234567) out[0] = s;
}

// half-kernel round-1 pattern: 2 CTAs/SM (99 KB smem), 256 threads, 4 columns x 32 loads
__global__ void __launch_bounds__(256, 2) k_half(const uint64_t *__restrict__ src, uint64_t *out) {
    extern __shared__ uint32_t dyn[];
    const size_t limb = blockIdx.y;
    const uint64_t *p = src + (limb << 15);
    uint64_t s = 0;
#pragma unroll 1
    for (int g = 0; g < 4; g++) {
        const int c = threadIdx.x + 256 * g;
        uint64_t v[32];
#pragma unroll
        for (int t = 0; t < 32; t++) v[t] = __ldg(p + t * 1024 + c);
#pragma unroll
        for (int t = 0; t < 32; t++) s += v[t];
    }
    dyn[threadIdx.x] = (uint32_t)s;
    if (s == 0x1234567) out[0] = s;
}

int main() {
    const int limbs = 4096;
    uint64_t *src, *out;
    cudaMalloc(&src, (size_t)limbs << 18);
    cudaMalloc(&out, 64);
    cudaMemset(src, 1, (size_t)limbs << 18);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaFuncSetAttribute(k_half, cudaFuncAttributeMaxDynamicSharedMemorySize, 101376);
    for (int rep = 0; rep < 2; rep++) {
        float ms;
        cudaEventRecord(a);
        k_ldg<<<dim3(8, limbs), 256>>>(src, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("ldg64 p1-tile : %.1f GB/s\n", (double)limbs * 262144 / (ms * 1e6));
        cudaEventRecord(a);
        k_bulk<<<dim3(8, limbs), 256>>>(src, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("bulk p1-tile  : %.1f GB/s  (%s)\n", (double)limbs * 262144 / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
        cudaEventRecord(a);
        k_half<<<dim3(1, limbs), 256, 101376>>>(src, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("half round-1  : %.1f GB/s\n", (double)limbs * 262144 / (ms * 1e6));
    }
    return 0;
}
