// tcgen05.mma kind::i8 probe: u8 x u8 -> s32 GEMMs with operands in shared memory (K-major,
// no-swizzle canonical layout) and the accumulator in TMEM, checked against the CPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tc_probe scripts/tc_probe.cu && /tmp/tc_probe
// Cases: M = 64 (two coefficient tiles interleaved in the lane halves of one column block) and
// M = 128, N = 48 / 64, K = 128 (4 MMAs of K = 32).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// canonical K-major no-swizzle layout of an R x 128 (bytes) operand: [R/8 groups][8 chunks][8 rows][16 B]
__host__ __device__ __forceinline__ uint32_t kmaj_off(int r, int k) {
    return (uint32_t)((r >> 3) * 1024 + (k >> 4) * 128 + (r & 7) * 16 + (k & 15));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);           // start address
    d |= (uint64_t)(128 >> 4) << 16;                  // LBO: next 16-byte K chunk
    d |= (uint64_t)(1024 >> 4) << 32;                 // SBO: next 8-row group
    d |= (uint64_t)1 << 46;                           // version (sm_100)
    return d;                                         // base offset 0, no swizzle
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
    return (2u << 4)              // D format S32
           | (0u << 7) | (0u << 10)  // A, B unsigned 8 bit
           | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int M, int N, int TILES>
__global__ void k_probe(const uint8_t *A, const uint8_t *Bm, int32_t *D) {
    // A: TILES x [M][128], B: TILES x [N][128] (row-major in global), D: TILES x [M][N]
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *sa = sm, *sb = sm + TILES * M * 128;
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < TILES * M * 128; i += blockDim.x) {
        int t = i / (M * 128), r = (i / 128) % M, k = i % 128;
        sa[t * M * 128 + kmaj_off(r, k)] = A[i];
    }
    for (int i = tid; i < TILES * N * 128; i += blockDim.x) {
        int t = i / (N * 128), r = (i / 128) % N, k = i % 128;
        sb[t * N * 128 + kmaj_off(r, k)] = Bm[i];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)),
                     "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tbase;
    if (tid == 0) {
        constexpr uint32_t id = idesc_i8(M, N);
        for (int t = 0; t < TILES; t++) {
            // M = 64: tile t -> lanes 16 (t % 2) of each subpartition, columns N (t / 2)
            const uint32_t dt = M == 64 ? tmem + ((uint32_t)(16 * (t & 1)) << 16) + (uint32_t)(N * (t >> 1))
                                        : tmem + (uint32_t)(N * t);
            for (int ks = 0; ks < 4; ks++) {
                const uint64_t da = sdesc(smem_u32(sa + t * M * 128 + ks * 256));
                const uint64_t db = sdesc(smem_u32(sb + t * N * 128 + ks * 256));
                const uint32_t acc = ks > 0;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dt),
                    "l"(da), "l"(db), "r"(id), "r"(acc));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&bar)));
    }
    {
        uint32_t ok = 0;
        while (!ok)
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                : "=r"(ok)
                : "r"(smem_u32(&bar)), "r"(0));
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp < 4) {  // warp w reads TMEM lanes [32 w, 32 w + 32)
        const int tcols = M == 64 ? N * ((TILES + 1) / 2) : N * TILES;
        for (int c0 = 0; c0 < tcols; c0 += 8) {
            uint32_t v[8];
            const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                           "=r"(v[7])
                         : "r"(ta));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            const int L = 32 * warp + lane;  // TMEM lane
            for (int e = 0; e < 8; e++) {
                const int col = c0 + e;
                int t, row, n = col % N;
                if (M == 64) {
                    if ((L & 31) >= 16 && TILES < 2) continue;
                    t = 2 * (col / N) + ((L & 31) >= 16);
                    row = (L & 15) + 16 * (L >> 5);
                } else {
                    t = col / N;
                    row = L;
                }
                if (t < TILES) D[(t * M + row) * N + n] = (int32_t)v[e];
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

template <int M, int N, int TILES>
int run() {
    std::vector<uint8_t> A(TILES * M * 128), B(TILES * N * 128);
    for (auto &x : A) x = rand() & 255;
    for (auto &x : B) x = rand() & 255;
    uint8_t *dA, *dB;
    int32_t *dD;
    cudaMalloc(&dA, A.size());
    cudaMalloc(&dB, B.size());
    cudaMalloc(&dD, TILES * M * N * 4);
    cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
    cudaMemset(dD, 0xFF, TILES * M * N * 4);
    const size_t smem = (size_t)TILES * (M + N) * 128;
    cudaFuncSetAttribute(k_probe<M, N, TILES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_probe<M, N, TILES><<<1, 256, smem>>>(dA, dB, dD);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<int32_t> D(TILES * M * N);
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    long bad = 0;
    for (int t = 0; t < TILES; t++)
        for (int m = 0; m < M; m++)
            for (int n = 0; n < N; n++) {
                int32_t want = 0;
                for (int k = 0; k < 128; k++) want += (int32_t)A[(t * M + m) * 128 + k] * B[(t * N + n) * 128 + k];
                if (D[(t * M + m) * N + n] != want) {
                    if (bad < 4)
                        printf("  mismatch t%d m%d n%d got %d want %d\n", t, m, n, D[(t * M + m) * N + n], want);
                    bad++;
                }
            }
    printf("M=%d N=%d tiles=%d: %s, %ld mismatches\n", M, N, TILES, cudaGetErrorString(e), bad);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
    return bad != 0 || e != cudaSuccess;
}

int main() {
    int f = 0;
    f |= run<64, 48, 1>();
    f |= run<64, 48, 4>();
    f |= run<128, 64, 2>();
    f |= run<128, 48, 1>();
    printf(f ? "FAIL\n" : "ALL OK\n");
    return f;
}
