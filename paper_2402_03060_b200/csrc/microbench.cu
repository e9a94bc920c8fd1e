// Integer-pipe peak microbenchmarks (the modmul roofline denominator).
//
// The engine's work is 64-bit modular multiply-accumulate built from 32-bit
// IMAD; there is no vendor-published "IMAD peak" for B200, so the bench
// measures it on the box: (1) raw 32-bit IMAD issue rate, (2) the rate of the
// engine's lazy 128-bit multiply-accumulate (Acc::mac) and (3) of a fully
// reduced 64-bit modular product (mulmod), all register-resident with 8
// independent chains per thread and a grid of 148 x 8 CTAs.
#include "ops.cuh"

namespace uh {
namespace {

__global__ void k_imad_peak(uint32_t *out, int iters, uint32_t seed) {
    uint32_t a[8];
#pragma unroll
    for (int i = 0; i < 8; i++) a[i] = seed + threadIdx.x * 8 + i;
    const uint32_t m = 0x9E3779B1u + blockIdx.x;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) a[i] = a[i] * m + 0x7F4A7C15u;
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s ^= a[i];
    if (s == 0x12345678u) out[0] = s;
}

__global__ void k_mac_peak(uint64_t *out, int iters, uint64_t seed) {
    Acc acc[8];
    uint64_t x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) {
        acc[i].zero();
        x[i] = (seed + threadIdx.x * 8 + i) & ((1ull << 60) - 1);
    }
    const uint64_t w = (0x0FEDCBA987654321ull + blockIdx.x) & ((1ull << 60) - 1);
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            acc[i].mac(x[i], w);
            x[i] ^= acc[i].lo64();  // keep operands live and varying (XOR: ALU pipe)
        }
    }
    uint64_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s ^= acc[i].lo64() ^ acc[i].hi64();
    if (s == 0x1234567812345678ull) out[0] = s;
}

__global__ void k_macc_peak(uint64_t *out, int iters, uint64_t seed) {  // plain-C MAC form
    Acc acc[8];
    uint64_t x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) {
        acc[i].zero();
        x[i] = (seed + threadIdx.x * 8 + i) & ((1ull << 60) - 1);
    }
    const uint64_t w = (0x0FEDCBA987654321ull + blockIdx.x) & ((1ull << 60) - 1);
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            acc[i].mac_c(x[i], w);
            x[i] ^= acc[i].lo64();
        }
    }
    uint64_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s ^= acc[i].lo64() ^ acc[i].hi64();
    if (s == 0x1234567812345678ull) out[0] = s;
}

__global__ void k_shoup_peak(uint64_t *out, int iters, uint64_t seed, Mod m) {  // lazy Shoup (NTT butterfly core)
    uint64_t x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = (seed + threadIdx.x * 8 + i) % m.q;
    const uint64_t w = m.r64, ws = m.r64s;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) x[i] = shoup_lazy(x[i], w, ws, m.q);
    }
    uint64_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s ^= x[i];
    if (s == 0x1234567812345678ull) out[0] = s;
}

__global__ void k_mulmod_peak(uint64_t *out, int iters, uint64_t seed, Mod m) {
    uint64_t x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = (seed + threadIdx.x * 8 + i) % m.q;
    const uint64_t w = (0x0FEDCBA987654321ull + blockIdx.x) % m.q;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) x[i] = mulmod(x[i], w, m);
    }
    uint64_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s ^= x[i];
    if (s == 0x1234567812345678ull) out[0] = s;
}

// exact modular multiply-accumulate on the FP64 pipe for q < 2^50:
// x*y = p + e exactly (fma), r = p - rint(p/q)*q + e exactly, sum r exactly (< 2^53)
__device__ __forceinline__ double fmac(double acc, double x, double y, double q, double qinv) {
    const double magic = 6755399441055744.0;  // 1.5 * 2^52: round-to-nearest integer trick
    double p = x * y;
    double e = fma(x, y, -p);
    double qt = fma(p, qinv, magic) - magic;
    double r = fma(-qt, q, p);
    return acc + (r + e);
}

__global__ void k_fp64mac_peak(double *out, int iters, double seed, double q, double qinv) {
    double acc[8], x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) {
        acc[i] = 0;
        x[i] = fmod(seed * (threadIdx.x * 8 + i + 1), q);
    }
    const double w = fmod(1234567.0 * (blockIdx.x + 3), q);
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            acc[i] = fmac(acc[i], x[i], w, q, qinv);
            x[i] = acc[i] > q ? x[i] - 1.0 : x[i] + 1.0;  // keep operands varying
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s += acc[i];
    if (s == 1.2345) out[0] = s;
}

__global__ void k_macs_peak(uint64_t *out, int iters, uint64_t seed) {  // split accumulator (AccS)
    AccS acc[8];
    uint64_t x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) {
        acc[i].zero();
        x[i] = (seed + threadIdx.x * 8 + i) & ((1ull << 60) - 1);
    }
    const uint64_t w = (0x0FEDCBA987654321ull + blockIdx.x) & ((1ull << 60) - 1);
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            acc[i].mac(x[i], w);
            x[i] ^= acc[i].a0;
        }
    }
    uint64_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s ^= acc[i].lo64() ^ acc[i].hi64();
    if (s == 0x1234567812345678ull) out[0] = s;
}

// both pipes: half the chains on IMAD (128-bit integer MAC), half on FP64
__global__ void k_mixed_peak(uint64_t *out, int iters, uint64_t seed, double q, double qinv) {
    Acc acc[4];
    uint64_t x[4];
    double facc[4], fx[4];
#pragma unroll
    for (int i = 0; i < 4; i++) {
        acc[i].zero();
        x[i] = (seed + threadIdx.x * 8 + i) & ((1ull << 60) - 1);
        facc[i] = 0;
        fx[i] = (double)((seed + threadIdx.x * 4 + i) % (uint64_t)q);
    }
    const uint64_t w = (0x0FEDCBA987654321ull + blockIdx.x) & ((1ull << 60) - 1);
    const double fw = 987654321.0 + blockIdx.x;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 4; i++) {
            acc[i].mac(x[i], w);
            x[i] ^= acc[i].lo64();
            facc[i] = fmac(facc[i], fx[i], fw, q, qinv);
            fx[i] = facc[i] > q ? fx[i] - 1.0 : fx[i] + 1.0;
        }
    }
    uint64_t s = 0;
#pragma unroll
    for (int i = 0; i < 4; i++) s ^= acc[i].lo64() ^ acc[i].hi64() ^ (uint64_t)facc[i];
    if (s == 0x1234567812345678ull) out[0] = s;
}

// narrow-operand MAC (AccN, limbs with q < 2^41): both factors below 2^41
__global__ void k_macn_peak(uint64_t *out, int iters, uint64_t seed) {
    AccN acc[8];
    uint64_t x[8];
    constexpr uint64_t M41 = (1ull << 41) - 1;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        acc[i].zero();
        x[i] = (seed + threadIdx.x * 8 + i) & M41;
    }
    const uint64_t w = (0x0FEDCBA987654321ull + blockIdx.x) & M41;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            acc[i].mac(x[i], w);
            x[i] ^= acc[i].a & M41;  // one 3-input LOP3 (ALU pipe)
        }
    }
    uint64_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s ^= acc[i].lo64() ^ acc[i].hi64();
    if (s == 0x1234567812345678ull) out[0] = s;
}

// split-FP64 MAC for operands below 2^40: x = xh 2^20 + xl, w = wh 2^20 + wl (20-bit halves held
// exactly in doubles); x w accumulates exactly in three FP64 sums (hh, mid, ll: 40-bit products,
// 2^12 of them fit 53 bits) with 4 DFMA and no carries.  SPLIT: x arrives as a 64-bit integer and
// is split per MAC (2 ALU + 2 DADD), w is pre-split (a bank operand); otherwise both are doubles.
template <bool SPLIT>
__global__ void k_fpsplit_peak(uint64_t *out, int iters, uint64_t seed) {
    double hh[8], mm[8], ll[8];
    uint64_t x[8];
    constexpr uint64_t M40 = (1ull << 40) - 1;
    const uint64_t w = (0x0FEDCBA987654321ull + blockIdx.x) & M40;
    const double wh = (double)(w >> 20), wl = (double)(w & 0xFFFFF);
    const double two52 = 4503599627370496.0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        hh[i] = mm[i] = ll[i] = 0.0;
        x[i] = (seed + threadIdx.x * 8 + i) & M40;
    }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            double xh, xl;
            if (SPLIT) {
                xl = __longlong_as_double((long long)((x[i] & 0xFFFFF) | 0x4330000000000000ull)) - two52;
                xh = __longlong_as_double((long long)((x[i] >> 20) | 0x4330000000000000ull)) - two52;
            } else {
                xl = __longlong_as_double((long long)x[i]);
                xh = xl;
            }
            hh[i] = fma(xh, wh, hh[i]);
            mm[i] = fma(xh, wl, mm[i]);
            mm[i] = fma(xl, wh, mm[i]);
            ll[i] = fma(xl, wl, ll[i]);
            if (SPLIT)
                x[i] ^= (uint64_t)__double_as_longlong(ll[i]) & M40;
            else
                x[i] ^= (uint64_t)__double_as_longlong(ll[i]) & 0x000FFFFF00000000ull;
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s += hh[i] + mm[i] + ll[i];
    if (s == 0.123) out[0] = 1;
}

// u8 tensor-core MACs through the legacy warp-level path the engine uses (mma.sync m16n8k32
// -> IMMA.16832): 8 independent accumulator tiles per warp, 16 * 8 * 32 MACs per instruction
__global__ void k_imma_peak(uint64_t *out, int iters, uint32_t seed) {
    uint32_t a[4], b[2];
#pragma unroll
    for (int i = 0; i < 4; i++) a[i] = seed * (threadIdx.x + i + 1);
#pragma unroll
    for (int i = 0; i < 2; i++) b[i] = seed ^ (threadIdx.x * 7 + i);
    int d[8][4] = {};
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int t = 0; t < 8; t++)
            asm volatile(
                "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};"
                : "+r"(d[t][0]), "+r"(d[t][1]), "+r"(d[t][2]), "+r"(d[t][3])
                : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    int s = 0;
#pragma unroll
    for (int t = 0; t < 8; t++) s += d[t][0] + d[t][1] + d[t][2] + d[t][3];
    if (s == 0x12345) out[0] = (uint64_t)s;
}

// FP64 pipe: dependent-free DFMA streams (8 chains per thread), one FMA per op
__global__ void k_dfma_peak(double *out, int iters, double seed) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = seed + threadIdx.x + i;
    const double a = 0.999999, b = 1e-7;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) x[i] = fma(x[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s += x[i];
    if (s == 1234.5) out[0] = s;
}

// tcgen05.mma kind::i8 throughput: one CTA per SM, one thread issuing M = 128, N = 256, K = 32
// MMAs from shared memory (K-major, no swizzle) into two alternating TMEM accumulators
__global__ void __launch_bounds__(128, 1) k_tc_peak(uint64_t *out, int iters) {
    __shared__ __align__(1024) uint8_t tiles[128 * 32 + 256 * 32];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    for (int i = threadIdx.x; i < (int)sizeof(tiles); i += blockDim.x) tiles[i] = (uint8_t)(i * 7);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const uint32_t bar_a = (uint32_t)__cvta_generic_to_shared(&bar);
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&tbase)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x == 0) {
        auto desc = [](uint32_t a) {
            return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)8 << 16) | ((uint64_t)16 << 32) | ((uint64_t)1 << 46);
        };
        const uint64_t da = desc((uint32_t)__cvta_generic_to_shared(tiles));
        const uint64_t db = desc((uint32_t)__cvta_generic_to_shared(tiles + 128 * 32));
        const uint32_t idesc = (2u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        for (int it = 0; it < iters; it++) {
            const uint32_t d = tbase + (uint32_t)(256 * (it & 1));
            const uint32_t acc = it > 1;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
                "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar_a));
    }
    {
        uint32_t ok = 0;
        while (!ok)
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                : "=r"(ok)
                : "r"(bar_a), "r"(0)
                : "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tbase + ((32u * (threadIdx.x >> 5)) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (v == 0x12345u) out[0] = v;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
}

template <class F> double time_ms(F &&launch) {
    cudaEvent_t a, b;
    UH_CHECK(cudaEventCreate(&a));
    UH_CHECK(cudaEventCreate(&b));
    launch();  // warm-up
    UH_CHECK(cudaEventRecord(a));
    launch();
    UH_CHECK(cudaEventRecord(b));
    UH_CHECK(cudaEventSynchronize(b));
    float ms = 0;
    UH_CHECK(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms;
}

}  // namespace

// rates[0] = IMAD/s, [1] = 128-bit MAC/s, [2] = reduced mulmod/s (60-bit prime), [3] MAC128 plain-C
// form, [4] lazy Shoup product, [5] exact FP64 modMAC, [6] mixed IMAD+FP64 MAC, [7] split-accumulator
// MAC, [8] narrow-operand MAC (q < 2^41), [9] u8 IMMA MAC/s (mma.sync), [10] FP64 FMA/s,
// [11] tcgen05 kind::i8 MAC/s, [12] split-FP64 MAC (one operand split per MAC), [13] split-FP64 MAC
// (both operands pre-split: 4 DFMA)
void bench_peaks(const Ctx &c, double *rates) {
    int sms = 0;
    UH_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
    const int blocks = sms * 8, threads = 256, iters = 4096;
    const double lanes = (double)blocks * threads;
    uint64_t *out = nullptr;
    UH_CHECK(cudaMalloc(&out, 64));
    Mod m;
    UH_CHECK(cudaMemcpy(&m, c.d_mods, sizeof(Mod), cudaMemcpyDeviceToHost));
    double ms = time_ms([&] { k_imad_peak<<<blocks, threads>>>((uint32_t *)out, iters, 7u); });
    rates[0] = lanes * iters * 8 / (ms * 1e-3);
    ms = time_ms([&] { k_mac_peak<<<blocks, threads>>>(out, iters, 7ull); });
    rates[1] = lanes * iters * 8 / (ms * 1e-3);
    ms = time_ms([&] { k_mulmod_peak<<<blocks, threads>>>(out, iters / 2, 7ull, m); });
    rates[2] = lanes * (iters / 2) * 8 / (ms * 1e-3);
    ms = time_ms([&] { k_macc_peak<<<blocks, threads>>>(out, iters, 7ull); });
    rates[3] = lanes * iters * 8 / (ms * 1e-3);
    ms = time_ms([&] { k_shoup_peak<<<blocks, threads>>>(out, iters, 7ull, m); });
    rates[4] = lanes * iters * 8 / (ms * 1e-3);
    const double q40 = 1099511623297.0;  // a 40-bit NTT prime
    ms = time_ms([&] { k_fp64mac_peak<<<blocks, threads>>>((double *)out, iters, 3.0, q40, 1.0 / q40); });
    rates[5] = lanes * iters * 8 / (ms * 1e-3);
    ms = time_ms([&] { k_mixed_peak<<<blocks, threads>>>(out, iters, 7ull, q40, 1.0 / q40); });
    rates[6] = lanes * iters * 8 / (ms * 1e-3);
    ms = time_ms([&] { k_macs_peak<<<blocks, threads>>>(out, iters, 7ull); });
    rates[7] = lanes * iters * 8 / (ms * 1e-3);
    ms = time_ms([&] { k_macn_peak<<<blocks, threads>>>(out, iters, 7ull); });
    rates[8] = lanes * iters * 8 / (ms * 1e-3);
    {  // rates[9]: u8 IMMA MACs/s (mma.sync), 8 warps x 4 CTAs per SM
        const int wb = sms * 4, wt = 256, wi = 1024;
        ms = time_ms([&] { k_imma_peak<<<wb, wt>>>(out, wi, 3u); });
        rates[9] = (double)wb * (wt / 32) * wi * 8 * (16.0 * 8 * 32) / (ms * 1e-3);
    }
    ms = time_ms([&] { k_dfma_peak<<<blocks, threads>>>((double *)out, iters, 1.0); });
    rates[10] = lanes * iters * 8 / (ms * 1e-3);  // FP64 FMA/s
    {  // rates[11]: tcgen05 kind::i8 MACs/s (M = 128, N = 256, K = 32 per instruction)
        const int ti = 2048;
        ms = time_ms([&] { k_tc_peak<<<sms, 128>>>(out, ti); });
        rates[11] = (double)sms * ti * (128.0 * 256 * 32) / (ms * 1e-3);
    }
    // rates[12]: split-FP64 MAC, one operand split per MAC; rates[13]: both operands pre-split
    ms = time_ms([&] { k_fpsplit_peak<true><<<blocks, threads>>>(out, iters, 7ull); });
    rates[12] = lanes * iters * 8 / (ms * 1e-3);
    ms = time_ms([&] { k_fpsplit_peak<false><<<blocks, threads>>>(out, iters, 7ull); });
    rates[13] = lanes * iters * 8 / (ms * 1e-3);
    UH_CHECK(cudaGetLastError());
    cudaFree(out);
}

}  // namespace uh
