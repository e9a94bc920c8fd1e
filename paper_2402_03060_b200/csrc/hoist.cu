// Generic hoisted rotation-MAC kernel (sm_100a): the one kernel behind every
// fused layer path.
//
//   acc[o][b] (QP basis) = sum over terms q of  M[o][q] (.) P * rot_{s_t}(ct_{i}[b])
//
// terms: dense  q = (i, t) for i < I, t < T      (conv: I x T taps, O outputs)
//        diag   q = i = t for i < I (= T)          (sum of differently shifted inputs)
// M: weight masks in the QP basis ([O][Q][L+1][N]), or none (M = 1).
// P * rot_s(ct) is never materialised: for each term the rotated, key-switched
// ciphertext in the QP basis is formed on the fly from the hoisted ModUp
// digits D of the input (a shifted read -- slot order turns X -> X^(5^s) into
// a cyclic shift of each half) and the Galois key of tap t:
//   v0 = P*c0[rot n] + sum_j D_j[rot n] * K_t[j][0],   v1 = sum_j D_j[rot n] * K_t[j][1]
// (shift 0: v = P * ct).  v is staged in shared memory for a tile of TB
// ciphertexts x 32 coefficients and immediately multiply-accumulated into
// every output's 128-bit accumulators, so each mask value read from HBM/L2
// serves 2*TB products and each key value TB ciphertexts.
//
// CTA: W warps; lane <-> coefficient n (coalesced 256-byte rows of every
// operand); grid = (B/TB tiles fastest, N/32 coefficient tiles, L+1 limbs),
// so CTAs sharing the same masks/keys run back to back and hit L2.
#include <type_traits>

#include "ops.cuh"

namespace uh {
namespace {

constexpr int kTBatch = 8;   // ciphertexts per CTA tile
constexpr int kTChunk = 3;   // terms staged per shared-memory chunk (768 items: 2 / 3 per thread at 12 / 8 warps)
constexpr int kFold = 56;    // terms between folds of the 128-bit accumulators

__device__ __forceinline__ uint32_t rot_index(uint32_t n, uint32_t half, uint32_t r) {
    uint32_t h = n >= half ? half : 0;
    uint32_t j = n - h + r;
    j = j >= half ? j - half : j;
    return h + j;
}

// lazily reduced (hi*2^64 + lo) mod q in [0, 4q)
__device__ __forceinline__ uint64_t reduce128_lazy(uint64_t hi, uint64_t lo, const Mod &m) {
    return shoup_lazy(hi, m.r64, m.r64s, m.q) + barrett_lite(lo, m);
}
// A phase-A key sum for a limb with q < 2^41 is below 25 * 2^82 < 2^87, so its high word
// is below 2^23 and (hi * (2^64 mod q) + lo) folds it to a 64-bit value congruent mod q
// with one 32x64 product -- no full reduction (the phase-B accumulators absorb values < 2^64).
__device__ __forceinline__ uint64_t fold64_small(uint64_t hi, uint64_t lo, const Mod &m) {
    const uint64_t p = (uint64_t)(uint32_t)hi * m.r64;
    const uint64_t v = lo + p;
    return v < p ? v + m.r64 : v;  // a wrap past 2^64 is worth 2^64 mod q
}
// phase-A term value: lazily reduced into [0, 2q) (60-bit limbs) or folded below 2^64 (q < 2^41);
// with the narrow-operand accumulator (AccN) the value must itself stay a narrow operand: [0, 2q)
template <class A>
__device__ __forceinline__ uint64_t term_value(const A &a, const Mod &m, bool smallq) {
    uint64_t h, l;
    a.value(h, l);
    if constexpr (std::is_same<A, AccN>::value) return barrett_lite(fold64_small(h, l, m), m);
    return smallq ? fold64_small(h, l, m) : csub(reduce128_lazy(h, l, m), 2 * m.q);
}
// fold a lazily accumulated 128-bit sum back to one word in [0, 4q)
template <class A>
__device__ __forceinline__ void acc_fold(A &a, const Mod &m) {
    uint64_t h, l;
    a.value(h, l);
    a.set(reduce128_lazy(h, l, m), 0);
}
// The accumulator type is chosen per limb (uniform per CTA): limbs with q < 2^41 take the
// narrow-operand form (AccN, 3 IMAD.WIDE + 1 IMAD per multiply-add), the 60-bit limbs
// (q_0, P) the full 128-bit one.
#ifndef UH_NARROW_MAC
#define UH_NARROW_MAC 1
#endif

constexpr int kMaxL = 12;  // phase-A digit loop fully unrolled (predicated) up to this many limbs

// Phase-A key-switch dot product of one rotated term:
//   a0 += sum_j D_j * K[j][0],  a1 += sum_j D_j * K[j][1]   (j < L digits)
// Loads are issued in groups of G digits (3G independent 64-bit loads in flight)
// before any of the group's products: a per-digit load->use chain would
// serialise L round trips to L2 (ncu: long-scoreboard on the first MAC).
#ifndef UH_KS_GROUP_WIDE
#define UH_KS_GROUP_WIDE 2
#endif
#ifndef UH_KS_GROUP_FOR
#define UH_KS_GROUP_FOR(PPW, W) \
    ((PPW) * (W) >= 96 || ((PPW) >= 4 && (W) != 8) ? UH_KS_GROUP_WIDE : ((W) == 8 && (PPW) == 2) ? 2 : 4)
#endif
#ifndef UH_WS_GROUP
#define UH_WS_GROUP 4
#endif
template <int G, class A>
__device__ __forceinline__ void ks_dot(A &a0, A &a1, const uint64_t *Di, uint32_t dstride,
                                       const uint64_t *k0, uint32_t ks, int L) {
#pragma unroll
    for (int j0 = 0; j0 < kMaxL; j0 += G) {
        if (j0 < L) {
            uint64_t d[G], x[G], y[G];
#pragma unroll
            for (int g = 0; g < G; g++) {
                const int j = j0 + g;
                const bool ok = j < L;
                d[g] = ok ? __ldg(Di + j * dstride) : 0;
                x[g] = ok ? __ldg(k0 + (2 * j) * ks) : 0;
                y[g] = ok ? __ldg(k0 + (2 * j + 1) * ks) : 0;
            }
#pragma unroll
            for (int g = 0; g < G; g++) {
                if (j0 + g < L) {
                    a0.mac(d[g], x[g]);
                    a1.mac(d[g], y[g]);
                }
            }
        }
    }
}

// 8-warp CTAs are capped at 64 registers (4 CTAs / SM), 24-warp CTAs at 85 (1 CTA / SM).
// All element offsets are 32-bit (the host checks every operand has < 2^32 elements).
constexpr int kMaxTerms = 512;  // per-term metadata staged in shared memory

// TB: ciphertexts per CTA tile (8; 4 lets two 12-warp CTAs share an SM, so one CTA's
// phase-A latency overlaps the other's phase B without any intra-CTA coupling)
template <int PPW, int W, int TB = kTBatch>
__global__ void __launch_bounds__(W * 32, W == 8 && PPW <= 2 ? 4 : (TB < 8 && W * 2 == TB * 6 ? 24 / W : 1))
    k_hoisted_mac(uint64_t *__restrict__ acc_out, const uint64_t *__restrict__ X, int xls,
                  const uint64_t *__restrict__ D, const uint64_t *__restrict__ masks,
                  const uint64_t *const *__restrict__ keys, const int32_t *__restrict__ key_limbs,
                  const int32_t *__restrict__ shifts, int B, int I, int T, int O, int diag, int L, int sp, int logn,
                  const Mod *__restrict__ mods, int z0 = 0, int zstep = 1) {
    __shared__ uint64_t sv[2][kTChunk][TB][2][32];
    __shared__ const uint64_t *s_key[kMaxTerms];
    __shared__ uint32_t s_shift[kMaxTerms];
    __shared__ uint32_t s_kstride[kMaxTerms];  // key limbs << logn: one key component
    const int LP = L + 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int b0 = blockIdx.x * TB;
    const uint32_t n = blockIdx.y * 32 + lane;
    const int k = z0 + blockIdx.z * zstep;
    const uint32_t N = 1u << logn, half = N >> 1;
    const Mod m = mods[limb_mod(k, L, 0, sp)];
    const bool qlimb = k < L;
    const bool smallq = (m.q >> 41) == 0 && L <= kMaxL;
    const uint64_t P = mods[sp].q;
    const uint64_t Pk = qlimb ? (P < m.q ? P : csub(barrett_lite(P, m), m.q)) : 0;
    const int Q = diag ? I : I * T;
    const int npairs = O * TB;
    for (int t = threadIdx.x; t < T; t += blockDim.x) {
        s_key[t] = keys[t];
        s_shift[t] = (uint32_t)shifts[t];
        s_kstride[t] = (uint32_t)key_limbs[t] << logn;
    }
    __syncthreads();

    auto body = [&](auto acc_tag) {
        using A = decltype(acc_tag);
        A acc[PPW][2];
#pragma unroll
        for (int j = 0; j < PPW; j++) {
            acc[j][0].zero();
            acc[j][1].zero();
        }
        // phase-A load group: bounded by the registers left next to the PPW accumulators
        constexpr int kKsGroup = UH_KS_GROUP_FOR(PPW, W);
        int since_fold = 0;
        int buf = 0;
        constexpr int ITEMS = kTChunk * TB / W;  // phase-A items per thread (1, 2 or 3)
        static_assert(ITEMS * W == kTChunk * TB, "phase-A items must tile the chunk");
        // a warp's PPW (output, ciphertext) pairs form a PO x PB block: each shared-memory v is
        // loaded once for PO outputs and each mask once for PB ciphertexts
        constexpr int PB = (PPW == 4 ? 2 : PPW) < TB ? (PPW == 4 ? 2 : PPW) : TB, PO = PPW / PB, WB = TB / PB;
        const int o_a = (warp / WB) * PO, b_a = (warp % WB) * PB;
        const bool warp_active = o_a < O && warp * PPW < npairs;
        const uint32_t dstride = (uint32_t)LP << logn;  // between digits of one D block
        const uint32_t mask_row = ((uint32_t)k << logn) + n;
        int i0 = 0, t0 = 0;  // (input, tap) of term q0, advanced incrementally (no runtime division)
        for (int q0 = 0; q0 < Q; q0 += kTChunk) {
            // prefetch this chunk's weight masks (consumed after the barrier, latency hidden by phase A)
            uint64_t mpre[kTChunk][PO];
#pragma unroll
            for (int qc = 0; qc < kTChunk; qc++)
#pragma unroll
                for (int d = 0; d < PO; d++)
                    mpre[qc][d] = (masks && warp_active && o_a + d < O && q0 + qc < Q)
                                      ? masks[(((uint32_t)(o_a + d) * Q + q0 + qc) * dstride) + mask_row]
                                      : 0;
            // ---- phase A: rotated, key-switched inputs of this chunk into shared memory ----
#pragma unroll
            for (int ii = 0; ii < ITEMS; ii++) {
                const int it = threadIdx.x + ii * W * 32;
                const int ln = it & 31, rest = it >> 5;
                const int bt = rest % TB, qc = rest / TB;
                const int q = q0 + qc, b = b0 + bt;
                uint64_t v0 = 0, v1 = 0;
                if (q < Q && b < B) {
                    int i, t;
                    if (diag) {
                        i = t = q;
                    } else {
                        i = i0;
                        t = t0 + qc;
                        while (t >= T) {
                            t -= T;
                            i++;
                        }
                    }
                    const uint32_t nn = blockIdx.y * 32 + ln;
                    const uint32_t ib = (uint32_t)(i * B + b);
                    const uint64_t *c0 = X + ((ib * 2 * (uint32_t)xls + (uint32_t)k) << logn);
                    const uint32_t r = s_shift[t];
                    if (r == 0) {
                        if (qlimb) {
                            v0 = mulmod(Pk, c0[nn], m);
                            v1 = mulmod(Pk, c0[((uint32_t)xls << logn) + nn], m);
                        }
                    } else {
                        const uint32_t src = rot_index(nn, half, r);
                        const uint64_t *Di = D + (((ib * (uint32_t)L) * LP + k) << logn) + src;
                        const uint32_t ks = s_kstride[t];
                        const uint64_t *k0 = s_key[t] + (qlimb ? ((uint32_t)k << logn) : ks - N) + nn;
                        A a0, a1;
                        a0.zero();
                        a1.zero();
                        ks_dot<kKsGroup>(a0, a1, Di, dstride, k0, ks, L);
                        if (qlimb) a0.mac(Pk, c0[src]);
                        v0 = term_value(a0, m, smallq);
                        v1 = term_value(a1, m, smallq);
                    }
                }
                sv[buf][qc][bt][0][ln] = v0;
                sv[buf][qc][bt][1][ln] = v1;
            }
            __syncthreads();
            // ---- phase B: multiply-accumulate into every (output, ciphertext) pair ----
            const int qn = min(kTChunk, Q - q0);
#pragma unroll
            for (int qc = 0; qc < kTChunk; qc++) {
                if (qc >= qn) break;
                if (warp_active) {
#pragma unroll
                    for (int db = 0; db < PB; db++) {
                        const int bt = b_a + db;
                        const uint64_t v0 = sv[buf][qc][bt][0][lane], v1 = sv[buf][qc][bt][1][lane];
#pragma unroll
                        for (int d = 0; d < PO; d++) {
                            const int j = d * PB + db;
                            if (masks) {
                                acc[j][0].mac(mpre[qc][d], v0);
                                acc[j][1].mac(mpre[qc][d], v1);
                            } else {
                                acc[j][0].add(v0);
                                acc[j][1].add(v1);
                            }
                        }
                    }
                }
                if (++since_fold == kFold) {
                    since_fold = 0;
#pragma unroll
                    for (int j = 0; j < PPW; j++)
                        for (int cc = 0; cc < 2; cc++) acc_fold(acc[j][cc], m);
                }
            }
            buf ^= 1;  // the other buffer is free: every thread passed the barrier after using it
            t0 += kTChunk;
            while (t0 >= T) {
                t0 -= T;
                i0++;
            }
        }
#pragma unroll
        for (int j = 0; j < PPW; j++) {
            const int o = o_a + j / PB, b = b0 + b_a + j % PB;
            if (warp_active && o < O) {
                if (b < B) {
                    uint64_t *dst = acc_out + (((uint32_t)(o * B + b) * 2 * LP + k) << logn) + n;
                    dst[0] = acc[j][0].reduce(m);
                    dst[dstride] = acc[j][1].reduce(m);
                }
            }
        }
    };
#if UH_NARROW_MAC
    if (smallq)
        body(AccN{});
    else
#endif
        body(Acc{});
}

// ---------------------------------------------------------------------------
// Pipelined variant: the next chunk's operands (hoisted digits at the rotated
// offsets, c0, and the Galois-key rows) are staged into shared memory with
// cp.async while the current chunk is multiply-accumulated, so phase A reads
// shared memory instead of waiting on L2/HBM.  Warp g of the chunk owns item
// group (term qc = g / 8, ciphertext bt = g % 8) for both copy and compute.
__device__ __forceinline__ void cp8(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int NW> __device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(NW)); }

template <int PPW, int W>
__global__ void __launch_bounds__(W * 32, 1)
    k_hoisted_mac_cp(uint64_t *__restrict__ acc_out, const uint64_t *__restrict__ X, int xls,
                     const uint64_t *__restrict__ D, const uint64_t *__restrict__ masks,
                     const uint64_t *const *__restrict__ keys, const int32_t *__restrict__ key_limbs,
                     const int32_t *__restrict__ shifts, int B, int I, int T, int O, int diag, int L, int sp,
                     int logn, const Mod *__restrict__ mods, int z0 = 0, int zstep = 1) {
    extern __shared__ uint64_t dyn[];
    __shared__ uint64_t sv[2][kTChunk][kTBatch][2][32];
    __shared__ const uint64_t *s_key[kMaxTerms];
    __shared__ uint32_t s_shift[kMaxTerms];
    __shared__ uint32_t s_kstride[kMaxTerms];
    const int LP = L + 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int b0 = blockIdx.x * kTBatch;
    const uint32_t n = blockIdx.y * 32 + lane;
    const int k = z0 + blockIdx.z * zstep;
    const uint32_t N = 1u << logn, half = N >> 1;
    const Mod m = mods[limb_mod(k, L, 0, sp)];
    const bool qlimb = k < L;
    const uint64_t P = mods[sp].q;
    const uint64_t Pk = qlimb ? (P < m.q ? P : csub(barrett_lite(P, m), m.q)) : 0;
    const bool smallq = (m.q >> 41) == 0 && L <= kMaxL;
    const int Q = diag ? I : I * T;
    const int npairs = O * kTBatch;
    for (int t = threadIdx.x; t < T; t += blockDim.x) {
        s_key[t] = keys[t];
        s_shift[t] = (uint32_t)shifts[t];
        s_kstride[t] = (uint32_t)key_limbs[t] << logn;
    }
    // stage layout (uint64 words): D [kTChunk][kTBatch][L][32], C [kTChunk][kTBatch][32], K [kTChunk][2L][32]
    const int szD = kTChunk * kTBatch * L * 32, szC = kTChunk * kTBatch * 32, szK = kTChunk * 2 * L * 32;
    const int stage = szD + szC + szK;
    __syncthreads();

    const uint32_t dstride = (uint32_t)LP << logn;
    // (input, tap) of a term q, from the running (i0, t0) of q0
    auto term_it = [&](int i0, int t0, int qc, int &i, int &t) {
        if (diag) {
            i = t = 0;  // set by caller
        } else {
            i = i0;
            t = t0 + qc;
            while (t >= T) {
                t -= T;
                i++;
            }
        }
    };
    auto issue = [&](int q0, int i0, int t0, int s) {
        uint64_t *sD = dyn + s * stage, *sC = sD + szD, *sK = sC + szC;
        for (int g = warp; g < kTChunk * kTBatch; g += W) {
            const int qc = g / kTBatch, bt = g % kTBatch, q = q0 + qc, b = b0 + bt;
            if (q >= Q || b >= B) continue;
            int i, t;
            term_it(i0, t0, qc, i, t);
            if (diag) i = t = q;
            const uint32_t ib = (uint32_t)(i * B + b);
            const uint64_t *c0 = X + ((ib * 2 * (uint32_t)xls + (uint32_t)k) << logn);
            const uint32_t r = s_shift[t];
            const uint32_t src = r ? rot_index(n, half, r) : n;
            uint64_t *dD = sD + ((qc * kTBatch + bt) * L) * 32 + lane;
            if (qlimb) cp8(sC + (qc * kTBatch + bt) * 32 + lane, c0 + src);
            if (r == 0) {
                if (qlimb) cp8(dD, c0 + ((uint32_t)xls << logn) + n);  // c1, unrotated
            } else {
                const uint64_t *Di = D + (((ib * (uint32_t)L) * LP + k) << logn) + src;
                for (int j = 0; j < L; j++) cp8(dD + j * 32, Di + j * dstride);
            }
        }
        for (int row = warp; row < kTChunk * 2 * L; row += W) {
            const int qc = row / (2 * L), jc = row % (2 * L), q = q0 + qc;
            if (q >= Q) continue;
            int i, t;
            term_it(i0, t0, qc, i, t);
            if (diag) t = q;
            if (s_shift[t] == 0) continue;
            const uint32_t ks = s_kstride[t];
            const uint64_t *k0 = s_key[t] + (qlimb ? ((uint32_t)k << logn) : ks - N) + n;
            cp8(sK + row * 32 + lane, k0 + jc * ks);
        }
    };

    Acc acc[PPW][2];
#pragma unroll
    for (int j = 0; j < PPW; j++) {
        acc[j][0].zero();
        acc[j][1].zero();
    }
    int since_fold = 0;
    int buf = 0;
    constexpr int PB = PPW == 4 ? 2 : PPW, PO = PPW / PB, WB = kTBatch / PB;
    const int o_a = (warp / WB) * PO, b_a = (warp % WB) * PB;
    const bool warp_active = o_a < O && warp * PPW < npairs;
    const uint32_t mask_row = ((uint32_t)k << logn) + n;
    int i0 = 0, t0 = 0;
    issue(0, 0, 0, 0);
    cp_commit();
    int st = 0;
    for (int q0 = 0; q0 < Q; q0 += kTChunk) {
        // next chunk's (i0, t0)
        int i1 = i0, t1 = t0 + kTChunk;
        while (t1 >= T) {
            t1 -= T;
            i1++;
        }
        if (q0 + kTChunk < Q) issue(q0 + kTChunk, i1, t1, st ^ 1);
        cp_commit();
        uint64_t mpre[kTChunk][PO];
#pragma unroll
        for (int qc = 0; qc < kTChunk; qc++)
#pragma unroll
            for (int d = 0; d < PO; d++)
                mpre[qc][d] = (masks && warp_active && o_a + d < O && q0 + qc < Q)
                                  ? masks[(((uint32_t)(o_a + d) * Q + q0 + qc) * dstride) + mask_row]
                                  : 0;
        cp_wait<1>();
        __syncthreads();
        // ---- phase A from shared memory ----
        const uint64_t *sD = dyn + st * stage, *sC = sD + szD, *sK = sC + szC;
        for (int g = warp; g < kTChunk * kTBatch; g += W) {
            const int qc = g / kTBatch, bt = g % kTBatch, q = q0 + qc, b = b0 + bt;
            uint64_t v0 = 0, v1 = 0;
            if (q < Q && b < B) {
                int i, t;
                term_it(i0, t0, qc, i, t);
                if (diag) t = q;
                const uint32_t r = s_shift[t];
                const uint64_t *dD = sD + ((qc * kTBatch + bt) * L) * 32 + lane;
                if (r == 0) {
                    if (qlimb) {
                        v0 = mulmod(Pk, sC[(qc * kTBatch + bt) * 32 + lane], m);
                        v1 = mulmod(Pk, dD[0], m);
                    }
                } else {
                    const uint64_t *kK = sK + (qc * 2 * L) * 32 + lane;
                    Acc a0, a1;
                    a0.zero();
                    a1.zero();
#pragma unroll 4
                    for (int j = 0; j < L; j++) {
                        const uint64_t d = dD[j * 32];
                        a0.mac(d, kK[(2 * j) * 32]);
                        a1.mac(d, kK[(2 * j + 1) * 32]);
                    }
                    if (qlimb) a0.mac(Pk, sC[(qc * kTBatch + bt) * 32 + lane]);
                    v0 = term_value(a0, m, smallq);
                    v1 = term_value(a1, m, smallq);
                }
            }
            sv[buf][qc][bt][0][lane] = v0;
            sv[buf][qc][bt][1][lane] = v1;
        }
        __syncthreads();
        // ---- phase B ----
        const int qn = min(kTChunk, Q - q0);
#pragma unroll
        for (int qc = 0; qc < kTChunk; qc++) {
            if (qc >= qn) break;
            if (warp_active) {
#pragma unroll
                for (int db = 0; db < PB; db++) {
                    const int bt = b_a + db;
                    const uint64_t v0 = sv[buf][qc][bt][0][lane], v1 = sv[buf][qc][bt][1][lane];
#pragma unroll
                    for (int d = 0; d < PO; d++) {
                        const int j = d * PB + db;
                        if (masks) {
                            acc[j][0].mac(mpre[qc][d], v0);
                            acc[j][1].mac(mpre[qc][d], v1);
                        } else {
                            acc[j][0].add(v0);
                            acc[j][1].add(v1);
                        }
                    }
                }
            }
            if (++since_fold == kFold) {
                since_fold = 0;
#pragma unroll
                for (int j = 0; j < PPW; j++)
                    for (int cc = 0; cc < 2; cc++) {
                        uint64_t rr = reduce128_lazy(acc[j][cc].hi64(), acc[j][cc].lo64(), m);
                        acc[j][cc].set(rr, 0);
                    }
            }
        }
        buf ^= 1;
        st ^= 1;
        i0 = i1;
        t0 = t1;
    }
    cp_wait<0>();
#pragma unroll
    for (int j = 0; j < PPW; j++) {
        const int o = o_a + j / PB, b = b0 + b_a + j % PB;
        if (warp_active && o < O && b < B) {
            uint64_t *dst = acc_out + (((uint32_t)(o * B + b) * 2 * LP + k) << logn) + n;
            dst[0] = acc[j][0].reduce(m);
            dst[dstride] = acc[j][1].reduce(m);        }
    }
}

// ---------------------------------------------------------------------------
// Direct variant for narrow layers (O <= 2: pooling rotation sums, flatten and
// FC stages): one thread per (ciphertext, limb, coefficient) walks all terms
// with everything in registers -- no shared-memory staging, no barriers.
// Without masks (rotation sums) the key products of every term accumulate into
// one 128-bit accumulator per component and are reduced once; with masks each
// term is reduced and multiply-accumulated into the O output accumulators.
// Warp w of the CTA serves ciphertext 8 * blockIdx.y + w at the same 32
// coefficients, so key and mask rows are shared through L1; the coefficient
// tile is the fastest grid dimension (rotated digit reads of neighbouring
// tiles hit L2).
#ifndef UH_DIRECT_CT_FAST
#define UH_DIRECT_CT_FAST 1  // ciphertext groups fastest in the grid (measured: conv1 16.0 vs 16.8 ms)
#endif
#ifndef UH_DIRECT_MINB
#define UH_DIRECT_MINB 4
#endif
#ifndef UH_DIRECT_G
#define UH_DIRECT_G 4
#endif
#ifndef UH_DIRECT_G4
#define UH_DIRECT_G4 4  // load group of the 3..4-output direct kernel (4: a few spills, measured faster than 2)
#endif
template <int OM, bool MASKS>
__global__ void __launch_bounds__(256, OM > 2 ? 3 : UH_DIRECT_MINB)
    k_hoisted_direct(uint64_t *__restrict__ acc_out, const uint64_t *__restrict__ X, int xls,
                     const uint64_t *__restrict__ D, const uint64_t *__restrict__ masks,
                     const uint64_t *const *__restrict__ keys, const int32_t *__restrict__ key_limbs,
                     const int32_t *__restrict__ shifts, int B, int I, int T, int O, int diag, int L, int sp,
                     int logn, const Mod *__restrict__ mods) {
    __shared__ const uint64_t *s_key[kMaxTerms];
    __shared__ uint32_t s_shift[kMaxTerms];
    __shared__ uint32_t s_kstride[kMaxTerms];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#if UH_DIRECT_CT_FAST
    const int b = blockIdx.x * 8 + warp;  // ciphertext groups fastest: CTAs sharing key rows run together
    const uint32_t n = blockIdx.y * 32 + lane;
#else
    const int b = blockIdx.y * 8 + warp;
    const uint32_t n = blockIdx.x * 32 + lane;
#endif
    const int k = blockIdx.z;
    const uint32_t N = 1u << logn, half = N >> 1;
    const int NT = diag == 2 ? I * T : T;  // per-term metadata entries
    for (int t = threadIdx.x; t < NT; t += blockDim.x) {
        s_key[t] = keys[t];
        s_shift[t] = (uint32_t)shifts[t];
        s_kstride[t] = (uint32_t)key_limbs[t] << logn;
    }
    __syncthreads();
    if (b >= B) return;
    const int LP = L + 1;
    const Mod m = mods[limb_mod(k, L, 0, sp)];
    const bool qlimb = k < L;
    const bool smallq = (m.q >> 41) == 0 && L <= kMaxL;
    const uint64_t P = mods[sp].q;
    const uint64_t Pk = qlimb ? (P < m.q ? P : csub(barrett_lite(P, m), m.q)) : 0;
    const int Q = diag == 1 ? I : I * T;
    const uint32_t dstride = (uint32_t)LP << logn;
    const uint32_t mask_row = ((uint32_t)k << logn) + n;
    auto body = [&](auto acc_tag) {
        using A = decltype(acc_tag);
        A acc[OM][2];
#pragma unroll
        for (int o = 0; o < OM; o++) {
            acc[o][0].zero();
            acc[o][1].zero();
        }
        int i = 0, t = 0, since = 0;
        for (int q = 0; q < Q; q++) {
            if (diag == 1) {
                i = t = q;
            } else if (diag == 2) {  // block-diagonal: input q / T with its own tap q
                t = q;
                i = q / T;
            }
            const uint32_t ib = (uint32_t)(i * B + b);
            const uint64_t *c0 = X + ((ib * 2 * (uint32_t)xls + (uint32_t)k) << logn);
            const uint32_t r = s_shift[t];
            uint64_t mk[OM];
            if (MASKS) {
#pragma unroll
                for (int o = 0; o < OM; o++)
                    mk[o] = o < O ? __ldg(masks + ((uint32_t)o * Q + q) * dstride + mask_row) : 0;
            }
            A a0, a1;
            a0.zero();
            a1.zero();
            if (r == 0) {
                if (qlimb) {
                    a0.mac(Pk, __ldg(c0 + n));
                    a1.mac(Pk, __ldg(c0 + ((uint32_t)xls << logn) + n));
                }
            } else {
                const uint32_t src = rot_index(n, half, r);
                const uint64_t *Di = D + (((ib * (uint32_t)L) * LP + k) << logn) + src;
                const uint32_t ks = s_kstride[t];
                const uint64_t *k0 = s_key[t] + (qlimb ? ((uint32_t)k << logn) : ks - N) + n;
                ks_dot<(OM > 2 ? UH_DIRECT_G4 : UH_DIRECT_G)>(a0, a1, Di, dstride, k0, ks, L);
                if (qlimb) a0.mac(Pk, __ldg(c0 + src));
            }
            if (MASKS) {
                const uint64_t v0 = term_value(a0, m, smallq);
                const uint64_t v1 = term_value(a1, m, smallq);
#pragma unroll
                for (int o = 0; o < OM; o++) {
                    acc[o][0].mac(mk[o], v0);
                    acc[o][1].mac(mk[o], v1);
                }
                if (++since == kFold) {
                    since = 0;
#pragma unroll
                    for (int o = 0; o < OM; o++)
                        for (int cc = 0; cc < 2; cc++) acc_fold(acc[o][cc], m);
                }
            } else {
                // fold the term's 128-bit sums (each < (2L + 1) q^2 < 2^125) into the running sum
                uint64_t h0, l0, h1, l1;
                a0.value(h0, l0);
                a1.value(h1, l1);
                const uint64_t v0 = smallq ? fold64_small(h0, l0, m) : reduce128_lazy(h0, l0, m);
                const uint64_t v1 = smallq ? fold64_small(h1, l1, m) : reduce128_lazy(h1, l1, m);
                acc[0][0].add(v0);
                acc[0][1].add(v1);
            }
            if (diag == 0 && ++t == T) {
                t = 0;
                i++;
            }
        }
#pragma unroll
        for (int o = 0; o < OM; o++) {
            if (o < O) {
                uint64_t *dst = acc_out + (((uint32_t)(o * B + b) * 2 * LP + k) << logn) + n;
                dst[0] = acc[o][0].reduce(m);
                dst[dstride] = acc[o][1].reduce(m);
            }
        }
    };
#if UH_NARROW_MAC
    if (smallq)
        body(AccN{});
    else
#endif
        body(Acc{});
}

}  // namespace

void hoisted_mac(const Ctx &c, uint64_t *acc, const uint64_t *X, int xls, const uint64_t *D, const uint64_t *masks,
                 const uint64_t *const *keys, const int32_t *key_limbs, const int32_t *shifts, int B, int I, int T,
                 int O, int diag, int level, cudaStream_t s) {
    const int L = level + 1;
    if (L > kMaxL) throw std::invalid_argument("hoisted kernel supports up to 12 live limbs");
    if ((diag == 2 ? I * T : T) > kMaxTerms) throw std::invalid_argument("hoisted kernel supports up to 512 taps");
    if (diag < 0 || diag > 2) throw std::invalid_argument("hoisted kernel: term mode must be 0, 1 or 2");
    if (diag == 2 && O > 2)
        throw std::invalid_argument("block-diagonal terms (per-input taps) are supported for up to 2 outputs");
    const double lim = 4294967295.0;  // 32-bit element offsets inside the kernel
    if ((double)I * B * 2 * xls * c.n > lim || (double)I * B * L * (L + 1) * c.n > lim ||
        (double)O * B * 2 * (L + 1) * c.n > lim || (double)O * (diag == 1 ? I : I * T) * (L + 1) * c.n > lim)
        throw std::invalid_argument("hoisted kernel operand exceeds 2^32 elements: split the batch");
    const int pairs = O * kTBatch;
    dim3 grid((B + kTBatch - 1) / kTBatch, (unsigned)(c.n / 32), L + 1);
    if (c.n < 32) throw std::invalid_argument("hoisted kernels need N >= 32");
    // warps x pairs-per-warp covering O * TB (output, ciphertext) pairs; every warp serves one output.
    // "wide" (default): 24 warps (register cap 85 -> 24 resident warps / SM for latency hiding);
    // "narrow": 8 or 12 warps with up to 8 pairs each (UH_HOIST_CFG=narrow).
    static const bool narrow = [] {
        const char *e = getenv("UH_HOIST_CFG");
        return e && std::string(e) == "narrow";
    }();
    // cp.async-pipelined variant: measured faster where phase A (key products over many
    // digits) dominates -- the 24-warp, 2-pair configuration (e.g. LeNet conv1 at level 7);
    // UH_HOIST_ASYNC=1 / 0 forces it on / off everywhere.
    static const int async_mode = [] {
        const char *e = getenv("UH_HOIST_ASYNC");
        return e ? (std::string(e) == "0" ? 0 : 1) : -1;
    }();
    auto go = [&](auto ppw_tag, auto w_tag) {
        constexpr int PP = decltype(ppw_tag)::value, WW = decltype(w_tag)::value;
        const bool async = async_mode >= 0 ? async_mode == 1 : (WW == 24 && PP == 2);
        if (async) {
            // two cp.async stages: D [3][8][L][32] + C [3][8][32] + K [3][2L][32] words each
            const size_t smem = 2 * (size_t)(kTChunk * kTBatch * L * 32 + kTChunk * kTBatch * 32 +
                                             kTChunk * 2 * L * 32) * sizeof(uint64_t);
            // opt in to > 48 KB dynamic shared memory once per device, at the largest L (12): 192 KB
            smem_optin(k_hoisted_mac_cp<PP, WW>,
                       2 * (size_t)(kTChunk * kTBatch * 12 * 32 + kTChunk * kTBatch * 32 + kTChunk * 2 * 12 * 32) *
                           sizeof(uint64_t));
            k_hoisted_mac_cp<PP, WW><<<grid, WW * 32, smem, s>>>(acc, X, xls, D, masks, keys, key_limbs, shifts, B,
                                                                 I, T, O, diag, L, c.sp(), (int)c.logn, c.d_mods);
        } else {
            k_hoisted_mac<PP, WW><<<grid, WW * 32, 0, s>>>(acc, X, xls, D, masks, keys, key_limbs, shifts, B, I, T,
                                                          O, diag, L, c.sp(), (int)c.logn, c.d_mods);
        }
    };
    using std::integral_constant;
    // narrow layers (O <= 2): direct register-only kernel (UH_HOIST_DIRECT=0 disables)
    static const bool direct_on = [] {
        const char *e = getenv("UH_HOIST_DIRECT");
        return !(e && std::string(e) == "0");
    }();
    // 3..4-output masked layers (e.g. LeNet conv1: phase-A heavy, 4 outputs) on the direct kernel:
    // measured conv1 layer 17.2 vs 21.5 ms (cp.async 24-warp kernel) at B = 64.  UH_HOIST_DIRECT4=0 disables.
    static const bool direct4 = [] {
        const char *e = getenv("UH_HOIST_DIRECT4");
        return !(e && std::string(e) == "0");
    }();
    if (direct4 && masks && O > 2 && O <= 4) {
        dim3 gd = UH_DIRECT_CT_FAST ? dim3((B + 7) / 8, (unsigned)(c.n / 32), L + 1)
                                    : dim3((unsigned)(c.n / 32), (B + 7) / 8, L + 1);
        k_hoisted_direct<4, true><<<gd, 256, 0, s>>>(acc, X, xls, D, masks, keys, key_limbs, shifts, B, I, T, O, diag,
                                                      L, c.sp(), (int)c.logn, c.d_mods);
        UH_LAUNCH_CHECK();
        return;
    }
    if ((direct_on || diag == 2) && O <= 2) {
        dim3 gd = UH_DIRECT_CT_FAST ? dim3((B + 7) / 8, (unsigned)(c.n / 32), L + 1)
                                    : dim3((unsigned)(c.n / 32), (B + 7) / 8, L + 1);
        if ((B + 7) / 8 > 65535 && !UH_DIRECT_CT_FAST)
            throw std::invalid_argument("hoisted kernel: batch too large for one launch");
        if (masks) {
            if (O == 1)
                k_hoisted_direct<1, true><<<gd, 256, 0, s>>>(acc, X, xls, D, masks, keys, key_limbs, shifts, B, I, T,
                                                              O, diag, L, c.sp(), (int)c.logn, c.d_mods);
            else
                k_hoisted_direct<2, true><<<gd, 256, 0, s>>>(acc, X, xls, D, masks, keys, key_limbs, shifts, B, I, T,
                                                              O, diag, L, c.sp(), (int)c.logn, c.d_mods);
        } else {
            if (O != 1) {
                // identical unmasked outputs: compute one, copy the rest
                k_hoisted_direct<1, false><<<gd, 256, 0, s>>>(acc, X, xls, D, masks, keys, key_limbs, shifts, B, I,
                                                               T, 1, diag, L, c.sp(), (int)c.logn, c.d_mods);
                UH_LAUNCH_CHECK();
                const size_t one = (size_t)B * 2 * (L + 1) * c.n;
                for (int o = 1; o < O; o++)
                    UH_CHECK(cudaMemcpyAsync(acc + o * one, acc, one * 8, cudaMemcpyDeviceToDevice, s));
                return;
            }
            k_hoisted_direct<1, false><<<gd, 256, 0, s>>>(acc, X, xls, D, masks, keys, key_limbs, shifts, B, I, T, 1,
                                                           diag, L, c.sp(), (int)c.logn, c.d_mods);
        }
        UH_LAUNCH_CHECK();
        return;
    }
    if (O <= 12) {
        // measured (B200, N=2^15): 24 warps win when phase B is heavy (O >= 3), 8-warp CTAs when it is not
        if (narrow || O <= 2) {
            const int ppw = pairs > 32 ? 8 : (pairs > 16 ? 4 : (pairs > 8 ? 2 : 1));
            if (ppw == 1) go(integral_constant<int, 1>(), integral_constant<int, 8>());
            else if (ppw == 2) go(integral_constant<int, 2>(), integral_constant<int, 8>());
            else if (ppw == 4) go(integral_constant<int, 4>(), integral_constant<int, 8>());
            else go(integral_constant<int, 8>(), integral_constant<int, 12>());
        } else {
            const int ppw = pairs > 48 ? 4 : (pairs > 24 ? 2 : 1);
            if (ppw == 1) go(integral_constant<int, 1>(), integral_constant<int, 24>());
            else if (ppw == 2) go(integral_constant<int, 2>(), integral_constant<int, 24>());
            else {
                // ciphertexts per CTA tile for the widest layers (UH_HOIST_TB): 2 (default: four
                // 6-warp CTAs per SM, so one CTA's phase-A latency overlaps the others' phase B
                // with no barrier coupling between them), 4 (two 12-warp CTAs), 1 (eight 3-warp
                // CTAs) or 8 (one 24-warp CTA).  Measured LeNet conv2 at B = 64 (B200):
                // 62.4 / 66.5 / 81.4 / 72.2 ms.
                static const int tbw = [] {
                    const char *e = getenv("UH_HOIST_TB");
                    return e ? atoi(e) : 2;
                }();
                if (tbw == 4 && O > 6) {
                    dim3 g4((B + 3) / 4, grid.y, grid.z);
                    k_hoisted_mac<4, 12, 4><<<g4, 12 * 32, 0, s>>>(acc, X, xls, D, masks, keys, key_limbs, shifts, B, I,
                                                                  T, O, diag, L, c.sp(), (int)c.logn, c.d_mods);
                } else if (tbw == 1 && O > 6) {
                    dim3 g1((unsigned)B, grid.y, grid.z);
                    k_hoisted_mac<4, 3, 1><<<g1, 3 * 32, 0, s>>>(acc, X, xls, D, masks, keys, key_limbs, shifts, B, I,
                                                                T, O, diag, L, c.sp(), (int)c.logn, c.d_mods);
                } else if (tbw == 2 && O > 6) {
                    dim3 g2((B + 1) / 2, grid.y, grid.z);
                    k_hoisted_mac<4, 6, 2><<<g2, 6 * 32, 0, s>>>(acc, X, xls, D, masks, keys, key_limbs, shifts, B, I,
                                                                T, O, diag, L, c.sp(), (int)c.logn, c.d_mods);
                } else {
                    go(integral_constant<int, 4>(), integral_constant<int, 24>());
                }
            }
        }
    } else {
        // very wide layers: split the outputs in groups of 12 (12 warps x 8 pairs)
        for (int o0 = 0; o0 < O; o0 += 12) {
            int oc = std::min(12, O - o0);
            hoisted_mac(c, acc + (size_t)o0 * B * 2 * (L + 1) * c.n, X, xls, D,
                        masks ? masks + (size_t)o0 * (diag ? I : I * T) * (L + 1) * c.n : nullptr, keys, key_limbs,
                        shifts, B, I, T, oc, diag, level, s);
        }
        return;
    }
    UH_LAUNCH_CHECK();
}

}  // namespace uh
