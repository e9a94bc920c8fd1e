// Hoisted rotation-MAC over a per-layer key bank, with compile-time strides
// (sm_100a).  Same algorithm and result as hoist.cu's k_hoisted_mac (dense
// terms, weight masks):
//
//   acc[o][b] (QP basis) = sum over terms q = (i, t) of  M[o][q] (.) P * rot_{s_t}(ct_i[b])
//
// What differs is the addressing.  The generic kernel takes one pointer per
// Galois key (keys generated at their first-use level, so every key has its own
// limb count) and runtime N / L, which costs ~2 integer instructions of address
// arithmetic per 64-bit operand load -- more issue slots than the modular
// multiply-accumulates themselves once they use the narrow-operand form.  Here
//   * the layer's keys are re-laid once into a bank kb[T][L+1][2L][N]
//     (limb-major, (digit, component) inner), truncated to the layer's level,
//     so the 2L key rows a thread needs for limb k sit at compile-time offsets
//     (2j + c) * N from one base pointer;
//   * L and N are template parameters, so the hoisted digits D_j (stride
//     (L+1) N), the masks (stride (L+1) N per term) and the c1 rows are all
//     immediate offsets as well;
//   * per-term offsets (input block, key block, shift) are tabulated once per
//     CTA in shared memory -- no (input, tap) decode in the loop.
// CTA tile: TB = 2 ciphertexts x 32 coefficients x one limb; W = 6 warps; a
// chunk of 3 terms is key-switched (phase A, one item per warp) into shared
// memory, then every warp multiply-accumulates its 2 outputs x 2 ciphertexts
// (phase B).  Four CTAs per SM overlap one CTA's phase-A latency with the
// others' phase B.
#include <type_traits>

#include "ops.cuh"

namespace uh {
namespace {

#ifndef UH_BANK_CHUNK
#define UH_BANK_CHUNK 3
#endif
#ifndef UH_BANK_TB
#define UH_BANK_TB 2
#endif
constexpr int kChunk = UH_BANK_CHUNK;        // terms per shared-memory chunk
constexpr int kFoldChunks = 54 / kChunk;     // 54 terms between folds of the 128-bit accumulators
constexpr int kBankMaxTerms = 512;
#ifndef UH_BANK_MINB
#define UH_BANK_MINB 3  // resident CTAs per SM requested from ptxas (3: 96 registers, no spills; measured 51.9 vs 52.8 ms at 4)
#endif
#ifndef UH_BANK_DIRECT_MINB
#define UH_BANK_DIRECT_MINB 4  // narrow layers (<= 2 outputs): 64 registers, no spills (flatten 22.2 vs 22.7 ms, pools -0.2 ms at B = 64)
#endif
#ifndef UH_BANK_DIRECT_G
#define UH_BANK_DIRECT_G 4  // digits per load group (measured G = 4 at 62 registers: narrow MAC calls 27.6 vs 28.0 ms)
#endif
#ifndef UH_BANK_DIRECT4_G
#define UH_BANK_DIRECT4_G 8  // 3-4-output layers (LeNet conv1): every digit's loads in flight
#endif
#ifndef UH_BANK_DIRECT4_MINB
#define UH_BANK_DIRECT4_MINB 2
#endif
#ifndef UH_BANK_G
#define UH_BANK_G 6  // phase-A load group (digits): all of a term's loads in flight for L <= 6
#endif

__device__ __forceinline__ uint32_t rot_index_b(uint32_t n, uint32_t half, uint32_t r) {
    uint32_t h = n >= half ? half : 0;
    uint32_t j = n - h + r;
    j = j >= half ? j - half : j;
    return h + j;
}
__device__ __forceinline__ uint64_t fold64_b(uint64_t hi, uint64_t lo, const Mod &m) {
    const uint64_t p = (uint64_t)(uint32_t)hi * m.r64;
    const uint64_t v = lo + p;
    return v < p ? v + m.r64 : v;
}
__device__ __forceinline__ uint64_t reduce128_lazy_b(uint64_t hi, uint64_t lo, const Mod &m) {
    return shoup_lazy(hi, m.r64, m.r64s, m.q) + barrett_lite(lo, m);
}

template <int L, int LOGN, int W, int TB, int G>
__global__ void __launch_bounds__(W * 32, UH_BANK_MINB)
    k_hoisted_bank(uint64_t *__restrict__ acc_out, const uint64_t *__restrict__ X, const uint64_t *__restrict__ D,
                   const uint64_t *__restrict__ masks, const uint64_t *__restrict__ kbank,
                   const int32_t *__restrict__ shifts, int B, int I, int T, int O, int sp,
                   const Mod *__restrict__ mods, int wide_only) {
    constexpr int LP = L + 1;
    constexpr uint32_t N = 1u << LOGN, half = N >> 1;
    constexpr uint32_t ROW = (uint32_t)LP << LOGN;  // one limb block: digit / mask term / key stride
    constexpr int PO = 2, PB = TB;                  // a warp: 2 outputs x TB ciphertexts
    static_assert(kChunk * TB == W, "phase A: one item per warp");
    __shared__ uint64_t sv[2][kChunk][TB][2][32];
    __shared__ uint32_t s_x[kBankMaxTerms], s_d[kBankMaxTerms], s_k[kBankMaxTerms], s_r[kBankMaxTerms];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int b0 = blockIdx.x * TB;
    const uint32_t n = blockIdx.y * 32 + lane;
    // wide_only: just the 60-bit limbs q_0 and P (the 40-bit ones run on hoist_imma.cu)
    const int k = wide_only ? (blockIdx.z ? L : 0) : (int)blockIdx.z;
    const Mod m = mods[k < L ? k : sp];
    const bool qlimb = k < L;
    const uint64_t P = mods[sp].q;
    const uint64_t Pk = qlimb ? (P < m.q ? P : csub(barrett_lite(P, m), m.q)) : 0;
    const int Q = I * T;
    // per-term element offsets: input block of X and D, key block, shift
    for (int q = threadIdx.x; q < Q; q += blockDim.x) {
        const int i = q / T, t = q - i * T;
        s_x[q] = (uint32_t)i * (uint32_t)B * (2u * L << LOGN);
        s_d[q] = (uint32_t)i * (uint32_t)B * ((uint32_t)L * LP << LOGN);
        s_k[q] = (uint32_t)t * ((uint32_t)LP * 2 * L << LOGN);
        s_r[q] = (uint32_t)shifts[t];
    }
    __syncthreads();
    const bool smallq = (m.q >> 41) == 0;

    // phase-A item of this warp: term qc = warp / TB, ciphertext b0 + warp % TB
    const int a_qc = warp / TB, a_bt = warp % TB, a_b = b0 + a_bt;
    const bool a_ok = a_b < B;
    const uint32_t xrow = ((uint32_t)a_b * 2 * L + k) << LOGN;           // c0 limb k of ciphertext a_b
    const uint32_t drow = ((uint32_t)a_b * L * LP + k) << LOGN;          // digit 0, limb k
    const uint32_t krow = (((uint32_t)(qlimb ? k : L)) * 2 * L << LOGN) + n;  // key rows of limb k
    // phase B: outputs o_a, o_a + 1 for all TB ciphertexts of the tile
    const int o_a = warp * PO;
    const bool o0 = o_a < O, o1 = o_a + 1 < O;
    const uint64_t *mrow0 = masks + (((uint32_t)o_a * Q) * ROW) + ((uint32_t)k << LOGN) + n;
    const uint64_t *mrow1 = mrow0 + (uint32_t)Q * ROW;

    auto body = [&](auto acc_tag) {
        using A = decltype(acc_tag);
        constexpr bool NARROW = std::is_same<A, AccN>::value;
        A acc[PO][PB][2];
#pragma unroll
        for (int d = 0; d < PO; d++)
#pragma unroll
            for (int e = 0; e < PB; e++) {
                acc[d][e][0].zero();
                acc[d][e][1].zero();
            }
        int buf = 0, fold = 0;
        for (int q0 = 0; q0 < Q; q0 += kChunk) {
            // weight masks of this chunk (consumed after the barrier; latency hidden by phase A)
            uint64_t mk[kChunk][PO];
#pragma unroll
            for (int qc = 0; qc < kChunk; qc++) {
                const bool ok = q0 + qc < Q;
                mk[qc][0] = ok && o0 ? __ldg(mrow0 + (uint32_t)(q0 + qc) * ROW) : 0;
                mk[qc][1] = ok && o1 ? __ldg(mrow1 + (uint32_t)(q0 + qc) * ROW) : 0;
            }
            // ---- phase A: P * rot(ct) of term q0 + a_qc for ciphertext a_b, limb k ----
            {
                const int q = q0 + a_qc;
                uint64_t v0 = 0, v1 = 0;
                if (q < Q && a_ok) {
                    const uint32_t r = s_r[q];
                    const uint64_t *c0 = X + s_x[q] + xrow;
                    if (r == 0) {
                        if (qlimb) {
                            v0 = mulmod(Pk, __ldg(c0 + n), m);
                            v1 = mulmod(Pk, __ldg(c0 + ((uint32_t)L << LOGN) + n), m);
                        }
                    } else {
                        const uint32_t src = rot_index_b(n, half, r);
                        const uint64_t *Dj = D + s_d[q] + drow + src;
                        const uint64_t *K = kbank + s_k[q] + krow;
                        A a0, a1;
                        a0.zero();
                        a1.zero();
                        // loads issued in groups of G digits (3G independent loads in flight)
#pragma unroll
                        for (int j0 = 0; j0 < L; j0 += G) {
                            uint64_t d[G], x[G], y[G];
#pragma unroll
                            for (int g = 0; g < G; g++) {
                                if (j0 + g < L) {
                                    d[g] = __ldg(Dj + (uint32_t)(j0 + g) * ROW);
                                    x[g] = __ldg(K + ((uint32_t)(2 * (j0 + g)) << LOGN));
                                    y[g] = __ldg(K + ((uint32_t)(2 * (j0 + g) + 1) << LOGN));
                                }
                            }
#pragma unroll
                            for (int g = 0; g < G; g++) {
                                if (j0 + g < L) {
                                    a0.mac(d[g], x[g]);
                                    a1.mac(d[g], y[g]);
                                }
                            }
                        }
                        if (qlimb) a0.mac(Pk, __ldg(c0 + src));
                        uint64_t h0, l0, h1, l1;
                        a0.value(h0, l0);
                        a1.value(h1, l1);
                        if (NARROW) {  // narrow phase-B operands: [0, 2q)
                            v0 = barrett_lite(fold64_b(h0, l0, m), m);
                            v1 = barrett_lite(fold64_b(h1, l1, m), m);
                        } else if (smallq) {
                            v0 = fold64_b(h0, l0, m);
                            v1 = fold64_b(h1, l1, m);
                        } else {
                            v0 = csub(reduce128_lazy_b(h0, l0, m), 2 * m.q);
                            v1 = csub(reduce128_lazy_b(h1, l1, m), 2 * m.q);
                        }
                    }
                }
                sv[buf][a_qc][a_bt][0][lane] = v0;
                sv[buf][a_qc][a_bt][1][lane] = v1;
            }
            __syncthreads();
            // ---- phase B ----
            if (o0) {
#pragma unroll
                for (int qc = 0; qc < kChunk; qc++) {
#pragma unroll
                    for (int e = 0; e < PB; e++) {
                        const uint64_t v0 = sv[buf][qc][e][0][lane], v1 = sv[buf][qc][e][1][lane];
#pragma unroll
                        for (int d = 0; d < PO; d++) {
                            acc[d][e][0].mac(mk[qc][d], v0);
                            acc[d][e][1].mac(mk[qc][d], v1);
                        }
                    }
                }
            }
            buf ^= 1;
            if (++fold == kFoldChunks) {
                fold = 0;
#pragma unroll
                for (int d = 0; d < PO; d++)
#pragma unroll
                    for (int e = 0; e < PB; e++)
#pragma unroll
                        for (int c = 0; c < 2; c++) {
                            uint64_t h, l;
                            acc[d][e][c].value(h, l);
                            acc[d][e][c].set(reduce128_lazy_b(h, l, m), 0);
                        }
            }
        }
#pragma unroll
        for (int d = 0; d < PO; d++) {
            const int o = o_a + d;
#pragma unroll
            for (int e = 0; e < PB; e++) {
                const int b = b0 + e;
                if (o < O && b < B) {
                    uint64_t *dst = acc_out + (((uint32_t)(o * B + b) * 2 * LP + k) << LOGN) + n;
                    dst[0] = acc[d][e][0].reduce(m);
                    dst[ROW] = acc[d][e][1].reduce(m);
                }
            }
        }
    };
    if (smallq)
        body(AccN{});
    else
        body(Acc{});
}

// ---------------------------------------------------------------------------
// Register-only variant for narrow layers (O <= 4 masked outputs, or unmasked
// rotation sums): one thread per (ciphertext, limb, coefficient) walks every
// term with everything in registers, as hoist.cu's k_hoisted_direct, over the
// same key bank and with compile-time strides.  Term modes: dense (q = i*T + t),
// diagonal (q = i = t) and block-diagonal (q = i*T + t', tap q) -- resolved
// once into the per-term offset tables.  Warp w of the CTA serves ciphertext
// 8 * blockIdx.x + w (ciphertext groups fastest in the grid: CTAs sharing the
// same key and mask rows run together).
//
// PRE (one masked output): the bank is a key-mask bank km[Q][L+1][2L+1][N] (k_km_bank) whose entry
// q holds the key rows of term q already multiplied by the term's mask, plus the row M_q * P, so
//   acc = sum_q sum_j rot(D_j) (M_q K_{q,j}) + (M_q P) rot(c0)
// needs no per-term reduction and no mask multiply: 2L + 1 MACs per term instead of 2L + 3 and two
// reductions.  Same canonical residues as the masked form (the sums agree mod q_k).
template <int L, int LOGN, int OM, bool MASKS, int G, int MINB, bool PRE = false>
__global__ void __launch_bounds__(256, MINB)
    k_direct_bank(uint64_t *__restrict__ acc_out, const uint64_t *__restrict__ X, const uint64_t *__restrict__ D,
                  const uint64_t *__restrict__ masks, const uint64_t *__restrict__ kbank,
                  const int32_t *__restrict__ shifts, int B, int I, int T, int O, int diag, int sp,
                  const Mod *__restrict__ mods) {
    static_assert(!PRE || (!MASKS && OM == 1), "key-mask bank: one output, masks folded into the bank");
    constexpr int LP = L + 1;
    constexpr int KR = PRE ? 2 * L + 1 : 2 * L;  // rows per (entry, limb) of the bank
    constexpr uint32_t N = 1u << LOGN, half = N >> 1;
    constexpr uint32_t ROW = (uint32_t)LP << LOGN;
    __shared__ uint32_t s_x[kBankMaxTerms], s_d[kBankMaxTerms], s_k[kBankMaxTerms], s_r[kBankMaxTerms];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int b = blockIdx.x * 8 + warp;
    const uint32_t n = blockIdx.y * 32 + lane;
    const int k = blockIdx.z;
    const int Q = diag == 1 ? I : I * T;
    for (int q = threadIdx.x; q < Q; q += blockDim.x) {
        int i, t;
        if (diag == 1) {
            i = t = q;
        } else {
            i = q / T;
            t = diag == 2 ? q : q - i * T;
        }
        s_x[q] = (uint32_t)i * (uint32_t)B * (2u * L << LOGN);
        s_d[q] = (uint32_t)i * (uint32_t)B * ((uint32_t)L * LP << LOGN);
        s_k[q] = (uint32_t)(PRE ? q : t) * ((uint32_t)LP * KR << LOGN);
        s_r[q] = (uint32_t)shifts[t];
    }
    __syncthreads();
    if (b >= B) return;
    const Mod m = mods[k < L ? k : sp];
    const bool qlimb = k < L;
    const bool smallq = (m.q >> 41) == 0;
    const uint64_t P = mods[sp].q;
    const uint64_t Pk = qlimb ? (P < m.q ? P : csub(barrett_lite(P, m), m.q)) : 0;
    const uint32_t xrow = ((uint32_t)b * 2 * L + k) << LOGN;
    const uint32_t drow = ((uint32_t)b * L * LP + k) << LOGN;
    const uint32_t krow = (((uint32_t)(qlimb ? k : L)) * KR << LOGN) + n;
    const uint64_t *mrow = masks + ((uint32_t)k << LOGN) + n;

    auto body = [&](auto acc_tag) {
        using A = decltype(acc_tag);
        constexpr bool NARROW = std::is_same<A, AccN>::value;
        A acc[OM][2];
#pragma unroll
        for (int o = 0; o < OM; o++) {
            acc[o][0].zero();
            acc[o][1].zero();
        }
        int since = 0;
        if constexpr (!MASKS) {
            // mask-free sums (and the key-mask bank): every term's MACs go straight into the running
            // sums; these fold back below 2^64 before the accumulator can overflow (narrow: the
            // x1 y1 word holds 2^14 products; wide: 256 products below 2^120)
            constexpr int kBudget = NARROW ? 8192 : 240;
            A &a0 = acc[0][0], &a1 = acc[0][1];
            for (int q = 0; q < Q; q++) {
                const uint32_t r = s_r[q];
                const uint64_t *c0 = X + s_x[q] + xrow;
                const uint64_t *K = kbank + s_k[q] + krow;
                if (since + 2 * L + 1 > kBudget) {
                    since = 0;
                    uint64_t h, l;
                    a0.value(h, l);
                    a0.set(smallq ? fold64_b(h, l, m) : reduce128_lazy_b(h, l, m), 0);
                    a1.value(h, l);
                    a1.set(smallq ? fold64_b(h, l, m) : reduce128_lazy_b(h, l, m), 0);
                }
                since += 2 * L + 1;
                if (r == 0) {
                    if (qlimb) {
                        const uint64_t pm = PRE ? __ldg(K + ((uint32_t)(2 * L) << LOGN)) : Pk;
                        a0.mac(pm, __ldg(c0 + n));
                        a1.mac(pm, __ldg(c0 + ((uint32_t)L << LOGN) + n));
                    }
                    continue;
                }
                const uint32_t src = rot_index_b(n, half, r);
                const uint64_t *Dj = D + s_d[q] + drow + src;
                uint64_t pm = Pk, cs = 0;
                if (qlimb) {
                    if (PRE) pm = __ldg(K + ((uint32_t)(2 * L) << LOGN));
                    cs = __ldg(c0 + src);
                }
#pragma unroll
                for (int j0 = 0; j0 < L; j0 += G) {
                    uint64_t d[G], x[G], y[G];
#pragma unroll
                    for (int g = 0; g < G; g++) {
                        if (j0 + g < L) {
                            d[g] = __ldg(Dj + (uint32_t)(j0 + g) * ROW);
                            x[g] = __ldg(K + ((uint32_t)(2 * (j0 + g)) << LOGN));
                            y[g] = __ldg(K + ((uint32_t)(2 * (j0 + g) + 1) << LOGN));
                        }
                    }
#pragma unroll
                    for (int g = 0; g < G; g++) {
                        if (j0 + g < L) {
                            a0.mac(d[g], x[g]);
                            a1.mac(d[g], y[g]);
                        }
                    }
                }
                if (qlimb) a0.mac(pm, cs);
            }
        }
        for (int q = 0; MASKS && q < Q; q++) {
            uint64_t mk[OM];
            if (MASKS) {
#pragma unroll
                for (int o = 0; o < OM; o++) mk[o] = o < O ? __ldg(mrow + (uint32_t)(o * Q + q) * ROW) : 0;
            }
            const uint32_t r = s_r[q];
            const uint64_t *c0 = X + s_x[q] + xrow;
            A a0, a1;
            a0.zero();
            a1.zero();
            if (r == 0) {
                if (qlimb) {
                    a0.mac(Pk, __ldg(c0 + n));
                    a1.mac(Pk, __ldg(c0 + ((uint32_t)L << LOGN) + n));
                }
            } else {
                const uint32_t src = rot_index_b(n, half, r);
                const uint64_t *Dj = D + s_d[q] + drow + src;
                const uint64_t *K = kbank + s_k[q] + krow;
#pragma unroll
                for (int j0 = 0; j0 < L; j0 += G) {
                    uint64_t d[G], x[G], y[G];
#pragma unroll
                    for (int g = 0; g < G; g++) {
                        if (j0 + g < L) {
                            d[g] = __ldg(Dj + (uint32_t)(j0 + g) * ROW);
                            x[g] = __ldg(K + ((uint32_t)(2 * (j0 + g)) << LOGN));
                            y[g] = __ldg(K + ((uint32_t)(2 * (j0 + g) + 1) << LOGN));
                        }
                    }
#pragma unroll
                    for (int g = 0; g < G; g++) {
                        if (j0 + g < L) {
                            a0.mac(d[g], x[g]);
                            a1.mac(d[g], y[g]);
                        }
                    }
                }
                if (qlimb) a0.mac(Pk, __ldg(c0 + src));
            }
            uint64_t h0, l0, h1, l1;
            a0.value(h0, l0);
            a1.value(h1, l1);
            if (MASKS) {
                uint64_t v0, v1;
                if (NARROW) {
                    v0 = barrett_lite(fold64_b(h0, l0, m), m);
                    v1 = barrett_lite(fold64_b(h1, l1, m), m);
                } else if (smallq) {
                    v0 = fold64_b(h0, l0, m);
                    v1 = fold64_b(h1, l1, m);
                } else {
                    v0 = csub(reduce128_lazy_b(h0, l0, m), 2 * m.q);
                    v1 = csub(reduce128_lazy_b(h1, l1, m), 2 * m.q);
                }
#pragma unroll
                for (int o = 0; o < OM; o++) {
                    acc[o][0].mac(mk[o], v0);
                    acc[o][1].mac(mk[o], v1);
                }
                if (++since == 54) {
                    since = 0;
#pragma unroll
                    for (int o = 0; o < OM; o++)
#pragma unroll
                        for (int c = 0; c < 2; c++) {
                            uint64_t h, l;
                            acc[o][c].value(h, l);
                            acc[o][c].set(reduce128_lazy_b(h, l, m), 0);
                        }
                }
            }
        }
#pragma unroll
        for (int o = 0; o < OM; o++) {
            if (o < O) {
                uint64_t *dst = acc_out + (((uint32_t)(o * B + b) * 2 * LP + k) << LOGN) + n;
                dst[0] = acc[o][0].reduce(m);
                dst[ROW] = acc[o][1].reduce(m);
            }
        }
    };
    if (smallq)
        body(AccN{});
    else
        body(Acc{});
}

template <int L, int OM, bool MASKS>
void launch_direct_bank(const Ctx &c, uint64_t *acc, const uint64_t *X, const uint64_t *D, const uint64_t *masks,
                        const uint64_t *kbank, const int32_t *shifts, int B, int I, int T, int O, int diag,
                        cudaStream_t s) {
    dim3 grid((unsigned)((B + 7) / 8), (unsigned)(c.n / 32), L + 1);
    // 4-output layers (LeNet conv1): all of a term's digit / key loads in flight at 2 CTAs per SM
    // (measured 13.5 vs 15.5 ms for conv1 at B = 64 with 3 CTAs and groups of 2); narrower
    // layers are unchanged by either knob
    constexpr int G = OM >= 4 ? UH_BANK_DIRECT4_G : UH_BANK_DIRECT_G;
    constexpr int MINB = OM >= 4 ? UH_BANK_DIRECT4_MINB : UH_BANK_DIRECT_MINB;
    k_direct_bank<L, 15, OM, MASKS, G, MINB><<<grid, 256, 0, s>>>(acc, X, D, masks, kbank, shifts, B, I, T, O, diag,
                                                                  c.sp(), c.d_mods);
    UH_LAUNCH_CHECK();
}

template <int L>
void direct_bank_L(const Ctx &c, uint64_t *acc, const uint64_t *X, const uint64_t *D, const uint64_t *masks,
                   const uint64_t *kbank, const int32_t *shifts, int B, int I, int T, int O, int diag, cudaStream_t s) {
    if (!masks) {
        launch_direct_bank<L, 1, false>(c, acc, X, D, masks, kbank, shifts, B, I, T, 1, diag, s);
        const size_t one = (size_t)B * 2 * (L + 1) * c.n;  // identical unmasked outputs: copies
        for (int o = 1; o < O; o++)
            UH_CHECK(cudaMemcpyAsync(acc + o * one, acc, one * 8, cudaMemcpyDeviceToDevice, s));
    } else if (O == 1) {
        launch_direct_bank<L, 1, true>(c, acc, X, D, masks, kbank, shifts, B, I, T, O, diag, s);
    } else if (O == 2) {
        launch_direct_bank<L, 2, true>(c, acc, X, D, masks, kbank, shifts, B, I, T, O, diag, s);
    } else {
        launch_direct_bank<L, 4, true>(c, acc, X, D, masks, kbank, shifts, B, I, T, O, diag, s);
    }
}

// Key-mask bank km[Q][L+1][2L+1][N] of a one-output masked layer: rows 2j + c of entry q are
// M_q (.) K_{t(q)}[j][c] (zero for a zero shift), row 2L is M_q * P on the q-limbs (zero on P).
// t(q) = q mod T for dense terms, q otherwise (diagonal / block-diagonal: one key entry per term).
__global__ void k_km_bank(uint64_t *__restrict__ km, const uint64_t *__restrict__ masks,
                          const uint64_t *__restrict__ kbank, const int32_t *__restrict__ shifts, int Q, int T,
                          int diag, int L, int logn, int sp, const Mod *__restrict__ mods) {
    const int LP = L + 1, KR = 2 * L + 1;
    const size_t N = (size_t)1 << logn;
    const size_t total = (size_t)Q * LP * KR * N;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
        const size_t n = idx & (N - 1);
        size_t r = idx >> logn;
        const int row = (int)(r % KR);
        r /= KR;
        const int k = (int)(r % LP), q = (int)(r / LP);
        const int t = diag == 0 ? q % T : q;
        const Mod m = mods[k < L ? k : sp];
        const uint64_t mk = masks[((size_t)q * LP + k) * N + n];
        uint64_t v = 0;
        if (row < 2 * L) {
            if (shifts[t] != 0) v = mulmod(mk, kbank[(((size_t)t * LP + k) * 2 * L + row) * N + n], m);
        } else if (k < L) {
            const uint64_t P = mods[sp].q;
            v = mulmod(mk, P < m.q ? P : csub(barrett_lite(P, m), m.q), m);
        }
        km[idx] = v;
    }
}

template <int L>
void launch_km(const Ctx &c, uint64_t *acc, const uint64_t *X, const uint64_t *D, const uint64_t *km,
               const int32_t *shifts, int B, int I, int T, int diag, cudaStream_t s) {
    dim3 grid((unsigned)((B + 7) / 8), (unsigned)(c.n / 32), L + 1);
    k_direct_bank<L, 15, 1, false, UH_BANK_DIRECT_G, UH_BANK_DIRECT_MINB, true><<<grid, 256, 0, s>>>(
        acc, X, D, nullptr, km, shifts, B, I, T, 1, diag, c.sp(), c.d_mods);
    UH_LAUNCH_CHECK();
}

template <int L>
void launch_bank(const Ctx &c, uint64_t *acc, const uint64_t *X, const uint64_t *D, const uint64_t *masks,
                 const uint64_t *kbank, const int32_t *shifts, int B, int I, int T, int O, cudaStream_t s,
                 int wide_only = 0) {
    constexpr int TB = UH_BANK_TB, W = kChunk * TB;  // phase A: one (term, ciphertext) item per warp
    // phase B: warp w owns outputs 2w, 2w + 1 -- the tile must have a warp for every output pair
    // (measured: every W >= 6 alternative -- chunk 2 x 3 ciphertexts, chunk 2 x 4 -- was slower)
    if (O > 2 * W) throw std::invalid_argument("key-bank tiled kernel: more outputs than 2 x warps per CTA");
    dim3 grid((unsigned)((B + TB - 1) / TB), (unsigned)(c.n / 32), wide_only ? 2 : L + 1);
    k_hoisted_bank<L, 15, W, TB, UH_BANK_G><<<grid, W * 32, 0, s>>>(acc, X, D, masks, kbank, shifts, B, I, T, O, c.sp(),
                                                          c.d_mods, wide_only);
    UH_LAUNCH_CHECK();
}

}  // namespace

// the tiled kernel over the 60-bit limbs (q_0, P) only -- hoist_imma.cu covers the rest
void hoisted_mac_bank_wide(const Ctx &c, uint64_t *acc, const uint64_t *X, const uint64_t *D, const uint64_t *masks,
                           const uint64_t *kbank, const int32_t *shifts, int B, int I, int T, int O, int level,
                           cudaStream_t s) {
    switch (level + 1) {
        case 2: launch_bank<2>(c, acc, X, D, masks, kbank, shifts, B, I, T, O, s, 1); break;
        case 3: launch_bank<3>(c, acc, X, D, masks, kbank, shifts, B, I, T, O, s, 1); break;
        case 4: launch_bank<4>(c, acc, X, D, masks, kbank, shifts, B, I, T, O, s, 1); break;
        case 5: launch_bank<5>(c, acc, X, D, masks, kbank, shifts, B, I, T, O, s, 1); break;
        case 6: launch_bank<6>(c, acc, X, D, masks, kbank, shifts, B, I, T, O, s, 1); break;
        case 7: launch_bank<7>(c, acc, X, D, masks, kbank, shifts, B, I, T, O, s, 1); break;
        case 8: launch_bank<8>(c, acc, X, D, masks, kbank, shifts, B, I, T, O, s, 1); break;
        case 9: launch_bank<9>(c, acc, X, D, masks, kbank, shifts, B, I, T, O, s, 1); break;
        case 10: launch_bank<10>(c, acc, X, D, masks, kbank, shifts, B, I, T, O, s, 1); break;
        default: throw std::invalid_argument("wide-limb hoisted kernel: 2 <= level + 1 <= 10");
    }
}

void km_bank(const Ctx &c, uint64_t *km, const uint64_t *masks, const uint64_t *kbank, const int32_t *shifts, int Q,
             int T, int diag, int level, cudaStream_t s) {
    const int L = level + 1;
    const size_t total = (size_t)Q * (L + 1) * (2 * L + 1) * c.n;
    const unsigned blocks = (unsigned)std::min<size_t>((total + 255) / 256, 148 * 32);
    k_km_bank<<<blocks, 256, 0, s>>>(km, masks, kbank, shifts, Q, T, diag, L, (int)c.logn, c.sp(), c.d_mods);
    UH_LAUNCH_CHECK();
}

// one masked output over a key-mask bank (every term mode): the register-only kernel, 2L + 1 MACs per term
void hoisted_mac_km(const Ctx &c, uint64_t *acc, const uint64_t *X, const uint64_t *D, const uint64_t *km,
                    const int32_t *shifts, int B, int I, int T, int diag, int level, cudaStream_t s) {
    if (!hoisted_bank_supported(c, level, 1))
        throw std::invalid_argument("key-mask bank kernel: needs N = 2^15, level + 1 <= 10");
    const int Q = diag == 1 ? I : I * T;
    if (Q > kBankMaxTerms) throw std::invalid_argument("key-mask bank kernel supports up to 512 terms");
    if (diag == 1 && I != T) throw std::invalid_argument("diagonal terms need I == T");
    const int L = level + 1;
    const double lim = 4294967295.0;  // 32-bit element offsets inside the kernel
    if ((double)I * B * 2 * L * c.n > lim || (double)I * B * L * (L + 1) * c.n > lim ||
        (double)B * 2 * (L + 1) * c.n > lim || (double)Q * (L + 1) * (2 * L + 1) * c.n > lim)
        throw std::invalid_argument("key-mask bank kernel operand exceeds 2^32 elements: split the batch");
#define UH_KM_CASE(LL) \
    case LL: launch_km<LL>(c, acc, X, D, km, shifts, B, I, T, diag, s); break;
    switch (L) {
        UH_KM_CASE(1)
        UH_KM_CASE(2)
        UH_KM_CASE(3)
        UH_KM_CASE(4)
        UH_KM_CASE(5)
        UH_KM_CASE(6)
        UH_KM_CASE(7)
        UH_KM_CASE(8)
        UH_KM_CASE(9)
        UH_KM_CASE(10)
        default: throw std::invalid_argument("key-mask bank kernel: level + 1 <= 10");
    }
#undef UH_KM_CASE
}

bool hoisted_bank_supported(const Ctx &c, int level, int O) {
    return c.logn == 15 && level >= 0 && level + 1 <= 10 && O >= 1 && O <= 12;
}

// dense masked terms with 7..12 outputs: the shared-memory tiled kernel; everything else
// (<= 4 masked outputs, unmasked rotation sums, diagonal / block-diagonal terms): the
// register-only kernel (5..6 masked outputs: the tiled kernel as well)
void hoisted_mac_bank(const Ctx &c, uint64_t *acc, const uint64_t *X, const uint64_t *D, const uint64_t *masks,
                      const uint64_t *kbank, const int32_t *shifts, int B, int I, int T, int O, int diag, int level,
                      cudaStream_t s) {
    if (!hoisted_bank_supported(c, level, O))
        throw std::invalid_argument("key-bank hoisted kernel: needs N = 2^15, level + 1 <= 10, 1 <= O <= 12");
    const int Q = diag == 1 ? I : I * T;
    if (Q > kBankMaxTerms || (diag == 2 ? I * T : diag == 1 ? I : T) > kBankMaxTerms)
        throw std::invalid_argument("key-bank hoisted kernel supports up to 512 terms");
    if (diag == 1 && I != T) throw std::invalid_argument("diagonal terms need I == T");
    const int L = level + 1;
    const int NT = diag == 2 ? I * T : (diag == 1 ? I : T);  // key-bank entries
    const double lim = 4294967295.0;  // 32-bit element offsets inside the kernels
    if ((double)I * B * 2 * L * c.n > lim || (double)I * B * L * (L + 1) * c.n > lim ||
        (double)O * B * 2 * (L + 1) * c.n > lim || (double)O * Q * (L + 1) * c.n > lim ||
        (double)NT * (L + 1) * 2 * L * c.n > lim)
        throw std::invalid_argument("key-bank hoisted kernel operand exceeds 2^32 elements: split the batch");
    const bool tiled = masks && diag == 0 && O > 4;
#define UH_BANK_CASE(LL)                                                                           \
    case LL:                                                                                       \
        if (tiled)                                                                                 \
            launch_bank<LL>(c, acc, X, D, masks, kbank, shifts, B, I, T, O, s);                    \
        else                                                                                       \
            direct_bank_L<LL>(c, acc, X, D, masks, kbank, shifts, B, I, T, O, diag, s);            \
        break;
    switch (L) {
        UH_BANK_CASE(1)
        UH_BANK_CASE(2)
        UH_BANK_CASE(3)
        UH_BANK_CASE(4)
        UH_BANK_CASE(5)
        UH_BANK_CASE(6)
        UH_BANK_CASE(7)
        UH_BANK_CASE(8)
        UH_BANK_CASE(9)
        UH_BANK_CASE(10)
        default: throw std::invalid_argument("key-bank hoisted kernel: level + 1 <= 10");
    }
#undef UH_BANK_CASE
}

}  // namespace uh
