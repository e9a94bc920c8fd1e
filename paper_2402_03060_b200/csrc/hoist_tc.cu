// Hoisted rotation-MAC with the weight-mask contraction on the 5th-generation tensor cores
// (tcgen05.mma kind::i8, accumulators in TMEM).  Same result, residue for residue, as
// hoist_bank.cu's IMAD kernel:
//
//   acc[o][b] (QP basis) = sum over terms q = (i, t) of  M[o][q] (.) P * rot_{s_t}(ct_i[b])
//
// For one coefficient n of one limb k the mask contraction is the integer GEMM
//   acc[o][j] = sum_q M[o][q][n] * V[q][j][n]          (j = ciphertext x component)
// whose A operand (the masks at n) is shared by every ciphertext.  Both factors are canonical
// residues split exactly into W bytes (W = 5 for the 40-bit limbs q_1..q_l, W = 8 for the
// 60-bit q_0 and P), so
//   acc = sum_{a,b < W} 2^(8(a+b)) sum_q M_a[o][q] V_b[q][j]
// with every inner sum a u8 x u8 dot product over <= 128 terms (< 2^23: exact in s32).
// Rows of the MMA are (output o, mask byte a) -- the A operand, pre-split once per layer into a
// per-coefficient tile in the UMMA canonical K-major layout (k_tc_bank) and brought into shared
// memory with one bulk copy (cp.async.bulk) per coefficient; columns are (value byte b,
// ciphertext, component) -- the B operand, written into shared memory by phase A.
//
// CTA tile: NC coefficients x CT ciphertexts x one limb, 256 threads.
//   phase A : every item (4 consecutive terms, ciphertext pair, coefficient) key-switches its
//             terms (hoisted digits x Galois-key bank + P c0, as hoist_bank.cu) and packs the
//             W bytes of its 4 x 4 values into 32-bit words (4 consecutive K per word) in the
//             B tiles;
//   phase B : one thread issues, per coefficient, Kpad / 32 tcgen05.mma (M = 64 or 128, N =
//             2 CT W rounded to 16, K = 32) into TMEM -- for M = 64 two coefficients share a
//             column block (TMEM lanes 0-15 / 16-31 of every subpartition) -- and commits to
//             an mbarrier;
//   epilogue: tcgen05.ld (32x32b) of each accumulator row, sum over the value bytes in
//             registers, sum over the mask bytes through shared memory, reduction mod q,
//             store.  Canonical residues: bit-identical to the IMAD kernel.
#include "ops.cuh"

namespace uh {
namespace {

constexpr int kTcMaxTerms = 128;  // 4 K-steps of 32
constexpr int kTcThreads = 256;
#ifndef UH_TC_TQ5
#define UH_TC_TQ5 4
#endif
#ifndef UH_TC_TQ8
#define UH_TC_TQ8 2
#endif
#ifndef UH_TC_NC8
#define UH_TC_NC8 4  // coefficients per CTA on the 60-bit limbs (TMEM: 64 columns each at M = 128)
#endif
#ifndef UH_TC_MINB8
#define UH_TC_MINB8 2
#endif

template <int W, int MP_, int NC_, int CT_>
struct TcCfg {
    static constexpr int MP = MP_;                       // MMA M (64 or 128)
    static constexpr int NC = NC_;                       // coefficients per CTA
    static constexpr int CT = CT_;                       // ciphertexts per CTA
    static constexpr int NCOL = 2 * CT * W;              // B rows used: (byte b, ciphertext, component)
    static constexpr int NP = (NCOL + 15) / 16 * 16;     // MMA N
    static constexpr int TPB = MP == 64 ? 2 : 1;         // coefficients per TMEM column block
    static constexpr int NBLK = (NC + TPB - 1) / TPB;    // column blocks
    static constexpr int TCOLS_USED = NBLK * NP;
    static constexpr int TCOLS = TCOLS_USED <= 32 ? 32 : TCOLS_USED <= 64 ? 64 : TCOLS_USED <= 128 ? 128
                                 : TCOLS_USED <= 256 ? 256 : 512;
    static_assert(TCOLS_USED <= 512, "TMEM");
    static_assert(CT % 2 == 0, "ciphertext pairs");
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
// UMMA canonical K-major, no swizzle: core matrices of 8 rows x 16 bytes, K chunks at 128 B,
// 8-row groups at kpad * 8 B (one group holds all kpad / 16 chunks)
__host__ __device__ __forceinline__ uint32_t tc_off(int r, int k, int kpad) {
    return (uint32_t)((r >> 3) * (kpad * 8) + (k >> 4) * 128 + (r & 7) * 16 + (k & 15));
}
__device__ __forceinline__ uint64_t tc_desc(uint32_t saddr, int kpad) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);  // start address
    d |= (uint64_t)(128 >> 4) << 16;                 // leading byte offset: next K chunk
    d |= (uint64_t)((kpad * 8) >> 4) << 32;          // stride byte offset: next 8-row group
    d |= (uint64_t)1 << 46;                          // descriptor version (sm_100)
    return d;                                        // base offset 0, SWIZZLE_NONE
}
__host__ __device__ constexpr uint32_t tc_idesc(int M, int N) {
    return (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);  // S32 <- U8 x U8, K-major
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
}
__device__ __forceinline__ uint32_t rot_index_t(uint32_t n, uint32_t half, uint32_t r) {
    uint32_t h = n >= half ? half : 0;
    uint32_t j = n - h + r;
    j = j >= half ? j - half : j;
    return h + j;
}
__device__ __forceinline__ uint64_t fold64_t(uint64_t hi, uint64_t lo, const Mod &m) {
    const uint64_t p = (uint64_t)(uint32_t)hi * m.r64;
    const uint64_t v = lo + p;
    return v < p ? v + m.r64 : v;
}
// (hi:lo) += t << sh, 0 <= sh < 64
__device__ __forceinline__ void add_shl(uint64_t &hi, uint64_t &lo, uint64_t t, int sh) {
    const uint64_t l = t << sh;
    const uint64_t h = sh ? t >> (64 - sh) : 0;
    lo += l;
    hi += h + (lo < l);
}
// A-operand bank: for every limb slot and coefficient a tile [MP rows][kpad] (canonical K-major
// layout) of mask bytes: row o W + a holds byte a of M[o][q][limb][n] at K = q (zero past Q and
// for rows >= O W).  Slots: W = 5 -> limbs 1..L-1, W = 8 -> limbs 0 and L (P).
template <int W, int MP>
__global__ void k_tc_bank(uint8_t *__restrict__ bank, const uint64_t *__restrict__ masks, int O, int Q, int L,
                          int logn, int kpad) {
    const uint32_t N = 1u << logn;
    const int nslots = W == 5 ? L - 1 : 2;
    const size_t words = (size_t)MP * kpad / 4;  // 32-bit words per tile
    const size_t total = (size_t)nslots * N * words;
    const size_t ROW = (size_t)(L + 1) << logn;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
        const size_t tile = idx / words;
        const int w = (int)(idx - tile * words);
        const int r = w / (kpad / 4), k0 = (w % (kpad / 4)) * 4;
        const uint32_t n = (uint32_t)(tile & (N - 1));
        const int slot = (int)(tile >> logn);
        const int limb = W == 5 ? slot + 1 : (slot ? L : 0);
        const int o = r / W, a = r % W;
        uint32_t v = 0;
        if (o < O) {
#pragma unroll
            for (int t = 0; t < 4; t++) {
                const int q = k0 + t;
                if (q < Q) {
                    const uint64_t mv = masks[((size_t)o * Q + q) * ROW + ((size_t)limb << logn) + n];
                    v |= (uint32_t)((mv >> (8 * a)) & 0xFF) << (8 * t);
                }
            }
        }
        *reinterpret_cast<uint32_t *>(bank + tile * (size_t)MP * kpad + tc_off(r, k0, kpad)) = v;
    }
}

template <int L, int LOGN, int W, class C>
__global__ void __launch_bounds__(kTcThreads, W == 5 ? 2 : UH_TC_MINB8)
    k_hoisted_tc(uint64_t *__restrict__ acc_out, const uint64_t *__restrict__ X, const uint64_t *__restrict__ D,
                 const uint8_t *__restrict__ bank, const uint64_t *__restrict__ kbank,
                 const int32_t *__restrict__ shifts, int B, int I, int T, int O, int sp,
                 const Mod *__restrict__ mods, int kpad) {
    constexpr int LP = L + 1;
    constexpr uint32_t N = 1u << LOGN, half = N >> 1;
    constexpr uint32_t ROW = (uint32_t)LP << LOGN;
    constexpr int MP = C::MP, NC = C::NC, CT = C::CT, NP = C::NP;
    extern __shared__ __align__(1024) uint8_t tsm[];
    uint8_t *sa = tsm;                                  // NC A tiles [MP][kpad]
    uint8_t *sb = tsm + (size_t)NC * MP * kpad;         // NC B tiles [NP][kpad]
    __shared__ uint32_t s_x[kTcMaxTerms], s_d[kTcMaxTerms], s_k[kTcMaxTerms], s_r[kTcMaxTerms];
    __shared__ __align__(8) uint64_t bar_a, bar_mma;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int b0 = blockIdx.x * CT;
    const uint32_t n0 = blockIdx.y * NC;
    const int slot = blockIdx.z;
    const int k = W == 5 ? 1 + slot : (slot ? L : 0);  // limb: q_1..q_{L-1}, or q_0 / P
    const bool qlimb = W == 5 || k < L;
    const Mod m = mods[qlimb ? k : sp];
    const uint64_t P = mods[sp].q;
    const uint64_t Pk = qlimb ? (P < m.q ? P : csub(barrett_lite(P, m), m.q)) : 0;
    const int Q = I * T;
    const uint32_t atile = (uint32_t)MP * kpad, btile = (uint32_t)NP * kpad;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                     "r"(C::TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 32) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar_a)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar_mma)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // the A tiles of this CTA's coefficients: one bulk copy each, overlapping phase A
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar_a)),
                     "r"((uint32_t)NC * atile)
                     : "memory");
        const uint8_t *src = bank + ((size_t)slot * N + n0) * atile;
        for (int c = 0; c < NC; c++)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(sa + c * atile)),
                "l"(src + (size_t)c * atile), "r"(atile), "r"(smem_u32(&bar_a))
                : "memory");
    }
    for (int q = tid; q < Q; q += kTcThreads) {
        const int i = q / T, t = q - i * T;
        s_x[q] = (uint32_t)i * (uint32_t)B * (2u * L << LOGN);
        s_d[q] = (uint32_t)i * (uint32_t)B * ((uint32_t)L * LP << LOGN);
        s_k[q] = (uint32_t)t * ((uint32_t)LP * 2 * L << LOGN);
        s_r[q] = (uint32_t)shifts[t];
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base;

    // ---- phase A: items (4 terms, ciphertext pair, coefficient) -> packed B-tile words ----
    {
        constexpr int NPAIR = CT / 2;
        // terms per item: 4 (one 32-bit B word per (value, byte)) on the 40-bit limbs; 2 (16-bit halves)
        // on the 60-bit limbs, whose 128-bit MACs make an item twice as long -- twice the items keeps
        // every thread busy (200 -> 400 items per CTA at the LeNet conv2 shape)
        constexpr int TQ = W == 5 ? UH_TC_TQ5 : UH_TC_TQ8;
        const int ngrp = (Q + TQ - 1) / TQ;
        const uint32_t krow = ((uint32_t)(qlimb ? k : L) * 2 * L) << LOGN;
        for (int it = tid; it < ngrp * NPAIR * NC; it += kTcThreads) {
            const int cf = it % NC, cp = (it / NC) % NPAIR, g = it / (NC * NPAIR);
            const int ba = b0 + 2 * cp;
            const bool oka = ba < B, okb = ba + 1 < B;
            const uint32_t n = n0 + cf;
            // B-tile words: wd[jj][b] = byte b of value jj for terms TQ g .. TQ g + TQ - 1 (term tq -> byte tq);
            // values jj: (ct a, c0), (ct a, c1), (ct b, c0), (ct b, c1)
            uint32_t wd[4][W];
#pragma unroll
            for (int jj = 0; jj < 4; jj++)
#pragma unroll
                for (int b = 0; b < W; b++) wd[jj][b] = 0;
#pragma unroll
            for (int tq = 0; tq < TQ; tq++) {
                const int q = TQ * g + tq;
                uint64_t v[4] = {0, 0, 0, 0};
                if (q < Q && oka) {
                const uint32_t r = s_r[q];
                const uint64_t *c0a = X + s_x[q] + (((uint32_t)ba * 2 * L + (qlimb ? k : 0)) << LOGN);
                const uint64_t *c0b = c0a + ((uint32_t)(2 * L) << LOGN);
                if (r == 0) {
                    if (qlimb) {
                        v[0] = mulmod(Pk, __ldg(c0a + n), m);
                        v[1] = mulmod(Pk, __ldg(c0a + ((uint32_t)L << LOGN) + n), m);
                        if (okb) {
                            v[2] = mulmod(Pk, __ldg(c0b + n), m);
                            v[3] = mulmod(Pk, __ldg(c0b + ((uint32_t)L << LOGN) + n), m);
                        }
                    }
                } else {
                const uint32_t src = rot_index_t(n, half, r);
                const uint64_t *Da = D + s_d[q] + (((uint32_t)ba * L * LP + k) << LOGN) + src;
                const uint64_t *Db = Da + ((uint32_t)(L * LP) << LOGN);
                const uint64_t *K = kbank + s_k[q] + krow + n;
                uint64_t da[L], db[L], x[L], y[L];
#pragma unroll
                for (int j = 0; j < L; j++) {
                    x[j] = __ldg(K + ((uint32_t)(2 * j) << LOGN));
                    y[j] = __ldg(K + ((uint32_t)(2 * j + 1) << LOGN));
                    da[j] = __ldg(Da + (uint32_t)j * ROW);
                    db[j] = okb ? __ldg(Db + (uint32_t)j * ROW) : 0;
                }
                const uint64_t csa = qlimb ? __ldg(c0a + src) : 0, csb = qlimb && okb ? __ldg(c0b + src) : 0;
                if constexpr (W == 5) {
                    AccN a0, a1, e0, e1;
                    a0.zero();
                    a1.zero();
                    e0.zero();
                    e1.zero();
#pragma unroll
                    for (int j = 0; j < L; j++) {
                        a0.mac(da[j], x[j]);
                        a1.mac(da[j], y[j]);
                        e0.mac(db[j], x[j]);
                        e1.mac(db[j], y[j]);
                    }
                    a0.mac(Pk, csa);
                    e0.mac(Pk, csb);
                    auto fin = [&](const AccN &acc) -> uint64_t {
                        uint64_t h, l;
                        acc.value(h, l);
                        return csub(barrett_lite(fold64_t(h, l, m), m), m.q);
                    };
                    v[0] = fin(a0);
                    v[1] = fin(a1);
                    if (okb) {
                        v[2] = fin(e0);
                        v[3] = fin(e1);
                    }
                } else {
                    Acc a0, a1, e0, e1;
                    a0.zero();
                    a1.zero();
                    e0.zero();
                    e1.zero();
#pragma unroll
                    for (int j = 0; j < L; j++) {
                        a0.mac(da[j], x[j]);
                        a1.mac(da[j], y[j]);
                        e0.mac(db[j], x[j]);
                        e1.mac(db[j], y[j]);
                    }
                    if (qlimb) {
                        a0.mac(Pk, csa);
                        e0.mac(Pk, csb);
                    }
                    v[0] = a0.reduce(m);
                    v[1] = a1.reduce(m);
                    if (okb) {
                        v[2] = e0.reduce(m);
                        v[3] = e1.reduce(m);
                    }
                }
                }
                }
#pragma unroll
                for (int jj = 0; jj < 4; jj++)
#pragma unroll
                    for (int b = 0; b < W; b++) wd[jj][b] |= (uint32_t)((v[jj] >> (8 * b)) & 0xFF) << (8 * tq);
            }
            // B rows: r = b * 2CT + (2 * ciphertext + component); K = terms 4g .. 4g + 3 in one word
            uint8_t *bt = sb + (size_t)cf * btile;
#pragma unroll
            for (int jj = 0; jj < 4; jj++) {
                const int j = 4 * cp + jj;  // (ciphertext 2 cp + jj / 2, component jj % 2)
#pragma unroll
                for (int b = 0; b < W; b++)
                    if constexpr (TQ == 4)
                        *reinterpret_cast<uint32_t *>(bt + tc_off(b * 2 * CT + j, 4 * g, kpad)) = wd[jj][b];
                    else if constexpr (TQ == 2)
                        *reinterpret_cast<uint16_t *>(bt + tc_off(b * 2 * CT + j, 2 * g, kpad)) = (uint16_t)wd[jj][b];
                    else
                        bt[tc_off(b * 2 * CT + j, g, kpad)] = (uint8_t)wd[jj][b];
            }
        }
        // K columns [TQ ngrp, kpad) of the B tiles are never written: their A bytes are zero
    }
    // generic-proxy smem writes -> visible to the tensor core (async proxy)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();

    // ---- phase B: one thread issues every MMA of the CTA ----
    if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        mbar_wait(smem_u32(&bar_a), 0);
        constexpr uint32_t idesc = tc_idesc(MP, NP);
        const int ks_n = kpad / 32;
        for (int c = 0; c < NC; c++) {
            const uint32_t dt = MP == 64 ? tmem + ((uint32_t)(16 * (c & 1)) << 16) + (uint32_t)(NP * (c >> 1))
                                         : tmem + (uint32_t)(NP * c);
            const uint32_t a0 = smem_u32(sa + c * atile), b0a = smem_u32(sb + c * btile);
            for (int ks = 0; ks < ks_n; ks++) {
                const uint64_t da = tc_desc(a0 + ks * 256, kpad), db = tc_desc(b0a + ks * 256, kpad);
                const uint32_t accum = ks > 0;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dt),
                    "l"(da), "l"(db), "r"(idesc), "r"(accum));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&bar_mma)));
    }
    mbar_wait(smem_u32(&bar_mma), 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    // ---- epilogue: TMEM rows -> sum over value bytes (registers) -> smem -> sum over mask bytes ----
    // Tb[c][row][j]: sum_b 2^(8b) C[row][(b, j)] for the accumulator row (o, a) (reuses the A/B tiles:
    // every MMA has completed).  W = 5: < 2^56, one word; W = 8: < 2^80, two words.
    constexpr int JN = 2 * CT;
    constexpr int TW = W == 5 ? 1 : 2;
    uint64_t *Tb = reinterpret_cast<uint64_t *>(tsm);
    const int sub = warp & 3;  // TMEM lanes [32 sub, 32 sub + 32)
    for (int blk = warp >> 2; blk < C::NBLK; blk += kTcThreads / 128) {
        uint32_t cv[C::NCOL];
#pragma unroll
        for (int c0 = 0; c0 < C::NCOL; c0 += 8) {
            const uint32_t ta = tmem + ((uint32_t)(32 * sub) << 16) + (uint32_t)(NP * blk + c0);
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(cv[c0]), "=r"(cv[c0 + 1]), "=r"(cv[c0 + 2]), "=r"(cv[c0 + 3]), "=r"(cv[c0 + 4]),
                           "=r"(cv[c0 + 5]), "=r"(cv[c0 + 6]), "=r"(cv[c0 + 7])
                         : "r"(ta));
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        int c, row;
        if (MP == 64) {
            c = 2 * blk + (lane >> 4);
            row = 16 * sub + (lane & 15);
        } else {
            c = blk;
            row = 32 * sub + lane;
        }
        if (c < NC && row < O * W) {
#pragma unroll
            for (int j = 0; j < JN; j++) {
                uint64_t hi = 0, lo = 0;
#pragma unroll
                for (int b = 0; b < W; b++) add_shl(hi, lo, (uint64_t)cv[b * JN + j], 8 * b);
                uint64_t *dst = Tb + (((size_t)c * MP + row) * JN + j) * TW;
                dst[0] = lo;
                if (TW == 2) dst[1] = hi;
            }
        }
    }
    __syncthreads();
    for (int it = tid; it < NC * O * JN; it += kTcThreads) {
        const int c = it % NC, j = (it / NC) % JN, o = it / (NC * JN);  // 4 coefficients: one 32-byte run
        const int b = b0 + j / 2;
        if (b >= B) continue;
        uint64_t r;
        if constexpr (W == 5) {  // sum_a 2^(8a) T_a < 2^89
            uint64_t hi = 0, lo = 0;
#pragma unroll
            for (int a = 0; a < W; a++) add_shl(hi, lo, Tb[(((size_t)c * MP + o * W + a) * JN + j)], 8 * a);
            r = reduce128(hi, lo, m);
        } else {  // T_a < 2^80: reduce each, then sum_a 2^(8a) (T_a mod q) < 2^119
            uint64_t hi = 0, lo = 0;
#pragma unroll
            for (int a = 0; a < W; a++) {
                const uint64_t *t = Tb + (((size_t)c * MP + o * W + a) * JN + j) * 2;
                add_shl(hi, lo, reduce128(t[1], t[0], m), 8 * a);
            }
            r = reduce128(hi, lo, m);
        }
        acc_out[((((uint32_t)o * B + b) * 2 + (j & 1)) * LP + k) * N + n0 + c] = r;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TCOLS));
}

// 40-bit limbs: 4 coefficients x 8 ciphertexts (M = 64, N = 80: two 80-column TMEM blocks,
// 72 KB of tiles); 60-bit limbs: 4 coefficients x 4 ciphertexts (N = 64).  Two CTAs per SM
// (TMEM: 256 columns each).
template <int L, int W, int MP>
void launch_tc(const Ctx &c, uint64_t *acc, const uint64_t *X, const uint64_t *D, const uint8_t *bank,
               const uint64_t *kbank, const int32_t *shifts, int B, int I, int T, int O, int kpad, cudaStream_t s) {
    using C = TcCfg<W, MP, W == 5 ? 4 : UH_TC_NC8, W == 5 ? 8 : 4>;
    const size_t smem = (size_t)C::NC * (MP + C::NP) * kpad;
    const size_t tb = (size_t)C::NC * MP * 2 * C::CT * (W == 5 ? 1 : 2) * 8;  // epilogue staging (reuses tiles)
    const size_t need = std::max(smem, tb);
    smem_optin(k_hoisted_tc<L, 15, W, C>, need);
    dim3 grid((unsigned)((B + C::CT - 1) / C::CT), (unsigned)(c.n / C::NC), W == 5 ? L - 1 : 2);
    k_hoisted_tc<L, 15, W, C><<<grid, kTcThreads, need, s>>>(acc, X, D, bank, kbank, shifts, B, I, T, O, c.sp(),
                                                             c.d_mods, kpad);
    UH_LAUNCH_CHECK();
}

inline int tc_kpad(int Q) { return (Q + 31) / 32 * 32; }
inline int tc_mp8(int O) { return O <= 8 ? 64 : 128; }

}  // namespace

// N = 2^15, 40-bit q_1..q_level and 60-bit q_0 / P, 1..12 dense masked outputs, <= 128 terms.
bool hoisted_tc_supported(const Ctx &c, int level, int O, int Q) {
    if (c.logn != 15 || level < 1 || level + 1 > 10 || O < 1 || O > 12 || Q < 1 || Q > kTcMaxTerms) return false;
    for (int k = 1; k <= level; k++)
        if (c.h_q[k] >> 40) return false;
    return (c.h_q[0] >> 40) && (c.h_q[c.count - 1] >> 40) && (c.h_q[0] >> 60) == 0 &&
           (c.h_q[c.count - 1] >> 60) == 0;
}

// bytes of the A-operand bank: the 40-bit-limb tiles followed by the 60-bit-limb tiles
size_t tc_bank_bytes(const Ctx &c, int level, int O, int Q) {
    const int kpad = tc_kpad(Q);
    return ((size_t)level * 64 + (size_t)2 * tc_mp8(O)) * kpad * c.n;
}

void tc_mask_bank(const Ctx &c, uint8_t *bank, const uint64_t *masks, int O, int Q, int level, cudaStream_t s) {
    const int L = level + 1, kpad = tc_kpad(Q);
    const size_t t5 = (size_t)(L - 1) * c.n * 64 * kpad / 4;
    k_tc_bank<5, 64><<<(unsigned)std::min<size_t>((t5 + 255) / 256, 148 * 32), 256, 0, s>>>(bank, masks, O, Q, L,
                                                                                          (int)c.logn, kpad);
    UH_LAUNCH_CHECK();
    uint8_t *b8 = bank + (size_t)(L - 1) * c.n * 64 * kpad;
    const int mp8 = tc_mp8(O);
    const size_t t8 = (size_t)2 * c.n * mp8 * kpad / 4;
    if (mp8 == 64)
        k_tc_bank<8, 64><<<(unsigned)std::min<size_t>((t8 + 255) / 256, 148 * 32), 256, 0, s>>>(b8, masks, O, Q, L,
                                                                                              (int)c.logn, kpad);
    else
        k_tc_bank<8, 128><<<(unsigned)std::min<size_t>((t8 + 255) / 256, 148 * 32), 256, 0, s>>>(b8, masks, O, Q, L,
                                                                                               (int)c.logn, kpad);
    UH_LAUNCH_CHECK();
}

void hoisted_mac_tc(const Ctx &c, uint64_t *acc, const uint64_t *X, const uint64_t *D, const uint8_t *bank,
                    const uint64_t *kbank, const int32_t *shifts, int B, int I, int T, int O, int level,
                    cudaStream_t s) {
    if (!hoisted_tc_supported(c, level, O, I * T))
        throw std::invalid_argument("tensor-core hoisted kernel: needs N = 2^15, 40-bit q_1..q_level, 60-bit q_0 / P, "
                                    "1 <= O <= 12, <= 128 terms");
    const int L = level + 1, kpad = tc_kpad(I * T);
    const double lim = 4294967295.0;
    if ((double)I * B * 2 * L * c.n > lim || (double)I * B * L * (L + 1) * c.n > lim ||
        (double)O * B * 2 * (L + 1) * c.n > lim || (double)T * (L + 1) * 2 * L * c.n > lim)
        throw std::invalid_argument("tensor-core hoisted kernel operand exceeds 2^32 elements: split the batch");
    const uint8_t *b8 = bank + (size_t)(L - 1) * c.n * 64 * kpad;
    const bool big = tc_mp8(O) == 128;
#define UH_TC_CASE(LL)                                                                              \
    case LL:                                                                                        \
        if (LL > 1) launch_tc<LL, 5, 64>(c, acc, X, D, bank, kbank, shifts, B, I, T, O, kpad, s);   \
        if (big)                                                                                    \
            launch_tc<LL, 8, 128>(c, acc, X, D, b8, kbank, shifts, B, I, T, O, kpad, s);            \
        else                                                                                        \
            launch_tc<LL, 8, 64>(c, acc, X, D, b8, kbank, shifts, B, I, T, O, kpad, s);             \
        break;
    switch (L) {
        UH_TC_CASE(2)
        UH_TC_CASE(3)
        UH_TC_CASE(4)
        UH_TC_CASE(5)
        UH_TC_CASE(6)
        UH_TC_CASE(7)
        UH_TC_CASE(8)
        UH_TC_CASE(9)
        UH_TC_CASE(10)
        default: throw std::invalid_argument("tensor-core hoisted kernel: 2 <= level + 1 <= 10");
    }
#undef UH_TC_CASE
}

}  // namespace uh
