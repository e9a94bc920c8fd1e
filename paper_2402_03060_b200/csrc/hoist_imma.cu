// Hoisted rotation-MAC with the weight-mask contraction on the tensor cores
// (mma.sync m16n8k32 u8 -> IMMA.16832 on sm_100a).  Same result as
// hoist_bank.cu's k_hoisted_bank, residue for residue:
//
//   acc[o][b] (QP basis) = sum over terms q = (i, t) of  M[o][q] (.) P * rot_{s_t}(ct_i[b])
//
// For a fixed coefficient n of a fixed limb k, phase B is a small integer GEMM
//   acc[o][j] = sum_q M[o][q][n] * V[q][j][n]      (j = ciphertext x component)
// whose A operand (the masks at n) is shared by every ciphertext.  Both factors
// are residues below q_k < 2^40 (the 40-bit limbs of the chain), so they split
// exactly into 5 bytes each, and
//   acc = sum_{a,b < 5} 2^(8(a+b)) * sum_q M_a[o][q] V_b[q][j]
// where each inner sum is a u8 x u8 dot product of length <= 256 (< 2^24 in
// s32: exact).  Rows of the MMA are (output, mask byte a), columns (value byte
// b, ciphertext, component); one m16n8k32 covers 3 outputs x 5 mask bytes by
// 8 columns by 32 terms.  The epilogue recombines the 25 byte products of each
// (output, column) in 128-bit integers and reduces mod q_k -- canonical, so the
// output is bit-identical to the IMAD kernel's.
//
// CTA tile: 8 coefficients x 4 ciphertexts x one 40-bit limb, 256 threads.
//   phase A : every (term, ciphertext, coefficient) item key-switches its term
//             (hoisted digits x Galois-key bank, + P c0, as hoist_bank.cu) and
//             writes the byte planes of the two results into shared memory, in
//             the B-fragment layout ([coefficient][byte][column][term]);
//   phase B : warp w takes (coefficient, m-tile) units; A fragments come from a
//             pre-split mask bank (16-byte loads, fragment order), B fragments
//             from shared memory; ceil(Q / 32) k-steps x 5 n-tiles of IMMA per unit, then
//             the byte recombination and the modular reduction per output.
// The 60-bit limbs (q_0, P) run k_hoisted_imma8 below (8-byte operands), or the IMAD key-bank kernel
// (hoisted_mac_bank_wide, hoist_bank.cu).  k_hoisted_imma_ta (further below) is this kernel with phase A
// on the tensor cores as well, the default where the level's digit bytes fit one k-step.
#include <cstdlib>
#include <type_traits>

#include "ops.cuh"

namespace uh {
namespace {

#ifndef UH_IMMA_NC
#define UH_IMMA_NC 8
#endif
#ifndef UH_IMMA_MINB
#define UH_IMMA_MINB 3
#endif
#ifndef UH_IMMA_MIN_O
#define UH_IMMA_MIN_O 5  // narrower layers stay on the register-only IMAD kernel
#endif
constexpr int kICT = 4;                     // ciphertexts per CTA
constexpr int kIJ = 2 * kICT;               // columns per value byte (ciphertext x component)
#ifndef UH_IMMA_NC_WIDE
#define UH_IMMA_NC_WIDE 4  // coefficients per CTA past 4 k-steps (keeps 3 CTAs / SM)
#endif
constexpr int kIMaxTerms = 256;             // 8 k-steps
// D = A x B (zero accumulator: the A fragment stays live for a second product)
__device__ __forceinline__ void imma0(int (&d)[4], const uint4 &a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%10,%10,%10};"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
        : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1), "r"(0));
}

// Byte width W = 5 of the 40-bit residues: 3 outputs x 5 mask bytes per 16-row m-tile, 4 m-tiles.
// NKS k-steps of 32 terms.  A B-plane row (coefficient, byte, column) holds 32 NKS terms + 16 bytes
// of pad: its word stride is 4 mod 8, so the 8 gid rows x 4 tig words of a fragment load hit 32
// distinct banks.
template <int W, int NKS> struct IW {
    static_assert(W == 5, "40-bit limbs only");
    static constexpr int NC = NKS > 4 ? UH_IMMA_NC_WIDE : UH_IMMA_NC;  // coefficients per CTA
    static constexpr int OPT = 3;                       // outputs per m-tile (m-tiles: ceil(O / 3))
    static constexpr int ROWB = NKS > 4 ? 32 * NKS + 16 : 144;  // bytes per B-plane row
    static constexpr int COEF = W * kIJ * ROWB + 4;     // coefficient stride of the B planes
    // C staging row stride (int32): 40 = 8 mod 32 puts both the fragment stores (4 rows per
    // half-warp) and the epilogue reads (rows o W + a of 3 outputs) on 32 distinct banks
    static constexpr int CS = W * 8;
    static constexpr size_t SMEM = (size_t)NC * COEF + 8 * 16 * CS * 4;
    static constexpr int MINB = UH_IMMA_MINB;           // resident CTAs per SM
};
constexpr int kIOPT = 3;
constexpr int kIMaxO = 48;                  // 16 m-tiles
__host__ __device__ constexpr int imma_mtiles(int O) { return (O + kIOPT - 1) / kIOPT; }

__device__ __forceinline__ uint32_t rot_index_i(uint32_t n, uint32_t half, uint32_t r) {
    uint32_t h = n >= half ? half : 0;
    uint32_t j = n - h + r;
    j = j >= half ? j - half : j;
    return h + j;
}
__device__ __forceinline__ uint64_t fold64_i(uint64_t hi, uint64_t lo, const Mod &m) {
    const uint64_t p = (uint64_t)(uint32_t)hi * m.r64;
    const uint64_t v = lo + p;
    return v < p ? v + m.r64 : v;
}

__device__ __forceinline__ void imma(int (&c)[4], const uint4 &a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}

// A-fragment mask bank [limb slot][N][m-tile][k-step][lane][4 words], ceil(O / 3) m-tiles: per
// coefficient, the (output x byte) x term matrix.  Row r of m-tile mt is output OPT mt + r / W,
// byte r % W (rows past OPT W and outputs >= O are zero).  Limb slots: limbs 1..L-1.
template <int W>
__global__ void k_imma_bank(uint32_t *__restrict__ ib, const uint64_t *__restrict__ masks, int O, int Q, int L,
                            int logn, int nks) {
    using C = IW<W, 1>;
    const uint32_t N = 1u << logn;
    const int nslots = L - 1;
    const int MT = imma_mtiles(O);
    const size_t total = (size_t)nslots * N * MT * nks * 32;
    const size_t ROW = (size_t)(L + 1) << logn;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
        const int lane = (int)(idx & 31);
        const int ks = (int)((idx >> 5) % nks);
        const size_t r0 = (idx >> 5) / nks;
        const int mt = (int)(r0 % MT);
        const size_t r1 = r0 / MT;
        const uint32_t n = (uint32_t)(r1 & (N - 1));
        const int slot = (int)(r1 >> logn);
        const int k = slot + 1;
        const int g = lane >> 2, tig = lane & 3;
        uint32_t w[4];
#pragma unroll
        for (int reg = 0; reg < 4; reg++) {
            const int row = g + (reg & 1) * 8;
            const int kb = ks * 32 + tig * 4 + (reg >> 1) * 16;
            const int o = mt * C::OPT + row / W, a = row % W;
            uint32_t v = 0;
            if (row < C::OPT * W && o < O) {
#pragma unroll
                for (int t = 0; t < 4; t++) {
                    const int q = kb + t;
                    if (q < Q) {
                        const uint64_t mv = masks[((size_t)o * Q + q) * ROW + ((size_t)k << logn) + n];
                        v |= (uint32_t)((mv >> (8 * a)) & 0xFF) << (8 * t);
                    }
                }
            }
            w[reg] = v;
        }
        reinterpret_cast<uint4 *>(ib)[(((r1 * MT + mt) * nks + ks) << 5) + lane] = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

template <int L, int LOGN, int NKS, int W>
__global__ void __launch_bounds__(256, IW<W, NKS>::MINB)
    k_hoisted_imma(uint64_t *__restrict__ acc_out, const uint64_t *__restrict__ X, const uint64_t *__restrict__ D,
                   const uint4 *__restrict__ ib, const uint64_t *__restrict__ kbank, const int32_t *__restrict__ shifts,
                   int B, int I, int T, int O, int sp, const Mod *__restrict__ mods) {
    using C = IW<W, NKS>;
    constexpr int kIRow = C::ROWB;
    constexpr int LP = L + 1;
    constexpr uint32_t N = 1u << LOGN, half = N >> 1;
    constexpr uint32_t ROW = (uint32_t)LP << LOGN;
    extern __shared__ __align__(16) unsigned char ism[];
    int *cst = reinterpret_cast<int *>(ism + (size_t)C::NC * C::COEF);
    __shared__ uint32_t s_x[32 * NKS], s_d[32 * NKS], s_k[32 * NKS], s_r[32 * NKS];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int b0 = blockIdx.x * kICT;
    const uint32_t n0 = blockIdx.y * C::NC;
    const int slot = blockIdx.z;
    const int k = 1 + slot;  // limb q_1..q_{L-1}
    constexpr bool qlimb = true;
    const Mod m = mods[k];
    const uint64_t P = mods[sp].q;
    const uint64_t Pk = P < m.q ? P : csub(barrett_lite(P, m), m.q);
    const int Q = I * T;
    for (int q = tid; q < Q; q += blockDim.x) {
        const int i = q / T, t = q - i * T;
        s_x[q] = (uint32_t)i * (uint32_t)B * (2u * L << LOGN);
        s_d[q] = (uint32_t)i * (uint32_t)B * ((uint32_t)L * LP << LOGN);
        s_k[q] = (uint32_t)t * ((uint32_t)LP * 2 * L << LOGN);
        s_r[q] = (uint32_t)shifts[t];
    }
    __syncthreads();

    // ---- phase A: key-switched P * rot(ct) per (term, ciphertext, coefficient) -> byte planes ----
    // one term per item (Q * 32 items over 256 threads: balanced to within one item per thread);
    // lanes = (ciphertext, coefficient), so the byte stores of a warp hit 32 distinct banks
    {
        // two ciphertexts per item: the Galois-key rows (2L loads) serve both -- a third fewer
        // loads through L1, which is the phase's limit (MIO throttle)
        constexpr int LH = 2 * C::NC;  // lanes per term: (ciphertext pair, coefficient)
        for (int it = tid; it < Q * LH; it += 256) {
            const int q = it / LH, cp = (it / C::NC) & 1, cf = it % C::NC;
            const int ba = b0 + 2 * cp;
            const bool oka = ba < B, okb = ba + 1 < B;
            const uint32_t n = n0 + cf;
            uint64_t v[2][2] = {{0, 0}, {0, 0}};
            const uint32_t r = s_r[q];
            const uint64_t *c0a = X + s_x[q] + (((uint32_t)ba * 2 * L + k) << LOGN);
            const uint64_t *c0b = c0a + ((uint32_t)(2 * L) << LOGN);
            if (r == 0) {
                if (oka && qlimb) {
                    v[0][0] = mulmod(Pk, __ldg(c0a + n), m);
                    v[0][1] = mulmod(Pk, __ldg(c0a + ((uint32_t)L << LOGN) + n), m);
                }
                if (okb && qlimb) {
                    v[1][0] = mulmod(Pk, __ldg(c0b + n), m);
                    v[1][1] = mulmod(Pk, __ldg(c0b + ((uint32_t)L << LOGN) + n), m);
                }
            } else if (oka) {
                const uint32_t src = rot_index_i(n, half, r);
                const uint64_t *Da = D + s_d[q] + (((uint32_t)ba * L * LP + k) << LOGN) + src;
                const uint64_t *Db = Da + ((uint32_t)(L * LP) << LOGN);
                const uint64_t *K = kbank + s_k[q] + ((uint32_t)k * 2 * L << LOGN) + n;
                uint64_t da[L], db[L], x[L], y[L];
#pragma unroll
                for (int j = 0; j < L; j++) {
                    x[j] = __ldg(K + ((uint32_t)(2 * j) << LOGN));
                    y[j] = __ldg(K + ((uint32_t)(2 * j + 1) << LOGN));
                    da[j] = __ldg(Da + (uint32_t)j * ROW);
                    db[j] = okb ? __ldg(Db + (uint32_t)j * ROW) : 0;
                }
                const uint64_t csa = qlimb ? __ldg(c0a + src) : 0, csb = qlimb && okb ? __ldg(c0b + src) : 0;
                using A = AccN;
                A a0, a1, e0, e1;
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
                auto fin = [&](const A &acc) -> uint64_t {
                    uint64_t h, l;
                    acc.value(h, l);
                    return csub(barrett_lite(fold64_i(h, l, m), m), m.q);
                };
                v[0][0] = fin(a0);
                v[0][1] = fin(a1);
                if (okb) {
                    v[1][0] = fin(e0);
                    v[1][1] = fin(e1);
                }
            }
            unsigned char *pl = ism + cf * C::COEF + (4 * cp) * kIRow + q;
#pragma unroll
            for (int bb = 0; bb < W; bb++)
#pragma unroll
                for (int e = 0; e < 4; e++) pl[bb * kIJ * kIRow + e * kIRow] = (unsigned char)(v[e >> 1][e & 1] >> (8 * bb));
        }
    }
    // terms [Q, 32 NKS) of the B planes are never written: their A bytes are zero (integer
    // products, so whatever the shared memory holds there contributes nothing)
    __syncthreads();

    // ---- phase B: IMMA per (coefficient, m-tile), byte recombination, reduction ----
    const int gid = lane >> 2, tig = lane & 3;
    int *cw = cst + warp * 16 * C::CS;
    const int nmt = imma_mtiles(O);
    for (int u = warp; u < C::NC * nmt; u += 8) {
        const int cf = u / nmt, mt = u - cf * nmt;
        const uint32_t n = n0 + cf;
        const uint4 *af = ib + ((((size_t)slot * N + n) * nmt + mt) * NKS << 5) + lane;
        uint4 A[NKS];
#pragma unroll
        for (int ks = 0; ks < NKS; ks++) A[ks] = __ldg(af + (ks << 5));
        int Cr[W][4];
#pragma unroll
        for (int nb = 0; nb < W; nb++) Cr[nb][0] = Cr[nb][1] = Cr[nb][2] = Cr[nb][3] = 0;
        const unsigned char *bp = ism + cf * C::COEF + gid * kIRow + tig * 4;
#pragma unroll
        for (int ks = 0; ks < NKS; ks++)
#pragma unroll
            for (int nb = 0; nb < W; nb++) {
                const unsigned char *p = bp + nb * kIJ * kIRow + ks * 32;
                imma(Cr[nb], A[ks], *reinterpret_cast<const uint32_t *>(p),
                     *reinterpret_cast<const uint32_t *>(p + 16));
            }
#pragma unroll
        for (int nb = 0; nb < W; nb++) {
            const int col = nb * 8 + tig * 2;
            *reinterpret_cast<int2 *>(cw + gid * C::CS + col) = make_int2(Cr[nb][0], Cr[nb][1]);
            *reinterpret_cast<int2 *>(cw + (gid + 8) * C::CS + col) = make_int2(Cr[nb][2], Cr[nb][3]);
        }
        __syncwarp();
        if (lane < C::OPT * 8) {
            const int ol = lane >> 3, j = lane & 7;
            const int o = mt * C::OPT + ol, b = b0 + (j >> 1);
            if (o < O && b < B) {
                uint64_t Ts[2 * W - 1];
#pragma unroll
                for (int s2 = 0; s2 < 2 * W - 1; s2++) Ts[s2] = 0;
#pragma unroll
                for (int a = 0; a < W; a++)
#pragma unroll
                    for (int nb = 0; nb < W; nb++) Ts[a + nb] += (uint32_t)cw[(ol * W + a) * C::CS + nb * 8 + j];
                // value = sum_s Ts[s] 2^(8 s) < 2^89: low part (s <= 4) and high part (s >= 5) * 2^40
                const uint64_t lo = Ts[0] + (Ts[1] << 8) + (Ts[2] << 16) + (Ts[3] << 24) + (Ts[4] << 32);
                const uint64_t hx = Ts[5] + (Ts[6] << 8) + (Ts[7] << 16) + (Ts[8] << 24);
                const uint64_t l2 = lo + (hx << 40);
                const uint64_t h2 = (hx >> 24) + (l2 < lo);
                const uint64_t r = reduce128(h2, l2, m);
                acc_out[((((uint32_t)o * B + b) * 2 + (j & 1)) * LP + k) * N + n] = r;
            }
        }
        __syncwarp();
    }
}

template <int L, int NKS, int W>
void launch_imma_k(const Ctx &c, uint64_t *acc, const uint64_t *X, const uint64_t *D, const uint32_t *ib,
                   const uint64_t *kbank, const int32_t *shifts, int B, int I, int T, int O, cudaStream_t s) {
    using C = IW<W, NKS>;
    smem_optin(k_hoisted_imma<L, 15, NKS, W>, C::SMEM);
    dim3 grid((unsigned)((B + kICT - 1) / kICT), (unsigned)(c.n / C::NC), L - 1);
    k_hoisted_imma<L, 15, NKS, W><<<grid, 256, C::SMEM, s>>>(acc, X, D, reinterpret_cast<const uint4 *>(ib), kbank,
                                                                shifts, B, I, T, O, c.sp(), c.d_mods);
    UH_LAUNCH_CHECK();
}

template <int L, int W>
void launch_imma(const Ctx &c, uint64_t *acc, const uint64_t *X, const uint64_t *D, const uint32_t *ib,
                 const uint64_t *kbank, const int32_t *shifts, int B, int I, int T, int O, cudaStream_t s) {
    const int nks = (I * T + 31) / 32;
    if (nks <= 1) launch_imma_k<L, 1, W>(c, acc, X, D, ib, kbank, shifts, B, I, T, O, s);
    else if (nks == 2) launch_imma_k<L, 2, W>(c, acc, X, D, ib, kbank, shifts, B, I, T, O, s);
    else if (nks == 3) launch_imma_k<L, 3, W>(c, acc, X, D, ib, kbank, shifts, B, I, T, O, s);
    else if (nks == 4) launch_imma_k<L, 4, W>(c, acc, X, D, ib, kbank, shifts, B, I, T, O, s);
    else if (nks == 5) launch_imma_k<L, 5, W>(c, acc, X, D, ib, kbank, shifts, B, I, T, O, s);
    else if (nks == 6) launch_imma_k<L, 6, W>(c, acc, X, D, ib, kbank, shifts, B, I, T, O, s);
    else if (nks == 7) launch_imma_k<L, 7, W>(c, acc, X, D, ib, kbank, shifts, B, I, T, O, s);
    else launch_imma_k<L, 8, W>(c, acc, X, D, ib, kbank, shifts, B, I, T, O, s);
}

// ---------------------------------------------------------------------------
// The 60-bit limbs q_0 and P: the same contraction with 8-byte operands.  Canonical residues
// below 2^60 and <= 256 terms keep sum_q M V <= 256 (q - 1)^2 < 2^128, so the 64 byte products of each
// (output, column) recombine exactly in 128 bits.  An m-tile is 2 outputs x 8 mask bytes; n-tiles
// are the 8 value bytes.  Phase A is hoist_bank.cu's 60-bit key switch (128-bit accumulators);
// the epilogue stages each warp's C fragments in shared memory and recombines every (output,
// column) on two lanes (4 mask bytes each), summed with one 128-bit shuffle.
#ifndef UH_IMMA8_NC
#define UH_IMMA8_NC 8  // coefficients per CTA up to 4 k-steps: 64-byte runs at 2 CTAs / SM (106 KB each) measured
#endif                 // 52.35 vs 53.3 ms for the LeNet conv2 call at B = 128 against 4 coefficients at 3 CTAs / SM
#ifndef UH_IMMA8_MINB
#define UH_IMMA8_MINB 2
#endif
#ifndef UH_IMMA8_NC_WIDE
#define UH_IMMA8_NC_WIDE 2  // past 4 k-steps (3 CTAs / SM)
#endif
constexpr int kI8MaxTerms = 256;  // (q - 1)^2 * 256 < 2^128 for q < 2^60
constexpr int kI8OPT = 2;
__host__ __device__ constexpr int imma8_mtiles(int O) { return (O + kI8OPT - 1) / kI8OPT; }
template <int NKS> struct IW8 {
    static constexpr int W = 8;
    static constexpr int NC = NKS > 4 ? UH_IMMA8_NC_WIDE : UH_IMMA8_NC;
    static constexpr int ROWB = NKS > 4 ? 32 * NKS + 16 : 144;  // terms + pad (word stride 4 mod 8)
    static constexpr int COEF = W * kIJ * ROWB + 4;
    // C staging: 16 rows x 64 columns per warp, the 8-column groups of row r rotated by 8 g(r),
    // g(4 q + i) = (i + q) mod 4 -- a Latin square, so both the fragment stores (4 consecutive rows
    // per half-warp) and the epilogue reads (rows i, i + 4, i + 8, i + 12) hit 32 distinct banks
    static constexpr int CS = 64;
    static constexpr size_t SMEM = (size_t)NC * COEF + 8 * 16 * CS * 4;
    static constexpr int MINB = NKS > 4 ? 3 : UH_IMMA8_MINB;  // the wide tiles keep 3 CTAs / SM
};
__device__ __forceinline__ int stage8_col(int row, int col) {
    const int g = ((row & 3) + (row >> 2)) & 3;
    return (col + 8 * g) & 63;
}

// A-fragment bank of the 60-bit limbs [slot 0: q_0, 1: P][N][m-tile][k-step][lane][4 words]:
// row r of m-tile mt is output 2 mt + r / 8, mask byte r % 8
__global__ void k_imma_bank8(uint32_t *__restrict__ ib, const uint64_t *__restrict__ masks, int O, int Q, int L,
                             int logn, int nks) {
    const uint32_t N = 1u << logn;
    const int MT = imma8_mtiles(O);
    const size_t total = (size_t)2 * N * MT * nks * 32;
    const size_t ROW = (size_t)(L + 1) << logn;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
        const int lane = (int)(idx & 31);
        const int ks = (int)((idx >> 5) % nks);
        const size_t r0 = (idx >> 5) / nks;
        const int mt = (int)(r0 % MT);
        const size_t r1 = r0 / MT;
        const uint32_t n = (uint32_t)(r1 & (N - 1));
        const int slot = (int)(r1 >> logn);
        const int k = slot ? L : 0;
        const int g = lane >> 2, tig = lane & 3;
        uint32_t w[4];
#pragma unroll
        for (int reg = 0; reg < 4; reg++) {
            const int row = g + (reg & 1) * 8;
            const int kb = ks * 32 + tig * 4 + (reg >> 1) * 16;
            const int o = mt * kI8OPT + (row >> 3), a = row & 7;
            uint32_t v = 0;
            if (o < O) {
#pragma unroll
                for (int t = 0; t < 4; t++) {
                    const int q = kb + t;
                    if (q < Q) {
                        const uint64_t mv = masks[((size_t)o * Q + q) * ROW + ((size_t)k << logn) + n];
                        v |= (uint32_t)((mv >> (8 * a)) & 0xFF) << (8 * t);
                    }
                }
            }
            w[reg] = v;
        }
        reinterpret_cast<uint4 *>(ib)[(((r1 * MT + mt) * nks + ks) << 5) + lane] = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

template <int L, int LOGN, int NKS>
__global__ void __launch_bounds__(256, IW8<NKS>::MINB)
    k_hoisted_imma8(uint64_t *__restrict__ acc_out, const uint64_t *__restrict__ X, const uint64_t *__restrict__ D,
                    const uint4 *__restrict__ ib, const uint64_t *__restrict__ kbank, const int32_t *__restrict__ shifts,
                    int B, int I, int T, int O, int sp, const Mod *__restrict__ mods) {
    using C = IW8<NKS>;
    constexpr int W = C::W;
    constexpr int kIRow = C::ROWB;
    constexpr int LP = L + 1;
    constexpr uint32_t N = 1u << LOGN, half = N >> 1;
    constexpr uint32_t ROW = (uint32_t)LP << LOGN;
    extern __shared__ __align__(16) unsigned char ism[];
    int *cst = reinterpret_cast<int *>(ism + (size_t)C::NC * C::COEF);
    __shared__ uint32_t s_x[32 * NKS], s_d[32 * NKS], s_k[32 * NKS], s_r[32 * NKS];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int b0 = blockIdx.x * kICT;
    const uint32_t n0 = blockIdx.y * C::NC;
    const int slot = blockIdx.z;  // 0: q_0, 1: P
    const int k = slot ? L : 0;   // QP-basis limb
    const bool qlimb = slot == 0;
    const Mod m = mods[qlimb ? 0 : sp];
    const uint64_t P = mods[sp].q;
    const uint64_t Pk = qlimb ? (P < m.q ? P : csub(barrett_lite(P, m), m.q)) : 0;
    const int Q = I * T;
    for (int q = tid; q < Q; q += blockDim.x) {
        const int i = q / T, t = q - i * T;
        s_x[q] = (uint32_t)i * (uint32_t)B * (2u * L << LOGN);
        s_d[q] = (uint32_t)i * (uint32_t)B * ((uint32_t)L * LP << LOGN);
        s_k[q] = (uint32_t)t * ((uint32_t)LP * 2 * L << LOGN);
        s_r[q] = (uint32_t)shifts[t];
    }
    __syncthreads();

    // ---- phase A: canonical P * rot(ct) per (term, ciphertext pair, coefficient) -> 8 byte planes ----
    {
        constexpr int LH = 2 * C::NC;
        for (int it = tid; it < Q * LH; it += 256) {
            const int q = it / LH, cp = (it / C::NC) & 1, cf = it % C::NC;
            const int ba = b0 + 2 * cp;
            const bool oka = ba < B, okb = ba + 1 < B;
            const uint32_t n = n0 + cf;
            uint64_t v[2][2] = {{0, 0}, {0, 0}};
            const uint32_t r = s_r[q];
            const uint64_t *c0a = X + s_x[q] + (((uint32_t)ba * 2 * L + k) << LOGN);
            const uint64_t *c0b = c0a + ((uint32_t)(2 * L) << LOGN);
            if (r == 0) {
                if (oka && qlimb) {
                    v[0][0] = mulmod(Pk, __ldg(c0a + n), m);
                    v[0][1] = mulmod(Pk, __ldg(c0a + ((uint32_t)L << LOGN) + n), m);
                }
                if (okb && qlimb) {
                    v[1][0] = mulmod(Pk, __ldg(c0b + n), m);
                    v[1][1] = mulmod(Pk, __ldg(c0b + ((uint32_t)L << LOGN) + n), m);
                }
            } else if (oka) {
                const uint32_t src = rot_index_i(n, half, r);
                const uint64_t *Da = D + s_d[q] + (((uint32_t)ba * L * LP + k) << LOGN) + src;
                const uint64_t *Db = Da + ((uint32_t)(L * LP) << LOGN);
                const uint64_t *K = kbank + s_k[q] + ((uint32_t)k * 2 * L << LOGN) + n;
                uint64_t da[L], db[L], x[L], y[L];
#pragma unroll
                for (int j = 0; j < L; j++) {
                    x[j] = __ldg(K + ((uint32_t)(2 * j) << LOGN));
                    y[j] = __ldg(K + ((uint32_t)(2 * j + 1) << LOGN));
                    da[j] = __ldg(Da + (uint32_t)j * ROW);
                    db[j] = okb ? __ldg(Db + (uint32_t)j * ROW) : 0;
                }
                // requested with the rest (left after the MAC loop, the compiler issues one of them there)
                const uint64_t csa = qlimb ? __ldg(c0a + src) : 0, csb = qlimb && okb ? __ldg(c0b + src) : 0;
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
                    if (okb) e0.mac(Pk, csb);
                }
                v[0][0] = a0.reduce(m);
                v[0][1] = a1.reduce(m);
                if (okb) {
                    v[1][0] = e0.reduce(m);
                    v[1][1] = e1.reduce(m);
                }
            }
            unsigned char *pl = ism + cf * C::COEF + (4 * cp) * kIRow + q;
#pragma unroll
            for (int bb = 0; bb < W; bb++)
#pragma unroll
                for (int e = 0; e < 4; e++) pl[bb * kIJ * kIRow + e * kIRow] = (unsigned char)(v[e >> 1][e & 1] >> (8 * bb));
        }
    }
    __syncthreads();

    // ---- phase B: IMMA per (coefficient, m-tile), staged recombination, reduction ----
    const int gid = lane >> 2, tig = lane & 3;
    int *cw = cst + warp * 16 * C::CS;
    const int nmt = imma8_mtiles(O);
    for (int u = warp; u < C::NC * nmt; u += 8) {
        const int cf = u / nmt, mt = u - cf * nmt;
        const uint32_t n = n0 + cf;
        const uint4 *af = ib + ((((size_t)slot * N + n) * nmt + mt) * NKS << 5) + lane;
        uint4 A[NKS];
#pragma unroll
        for (int ks = 0; ks < NKS; ks++) A[ks] = __ldg(af + (ks << 5));
        int Cr[W][4];
#pragma unroll
        for (int nb = 0; nb < W; nb++) Cr[nb][0] = Cr[nb][1] = Cr[nb][2] = Cr[nb][3] = 0;
        const unsigned char *bp = ism + cf * C::COEF + gid * kIRow + tig * 4;
#pragma unroll
        for (int ks = 0; ks < NKS; ks++)
#pragma unroll
            for (int nb = 0; nb < W; nb++) {
                const unsigned char *p = bp + nb * kIJ * kIRow + ks * 32;
                imma(Cr[nb], A[ks], *reinterpret_cast<const uint32_t *>(p),
                     *reinterpret_cast<const uint32_t *>(p + 16));
            }
#pragma unroll
        for (int nb = 0; nb < W; nb++) {
            const int col = nb * 8 + tig * 2;
            *reinterpret_cast<int2 *>(cw + gid * C::CS + stage8_col(gid, col)) = make_int2(Cr[nb][0], Cr[nb][1]);
            *reinterpret_cast<int2 *>(cw + (gid + 8) * C::CS + stage8_col(gid + 8, col)) =
                make_int2(Cr[nb][2], Cr[nb][3]);
        }
        __syncwarp();
        {
            // lane pair (2 pr, 2 pr + 1): output 2 mt + ol, column j; half h sums mask bytes 4h..4h+3
            const int pr = lane >> 1, h = lane & 1;
            const int ol = pr >> 3, j = pr & 7;
            uint32_t Ts[11];
#pragma unroll
            for (int s2 = 0; s2 < 11; s2++) Ts[s2] = 0;
#pragma unroll
            for (int a4 = 0; a4 < 4; a4++)
#pragma unroll
                for (int nb = 0; nb < W; nb++) {
                    const int row = ol * 8 + 4 * h + a4;
                    Ts[a4 + nb] += (uint32_t)cw[row * C::CS + stage8_col(row, nb * 8 + j)];
                }
            // value of this half = 2^(32 h) sum_s Ts[s] 2^(8 s)  (Ts < 2^25: the half sum < 2^106)
            u128 v = 0;
#pragma unroll
            for (int s2 = 0; s2 < 11; s2++) v += (u128)Ts[s2] << (8 * s2);
            v <<= 32 * h;
            uint64_t lo = (uint64_t)v, hi = (uint64_t)(v >> 64);
            const uint64_t lo2 = __shfl_xor_sync(0xffffffffu, lo, 1), hi2 = __shfl_xor_sync(0xffffffffu, hi, 1);
            lo += lo2;
            hi += hi2 + (lo < lo2);
            const int o = mt * kI8OPT + ol, b = b0 + (j >> 1);
            if (h == 0 && o < O && b < B)
                acc_out[((((uint32_t)o * B + b) * 2 + (j & 1)) * LP + k) * N + n] = reduce128(hi, lo, m);
        }
        __syncwarp();
    }
}

template <int L, int NKS>
void launch_imma8_k(const Ctx &c, uint64_t *acc, const uint64_t *X, const uint64_t *D, const uint32_t *ib8,
                    const uint64_t *kbank, const int32_t *shifts, int B, int I, int T, int O, cudaStream_t s) {
    using C = IW8<NKS>;
    smem_optin(k_hoisted_imma8<L, 15, NKS>, C::SMEM);
    dim3 grid((unsigned)((B + kICT - 1) / kICT), (unsigned)(c.n / C::NC), 2);
    k_hoisted_imma8<L, 15, NKS><<<grid, 256, C::SMEM, s>>>(acc, X, D, reinterpret_cast<const uint4 *>(ib8), kbank,
                                                             shifts, B, I, T, O, c.sp(), c.d_mods);
    UH_LAUNCH_CHECK();
}

template <int L>
void launch_imma8(const Ctx &c, uint64_t *acc, const uint64_t *X, const uint64_t *D, const uint32_t *ib8,
                  const uint64_t *kbank, const int32_t *shifts, int B, int I, int T, int O, cudaStream_t s) {
    const int nks = (I * T + 31) / 32;
    if (nks <= 1) launch_imma8_k<L, 1>(c, acc, X, D, ib8, kbank, shifts, B, I, T, O, s);
    else if (nks == 2) launch_imma8_k<L, 2>(c, acc, X, D, ib8, kbank, shifts, B, I, T, O, s);
    else if (nks == 3) launch_imma8_k<L, 3>(c, acc, X, D, ib8, kbank, shifts, B, I, T, O, s);
    else if (nks == 4) launch_imma8_k<L, 4>(c, acc, X, D, ib8, kbank, shifts, B, I, T, O, s);
    else if (nks == 5) launch_imma8_k<L, 5>(c, acc, X, D, ib8, kbank, shifts, B, I, T, O, s);
    else if (nks == 6) launch_imma8_k<L, 6>(c, acc, X, D, ib8, kbank, shifts, B, I, T, O, s);
    else if (nks == 7) launch_imma8_k<L, 7>(c, acc, X, D, ib8, kbank, shifts, B, I, T, O, s);
    else launch_imma8_k<L, 8>(c, acc, X, D, ib8, kbank, shifts, B, I, T, O, s);
}

// the 60-bit limbs on the 8-byte IMMA kernel: every term count up to 128, q_0 and P below 2^60
bool imma8_ok(const Ctx &c, int Q) {
    if (Q > kI8MaxTerms) return false;
    const char *e = getenv("UH_IMMA8");
    if (e && e[0] == '0') return false;
    return !(c.h_q[0] >> 60) && !(c.h_q[c.count - 1] >> 60);
}


// ---------------------------------------------------------------------------
// Phase A on the tensor cores too (40-bit limbs, 5 (level + 1) <= 32).  The key switch of a term,
//   V[b][c] = sum_j D_j[b][n + s] K_{t,j,c}[n]  (mod q),
// splits D_j into bytes d_{j,a} and folds the byte weight into the key,
//   V = sum_{(j,a)} d_{j,a}[b] * K'_{(j,a),c},   K' = 2^(8a) K_{t,j,c} mod q  (again 5 bytes e),
// so for one (term, coefficient) the sums S_e[b][c] = sum_{(j,a)} d_{j,a}[b] byte_e(K'_{(j,a),c}) are ONE
// m16n8k32 per component: rows = 16 ciphertexts, K = the 5 L <= 32 digit bytes, columns = the 5 key
// bytes (+3 zero).  V = sum_e 2^(8e) S_e < 2^54 is recombined on the quad that holds a row
// (three 32-bit shuffles), P * c0 (pre-multiplied once per call) is added, one Barrett reduction
// gives the canonical residue -- the same value the IMAD phase A produces -- and its bytes go to
// the phase-B planes.  Operands: dp = the ModUp digits re-laid as bytes [slot][N][I * B][32]
// (k_ta_digits), kt = the key bank in B-fragment order [slot][N][T][lane][4 words] (k_ta_bank,
// once per layer), pc = P * (c0, c1) [I * B][2][slot][N].
// CTA tile: 16 ciphertexts x NC coefficients x one 40-bit limb; phase B as k_hoisted_imma over the
// tile's 32 columns (four n-tile groups per A-fragment load).
#ifndef UH_IMMA_TA_NC
#define UH_IMMA_TA_NC 2
#endif
#ifndef UH_IMMA_TA_MINB
#define UH_IMMA_TA_MINB 3
#endif
constexpr int kTCT = 16;
template <int NKS> struct IWT {
    static constexpr int W = 5, NC = UH_IMMA_TA_NC, OPT = 3;
    static constexpr int ROWB = NKS > 4 ? 32 * NKS + 16 : 144;  // bytes per B-plane row (terms + pad)
    static constexpr int GRP = 8 * ROWB + 4;   // one n-tile (8 columns) + a word: the 4 groups sit on distinct banks
    static constexpr int PLANE = 4 * GRP;      // 32 columns (ciphertext, component) of one byte
    static constexpr int COEF = W * PLANE;
    static constexpr int CS = W * 8;
    static constexpr size_t SMEM = (size_t)NC * COEF + 8 * 16 * CS * 4;
};

// Operand re-layout for the tensor-core phase A, one pass over the ModUp digits and c0:
//   dp[slot][n][r][32]: digit bytes, r = i * B + b; byte 5 j + a = byte a of D[i][b][j][1 + slot][n]
//   pc[slot][n][r]    : P * c0 = P * X[r][0][1 + slot][n] mod q_{1+slot}
// (ciphertext innermost: the 16 ciphertexts of a phase-A unit read whole lines).  A CTA transposes a
// 32-coefficient x 32-ciphertext tile through shared memory: coalesced limb reads (lanes = n), coalesced
// row writes (lanes = consecutive words of one coefficient's 32 rows); the tile's row strides (257 / 65
// words) keep both sides bank-conflict-free.
template <int L>
__global__ void __launch_bounds__(256)
    k_ta_pack(unsigned char *__restrict__ dp, uint64_t *__restrict__ pc, const uint64_t *__restrict__ D,
              const uint64_t *__restrict__ X, int R, int logn, int sp, const Mod *__restrict__ mods) {
    __shared__ uint32_t tw[32 * 257];
    __shared__ uint32_t tp[32 * 65];
    const size_t N = (size_t)1 << logn;
    const int LP = L + 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t n0 = (size_t)blockIdx.x * 32;
    const int r0 = blockIdx.y * 32, slot = blockIdx.z, k = 1 + slot;
    const Mod m = mods[k];
    const uint64_t P = mods[sp].q;
    const uint64_t Pk = P < m.q ? P : csub(barrett_lite(P, m), m.q);
#pragma unroll
    for (int rr = 0; rr < 4; rr++) {
        const int rl = warp + 8 * rr, r = r0 + rl;
        uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        uint64_t pv = 0;
        if (r < R) {
            uint64_t d[L];
#pragma unroll
            for (int j = 0; j < L; j++) d[j] = D[(((size_t)r * L + j) * LP + k) * N + n0 + lane];
            const uint64_t x0 = X[((size_t)r * 2 * L + k) * N + n0 + lane];
            // the 40-bit digits concatenated little-endian: digit j occupies bits [40 j, 40 j + 40)
#pragma unroll
            for (int j = 0; j < L; j++) {
                const int bit = 40 * j, wi = bit >> 5, sh = bit & 31;  // compile-time
                const uint64_t lo = d[j] << sh;                         // bits of words wi, wi + 1
                w[wi] |= (uint32_t)lo;
                w[wi + 1] |= (uint32_t)(lo >> 32);
                if (sh > 24) w[wi + 2] |= (uint32_t)(d[j] >> (64 - sh));  // spill past two words
            }
            pv = mulmod(Pk, x0, m);
        }
#pragma unroll
        for (int i = 0; i < 8; i++) tw[lane * 257 + rl * 8 + i] = w[i];
        tp[lane * 65 + rl * 2] = (uint32_t)pv;
        tp[lane * 65 + rl * 2 + 1] = (uint32_t)(pv >> 32);
    }
    __syncthreads();
    uint32_t *dpw = reinterpret_cast<uint32_t *>(dp);
    uint32_t *pcw = reinterpret_cast<uint32_t *>(pc);
#pragma unroll
    for (int nn = 0; nn < 4; nn++) {
        const int nl = warp + 8 * nn;
        const size_t row = ((size_t)slot * N + n0 + nl) * R + r0;  // first row of this coefficient's tile
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const int idx = lane + 32 * i;  // word of the 32 rows x 8 words
            if (r0 + (idx >> 3) < R) dpw[row * 8 + idx] = tw[nl * 257 + idx];
        }
#pragma unroll
        for (int i = 0; i < 2; i++) {
            const int idx = lane + 32 * i;
            if (r0 + (idx >> 1) < R) pcw[row * 2 + idx] = tp[nl * 65 + idx];
        }
    }
}

// x mod q in [0, 2q) for x < 2^56 and 2^39 < q < 2^40 (bar = floor(2^64 / q) < 2^25): the high word of
// x * bar from two 32 x 32 products
__device__ __forceinline__ uint64_t barrett_small(uint64_t x, uint32_t bar, uint64_t q) {
    const uint32_t x0 = (uint32_t)x, x1 = (uint32_t)(x >> 32);
    const uint64_t t = (uint64_t)x0 * bar;
    const uint64_t u = (uint64_t)x1 * bar + (t >> 32);
    const uint32_t qh = (uint32_t)(u >> 32);
    return x - (uint64_t)qh * q;
}

// key bank in B-fragment order: kt[slot][n][t][lane] = (comp 0: b0, b1; comp 1: b0, b1).  Lane (g, tig)
// holds column e = g (key byte) and the digit-byte positions 8 tig + x (b0) and 8 tig + 4 + x (b1), x < 4
// -- the bytes of a dp row a lane loads as its A fragment (one 8-byte load per row).
__global__ void k_ta_bank(uint4 *__restrict__ kt, const uint64_t *__restrict__ kbank, const int32_t *__restrict__ shifts,
                          int T, int L, int logn, const Mod *__restrict__ mods) {
    const size_t N = (size_t)1 << logn;
    const int NS = L - 1, LP = L + 1;
    const size_t total = (size_t)NS * N * T * 32;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
        const int lane = (int)(idx & 31);
        const size_t r0 = idx >> 5;
        const int t = (int)(r0 % T);
        const size_t r1 = r0 / T;
        const size_t n = r1 & (N - 1);
        const int slot = (int)(r1 >> logn), k = 1 + slot;
        const int g = lane >> 2, tig = lane & 3;
        const Mod m = mods[k];
        uint32_t w[4] = {0, 0, 0, 0};
        if (g < 5 && shifts[t] != 0) {
#pragma unroll
            for (int reg = 0; reg < 2; reg++)
#pragma unroll
                for (int x = 0; x < 4; x++) {
                    const int pos = 8 * tig + 4 * reg + x;
                    const int j = pos / 5, a = pos - 5 * j;
                    if (j < L) {
#pragma unroll
                        for (int c = 0; c < 2; c++) {
                            const uint64_t kv = kbank[(((size_t)t * LP + k) * 2 * L + 2 * j + c) * N + n];
                            const uint64_t kw = mulmod(kv, (uint64_t)1 << (8 * a), m);  // 2^(8a) < q
                            w[2 * c + reg] |= (uint32_t)((kw >> (8 * g)) & 0xFF) << (8 * x);
                        }
                    }
                }
        }
        kt[idx] = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

template <int L, int LOGN, int NKS>
__global__ void __launch_bounds__(256, UH_IMMA_TA_MINB)
    k_hoisted_imma_ta(uint64_t *__restrict__ acc_out, const uint64_t *__restrict__ X,
                      const unsigned char *__restrict__ dp, const uint64_t *__restrict__ pc,
                      const uint4 *__restrict__ ib, const uint4 *__restrict__ kt, const int32_t *__restrict__ shifts,
                      int B, int I, int T, int O, int sp, const Mod *__restrict__ mods) {
    using C = IWT<NKS>;
    constexpr int W = C::W;
    constexpr int LP = L + 1;
    constexpr uint32_t N = 1u << LOGN, half = N >> 1;
    static_assert(5 * L <= 32, "one k-step holds the digit bytes");
    extern __shared__ __align__(16) unsigned char ism[];
    int *cst = reinterpret_cast<int *>(ism + (size_t)C::NC * C::COEF);
    __shared__ uint32_t s_ib[32 * NKS], s_t[32 * NKS], s_r[32 * NKS];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gid = lane >> 2, tig = lane & 3;
    const int b0 = blockIdx.x * kTCT;
    const uint32_t n0 = blockIdx.y * C::NC;
    const int slot = blockIdx.z;
    const int k = 1 + slot;
    const Mod m = mods[k];
    const int Q = I * T;
    const uint32_t R = (uint32_t)I * B;
    for (int q = tid; q < Q; q += blockDim.x) {
        const int i = q / T, t = q - i * T;
        s_ib[q] = (uint32_t)i * B;
        s_t[q] = t;
        s_r[q] = (uint32_t)shifts[t];
    }
    __syncthreads();

    // ---- phase A: one (term, coefficient) unit per warp iteration ----
    {
        // after the quad exchange lane (gid, tig) owns ciphertext gid + 8 (tig >> 1), component tig & 1
        const int ctl = gid + 8 * (tig >> 1), comp = tig & 1;
        const int b = b0 + ctl;
        const int col = 2 * ctl + comp;
        const bool rowa = b0 + gid < B, rowb = b0 + gid + 8 < B, pc_on = comp == 0 && b < B;
        unsigned char *plane = ism + (col >> 3) * C::GRP + (col & 7) * C::ROWB;
        // per-lane bases; the per-unit offsets fit 32 bits (checked on the host)
        const unsigned char *dbase = dp + ((size_t)slot * N * R + b0 + gid) * 32 + tig * 8;
        const uint4 *kbase = kt + (((size_t)slot * N + n0) * T << 5) + lane;
        const uint64_t *pbase = pc + (size_t)slot * N * R + b;
        const uint32_t bar = (uint32_t)m.bar;
        const bool t1 = tig & 1, t2 = tig & 2;
        const uint64_t P = mods[sp].q;
        const uint64_t Pk = P < m.q ? P : csub(barrett_lite(P, m), m.q);
        // operands of one (term q, coefficient n0 + cf) unit, loaded ahead of the arithmetic so the two
        // units of an iteration have their loads in flight together
        struct Unit {
            uint2 ra, rb;
            uint4 kb;
            uint64_t pcv;  // P c0 at the rotated slot (component-0 lanes); for a zero shift: the c value itself
            bool zero;
        };
        auto load = [&](int q, int cf) -> Unit {
            Unit w;
            const uint32_t n = n0 + cf;
            const uint32_t r = s_r[q];
            const uint32_t ib0 = s_ib[q];
            w.zero = r == 0;
            w.ra = w.rb = make_uint2(0, 0);
            w.kb = make_uint4(0, 0, 0, 0);
            w.pcv = 0;
            if (w.zero) {
                if (b < B) w.pcv = __ldg(X + (((size_t)(ib0 + b) * 2 + comp) * L + k) * N + n);
                return w;
            }
            const uint32_t src = rot_index_i(n, half, r);
            const unsigned char *drow = dbase + (size_t)((src * R + ib0) << 5);
            if (rowa) w.ra = __ldg(reinterpret_cast<const uint2 *>(drow));
            if (rowb) w.rb = __ldg(reinterpret_cast<const uint2 *>(drow + 8 * 32));
            if (gid < 5) w.kb = __ldg(kbase + ((cf * (uint32_t)T + s_t[q]) << 5));  // columns 5..7: zero padding
            if (pc_on) w.pcv = __ldg(pbase + (size_t)(src * R + ib0));
            return w;
        };
        // the canonical key-switched value of the unit for this lane's (ciphertext, component)
        auto compute = [&](const Unit &w) -> uint64_t {
            if (w.zero) return b < B ? mulmod(Pk, w.pcv, m) : 0;  // warp-uniform branch
            const uint4 af = make_uint4(w.ra.x, w.rb.x, w.ra.y, w.rb.y);
            int c0[4], c1[4];
            imma0(c0, af, w.kb.x, w.kb.y);
            imma0(c1, af, w.kb.z, w.kb.w);
            // this lane's share (key bytes 2 tig, 2 tig + 1) of the four (row, component) values
            const uint32_t p0 = (uint32_t)c0[0] + ((uint32_t)c0[1] << 8);  // row gid,     component 0
            const uint32_t p1 = (uint32_t)c1[0] + ((uint32_t)c1[1] << 8);  // row gid,     component 1
            const uint32_t p2 = (uint32_t)c0[2] + ((uint32_t)c0[3] << 8);  // row gid + 8, component 0
            const uint32_t p3 = (uint32_t)c1[2] + ((uint32_t)c1[3] << 8);  // row gid + 8, component 1
            // quad exchange: lane tig owns value tig.  Round d sends e_d = p[(tig - d) & 3] to lane tig - d
            // and receives lane tig + d's share.  With b = (p0, p3, p2, p1), e_d = b[(d - tig) & 3]: a
            // barrel rotation of b by tig & 1, then by tig & 2
            const uint32_t a0 = t1 ? p1 : p0, a1 = t1 ? p0 : p3, a2 = t1 ? p3 : p2, a3 = t1 ? p2 : p1;
            const uint32_t e0 = t2 ? a2 : a0, e1 = t2 ? a3 : a1, e2 = t2 ? a0 : a2, e3 = t2 ? a1 : a3;
            const uint32_t g1 = __shfl_sync(0xffffffffu, e1, (lane & ~3) | ((tig + 1) & 3));
            const uint32_t g2 = __shfl_sync(0xffffffffu, e2, (lane & ~3) | ((tig + 2) & 3));
            const uint32_t g3 = __shfl_sync(0xffffffffu, e3, (lane & ~3) | ((tig + 3) & 3));
            // shares by source lane, S[s] = g[(s - tig) & 3] (g_0 = e0): the same rotation applied to the
            // received shares; lane 3's share is zero (key-byte columns 6, 7), so sources 0, 1, 2 are placed
            const uint32_t h0 = t1 ? g3 : e0, h1 = t1 ? e0 : g1, h2 = t1 ? g1 : g2, h3 = t1 ? g2 : g3;
            const uint32_t s0 = t2 ? h2 : h0, s1 = t2 ? h3 : h1, s2 = t2 ? h0 : h2;
            const uint64_t v = (uint64_t)s0 + ((uint64_t)s1 << 16) + ((uint64_t)s2 << 32) + w.pcv;
            return csub(barrett_small(v, bar, m.q), m.q);
        };
        const int QP = (Q + 1) >> 1;
        for (int u = warp; u < QP * C::NC; u += 8) {
            const int qp = u / C::NC, cf = u - qp * C::NC;
            const int q = 2 * qp;
            const bool two = q + 1 < Q;  // warp-uniform
            const Unit wa = load(q, cf);
            Unit wb;
            if (two) wb = load(q + 1, cf);
            const uint64_t va = compute(wa);
            const uint64_t vb = two ? compute(wb) : 0;
            unsigned char *pl = plane + cf * C::COEF + q;
            const uint32_t al = (uint32_t)va, bl = (uint32_t)vb;
            *reinterpret_cast<unsigned short *>(pl) = (unsigned short)__byte_perm(al, bl, 0x0040);
            *reinterpret_cast<unsigned short *>(pl + C::PLANE) = (unsigned short)__byte_perm(al, bl, 0x0051);
            *reinterpret_cast<unsigned short *>(pl + 2 * C::PLANE) = (unsigned short)__byte_perm(al, bl, 0x0062);
            *reinterpret_cast<unsigned short *>(pl + 3 * C::PLANE) = (unsigned short)__byte_perm(al, bl, 0x0073);
            *reinterpret_cast<unsigned short *>(pl + 4 * C::PLANE) =
                (unsigned short)(((uint32_t)(va >> 32) & 0xFF) | (((uint32_t)(vb >> 32) & 0xFF) << 8));
        }
    }
    __syncthreads();

    // ---- phase B: IMMA per (coefficient, m-tile, column group), byte recombination, reduction ----
    int *cw = cst + warp * 16 * C::CS;
    const int nmt = imma_mtiles(O);
    for (int u = warp; u < C::NC * nmt; u += 8) {
        const int cf = u / nmt, mt = u - cf * nmt;
        const uint32_t n = n0 + cf;
        const uint4 *af = ib + ((((size_t)slot * N + n) * nmt + mt) * NKS << 5) + lane;
        uint4 A[NKS];
#pragma unroll
        for (int ks = 0; ks < NKS; ks++) A[ks] = __ldg(af + (ks << 5));
#pragma unroll 1
        for (int cg = 0; cg < 4; cg++) {
            if (b0 + 4 * cg >= B) break;
            int Cr[W][4];
#pragma unroll
            for (int nb = 0; nb < W; nb++) Cr[nb][0] = Cr[nb][1] = Cr[nb][2] = Cr[nb][3] = 0;
            const unsigned char *bp = ism + cf * C::COEF + cg * C::GRP + gid * C::ROWB + tig * 4;
#pragma unroll
            for (int ks = 0; ks < NKS; ks++)
#pragma unroll
                for (int nb = 0; nb < W; nb++) {
                    const unsigned char *p = bp + nb * C::PLANE + ks * 32;
                    imma(Cr[nb], A[ks], *reinterpret_cast<const uint32_t *>(p),
                         *reinterpret_cast<const uint32_t *>(p + 16));
                }
#pragma unroll
            for (int nb = 0; nb < W; nb++) {
                const int cc = nb * 8 + tig * 2;
                *reinterpret_cast<int2 *>(cw + gid * C::CS + cc) = make_int2(Cr[nb][0], Cr[nb][1]);
                *reinterpret_cast<int2 *>(cw + (gid + 8) * C::CS + cc) = make_int2(Cr[nb][2], Cr[nb][3]);
            }
            __syncwarp();
            if (lane < C::OPT * 8) {
                const int ol = lane >> 3, j = lane & 7;
                const int o = mt * C::OPT + ol, b = b0 + 4 * cg + (j >> 1);
                if (o < O && b < B) {
                    uint64_t Ts[2 * W - 1];
#pragma unroll
                    for (int s2 = 0; s2 < 2 * W - 1; s2++) Ts[s2] = 0;
#pragma unroll
                    for (int a = 0; a < W; a++)
#pragma unroll
                        for (int nb = 0; nb < W; nb++) Ts[a + nb] += (uint32_t)cw[(ol * W + a) * C::CS + nb * 8 + j];
                    const uint64_t lo = Ts[0] + (Ts[1] << 8) + (Ts[2] << 16) + (Ts[3] << 24) + (Ts[4] << 32);
                    const uint64_t hx = Ts[5] + (Ts[6] << 8) + (Ts[7] << 16) + (Ts[8] << 24);
                    const uint64_t l2 = lo + (hx << 40);
                    const uint64_t h2 = (hx >> 24) + (l2 < lo);
                    acc_out[((((uint32_t)o * B + b) * 2 + (j & 1)) * LP + k) * N + n] = reduce128(h2, l2, m);
                }
            }
            __syncwarp();
        }
    }
}

template <int L, int NKS>
void launch_imma_ta_k(const Ctx &c, uint64_t *acc, const uint64_t *X, const unsigned char *dp, const uint64_t *pc,
                      const uint32_t *ib,
                      const uint4 *kt, const int32_t *shifts, int B, int I, int T, int O, cudaStream_t s) {
    using C = IWT<NKS>;
    smem_optin(k_hoisted_imma_ta<L, 15, NKS>, C::SMEM);
    dim3 grid((unsigned)((B + kTCT - 1) / kTCT), (unsigned)(c.n / C::NC), L - 1);
    k_hoisted_imma_ta<L, 15, NKS><<<grid, 256, C::SMEM, s>>>(acc, X, dp, pc, reinterpret_cast<const uint4 *>(ib), kt,
                                                               shifts, B, I, T, O, c.sp(), c.d_mods);
    UH_LAUNCH_CHECK();
}

template <int L>
void launch_imma_ta(const Ctx &c, uint64_t *acc, const uint64_t *X, const unsigned char *dp, const uint64_t *pc,
                    const uint32_t *ib,
                    const uint4 *kt, const int32_t *shifts, int B, int I, int T, int O, cudaStream_t s) {
    const int nks = (I * T + 31) / 32;
    if (nks <= 1) launch_imma_ta_k<L, 1>(c, acc, X, dp, pc, ib, kt, shifts, B, I, T, O, s);
    else if (nks == 2) launch_imma_ta_k<L, 2>(c, acc, X, dp, pc, ib, kt, shifts, B, I, T, O, s);
    else if (nks == 3) launch_imma_ta_k<L, 3>(c, acc, X, dp, pc, ib, kt, shifts, B, I, T, O, s);
    else launch_imma_ta_k<L, 4>(c, acc, X, dp, pc, ib, kt, shifts, B, I, T, O, s);
}

}  // namespace

// Applicable when N = 2^15, the level has 40-bit limbs q_1..q_{L-1} (< 2^40) and 60-bit
// q_0 and P, 5..48 dense masked outputs and at most 256 terms.
bool hoisted_imma_supported(const Ctx &c, int level, int O, int Q) {
    if (c.logn != 15 || level < 2 || level + 1 > 10 || O < UH_IMMA_MIN_O || O > kIMaxO || Q < 1 || Q > kIMaxTerms)
        return false;
    for (int k = 1; k <= level; k++)
        if (c.h_q[k] >> 40) return false;
    return (c.h_q[0] >> 40) && (c.h_q[c.count - 1] >> 40);
}

// uint32 words of the 40-bit-limb bank
static size_t imma_bank5_words(const Ctx &c, int level, int O, int Q) {
    const int nks = (Q + 31) / 32;
    return (size_t)level * imma_mtiles(O) * c.n * nks * 32 * 4;
}
// the whole bank: the 40-bit limbs' part, then (when the 60-bit limbs run the 8-byte kernel) q_0 / P's
size_t imma_bank_words(const Ctx &c, int level, int O, int Q) {
    const int nks = (Q + 31) / 32;
    return imma_bank5_words(c, level, O, Q) + (imma8_ok(c, Q) ? (size_t)2 * imma8_mtiles(O) * c.n * nks * 32 * 4 : 0);
}

void imma_mask_bank(const Ctx &c, uint32_t *ib, const uint64_t *masks, int O, int Q, int level, cudaStream_t s) {
    const int L = level + 1, nks = (Q + 31) / 32;
    const size_t t5 = (size_t)(L - 1) * c.n * imma_mtiles(O) * nks * 32;
    k_imma_bank<5><<<(unsigned)std::min<size_t>((t5 + 255) / 256, 148 * 32), 256, 0, s>>>(ib, masks, O, Q, L,
                                                                                         (int)c.logn, nks);
    UH_LAUNCH_CHECK();
    if (imma8_ok(c, Q)) {
        const size_t t8 = (size_t)2 * c.n * imma8_mtiles(O) * nks * 32;
        k_imma_bank8<<<(unsigned)std::min<size_t>((t8 + 255) / 256, 148 * 32), 256, 0, s>>>(
            ib + imma_bank5_words(c, level, O, Q), masks, O, Q, L, (int)c.logn, nks);
        UH_LAUNCH_CHECK();
    }
}

void hoisted_mac_bank_wide(const Ctx &c, uint64_t *acc, const uint64_t *X, const uint64_t *D, const uint64_t *masks,
                           const uint64_t *kbank, const int32_t *shifts, int B, int I, int T, int O, int level,
                           cudaStream_t s);


void hoisted_mac_imma(const Ctx &c, uint64_t *acc, const uint64_t *X, const uint64_t *D, const uint64_t *masks,
                      const uint32_t *ib, const uint64_t *kbank, const int32_t *shifts, int B, int I, int T, int O,
                      int level, cudaStream_t s) {
    if (!hoisted_imma_supported(c, level, O, I * T))
        throw std::invalid_argument("IMMA hoisted kernel: needs N = 2^15, 40-bit q_1..q_level, 5 <= O <= 48, <= 256 terms");
    const double lim = 4294967295.0;
    const int L = level + 1;
    if ((double)I * B * 2 * L * c.n > lim || (double)I * B * L * (L + 1) * c.n > lim ||
        (double)O * B * 2 * (L + 1) * c.n > lim)
        throw std::invalid_argument("IMMA hoisted kernel operand exceeds 2^32 elements: split the batch");
    // q_0 and P on the IMAD key-bank kernel (the tcgen05 kernel on these limbs alone measured 16.2-16.5 ms
    // vs 13.6 ms at the LeNet conv2 shape: its 2-4-coefficient tiles cannot coalesce phase A's loads),
    // in groups of <= 12 outputs (its register tile); the 40-bit limbs take every output in one pass,
    // so their key switching (phase A) is done once for all of them
    // -- or on the 8-byte IMMA kernel (every output in one pass)
    if (imma8_ok(c, I * T)) {
        const uint32_t *ib8 = ib + imma_bank5_words(c, level, O, I * T);
#define UH_IMMA8_CASE(LL)                                                    \
    case LL:                                                                 \
        launch_imma8<LL>(c, acc, X, D, ib8, kbank, shifts, B, I, T, O, s);   \
        break;
        switch (L) {
            UH_IMMA8_CASE(3)
            UH_IMMA8_CASE(4)
            UH_IMMA8_CASE(5)
            UH_IMMA8_CASE(6)
            UH_IMMA8_CASE(7)
            UH_IMMA8_CASE(8)
            UH_IMMA8_CASE(9)
            UH_IMMA8_CASE(10)
            default: throw std::invalid_argument("IMMA hoisted kernel: 3 <= level + 1 <= 10");
        }
#undef UH_IMMA8_CASE
    } else {
        const size_t LPN = (size_t)(L + 1) * c.n;
        for (int o0 = 0; o0 < O; o0 += 12)
            hoisted_mac_bank_wide(c, acc + (size_t)o0 * B * 2 * LPN, X, D, masks + (size_t)o0 * I * T * LPN, kbank,
                                  shifts, B, I, T, std::min(12, O - o0), level, s);
    }
#define UH_IMMA_CASE(LL)                                                    \
    case LL:                                                                \
        launch_imma<LL, 5>(c, acc, X, D, ib, kbank, shifts, B, I, T, O, s); \
        break;
    switch (L) {
        UH_IMMA_CASE(3)
        UH_IMMA_CASE(4)
        UH_IMMA_CASE(5)
        UH_IMMA_CASE(6)
        UH_IMMA_CASE(7)
        UH_IMMA_CASE(8)
        UH_IMMA_CASE(9)
        UH_IMMA_CASE(10)
        default: throw std::invalid_argument("IMMA hoisted kernel: 3 <= level + 1 <= 10");
    }
#undef UH_IMMA_CASE
}


// Tensor-core phase A (k_hoisted_imma_ta): the IMMA shapes with 5 (level + 1) <= 32 digit bytes and
// at most 128 terms (the phase-B planes of 32 columns at 3 CTAs / SM).
bool hoisted_imma_ta_supported(const Ctx &c, int level, int O, int Q) {
    return hoisted_imma_supported(c, level, O, Q) && 5 * (level + 1) <= 32 && Q <= 128 && imma8_ok(c, Q);
}
size_t imma_ta_bank_bytes(const Ctx &c, int level, int T) { return (size_t)level * c.n * T * 32 * 16; }
void imma_ta_bank(const Ctx &c, uint8_t *kt, const uint64_t *kbank, const int32_t *shifts, int T, int level,
                  cudaStream_t s) {
    const size_t total = (size_t)level * c.n * T * 32;
    k_ta_bank<<<(unsigned)std::min<size_t>((total + 255) / 256, 148 * 32), 256, 0, s>>>(
        reinterpret_cast<uint4 *>(kt), kbank, shifts, T, level + 1, (int)c.logn, c.d_mods);
    UH_LAUNCH_CHECK();
}

void hoisted_mac_imma_ta(const Ctx &c, uint64_t *acc, const uint64_t *X, const uint64_t *D, const uint32_t *ib,
                         const uint8_t *kt, const uint64_t *kbank, const int32_t *shifts, int B, int I, int T, int O,
                         int level, cudaStream_t s) {
    if (!hoisted_imma_ta_supported(c, level, O, I * T))
        throw std::invalid_argument("tensor-core phase A: needs the IMMA shape with level + 1 <= 6 and <= 128 terms");
    const int L = level + 1, R = I * B;
    const double lim = 4294967295.0;
    if ((double)I * B * 2 * L * c.n > lim || (double)I * B * L * (L + 1) * c.n > lim ||
        (double)O * B * 2 * (L + 1) * c.n > lim)
        throw std::invalid_argument("IMMA hoisted kernel operand exceeds 2^32 elements: split the batch");
    // q_0 and P: the 8-byte IMMA kernel (IMAD phase A on the 60-bit limbs)
    const uint32_t *ib8 = ib + imma_bank5_words(c, level, O, I * T);
    // 32-bit per-unit offsets inside the kernel: digit bytes of one limb, the key fragments of one
    // limb's coefficient tile, the P c0 rows
    if ((double)c.n * R * 32 > lim || (double)c.n * T * 32 > lim || (double)R * level * c.n > lim)
        throw std::invalid_argument("tensor-core phase A operand exceeds 2^32 elements: split the batch");
    Scratch dp((size_t)level * c.n * R * 32, s), pc((size_t)R * level * c.n * 8, s);
    {
        dim3 grid((unsigned)(c.n / 32), (unsigned)((R + 31) / 32), (unsigned)level);
#define UH_TA_PACK(LL)                                                                                         \
    case LL:                                                                                                   \
        k_ta_pack<LL><<<grid, 256, 0, s>>>(dp.as<unsigned char>(), pc.as<uint64_t>(), D, X, R, (int)c.logn,    \
                                           c.sp(), c.d_mods);                                                  \
        break;
        switch (L) {
            UH_TA_PACK(3)
            UH_TA_PACK(4)
            UH_TA_PACK(5)
            UH_TA_PACK(6)
            default: throw std::invalid_argument("tensor-core phase A: 3 <= level + 1 <= 6");
        }
#undef UH_TA_PACK
        UH_LAUNCH_CHECK();
    }
#define UH_TA_CASE(LL)                                                                                      \
    case LL:                                                                                                \
        launch_imma8<LL>(c, acc, X, D, ib8, kbank, shifts, B, I, T, O, s);                                  \
        launch_imma_ta<LL>(c, acc, X, dp.as<unsigned char>(), pc.as<uint64_t>(), ib,                        \
                           reinterpret_cast<const uint4 *>(kt), shifts, B, I, T, O, s);                     \
        break;
    switch (L) {
        UH_TA_CASE(3)
        UH_TA_CASE(4)
        UH_TA_CASE(5)
        UH_TA_CASE(6)
        default: throw std::invalid_argument("tensor-core phase A: 3 <= level + 1 <= 6");
    }
#undef UH_TA_CASE
}

}  // namespace uh
