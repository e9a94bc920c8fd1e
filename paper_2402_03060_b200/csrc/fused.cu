// Hoisted, fused layer kernels (sm_100a).
//
// Convolution (reference layers.py:134-197) and average pooling
// (layers.py:200-227) are sums of masked rotations of the same few input
// ciphertexts.  Instead of key-switching every rotation separately
// (ModUp + inner product + ModDown per rotation, then a rescale per masked
// product), the engine
//   1. ModUps each input's c1 ONCE (hoisting: the digit decomposition uses a
//      centred lift, so it commutes with the Galois automorphism and the
//      rotated decomposition is just a shifted read of the unrotated one),
//   2. for every tap forms the rotated, key-switched ciphertext in the QP
//      basis on the fly -- P*rot(c0) + <rot(D), K_t> and <rot(D), K_t> --
//      and immediately multiply-accumulates it with every output channel's
//      plaintext weight mask (still in the QP basis, lazily in 128 bits),
//   3. leaves one ModDown (and one rescale) per output channel to the caller.
// Nothing per-rotation ever touches HBM; the inputs (D, c0), keys and masks
// are read once per tile.
#include "ops.cuh"

namespace uh {

namespace {

constexpr int kTB = 256;

inline int grid_for(size_t total) {
    size_t g = (total + kTB - 1) / kTB;
    const size_t cap = 148u * 32u;
    return (int)(g < cap ? (g ? g : 1) : cap);
}

__device__ __forceinline__ uint32_t rot_index(uint32_t n, uint32_t half, uint32_t r) {
    uint32_t h = n >= half ? half : 0;
    uint32_t j = n - h + r;
    j = j >= half ? j - half : j;
    return h + j;
}

__device__ __forceinline__ uint64_t p_mod(const Mod &m, uint64_t P) {
    return P < m.q ? P : csub(barrett_lite(P, m), m.q);
}

// acc[o][b][c][k][n] (QP basis, o in [o0, o0+OC)) =
//   sum_{i,t} M[o][i][t][k][n] * v_{i,t}[b][c][k][n]
// v_{i,t} = key-switched rotation by shifts[t] of input ct (i, b), times P.
template <int OC>
__global__ void __launch_bounds__(kTB) k_conv_mac(uint64_t *__restrict__ acc_out, const uint64_t *__restrict__ X,
                                                 int xls, const uint64_t *__restrict__ D,
                                                 const uint64_t *__restrict__ masks,
                                                 const uint64_t *const *__restrict__ keys, const int32_t *__restrict__ key_limbs,
                                                 const int32_t *__restrict__ shifts, int B, int I, int T, int O,
                                                 int o0, int L, int sp, int fold_every, int logn,
                                                 const Mod *__restrict__ mods) {
    const int LP = L + 1;
    const size_t N = (size_t)1 << logn, nmask = N - 1;
    const uint32_t half = (uint32_t)(N >> 1);
    const size_t total = (size_t)B * LP * N;
    const uint64_t P = mods[sp].q;
    const size_t mstride_o = (size_t)I * T * LP * N;  // distance between consecutive output masks
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        const size_t n = idx & nmask, t = idx >> logn;
        const int k = (int)(t % LP);
        const size_t b = t / LP;
        const Mod m = mods[limb_mod(k, L, 0, sp)];
        const bool qlimb = k < L;
        const uint64_t Pk = qlimb ? p_mod(m, P) : 0;

        Acc acc[OC][2];
#pragma unroll
        for (int o = 0; o < OC; o++) {
            acc[o][0].zero();
            acc[o][1].zero();
        }
        int since_fold = 0;  // products accumulated since the last fold (<= 60 keeps 128 bits safe)
        for (int i = 0; i < I; i++) {
            const uint64_t *c0 = X + (((size_t)(i * B + b) * 2 * xls) << logn);
            const uint64_t *c1 = c0 + ((size_t)xls << logn);
            const uint64_t *Di = D + (((size_t)(i * B + b) * L * LP) << logn);
            for (int tt = 0; tt < T; tt++) {
                const uint32_t r = (uint32_t)shifts[tt];
                uint64_t v0, v1;
                if (r == 0) {
                    v0 = qlimb ? mulmod(Pk, c0[((size_t)k << logn) | n], m) : 0;
                    v1 = qlimb ? mulmod(Pk, c1[((size_t)k << logn) | n], m) : 0;
                } else {
                    const size_t src = rot_index((uint32_t)n, half, r);
                    const uint64_t *key = keys[tt];
                    const int kl = key_limbs[tt], kk = qlimb ? k : kl - 1;
                    Acc a0, a1;
                    a0.zero();
                    a1.zero();
                    for (int j = 0; j < L; j++) {
                        const uint64_t d = Di[(((size_t)j * LP + k) << logn) | src];
                        a0.mac(d, key[((((size_t)j * 2 + 0) * kl + kk) << logn) | n]);
                        a1.mac(d, key[((((size_t)j * 2 + 1) * kl + kk) << logn) | n]);
                    }
                    if (qlimb) a0.mac(Pk, c0[((size_t)k << logn) | src]);
                    v0 = a0.reduce(m);
                    v1 = a1.reduce(m);
                }
                const uint64_t *Mt = masks + ((((size_t)((o0 * I + i) * T + tt) * LP + k)) << logn) + n;
#pragma unroll
                for (int o = 0; o < OC; o++) {
                    if (o0 + o < O) {
                        const uint64_t mv = Mt[o * mstride_o];
                        acc[o][0].mac(mv, v0);
                        acc[o][1].mac(mv, v1);
                    }
                }
                if (++since_fold == fold_every) {  // keep the 128-bit sums clear of overflow on 61-bit primes
                    since_fold = 0;
#pragma unroll
                    for (int o = 0; o < OC; o++)
                        for (int c = 0; c < 2; c++) {
                            uint64_t rr = acc[o][c].reduce(m);
                            acc[o][c].lo = rr;
                            acc[o][c].hi = 0;
                        }
                }
            }
        }
#pragma unroll
        for (int o = 0; o < OC; o++) {
            if (o0 + o < O) {
                uint64_t *dst = acc_out + ((((size_t)((o0 + o) * B + b) * 2) * LP + k) << logn) + n;
                dst[0] = acc[o][0].reduce(m);
                dst[(size_t)LP << logn] = acc[o][1].reduce(m);
            }
        }
    }
}

// Hoisted rotation sum (average pooling): out[ch][b] (QP) = sum_t rot_{shifts[t]}(ct[ch][b]) * P.
__global__ void __launch_bounds__(kTB) k_rot_sum(uint64_t *__restrict__ out, const uint64_t *__restrict__ X, int xls,
                                                const uint64_t *__restrict__ D,
                                                const uint64_t *const *__restrict__ keys, const int32_t *__restrict__ key_limbs,
                                                const int32_t *__restrict__ shifts, int B, int C, int T, int L, int sp,
                                                int logn, const Mod *__restrict__ mods) {
    const int fold_taps = 60 / L > 0 ? 60 / L : 1;  // <= 60 products per 128-bit sum
    const int LP = L + 1;
    const size_t N = (size_t)1 << logn, nmask = N - 1;
    const uint32_t half = (uint32_t)(N >> 1);
    const size_t total = (size_t)C * B * LP * N;
    const uint64_t P = mods[sp].q;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        const size_t n = idx & nmask, t = idx >> logn;
        const int k = (int)(t % LP);
        const size_t cb = t / LP;  // ch * B + b
        const Mod m = mods[limb_mod(k, L, 0, sp)];
        const bool qlimb = k < L;
        const uint64_t Pk = qlimb ? p_mod(m, P) : 0;

        const uint64_t *c0 = X + ((cb * 2 * xls) << logn);
        const uint64_t *c1 = c0 + ((size_t)xls << logn);
        const uint64_t *Di = D + ((cb * L * LP) << logn);
        Acc a0, a1;
        a0.zero();
        a1.zero();
        uint64_t c0sum = 0, c1sum = 0;  // sums of < 2^62 values, folded every few taps
        for (int tt = 0; tt < T; tt++) {
            const uint32_t r = (uint32_t)shifts[tt];
            const size_t src = rot_index((uint32_t)n, half, r);
            if (qlimb) c0sum = addmod(c0sum, c0[((size_t)k << logn) | src], m.q);
            if (r == 0) {
                if (qlimb) c1sum = addmod(c1sum, c1[((size_t)k << logn) | n], m.q);
                continue;
            }
            const uint64_t *key = keys[tt];
            const int kl = key_limbs[tt], kk = qlimb ? k : kl - 1;
            for (int j = 0; j < L; j++) {
                const uint64_t d = Di[(((size_t)j * LP + k) << logn) | src];
                a0.mac(d, key[((((size_t)j * 2 + 0) * kl + kk) << logn) | n]);
                a1.mac(d, key[((((size_t)j * 2 + 1) * kl + kk) << logn) | n]);
            }
            if (tt % fold_taps == fold_taps - 1) {
                uint64_t r0 = a0.reduce(m), r1 = a1.reduce(m);
                a0.lo = r0; a0.hi = 0;
                a1.lo = r1; a1.hi = 0;
            }
        }
        if (qlimb) {
            a0.mac(Pk, c0sum);
            a1.mac(Pk, c1sum);
        }
        uint64_t *dst = out + (((cb * 2) * LP + k) << logn) + n;
        dst[0] = a0.reduce(m);
        dst[(size_t)LP << logn] = a1.reduce(m);
    }
}

}  // namespace

void conv_hoisted_mac(const Ctx &c, uint64_t *acc, const uint64_t *X, int xls, const uint64_t *D,
                      const uint64_t *masks, const uint64_t *const *keys, const int32_t *key_limbs, const int32_t *shifts, int B,
                      int I, int T, int O, int level, cudaStream_t s) {
    int L = level + 1;
    size_t total = (size_t)B * (L + 1) * c.n;
    // 128-bit accumulators hold >= 64 products of (< 2^61) x (< 2^61); fold per input channel group
    int fold_every = 60;  // taps between folds of the mask accumulators
    for (int o0 = 0; o0 < O; o0 += 8) {
        int left = O - o0;
        if (left > 4) {
            k_conv_mac<8><<<grid_for(total), kTB, 0, s>>>(acc, X, xls, D, masks, keys, key_limbs, shifts, B, I, T, O,
                                                          o0, L, c.sp(), fold_every, (int)c.logn, c.d_mods);
        } else if (left > 2) {
            k_conv_mac<4><<<grid_for(total), kTB, 0, s>>>(acc, X, xls, D, masks, keys, key_limbs, shifts, B, I, T, O,
                                                          o0, L, c.sp(), fold_every, (int)c.logn, c.d_mods);
        } else {
            k_conv_mac<2><<<grid_for(total), kTB, 0, s>>>(acc, X, xls, D, masks, keys, key_limbs, shifts, B, I, T, O,
                                                          o0, L, c.sp(), fold_every, (int)c.logn, c.d_mods);
        }
        UH_LAUNCH_CHECK();
    }
}

void rot_sum_hoisted(const Ctx &c, uint64_t *out, const uint64_t *X, int xls, const uint64_t *D,
                     const uint64_t *const *keys, const int32_t *key_limbs, const int32_t *shifts, int B, int C, int T, int level,
                     cudaStream_t s) {
    int L = level + 1;
    size_t total = (size_t)C * B * (L + 1) * c.n;
    k_rot_sum<<<grid_for(total), kTB, 0, s>>>(out, X, xls, D, keys, key_limbs, shifts, B, C, T, L, c.sp(),
                                              (int)c.logn, c.d_mods);
    UH_LAUNCH_CHECK();
}

}  // namespace uh
