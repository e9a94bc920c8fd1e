// Job description of the register-tiled two-pass NTT (ntt_fast.cu).
#pragma once
#include "engine.cuh"

namespace uh {

enum NttMode : int { NTT_PLAIN = 0, NTT_MODUP = 1, NTT_DIVIDE = 2, NTT_DIVIDE2 = 3 };

// One launch transforms `limbs` limbs; limb f is decoded per mode:
//  PLAIN : p = f / nl, k = f % nl; modulus limb_mod(k, nq, base, sp);
//          src row  src + (p * src_ps + k) * N,  dst row dst + (p * dst_ps + k) * N.
//  MODUP : (p, j, k') = f over [n][L][L], k = k' + (k' >= j) skips the diagonal;
//          modulus limb_mod(k, L, 0, sp); forward input centred(src[p * L + j], q_j);
//          dst row dst + ((p * L + j) * (L + 1) + k) * N.
//  DIVIDE: p = f / nl, k = f % nl, modulus k; forward input centred(src[p], q_top);
//          epilogue dst[p][k] = (in[p][k] - y) * q_top^-1 (rows at p * dst_ps / p * in_ps).
//  DIVIDE2 (fused ModDown + rescale, division by q_top * P): src rows [p][2] hold, per
//          coefficient, y | neg << 63 and x mod P, where x = (x mod P) + P y is the CRT
//          lift of (x mod q_top, x mod P) and neg marks its centred representative as
//          negative (prepared by ops.cu k_crt2_pre); forward input = that centred value
//          reduced into q_k; epilogue dst[p][k] = (in[p][k] - y) * (q_top P)^-1.
struct NttJob {
    int mode = NTT_PLAIN;
    int f0 = 0;  // first limb of this launch (chunked launches)
    int nl = 1, nq = 1, base = 0, sp = 0;
    const uint64_t *src = nullptr;
    int src_ps = 1;
    uint64_t *dst = nullptr;
    int dst_ps = 1;
    int L = 0;
    const uint64_t *in = nullptr;
    int in_ps = 1;
    int top_mod = 0, count = 0;
    const uint64_t *inv = nullptr, *invs = nullptr;
    const uint64_t *inv2 = nullptr, *inv2s = nullptr;  // DIVIDE2: (q_top * P)^-1 mod q_k (Shoup pairs)
    const ulonglong2 *pmod = nullptr;  // DIVIDE2: (P mod q_i, Shoup companion) per modulus
    // DIVIDE2: optional plaintext rows added to the even polynomials (c0) in the epilogue -- the conv
    // bias: bias[p / bias_group][nl][N], one row set per bias_group polynomials
    const uint64_t *bias = nullptr;
    int bias_group = 1;
    // inverse, PLAIN: optional copy of every input limb (p, k) to diag[((p * nl + k) * (nl + 1) + k)][N] --
    // the diagonal of a ModUp output, written while the limb streams through the first pass
    uint64_t *diag = nullptr;
};

bool ntt_fast_supported(const Ctx &c);
void ntt_fast_forward(const Ctx &c, const NttJob &J, int limbs, cudaStream_t s);
void ntt_fast_inverse(const Ctx &c, const NttJob &J, int limbs, cudaStream_t s);

}  // namespace uh
