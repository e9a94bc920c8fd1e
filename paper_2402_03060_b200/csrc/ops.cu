// RNS-CKKS operations on batches of ciphertexts (sm_100a): elementwise
// arithmetic, rescale / ModDown (divide by the top prime), ModUp, the
// key-switching inner product with the Galois automorphism folded into its
// reads (slot order makes X -> X^(5^r) a cyclic shift of each half), rotation,
// ct x pt and ct x ct (+ relinearisation) followed by rescale.
//
// Definitions follow oracle/ckks_oracle.c exactly (centred lifts, digit
// decomposition one digit per q_j, special prime P), so results are bit-exact
// against the oracle on every residue.
#include "ops.cuh"
#include "ntt_fast.cuh"

namespace uh {

namespace {

constexpr int kTB = 256;

inline int grid_for(size_t total, int tb = kTB) {
    size_t g = (total + tb - 1) / tb;
    const size_t cap = 148u * 64u;  // grid-stride beyond ~64 CTAs / SM
    return (int)(g < cap ? (g ? g : 1) : cap);
}

__device__ __forceinline__ uint32_t rot_index(uint32_t n, uint32_t half, uint32_t r) {
    uint32_t h = n >= half ? half : 0;
    uint32_t j = n - h + r;
    j = j >= half ? j - half : j;
    return h + j;
}

__global__ void k_elementwise(int op, uint64_t *out, const uint64_t *a, const uint64_t *b, int n_polys, int b_polys,
                              int b_div, int nl, int nq, int sp, int out_ps, int a_ps, int b_ps, int logn,
                              const Mod *__restrict__ mods) {
    size_t total = ((size_t)n_polys * nl) << logn;
    size_t nmask = ((size_t)1 << logn) - 1;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        size_t n = idx & nmask, t = idx >> logn;
        int k = (int)(t % nl), p = (int)(t / nl);
        const Mod &m = mods[limb_mod(k, nq, 0, sp)];
        size_t oi = (((size_t)p * out_ps + k) << logn) | n;
        uint64_t av = a[(((size_t)p * a_ps + k) << logn) | n];
        uint64_t bv = 0;
        if (op != OP_NEG && op != OP_COPY) bv = b[(((size_t)((p / b_div) % b_polys) * b_ps + k) << logn) | n];
        uint64_t r;
        switch (op) {
            case OP_ADD: r = addmod(av, bv, m.q); break;
            case OP_SUB: r = submod(av, bv, m.q); break;
            case OP_MUL: r = mulmod(av, bv, m); break;
            case OP_MAC: r = addmod(out[oi], mulmod(av, bv, m), m.q); break;
            case OP_NEG: r = av ? m.q - av : 0; break;
            default: r = av; break;
        }
        out[oi] = r;
    }
}

// dst[p][n] = src[p][limb]  (gather one limb of every poly into a compact list)
// D[p][j][j] = in[p][j]: the diagonal ModUp limb is the (evaluation-form) input limb itself
__global__ void k_modup_diag(uint64_t *D, const uint64_t *in, int n_polys, int L, int in_ps, int logn) {
    size_t total = ((size_t)n_polys * L) << logn;
    size_t nmask = ((size_t)1 << logn) - 1;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        size_t n = idx & nmask, t = idx >> logn;
        size_t j = t % L, p = t / L;
        D[((((p * L + j) * (L + 1)) + j) << logn) | n] = in[((p * in_ps + j) << logn) | n];
    }
}

// diagonal of the ModUp output: D[p][j][j] = in[p][j]; 16-byte vector copies, grid (N / 512, L, polys)
__global__ void __launch_bounds__(256) k_modup_diag2(uint64_t *__restrict__ D, const uint64_t *__restrict__ in, int L,
                                                     int in_ps, int logn) {
    const size_t p = blockIdx.z, j = blockIdx.y;
    const size_t n = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 2;
    const ulonglong2 v = *reinterpret_cast<const ulonglong2 *>(in + ((p * in_ps + j) << logn) + n);
    *reinterpret_cast<ulonglong2 *>(D + (((p * L + j) * (L + 1) + j) << logn) + n) = v;
}

__global__ void k_gather_limb(uint64_t *dst, const uint64_t *src, int n_polys, int limb, int src_ps, int logn) {
    size_t total = (size_t)n_polys << logn;
    size_t nmask = ((size_t)1 << logn) - 1;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        size_t n = idx & nmask, p = idx >> logn;
        dst[idx] = src[((p * src_ps + limb) << logn) | n];
    }
}

// T[p][k][n] = centred(top[p][n], q_top) mod q_k,  k < nl
__global__ void k_expand_centred(uint64_t *T, const uint64_t *top, int n_polys, int nl, int top_mod, int logn,
                                 const Mod *__restrict__ mods) {
    size_t total = ((size_t)n_polys * nl) << logn;
    size_t nmask = ((size_t)1 << logn) - 1;
    uint64_t qt = mods[top_mod].q;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        size_t n = idx & nmask, t = idx >> logn;
        int k = (int)(t % nl);
        size_t p = t / nl;
        T[idx] = centred_to(top[(p << logn) | n], qt, mods[k]);
    }
}

// out[p][k] = (in[p][k] - T[p][k]) * q_top^-1 mod q_k
__global__ void k_divide_finish(uint64_t *out, const uint64_t *in, const uint64_t *T, int n_polys, int nl,
                                int top_mod, int count, int out_ps, int in_ps, int logn, const Mod *__restrict__ mods,
                                const uint64_t *__restrict__ inv, const uint64_t *__restrict__ invs) {
    size_t total = ((size_t)n_polys * nl) << logn;
    size_t nmask = ((size_t)1 << logn) - 1;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        size_t n = idx & nmask, t = idx >> logn;
        int k = (int)(t % nl);
        size_t p = t / nl;
        uint64_t q = mods[k].q;
        uint64_t w = inv[(size_t)k * count + top_mod], ws = invs[(size_t)k * count + top_mod];
        uint64_t x = in[((p * in_ps + k) << logn) | n];
        out[((p * out_ps + k) << logn) | n] = shoup(submod(x, T[idx], q), w, ws, q);
    }
}

// D[p][j][k][n] = centred(C[p][j][n], q_j) mod p_k, k over (q_0..q_{L-1}, P)
__global__ void k_modup_expand(uint64_t *D, const uint64_t *C, int n_polys, int L, int sp, int logn,
                               const Mod *__restrict__ mods) {
    size_t total = ((size_t)n_polys * L * (L + 1)) << logn;
    size_t nmask = ((size_t)1 << logn) - 1;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        size_t n = idx & nmask, t = idx >> logn;
        int k = (int)(t % (L + 1));
        size_t pj = t / (L + 1);  // p * L + j
        int j = (int)(pj % L);
        uint64_t x = C[(pj << logn) | n];
        D[idx] = (k == j) ? x : centred_to(x, mods[j].q, mods[limb_mod(k, L, 0, sp)]);
    }
}

__global__ void k_key_inner(uint64_t *u, const uint64_t *D, const uint64_t *key, int key_limbs, int n_polys, int L,
                            int sp, uint32_t r, int logn, const Mod *__restrict__ mods) {
    const int LP = L + 1;
    size_t total = ((size_t)n_polys * LP) << logn;
    size_t nmask = ((size_t)1 << logn) - 1;
    uint32_t half = 1u << (logn - 1);
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        size_t n = idx & nmask, t = idx >> logn;
        int k = (int)(t % LP);
        size_t p = t / LP;
        const Mod &m = mods[limb_mod(k, L, 0, sp)];
        int kk = k < L ? k : key_limbs - 1;
        size_t src = rot_index((uint32_t)n, half, r);
        Acc a0, a1;
        a0.zero();
        a1.zero();
        for (int j = 0; j < L; j++) {
            uint64_t d = D[((((p * L + j) * LP) + k) << logn) | src];
            a0.mac(d, key[((((size_t)j * 2 + 0) * key_limbs + kk) << logn) | n]);
            a1.mac(d, key[((((size_t)j * 2 + 1) * key_limbs + kk) << logn) | n]);
        }
        u[((((p * 2 + 0) * LP) + k) << logn) | n] = a0.reduce(m);
        u[((((p * 2 + 1) * LP) + k) << logn) | n] = a1.reduce(m);
    }
}

// Key-switch inner product, one thread per coefficient: grid (N / 256, L + 1 limbs, polys);
// digit and key loads issued in groups of 4 (independent loads in flight, no division in
// the index math).  With `t` (relinearisation) the epilogue also adds (P mod q_k) * t[p][c][k]
// for the q-limbs, i.e. u + P * (d0, d1) in the QP basis, saving a pass over u.
__global__ void __launch_bounds__(256) k_key_inner2(uint64_t *__restrict__ u, const uint64_t *__restrict__ D,
                                                     const uint64_t *__restrict__ key, int key_limbs, int L, int sp,
                                                     uint32_t r, int logn, const Mod *__restrict__ mods,
                                                     const uint64_t *__restrict__ t,
                                                     const ulonglong2 *__restrict__ pmod) {
    const int LP = L + 1;
    const uint32_t n = blockIdx.x * blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    const size_t p = blockIdx.z;
    const uint32_t half = 1u << (logn - 1);
    const Mod m = mods[limb_mod(k, L, 0, sp)];
    const int kk = k < L ? k : key_limbs - 1;
    const uint32_t src = rot_index(n, half, r);
    const uint64_t *Dp = D + (((p * L) * LP + k) << logn) + src;
    const size_t dstr = (size_t)LP << logn, kstr = (size_t)key_limbs << logn;
    const uint64_t *K0 = key + ((size_t)kk << logn) + n;
    // relinearisation addend, loaded up front (its latency overlaps the digit loads)
    uint64_t t0 = 0, t1 = 0;
    const bool addp = t && k < L;
    if (addp) {
        t0 = __ldg(t + (((p * 2 + 0) * L + k) << logn) + n);
        t1 = __ldg(t + (((p * 2 + 1) * L + k) << logn) + n);
    }
    Acc a0, a1;
    a0.zero();
    a1.zero();
#ifndef UH_KI_G
#define UH_KI_G 4
#endif
    constexpr int G = UH_KI_G;
    for (int j0 = 0; j0 < L; j0 += G) {
        uint64_t d[G], x[G], y[G];
#pragma unroll
        for (int g = 0; g < G; g++) {
            const int j = j0 + g;
            const bool ok = j < L;
            d[g] = ok ? __ldg(Dp + j * dstr) : 0;
            x[g] = ok ? __ldg(K0 + (2 * j) * kstr) : 0;
            y[g] = ok ? __ldg(K0 + (2 * j + 1) * kstr) : 0;
        }
#pragma unroll
        for (int g = 0; g < G; g++) {
            a0.mac(d[g], x[g]);
            a1.mac(d[g], y[g]);
        }
    }
    uint64_t v0 = a0.reduce(m), v1 = a1.reduce(m);
    if (addp) {
        const ulonglong2 pk = pmod[k];
        v0 = addmod(v0, shoup(t0, pk.x, pk.y, m.q), m.q);
        v1 = addmod(v1, shoup(t1, pk.x, pk.y, m.q), m.q);
    }
    u[(((p * 2 + 0) * LP + k) << logn) + n] = v0;
    u[(((p * 2 + 1) * LP + k) << logn) + n] = v1;
}

// Same product with compile-time L and N (N = 2^15): no predicated digit groups, all 3L
// operand loads in flight at once, and the narrow-operand accumulator (AccN) for limbs
// with q < 2^41.  Grid (N / 256, L + 1, polys) as k_key_inner2.
template <int L, int LOGN>
__global__ void __launch_bounds__(256) k_key_inner_l(uint64_t *__restrict__ u, const uint64_t *__restrict__ D,
                                                     const uint64_t *__restrict__ key, int key_limbs, int sp,
                                                     uint32_t r, const Mod *__restrict__ mods,
                                                     const uint64_t *__restrict__ t,
                                                     const ulonglong2 *__restrict__ pmod,
                                                     const uint64_t *__restrict__ diag) {
    // diag != nullptr: the ModUp left its diagonal limbs D[p][k][k] unwritten; they are the input
    // polys' own limbs diag[p][k] (the relinearisation's d2 in evaluation form)
    constexpr int LP = L + 1;
    constexpr uint32_t half = 1u << (LOGN - 1);
    const uint32_t n = blockIdx.x * blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    const uint32_t p = blockIdx.z;
    const Mod m = mods[k < L ? k : sp];
    const int kk = k < L ? k : key_limbs - 1;
    const uint32_t src = rot_index(n, half, r);
    const uint64_t *Dp = D + (((size_t)p * L * LP + k) << LOGN) + src;
    const size_t kstr = (size_t)key_limbs << LOGN;
    const uint64_t *K0 = key + ((size_t)kk << LOGN) + n;
    const bool addp = t && k < L;
    uint64_t t0 = 0, t1 = 0;
    if (addp) {
        t0 = __ldg(t + (((size_t)(p * 2 + 0) * L + k) << LOGN) + n);
        t1 = __ldg(t + (((size_t)(p * 2 + 1) * L + k) << LOGN) + n);
    }
    uint64_t d[L], x[L], y[L];
#pragma unroll
    for (int j = 0; j < L; j++) {
        d[j] = diag && j == k ? __ldg(diag + (((size_t)p * L + k) << LOGN) + src) : __ldg(Dp + ((size_t)j * LP << LOGN));
        x[j] = __ldg(K0 + (2 * j) * kstr);
        y[j] = __ldg(K0 + (2 * j + 1) * kstr);
    }
    auto dot = [&](auto tag, uint64_t &v0, uint64_t &v1) {
        decltype(tag) a0, a1;
        a0.zero();
        a1.zero();
#pragma unroll
        for (int j = 0; j < L; j++) {
            a0.mac(d[j], x[j]);
            a1.mac(d[j], y[j]);
        }
        v0 = a0.reduce(m);
        v1 = a1.reduce(m);
    };
    uint64_t v0, v1;
    if ((m.q >> 41) == 0)
        dot(AccN{}, v0, v1);
    else
        dot(Acc{}, v0, v1);
    if (addp) {
        const ulonglong2 pk = pmod[k];
        v0 = addmod(v0, shoup(t0, pk.x, pk.y, m.q), m.q);
        v1 = addmod(v1, shoup(t1, pk.x, pk.y, m.q), m.q);
    }
    u[(((size_t)(p * 2 + 0) * LP + k) << LOGN) + n] = v0;
    u[(((size_t)(p * 2 + 1) * LP + k) << LOGN) + n] = v1;
}

// out c0 = rot(in c0) + ks0, c1 = ks1
__global__ void k_rot_finish(uint64_t *out, const uint64_t *in, const uint64_t *ks, int B, int L, int out_ls,
                             int in_ls, uint32_t r, int logn, const Mod *__restrict__ mods) {
    size_t total = ((size_t)B * 2 * L) << logn;
    size_t nmask = ((size_t)1 << logn) - 1;
    uint32_t half = 1u << (logn - 1);
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        size_t n = idx & nmask, t = idx >> logn;
        int k = (int)(t % L);
        size_t bc = t / L;  // b * 2 + comp
        int comp = (int)(bc & 1);
        size_t b = bc >> 1;
        uint64_t v = ks[idx];
        if (comp == 0) {
            uint64_t x = in[(((b * 2) * in_ls + k) << logn) | rot_index((uint32_t)n, half, r)];
            v = addmod(v, x, mods[k].q);
        }
        out[((bc * out_ls + k) << logn) | n] = v;
    }
}

// tensor product: T[b][0] = a0 b0, T[b][1] = a0 b1 + a1 b0, D2[b] = a1 b1
__global__ void k_tensor(uint64_t *T, uint64_t *D2, const uint64_t *a, const uint64_t *b, int B, int L, int a_ls,
                         int b_ls, int logn, const Mod *__restrict__ mods) {
    size_t total = ((size_t)B * L) << logn;
    size_t nmask = ((size_t)1 << logn) - 1;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        size_t n = idx & nmask, t = idx >> logn;
        int k = (int)(t % L);
        size_t bb = t / L;
        const Mod &m = mods[k];
        uint64_t a0 = a[(((bb * 2) * a_ls + k) << logn) | n], a1 = a[(((bb * 2 + 1) * a_ls + k) << logn) | n];
        uint64_t b0 = b[(((bb * 2) * b_ls + k) << logn) | n], b1 = b[(((bb * 2 + 1) * b_ls + k) << logn) | n];
        Acc d1;
        d1.zero();
        d1.mac(a0, b1);
        d1.mac(a1, b0);
        T[(((bb * 2) * L + k) << logn) | n] = mulmod(a0, b0, m);
        T[(((bb * 2 + 1) * L + k) << logn) | n] = d1.reduce(m);
        D2[idx] = mulmod(a1, b1, m);
    }
}

// k_tensor on a 3-D grid (N / 256, L, B): one thread per coefficient, limb-uniform modulus, no division
__global__ void __launch_bounds__(256) k_tensor2(uint64_t *__restrict__ T, uint64_t *__restrict__ D2,
                                                 const uint64_t *__restrict__ a, const uint64_t *__restrict__ b, int L,
                                                 int a_ls, int b_ls, int logn, const Mod *__restrict__ mods) {
    const size_t n = (size_t)blockIdx.x * blockDim.x + threadIdx.x, bb = blockIdx.z;
    const int k = blockIdx.y;
    const Mod m = mods[k];
    const uint64_t a0 = __ldg(a + (((bb * 2) * a_ls + k) << logn) + n);
    const uint64_t a1 = __ldg(a + (((bb * 2 + 1) * a_ls + k) << logn) + n);
    const uint64_t b0 = __ldg(b + (((bb * 2) * b_ls + k) << logn) + n);
    const uint64_t b1 = __ldg(b + (((bb * 2 + 1) * b_ls + k) << logn) + n);
    Acc d1;
    d1.zero();
    d1.mac(a0, b1);
    d1.mac(a1, b0);
    T[(((bb * 2) * L + k) << logn) + n] = mulmod(a0, b0, m);
    T[(((bb * 2 + 1) * L + k) << logn) + n] = d1.reduce(m);
    D2[((bb * L + k) << logn) + n] = mulmod(a1, b1, m);
}

// the square (a == b): (a0^2, 2 a0 a1, a1^2), two coefficients per thread (16-byte loads / stores);
// grid (N / 512, L, B)
__global__ void __launch_bounds__(256) k_tensor2_sq(uint64_t *__restrict__ T, uint64_t *__restrict__ D2,
                                                    const uint64_t *__restrict__ a, int L, int a_ls, int logn,
                                                    const Mod *__restrict__ mods) {
    const size_t n = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 2, bb = blockIdx.z;
    const int k = blockIdx.y;
    const Mod m = mods[k];
    const ulonglong2 a0 = __ldg(reinterpret_cast<const ulonglong2 *>(a + (((bb * 2) * a_ls + k) << logn) + n));
    const ulonglong2 a1 = __ldg(reinterpret_cast<const ulonglong2 *>(a + (((bb * 2 + 1) * a_ls + k) << logn) + n));
    auto twice = [&](uint64_t x, uint64_t y) {  // 2 x y mod q, canonical
        const uint64_t v = mulmod(x, y, m);
        return csub(v + v, m.q);
    };
    *reinterpret_cast<ulonglong2 *>(T + (((bb * 2) * L + k) << logn) + n) =
        make_ulonglong2(mulmod(a0.x, a0.x, m), mulmod(a0.y, a0.y, m));
    *reinterpret_cast<ulonglong2 *>(T + (((bb * 2 + 1) * L + k) << logn) + n) =
        make_ulonglong2(twice(a0.x, a1.x), twice(a0.y, a1.y));
    *reinterpret_cast<ulonglong2 *>(D2 + ((bb * L + k) << logn) + n) =
        make_ulonglong2(mulmod(a1.x, a1.x, m), mulmod(a1.y, a1.y, m));
}

// u[p][k] += (P mod q_k) * t[p][k] for the q-limbs k < L of QP-basis polys (u has L + 1 limbs, t has L)
__global__ void k_add_pscaled(uint64_t *u, const uint64_t *t, int n_polys, int L, int sp, int logn,
                              const Mod *__restrict__ mods, const ulonglong2 *__restrict__ pmod) {
    size_t total = ((size_t)n_polys * L) << logn;
    size_t nmask = ((size_t)1 << logn) - 1;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        size_t n = idx & nmask, r = idx >> logn;
        int k = (int)(r % L);
        size_t p = r / L;
        const uint64_t q = mods[k].q;
        const ulonglong2 pk = pmod[k];
        uint64_t &x = u[((p * (L + 1) + k) << logn) | n];
        x = addmod(x, shoup(t[idx], pk.x, pk.y, q), q);
    }
}
}  // namespace

void elementwise(const Ctx &c, int op, uint64_t *out, const uint64_t *a, const uint64_t *b, int n_polys, int b_polys,
                 int nl, int nq, int out_ps, int a_ps, int b_ps, cudaStream_t s) {
    size_t total = ((size_t)n_polys * nl) << c.logn;
    if (!total) return;
    int b_div = 1;
    if (b_polys < 0) {  // broadcast b over the two components of each ciphertext
        b_polys = -b_polys;
        b_div = 2;
    }
    k_elementwise<<<grid_for(total), kTB, 0, s>>>(op, out, a, b, n_polys, b_polys > 0 ? b_polys : 1, b_div, nl, nq,
                                                 c.sp(), out_ps, a_ps, b_ps, (int)c.logn, c.d_mods);
    UH_LAUNCH_CHECK();
}

void elementwise_grouped(const Ctx &c, int op, uint64_t *out, const uint64_t *a, const uint64_t *b, int n_polys,
                         int b_polys, int group, int nl, int nq, int out_ps, int a_ps, int b_ps, cudaStream_t s) {
    size_t total = ((size_t)n_polys * nl) << c.logn;
    if (!total) return;
    k_elementwise<<<grid_for(total), kTB, 0, s>>>(op, out, a, b, n_polys, b_polys, group, nl, nq, c.sp(), out_ps, a_ps,
                                                 b_ps, (int)c.logn, c.d_mods);
    UH_LAUNCH_CHECK();
}

void divide_top(const Ctx &c, uint64_t *out, const uint64_t *in, int n_polys, int nl, int top_mod, int out_ps,
                int in_ps, cudaStream_t s) {
    if (!n_polys) return;
    size_t N = c.n;
    bool is_sp = top_mod == c.sp();
    if (ntt_fast_supported(c)) {
        Scratch top((size_t)n_polys * N * 8, s);
        NttJob Ji;  // top limb -> coefficients
        Ji.nl = 1;
        Ji.nq = is_sp ? 0 : 1;
        Ji.base = is_sp ? 0 : top_mod;
        Ji.sp = c.sp();
        Ji.src = in + (size_t)nl * N;
        Ji.src_ps = in_ps;
        Ji.dst = top.as<uint64_t>();
        Ji.dst_ps = 1;
        ntt_fast_inverse(c, Ji, n_polys, s);
        if (nl == 0) return;
        NttJob Jf;  // centred lift into every lower limb, NTT, (in - t) * q_top^-1 epilogue
        Jf.mode = NTT_DIVIDE;
        Jf.nl = nl;
        Jf.nq = nl;
        Jf.sp = c.sp();
        Jf.src = top.as<uint64_t>();
        Jf.dst = out;
        Jf.dst_ps = out_ps;
        Jf.in = in;
        Jf.in_ps = in_ps;
        Jf.top_mod = top_mod;
        Jf.count = (int)c.count;
        Jf.inv = c.d_inv;
        Jf.invs = c.d_invs;
        ntt_fast_forward(c, Jf, n_polys * nl, s);
        return;
    }
    Scratch top((size_t)n_polys * N * 8, s), T((size_t)n_polys * nl * N * 8, s);
    k_gather_limb<<<grid_for((size_t)n_polys * N), kTB, 0, s>>>(top.as<uint64_t>(), in, n_polys, nl, in_ps,
                                                                 (int)c.logn);
    UH_LAUNCH_CHECK();
    ntt_inverse(c, top.as<uint64_t>(), n_polys, 1, is_sp ? 0 : 1, is_sp ? 0 : top_mod, 1, s);
    if (nl == 0) return;
    k_expand_centred<<<grid_for((size_t)n_polys * nl * N), kTB, 0, s>>>(T.as<uint64_t>(), top.as<uint64_t>(), n_polys,
                                                                        nl, top_mod, (int)c.logn, c.d_mods);
    UH_LAUNCH_CHECK();
    ntt_forward(c, T.as<uint64_t>(), n_polys, nl, nl, 0, nl, s);
    k_divide_finish<<<grid_for((size_t)n_polys * nl * N), kTB, 0, s>>>(out, in, T.as<uint64_t>(), n_polys, nl, top_mod,
                                                                       (int)c.count, out_ps, in_ps, (int)c.logn,
                                                                       c.d_mods, c.d_inv, c.d_invs);
    UH_LAUNCH_CHECK();
}

namespace {
// Per coefficient of the (x mod q_t, x mod P) rows: y = (a - b) P^-1 mod q_t, so x = b + P y,
// and whether the centred representative of x (in (-q_t P / 2, q_t P / 2]) is negative;
// stored in place of a as y | neg << 63.  Done once here instead of once per target limb
// in the DIVIDE2 forward NTT.
__global__ void k_crt2_pre(uint64_t *top, int n_polys, int logn, Mod mt, uint64_t P, ulonglong2 pinv) {
    const size_t total = (size_t)n_polys << logn, nmask = ((size_t)1 << logn) - 1;
    const uint64_t qt = mt.q, h = (qt - 1) >> 1, ph = (P - 1) / 2;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        const size_t p = idx >> logn, n = idx & nmask;
        uint64_t *a = top + ((2 * p) << logn) + n;
        const uint64_t b = a[(size_t)1 << logn];
        const uint64_t bt = b < qt ? b : csub(barrett_lite(b, mt), qt);
        const uint64_t y = shoup(submod(*a, bt, qt), pinv.x, pinv.y, qt);
        const bool neg = y > h || (y == h && b > ph);
        *a = y | ((uint64_t)neg << 63);
    }
}
}  // namespace

void divide_top2(const Ctx &c, uint64_t *out, const uint64_t *in, int n_polys, int level, int out_ps, int in_ps,
                 cudaStream_t s, const uint64_t *bias, int bias_group) {
    if (!n_polys) return;
    const size_t N = c.n;
    if (bias && (!ntt_fast_supported(c) || level == 0 || bias_group < 1))
        throw std::invalid_argument("fused bias needs the fast NTT (2^13 <= N <= 2^15) and level >= 1");
    if (!ntt_fast_supported(c)) {  // small N: the two divisions in sequence
        Scratch t((size_t)n_polys * (level + 1) * N * 8, s);
        divide_top(c, t.as<uint64_t>(), in, n_polys, level + 1, c.sp(), level + 1, in_ps, s);
        divide_top(c, out, t.as<uint64_t>(), n_polys, level, level, out_ps, level + 1, s);
        return;
    }
    Scratch top((size_t)n_polys * 2 * N * 8, s);
    NttJob Ji;  // limbs q_level and P -> coefficients, [p][2][N]
    Ji.nl = 2;
    Ji.nq = 1;
    Ji.base = level;
    Ji.sp = c.sp();
    Ji.src = in + (size_t)level * N;
    Ji.src_ps = in_ps;
    Ji.dst = top.as<uint64_t>();
    Ji.dst_ps = 2;
    ntt_fast_inverse(c, Ji, n_polys * 2, s);
    if (level == 0) return;
    {
        const int cnt = (int)c.count, sp = c.sp();
        const Mod mt = c.h_mods[level];
        const ulonglong2 pinv = make_ulonglong2(c.h_inv[(size_t)level * cnt + sp], c.h_invs[(size_t)level * cnt + sp]);
        k_crt2_pre<<<grid_for((size_t)n_polys * N), kTB, 0, s>>>(top.as<uint64_t>(), n_polys, (int)c.logn, mt,
                                                                 c.h_q[sp], pinv);
        UH_LAUNCH_CHECK();
    }
    NttJob Jf;
    Jf.mode = NTT_DIVIDE2;
    Jf.nl = level;
    Jf.nq = level;
    Jf.sp = c.sp();
    Jf.src = top.as<uint64_t>();
    Jf.dst = out;
    Jf.dst_ps = out_ps;
    Jf.in = in;
    Jf.in_ps = in_ps;
    Jf.top_mod = level;
    Jf.count = (int)c.count;
    Jf.inv = c.d_inv;
    Jf.invs = c.d_invs;
    Jf.inv2 = c.d_inv2;
    Jf.inv2s = c.d_inv2s;
    Jf.bias = bias;
    Jf.bias_group = bias ? bias_group : 1;
    Jf.pmod = c.d_pmod;
    ntt_fast_forward(c, Jf, n_polys * level, s);
}

#ifndef UH_MODUP_DIAG_IN_NTT
#define UH_MODUP_DIAG_IN_NTT 1
#endif
void modup(const Ctx &c, uint64_t *D, const uint64_t *in, int n_polys, int level, int in_ps, cudaStream_t s,
           bool diag) {
    int L = level + 1;
    size_t N = c.n;
    Scratch C((size_t)n_polys * L * N * 8, s);
    if (ntt_fast_supported(c)) {
        NttJob Ji;  // every digit to coefficients (strided in -> compact C)
        Ji.nl = L;
        Ji.nq = L;
        Ji.sp = c.sp();
        Ji.src = in;
        Ji.src_ps = in_ps;
        Ji.dst = C.as<uint64_t>();
        Ji.dst_ps = L;
        const bool diag_in_ntt = diag && UH_MODUP_DIAG_IN_NTT;
        if (diag_in_ntt) Ji.diag = D;  // D[p][j][j] = in[p][j], written by the inverse NTT's first pass
        ntt_fast_inverse(c, Ji, n_polys * L, s);
        if (diag_in_ntt) diag = false;
        NttJob Jf;  // centred lift of digit j into every QP limb, fused into the forward NTT's loads
        Jf.mode = NTT_MODUP;
        Jf.L = L;
        Jf.sp = c.sp();
        Jf.src = C.as<uint64_t>();
        Jf.dst = D;
        ntt_fast_forward(c, Jf, n_polys * L * L, s);
        if (!diag) return;  // the consumer reads the diagonal limbs from `in` itself
        if (N >= 512 && n_polys <= 65535) {
            k_modup_diag2<<<dim3((unsigned)(N / 512), L, n_polys), 256, 0, s>>>(D, in, L, in_ps, (int)c.logn);
        } else {
            k_modup_diag<<<grid_for((size_t)n_polys * L * N), kTB, 0, s>>>(D, in, n_polys, L, in_ps, (int)c.logn);
        }
        UH_LAUNCH_CHECK();
        return;
    }
    elementwise(c, OP_COPY, C.as<uint64_t>(), in, nullptr, n_polys, 1, L, L, L, in_ps, 0, s);
    ntt_inverse(c, C.as<uint64_t>(), n_polys, L, L, 0, L, s);
    size_t total = (size_t)n_polys * L * (L + 1) * N;
    k_modup_expand<<<grid_for(total), kTB, 0, s>>>(D, C.as<uint64_t>(), n_polys, L, c.sp(), (int)c.logn, c.d_mods);
    UH_LAUNCH_CHECK();
    ntt_forward(c, D, n_polys * L, L + 1, L, 0, L + 1, s);
}

#ifndef UH_KI_FIXED
#define UH_KI_FIXED 1
#endif
static bool key_inner_fixed(const Ctx &c, int L) { return UH_KI_FIXED && c.logn == 15 && L <= 10; }
// diag: the ModUp input polys when the ModUp skipped its diagonal copy (only with key_inner_fixed(c, L))
static void key_inner_impl(const Ctx &c, uint64_t *u, const uint64_t *D, const uint64_t *key, int key_limbs,
                           int n_polys, int level, int64_t r, const uint64_t *t, cudaStream_t s,
                           const uint64_t *diag = nullptr) {
    int L = level + 1;
    int64_t half = c.n / 2;
    uint32_t rr = (uint32_t)(((r % half) + half) % half);
    if (key_inner_fixed(c, L)) {
        for (int p0 = 0; p0 < n_polys; p0 += 65535) {
            const int np = std::min(65535, n_polys - p0);
            dim3 g((unsigned)(c.n / 256), L + 1, np);
            uint64_t *up = u + (size_t)p0 * 2 * (L + 1) * c.n;
            const uint64_t *Dp = D + (size_t)p0 * L * (L + 1) * c.n;
            const uint64_t *dg = diag ? diag + (size_t)p0 * L * c.n : nullptr;
            const uint64_t *tp = t ? t + (size_t)p0 * 2 * L * c.n : nullptr;
#define UH_KI_CASE(LL)                                                                                          \
    case LL:                                                                                                    \
        k_key_inner_l<LL, 15><<<g, 256, 0, s>>>(up, Dp, key, key_limbs, c.sp(), rr, c.d_mods, tp, c.d_pmod, dg); \
        break;
            switch (L) {
                UH_KI_CASE(1) UH_KI_CASE(2) UH_KI_CASE(3) UH_KI_CASE(4) UH_KI_CASE(5)
                UH_KI_CASE(6) UH_KI_CASE(7) UH_KI_CASE(8) UH_KI_CASE(9) UH_KI_CASE(10)
            }
#undef UH_KI_CASE
            UH_LAUNCH_CHECK();
        }
        return;
    }
    if (diag) throw std::logic_error("diagonal-free ModUp needs the fixed-L key inner product");
    if (c.n >= 256) {
        for (int p0 = 0; p0 < n_polys; p0 += 65535) {
            const int np = std::min(65535, n_polys - p0);
            dim3 g((unsigned)(c.n / 256), L + 1, np);
            k_key_inner2<<<g, 256, 0, s>>>(u + (size_t)p0 * 2 * (L + 1) * c.n, D + (size_t)p0 * L * (L + 1) * c.n,
                                           key, key_limbs, L, c.sp(), rr, (int)c.logn, c.d_mods,
                                           t ? t + (size_t)p0 * 2 * L * c.n : nullptr, c.d_pmod);
            UH_LAUNCH_CHECK();
        }
        return;
    }
    size_t total = (size_t)n_polys * (L + 1) * c.n;
    k_key_inner<<<grid_for(total), kTB, 0, s>>>(u, D, key, key_limbs, n_polys, L, c.sp(), rr, (int)c.logn, c.d_mods);
    UH_LAUNCH_CHECK();
    if (t) {
        k_add_pscaled<<<grid_for((size_t)n_polys * 2 * L * c.n), kTB, 0, s>>>(u, t, 2 * n_polys, L, c.sp(),
                                                                              (int)c.logn, c.d_mods, c.d_pmod);
        UH_LAUNCH_CHECK();
    }
}

void key_inner(const Ctx &c, uint64_t *u, const uint64_t *D, const uint64_t *key, int key_limbs, int n_polys,
               int level, int64_t r, cudaStream_t s) {
    key_inner_impl(c, u, D, key, key_limbs, n_polys, level, r, nullptr, s);
}

void keyswitch(const Ctx &c, uint64_t *out, const uint64_t *d, int n_polys, int level, int d_ps, const uint64_t *key,
               int key_limbs, int64_t r, cudaStream_t s) {
    int L = level + 1;
    size_t N = c.n;
    Scratch D((size_t)n_polys * L * (L + 1) * N * 8, s), u((size_t)n_polys * 2 * (L + 1) * N * 8, s);
    modup(c, D.as<uint64_t>(), d, n_polys, level, d_ps, s);
    key_inner(c, u.as<uint64_t>(), D.as<uint64_t>(), key, key_limbs, n_polys, level, r, s);
    divide_top(c, out, u.as<uint64_t>(), n_polys * 2, L, c.sp(), L, L + 1, s);
}

void ct_rotate(const Ctx &c, uint64_t *out, const uint64_t *in, int B, int level, int out_ls, int in_ls,
               const uint64_t *key, int key_limbs, int64_t r, cudaStream_t s) {
    int L = level + 1;
    int64_t half = c.n / 2;
    uint32_t rr = (uint32_t)(((r % half) + half) % half);
    if (rr == 0) {
        elementwise(c, OP_COPY, out, in, nullptr, 2 * B, 1, L, L, out_ls, in_ls, 0, s);
        return;
    }
    size_t N = c.n;
    Scratch ks((size_t)B * 2 * L * N * 8, s);
    keyswitch(c, ks.as<uint64_t>(), in + (size_t)in_ls * N, B, level, 2 * in_ls, key, key_limbs, rr, s);
    k_rot_finish<<<grid_for((size_t)B * 2 * L * N), kTB, 0, s>>>(out, in, ks.as<uint64_t>(), B, L, out_ls, in_ls, rr,
                                                                 (int)c.logn, c.d_mods);
    UH_LAUNCH_CHECK();
}

// ct_rotate with the ModUp digits of in's c1 supplied (D [B][L][L+1][N], from uh_modup): the key
// product with the Galois shift folded, ModDown, and rot(c0) + ks0.  Bit-identical to ct_rotate
// (the centred digit lift commutes with the automorphism), at the cost of a key product and a
// ModDown instead of a full key switch -- the op-level backend reuses D across the rotations of
// one ciphertext (automatic hoisting of the reference's per-tap rotate calls).
void ct_rotate_hoisted(const Ctx &c, uint64_t *out, const uint64_t *in, const uint64_t *D, int B, int level,
                       int out_ls, int in_ls, const uint64_t *key, int key_limbs, int64_t r, cudaStream_t s) {
    int L = level + 1;
    int64_t half = c.n / 2;
    uint32_t rr = (uint32_t)(((r % half) + half) % half);
    if (rr == 0) {
        elementwise(c, OP_COPY, out, in, nullptr, 2 * B, 1, L, L, out_ls, in_ls, 0, s);
        return;
    }
    size_t N = c.n;
    Scratch u((size_t)B * 2 * (L + 1) * N * 8, s), ks((size_t)B * 2 * L * N * 8, s);
    key_inner(c, u.as<uint64_t>(), D, key, key_limbs, B, level, rr, s);
    divide_top(c, ks.as<uint64_t>(), u.as<uint64_t>(), B * 2, L, c.sp(), L, L + 1, s);
    k_rot_finish<<<grid_for((size_t)B * 2 * L * N), kTB, 0, s>>>(out, in, ks.as<uint64_t>(), B, L, out_ls, in_ls, rr,
                                                                 (int)c.logn, c.d_mods);
    UH_LAUNCH_CHECK();
}

void ct_rescale(const Ctx &c, uint64_t *out, const uint64_t *in, int B, int level, int out_ls, int in_ls,
                cudaStream_t s) {
    divide_top(c, out, in, 2 * B, level, level, out_ls, in_ls, s);
}

void ct_mul_relin_rescale(const Ctx &c, uint64_t *out, const uint64_t *a, const uint64_t *b, int B, int level,
                          int out_ls, int a_ls, int b_ls, const uint64_t *rk, int rk_limbs, cudaStream_t s) {
    int L = level + 1;
    size_t N = c.n;
    Scratch T((size_t)B * 2 * L * N * 8, s), D2((size_t)B * L * N * 8, s), KS((size_t)B * 2 * L * N * 8, s);
    if (N >= 256 && B <= 65535)
        k_tensor2<<<dim3((unsigned)(N / 256), L, B), 256, 0, s>>>(T.as<uint64_t>(), D2.as<uint64_t>(), a, b, L, a_ls,
                                                                  b_ls, (int)c.logn, c.d_mods);
    else
        k_tensor<<<grid_for((size_t)B * L * N), kTB, 0, s>>>(T.as<uint64_t>(), D2.as<uint64_t>(), a, b, B, L, a_ls,
                                                             b_ls, (int)c.logn, c.d_mods);
    UH_LAUNCH_CHECK();
    keyswitch(c, KS.as<uint64_t>(), D2.as<uint64_t>(), B, level, L, rk, rk_limbs, 0, s);
    elementwise(c, OP_ADD, T.as<uint64_t>(), T.as<uint64_t>(), KS.as<uint64_t>(), 2 * B, 2 * B, L, L, L, L, L, s);
    divide_top(c, out, T.as<uint64_t>(), 2 * B, level, level, out_ls, L, s);
}


void ct_mul_relin_rescale_fused(const Ctx &c, uint64_t *out, const uint64_t *a, const uint64_t *b, int B, int level,
                                int out_ls, int a_ls, int b_ls, const uint64_t *rk, int rk_limbs, cudaStream_t s) {
    int L = level + 1;
    size_t N = c.n;
    Scratch T((size_t)B * 2 * L * N * 8, s), D2((size_t)B * L * N * 8, s);
    if (a == b && a_ls == b_ls && N >= 512 && B <= 65535)  // the square activation
        k_tensor2_sq<<<dim3((unsigned)(N / 512), L, B), 256, 0, s>>>(T.as<uint64_t>(), D2.as<uint64_t>(), a, L, a_ls,
                                                                     (int)c.logn, c.d_mods);
    else if (N >= 256 && B <= 65535)
        k_tensor2<<<dim3((unsigned)(N / 256), L, B), 256, 0, s>>>(T.as<uint64_t>(), D2.as<uint64_t>(), a, b, L, a_ls,
                                                                  b_ls, (int)c.logn, c.d_mods);
    else
        k_tensor<<<grid_for((size_t)B * L * N), kTB, 0, s>>>(T.as<uint64_t>(), D2.as<uint64_t>(), a, b, B, L, a_ls,
                                                             b_ls, (int)c.logn, c.d_mods);
    UH_LAUNCH_CHECK();
    Scratch D((size_t)B * L * (L + 1) * N * 8, s), u((size_t)B * 2 * (L + 1) * N * 8, s);
    // u = <D, rk> + P * (d0, d1): the relinearised product times P, in the QP basis (the ModUp's
    // diagonal limbs are d2's own limbs: read in place instead of copied)
    const bool skip = ntt_fast_supported(c) && key_inner_fixed(c, L);
    modup(c, D.as<uint64_t>(), D2.as<uint64_t>(), B, level, L, s, !skip);
    key_inner_impl(c, u.as<uint64_t>(), D.as<uint64_t>(), rk, rk_limbs, B, level, 0, T.as<uint64_t>(), s,
                   skip ? D2.as<uint64_t>() : nullptr);
    divide_top2(c, out, u.as<uint64_t>(), 2 * B, level, out_ls, L + 1, s);
}

void ct_mul_plain_rescale(const Ctx &c, uint64_t *out, const uint64_t *ct, const uint64_t *pt, int B, int level,
                          int out_ls, int ct_ls, int pt_ls, int pt_batched, cudaStream_t s) {
    int L = level + 1;
    size_t N = c.n;
    Scratch T((size_t)B * 2 * L * N * 8, s);
    elementwise(c, OP_MUL, T.as<uint64_t>(), ct, pt, 2 * B, pt_batched ? -B : 1, L, L, L, ct_ls, pt_ls, s);
    divide_top(c, out, T.as<uint64_t>(), 2 * B, level, level, out_ls, L, s);
}

}  // namespace uh
