// Secret key, key-switching keys, encryption, decryption and the canonical
// embedding (encode / decode).  Randomness comes from the counter-based RNG
// in common.cuh, whose definition is shared bit-for-bit with the CPU oracle,
// so seeded keys, masks and noise are identical on both sides.
#include "ops.cuh"

namespace uh {

namespace {

constexpr int kTB = 256;
inline int grid_for(size_t total) {
    size_t g = (total + kTB - 1) / kTB;
    const size_t cap = 148u * 64u;
    return (int)(g < cap ? (g ? g : 1) : cap);
}

__device__ __forceinline__ uint64_t sample_uniform(uint64_t st, int mod_idx, size_t n, int logn, const Mod &m) {
    uint64_t ctr = (((uint64_t)mod_idx << logn) + n) * 2;
    return reduce128(rng_draw(st, ctr), rng_draw(st, ctr + 1), m);
}
__device__ __forceinline__ int64_t sample_cbd(uint64_t st, size_t n) {
    uint64_t h = rng_draw(st, n);
    return (int64_t)__popcll(h & 0x1FFFFFULL) - (int64_t)__popcll((h >> 21) & 0x1FFFFFULL);
}
__device__ __forceinline__ uint64_t signed_to(int64_t v, const Mod &m) {
    if (v >= 0) return (uint64_t)v < m.q ? (uint64_t)v : csub(barrett_lite((uint64_t)v, m), m.q);
    uint64_t a = (uint64_t)(-(v + 1)) + 1;  // |v|, safe for INT64_MIN
    uint64_t r = a < m.q ? a : csub(barrett_lite(a, m), m.q);
    return r ? m.q - r : 0;
}

// secret: ternary coefficients written into every modulus (count limbs)
__global__ void k_secret(uint64_t *s, uint64_t st, int count, int logn, const Mod *__restrict__ mods) {
    size_t total = (size_t)count << logn;
    size_t nmask = ((size_t)1 << logn) - 1;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        size_t n = idx & nmask;
        int m = (int)(idx >> logn);
        int64_t v = (int64_t)(rng_draw(st, n) % 3) - 1;
        s[idx] = signed_to(v, mods[m]);
    }
}

// key material for digits j < L over limbs (q_0..q_{L-1}, P): a into key[j][1], noise into E[j]
__global__ void k_ksk_sample(uint64_t *key, uint64_t *E, uint64_t seed, uint64_t key_id, int L, int sp, int logn,
                             const Mod *__restrict__ mods) {
    const int LP = L + 1;
    size_t total = ((size_t)L * LP) << logn;
    size_t nmask = ((size_t)1 << logn) - 1;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        size_t n = idx & nmask, t = idx >> logn;
        int k = (int)(t % LP);
        int j = (int)(t / LP);
        int mk = limb_mod(k, L, 0, sp);
        const Mod &m = mods[mk];
        uint64_t sa = rng_stream(seed, TAG_KSK_A, key_id, (uint64_t)j);
        uint64_t se = rng_stream(seed, TAG_KSK_E, key_id, (uint64_t)j);
        key[((((size_t)j * 2 + 1) * LP + k) << logn) | n] = sample_uniform(sa, mk, n, logn, m);
        E[idx] = signed_to(sample_cbd(se, n), m);
    }
}

// b_j = E_j - a_j * s + [k == j] (P mod q_j) * s_from
__global__ void k_ksk_finish(uint64_t *key, const uint64_t *E, const uint64_t *s, const uint64_t *s_from, int L,
                             int sp, int logn, const Mod *__restrict__ mods) {
    const int LP = L + 1;
    size_t total = ((size_t)L * LP) << logn;
    size_t nmask = ((size_t)1 << logn) - 1;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        size_t n = idx & nmask, t = idx >> logn;
        int k = (int)(t % LP);
        int j = (int)(t / LP);
        int mk = limb_mod(k, L, 0, sp);
        const Mod &m = mods[mk];
        uint64_t a = key[((((size_t)j * 2 + 1) * LP + k) << logn) | n];
        uint64_t sv = s[((size_t)mk << logn) | n];
        uint64_t b = submod(E[idx], mulmod(a, sv, m), m.q);
        if (k == j) {
            uint64_t pm = mods[sp].q;
            pm = pm < m.q ? pm : csub(barrett_lite(pm, m), m.q);
            b = addmod(b, mulmod(pm, s_from[((size_t)mk << logn) | n], m), m.q);
        }
        key[((((size_t)j * 2 + 0) * LP + k) << logn) | n] = b;
    }
}

__global__ void k_rotate_rows(uint64_t *out, const uint64_t *in, int rows, uint32_t r, int logn) {
    size_t total = (size_t)rows << logn;
    size_t nmask = ((size_t)1 << logn) - 1;
    uint32_t half = 1u << (logn - 1);
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        uint32_t n = (uint32_t)(idx & nmask);
        uint32_t h = n >= half ? half : 0;
        uint32_t j = n - h + r;
        j = j >= half ? j - half : j;
        out[idx] = in[(idx & ~nmask) | (h + j)];
    }
}

__global__ void k_square_rows(uint64_t *out, const uint64_t *in, int rows, int logn, const Mod *__restrict__ mods) {
    size_t total = (size_t)rows << logn;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        const Mod &m = mods[idx >> logn];
        out[idx] = mulmod(in[idx], in[idx], m);
    }
}

// encryption noise e (coefficient form, per limb) and uniform a (evaluation form) into out c1
__global__ void k_enc_sample(uint64_t *E, uint64_t *out, int B, int L, int out_ls, uint64_t seed, uint64_t id0,
                             int logn, const Mod *__restrict__ mods) {
    size_t total = ((size_t)B * L) << logn;
    size_t nmask = ((size_t)1 << logn) - 1;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        size_t n = idx & nmask, t = idx >> logn;
        int k = (int)(t % L);
        size_t b = t / L;
        const Mod &m = mods[k];
        uint64_t sa = rng_stream(seed, TAG_ENC_A, id0 + b, 0);
        uint64_t se = rng_stream(seed, TAG_ENC_E, id0 + b, 0);
        out[(((b * 2 + 1) * out_ls + k) << logn) | n] = sample_uniform(sa, k, n, logn, m);
        E[idx] = signed_to(sample_cbd(se, n), m);
    }
}

// c0 = e - a * s + m
__global__ void k_enc_finish(uint64_t *out, const uint64_t *E, const uint64_t *pt, const uint64_t *s, int B, int L,
                             int out_ls, int pt_ls, int pt_batched, int logn, const Mod *__restrict__ mods) {
    size_t total = ((size_t)B * L) << logn;
    size_t nmask = ((size_t)1 << logn) - 1;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        size_t n = idx & nmask, t = idx >> logn;
        int k = (int)(t % L);
        size_t b = t / L;
        const Mod &m = mods[k];
        uint64_t a = out[(((b * 2 + 1) * out_ls + k) << logn) | n];
        uint64_t mv = pt[(((pt_batched ? b : 0) * pt_ls + k) << logn) | n];
        uint64_t v = submod(E[idx], mulmod(a, s[((size_t)k << logn) | n], m), m.q);
        out[(((b * 2) * out_ls + k) << logn) | n] = addmod(v, mv, m.q);
    }
}

// M[b] = c0[b][0] + c1[b][0] * s[0]
__global__ void k_dec_limb0(uint64_t *M, const uint64_t *ct, const uint64_t *s, int B, int ct_ls, int logn,
                            const Mod *__restrict__ mods) {
    size_t total = (size_t)B << logn;
    size_t nmask = ((size_t)1 << logn) - 1;
    const Mod &m = mods[0];
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        size_t n = idx & nmask, b = idx >> logn;
        uint64_t c0 = ct[(((b * 2) * ct_ls) << logn) | n], c1 = ct[(((b * 2 + 1) * ct_ls) << logn) | n];
        M[idx] = addmod(c0, mulmod(c1, s[n], m), m.q);
    }
}

__global__ void k_centred_double(double *out, const uint64_t *M, size_t total, const Mod *__restrict__ mods) {
    uint64_t q = mods[0].q;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        uint64_t x = M[idx];
        out[idx] = x > (q - 1) / 2 ? -(double)(q - x) : (double)x;
    }
}

__global__ void k_from_signed(uint64_t *out, const int64_t *coef, int n_polys, int nl, int nq, int sp, int out_ps,
                              int logn, const Mod *__restrict__ mods) {
    size_t total = ((size_t)n_polys * nl) << logn;
    size_t nmask = ((size_t)1 << logn) - 1;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        size_t n = idx & nmask, t = idx >> logn;
        int k = (int)(t % nl);
        size_t p = t / nl;
        out[((p * out_ps + k) << logn) | n] = signed_to(coef[(p << logn) | n], mods[limb_mod(k, nq, 0, sp)]);
    }
}

}  // namespace

void secret_gen(const Ctx &c, uint64_t *s_eval, uint64_t seed, cudaStream_t st) {
    uint64_t stream = rng_stream(seed, TAG_SECRET, 0, 0);
    k_secret<<<grid_for((size_t)c.count * c.n), kTB, 0, st>>>(s_eval, stream, (int)c.count, (int)c.logn, c.d_mods);
    UH_LAUNCH_CHECK();
    ntt_forward(c, s_eval, 1, (int)c.count, (int)c.count - 1, 0, (int)c.count, st);
}

void switch_keygen(const Ctx &c, uint64_t *key, const uint64_t *s_eval, const uint64_t *s_from_eval, uint64_t seed,
                   uint64_t key_id, int level, cudaStream_t st) {
    int L = level + 1;
    size_t N = c.n;
    Scratch E((size_t)L * (L + 1) * N * 8, st);
    k_ksk_sample<<<grid_for((size_t)L * (L + 1) * N), kTB, 0, st>>>(key, E.as<uint64_t>(), seed, key_id, L, c.sp(),
                                                                    (int)c.logn, c.d_mods);
    UH_LAUNCH_CHECK();
    ntt_forward(c, E.as<uint64_t>(), L, L + 1, L, 0, L + 1, st);
    k_ksk_finish<<<grid_for((size_t)L * (L + 1) * N), kTB, 0, st>>>(key, E.as<uint64_t>(), s_eval, s_from_eval, L,
                                                                    c.sp(), (int)c.logn, c.d_mods);
    UH_LAUNCH_CHECK();
}

void galois_keygen(const Ctx &c, uint64_t *key, const uint64_t *s_eval, uint64_t seed, int64_t r, int level,
                   cudaStream_t st) {
    int64_t half = c.n / 2;
    uint64_t rr = (uint64_t)(((r % half) + half) % half);
    uint64_t g = 1, two_n = 2ull * c.n;
    for (uint64_t i = 0; i < rr; i++) g = g * 5 % two_n;
    Scratch S((size_t)c.count * c.n * 8, st);
    k_rotate_rows<<<grid_for((size_t)c.count * c.n), kTB, 0, st>>>(S.as<uint64_t>(), s_eval, (int)c.count,
                                                                   (uint32_t)rr, (int)c.logn);
    UH_LAUNCH_CHECK();
    switch_keygen(c, key, s_eval, S.as<uint64_t>(), seed, g, level, st);
}

void relin_keygen(const Ctx &c, uint64_t *key, const uint64_t *s_eval, uint64_t seed, int level, cudaStream_t st) {
    Scratch S((size_t)c.count * c.n * 8, st);
    k_square_rows<<<grid_for((size_t)c.count * c.n), kTB, 0, st>>>(S.as<uint64_t>(), s_eval, (int)c.count,
                                                                   (int)c.logn, c.d_mods);
    UH_LAUNCH_CHECK();
    switch_keygen(c, key, s_eval, S.as<uint64_t>(), seed, 2, level, st);
}

void encrypt(const Ctx &c, uint64_t *out, const uint64_t *pt, const uint64_t *s_eval, int B, int level, int out_ls,
             int pt_ls, uint64_t seed, uint64_t ct_id0, cudaStream_t st) {
    int L = level + 1;
    size_t N = c.n;
    Scratch E((size_t)B * L * N * 8, st);
    k_enc_sample<<<grid_for((size_t)B * L * N), kTB, 0, st>>>(E.as<uint64_t>(), out, B, L, out_ls, seed, ct_id0,
                                                              (int)c.logn, c.d_mods);
    UH_LAUNCH_CHECK();
    ntt_forward(c, E.as<uint64_t>(), B, L, L, 0, L, st);
    int pt_batched = pt_ls < 0 ? 0 : 1;
    if (pt_ls < 0) pt_ls = -pt_ls;
    k_enc_finish<<<grid_for((size_t)B * L * N), kTB, 0, st>>>(out, E.as<uint64_t>(), pt, s_eval, B, L, out_ls, pt_ls,
                                                              pt_batched, (int)c.logn, c.d_mods);
    UH_LAUNCH_CHECK();
}

void decrypt_coeffs(const Ctx &c, double *out, const uint64_t *ct, const uint64_t *s_eval, int B, int ct_ls,
                    cudaStream_t st) {
    size_t N = c.n;
    Scratch M((size_t)B * N * 8, st);
    k_dec_limb0<<<grid_for((size_t)B * N), kTB, 0, st>>>(M.as<uint64_t>(), ct, s_eval, B, ct_ls, (int)c.logn,
                                                         c.d_mods);
    UH_LAUNCH_CHECK();
    ntt_inverse(c, M.as<uint64_t>(), B, 1, 1, 0, 1, st);
    k_centred_double<<<grid_for((size_t)B * N), kTB, 0, st>>>(out, M.as<uint64_t>(), (size_t)B * N, c.d_mods);
    UH_LAUNCH_CHECK();
}

void from_signed(const Ctx &c, uint64_t *out, const int64_t *coef, int n_polys, int nq, int special, int out_ps,
                 cudaStream_t s) {
    int nl = nq + (special ? 1 : 0);
    k_from_signed<<<grid_for((size_t)n_polys * nl * c.n), kTB, 0, s>>>(out, coef, n_polys, nl, nq, c.sp(), out_ps,
                                                                      (int)c.logn, c.d_mods);
    UH_LAUNCH_CHECK();
    ntt_forward(c, out, n_polys, nl, nq, 0, out_ps, s);
}

}  // namespace uh
