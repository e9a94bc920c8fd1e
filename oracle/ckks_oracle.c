/*
 * CPU restatement of the RNS-CKKS arithmetic behind the reference's operator
 * boundary -- TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library, and only as the checker (never as the product).
 *
 * What it restates.  The reference package (pkg/src/slotcnn/he_backend.py) is
 * a slot simulator; the arithmetic the paper actually timed lived in
 * SEAL-Python -> Microsoft SEAL (version unpinned,
 * not vendored: pkg/.gitignore:2).  This file restates SEAL's published
 * RNS-CKKS algorithms in plain C with unsigned __int128 arithmetic:
 *   - negacyclic NTT over each RNS prime (evaluation at the odd powers of a
 *     primitive 2N-th root psi), output in "slot order" (see params.py
 *     slot_tables): the representation every other op works in;
 *   - Galois automorphism X -> X^(5^r)  == reference rotate, he_backend.py:249-253;
 *   - hybrid key switching with one special prime P and one digit per q_j
 *     (ModUp by centred lift, key inner product, ModDown by centred lift);
 *   - rescale by the top prime (centred lift)  == the level-1 of
 *     mul_plain / mul_cipher, he_backend.py:226-247;
 *   - the counter-based RNG (SplitMix64 finaliser) used for secret key,
 *     key-switching keys and encryption randomness, so a seeded GPU run and a
 *     seeded oracle run draw identical keys, masks and noise.
 * Every result is a canonical residue in [0, q): any correct implementation
 * of the same definitions produces identical bits, which is what the parity
 * tests compare.
 *
 * Residue-level parity against the reference itself is UNPINNED (no RNS code
 * exists in /root/reference); this oracle is pinned by known-answer tests
 * (naive O(N^2) evaluation, big-integer CRT rescale/ModDown, decrypt of
 * rotations == np.roll) in tests/test_oracle_kat.py, and at slot level by
 * golden vectors generated from the reference simulator (tests/golden/).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

#define OR_API __attribute__((visibility("default")))

static inline uint64_t mulmod(uint64_t a, uint64_t b, uint64_t q) {
    return (uint64_t)(((u128)a * b) % q);
}
static inline uint64_t addmod(uint64_t a, uint64_t b, uint64_t q) {
    uint64_t s = a + b;
    return s >= q ? s - q : s;
}
static inline uint64_t submod(uint64_t a, uint64_t b, uint64_t q) {
    return a >= b ? a - b : a + q - b;
}
static uint64_t powmod(uint64_t b, uint64_t e, uint64_t q) {
    uint64_t r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = mulmod(r, b, q);
        b = mulmod(b, b, q);
        e >>= 1;
    }
    return r;
}
static uint64_t invmod(uint64_t a, uint64_t q) { return powmod(a, q - 2, q); }
/* x * w mod q via Shoup's precomputed quotient ws = floor(w * 2^64 / q); exact, canonical output */
static inline uint64_t shoupmul(uint64_t x, uint64_t w, uint64_t ws, uint64_t q) {
    uint64_t qh = (uint64_t)(((u128)x * ws) >> 64);
    uint64_t r = x * w - qh * q;
    return r >= q ? r - q : r;
}

/* signed value -> residue mod q */
static inline uint64_t from_signed(int64_t v, uint64_t q) {
    if (v >= 0) return (uint64_t)v % q;
    uint64_t m = (uint64_t)(-(v + 1)) % q; /* -(v+1) >= 0, avoids INT64_MIN overflow */
    return q - 1 - m;
}
/* centred lift of x in [0,p): value in (-p/2, p/2), then reduced mod q */
static inline uint64_t centred_to(uint64_t x, uint64_t p, uint64_t q) {
    if (x > (p - 1) / 2) return submod(0, (p - x) % q, q);
    return x % q;
}

/* -- RNG (counter based; identical definition in csrc/rng.cuh) ------------- */
OR_API uint64_t or_mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
OR_API uint64_t or_stream(uint64_t seed, uint64_t tag, uint64_t a, uint64_t b) {
    return or_mix64(or_mix64(or_mix64(or_mix64(seed) ^ tag) ^ a) ^ b);
}
static inline uint64_t draw(uint64_t stream, uint64_t i) { return or_mix64(stream ^ or_mix64(i)); }

/* -- context ---------------------------------------------------------------- */
#include "ckks_oracle.h"

static uint32_t brv(uint32_t x, uint32_t bits) {
    uint32_t r = 0;
    for (uint32_t i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

OR_API or_ctx *or_create(uint32_t n, const uint64_t *moduli, const uint64_t *psi, uint32_t count,
                         const int32_t *slot_of_brv) {
    or_ctx *c = (or_ctx *)calloc(1, sizeof(or_ctx));
    c->n = n;
    c->count = count;
    while ((1u << c->logn) < n) c->logn++;
    c->q = (uint64_t *)malloc(sizeof(uint64_t) * count);
    c->psi = (uint64_t *)malloc(sizeof(uint64_t) * count);
    c->n_inv = (uint64_t *)malloc(sizeof(uint64_t) * count);
    c->psi_rev = (uint64_t *)malloc(sizeof(uint64_t) * count * n);
    c->ipsi_rev = (uint64_t *)malloc(sizeof(uint64_t) * count * n);
    c->psi_sh = (uint64_t *)malloc(sizeof(uint64_t) * count * n);
    c->ipsi_sh = (uint64_t *)malloc(sizeof(uint64_t) * count * n);
    c->slot_of_brv = (int32_t *)malloc(sizeof(int32_t) * n);
    memcpy(c->slot_of_brv, slot_of_brv, sizeof(int32_t) * n);
    for (uint32_t m = 0; m < count; m++) {
        uint64_t q = moduli[m];
        c->q[m] = q;
        c->psi[m] = psi[m];
        c->n_inv[m] = invmod(n, q);
        uint64_t ip = invmod(psi[m], q);
        for (uint32_t i = 0; i < n; i++) {
            uint32_t e = brv(i, c->logn);
            c->psi_rev[(size_t)m * n + i] = powmod(psi[m], e, q);
            c->ipsi_rev[(size_t)m * n + i] = powmod(ip, e, q);
            c->psi_sh[(size_t)m * n + i] = (uint64_t)(((u128)c->psi_rev[(size_t)m * n + i] << 64) / q);
            c->ipsi_sh[(size_t)m * n + i] = (uint64_t)(((u128)c->ipsi_rev[(size_t)m * n + i] << 64) / q);
        }
    }
    return c;
}

OR_API void or_destroy(or_ctx *c) {
    if (!c) return;
    free(c->q); free(c->psi); free(c->n_inv); free(c->psi_rev); free(c->ipsi_rev);
    free(c->psi_sh); free(c->ipsi_sh);
    free(c->slot_of_brv); free(c);
}

/* -- NTT --------------------------------------------------------------------- */
/* Coefficients (natural order) -> slot-order evaluations, one limb, modulus m. */
OR_API void or_ntt(const or_ctx *c, uint32_t m, uint64_t *a) {
    const uint32_t n = c->n;
    const uint64_t q = c->q[m];
    const uint64_t *w = c->psi_rev + (size_t)m * n, *ws = c->psi_sh + (size_t)m * n;
    uint64_t *tmp = (uint64_t *)malloc(sizeof(uint64_t) * n);
    memcpy(tmp, a, sizeof(uint64_t) * n);
    for (uint32_t len = 1, t = n / 2; len < n; len <<= 1, t >>= 1) {
        for (uint32_t i = 0; i < len; i++) {
            uint64_t wi = w[len + i], wsi = ws[len + i];
            for (uint32_t j = 2 * i * t; j < 2 * i * t + t; j++) {
                uint64_t u = tmp[j], v = shoupmul(tmp[j + t], wi, wsi, q);
                tmp[j] = addmod(u, v, q);
                tmp[j + t] = submod(u, v, q);
            }
        }
    }
    for (uint32_t k = 0; k < n; k++) a[c->slot_of_brv[k]] = tmp[k];
    free(tmp);
}

/* Slot-order evaluations -> coefficients. */
OR_API void or_intt(const or_ctx *c, uint32_t m, uint64_t *a) {
    const uint32_t n = c->n;
    const uint64_t q = c->q[m];
    const uint64_t *w = c->ipsi_rev + (size_t)m * n, *ws = c->ipsi_sh + (size_t)m * n;
    uint64_t *tmp = (uint64_t *)malloc(sizeof(uint64_t) * n);
    for (uint32_t k = 0; k < n; k++) tmp[k] = a[c->slot_of_brv[k]];
    for (uint32_t len = n / 2, t = 1; len >= 1; len >>= 1, t <<= 1) {
        for (uint32_t i = 0; i < len; i++) {
            uint64_t wi = w[len + i], wsi = ws[len + i];
            for (uint32_t j = 2 * i * t; j < 2 * i * t + t; j++) {
                uint64_t u = tmp[j], v = tmp[j + t];
                tmp[j] = addmod(u, v, q);
                tmp[j + t] = shoupmul(submod(u, v, q), wi, wsi, q);
            }
        }
        if (len == 1) break;
    }
    for (uint32_t k = 0; k < n; k++) a[k] = mulmod(tmp[k], c->n_inv[m], q);
    free(tmp);
}

/* O(N^2) definition of the slot-order NTT, for known-answer tests. */
OR_API void or_ntt_naive(const or_ctx *c, uint32_t m, const uint64_t *a, uint64_t *out) {
    const uint32_t n = c->n, half = n / 2;
    const uint64_t q = c->q[m], two_n = 2 * (uint64_t)n;
    uint64_t e = 1;
    for (uint32_t j = 0; j < (half ? half : 1); j++) {
        for (int side = 0; side < 2; side++) {
            uint64_t ex = side == 0 ? e : two_n - e;
            uint64_t x = powmod(c->psi[m], ex, q), xp = 1, acc = 0;
            for (uint32_t i = 0; i < n; i++) {
                acc = addmod(acc, mulmod(a[i], xp, q), q);
                xp = mulmod(xp, x, q);
            }
            out[side * half + j] = acc;
        }
        e = e * 5 % two_n;
    }
}

/* -- elementwise over RNS polynomials ----------------------------------------
 * A polynomial is [L][n] with limb l reduced modulo moduli[mods[l]]. */
OR_API void or_add(const or_ctx *c, uint64_t *out, const uint64_t *a, const uint64_t *b,
                   const int32_t *mods, uint32_t L) {
    for (uint32_t l = 0; l < L; l++) {
        uint64_t q = c->q[mods[l]];
        for (uint32_t i = 0; i < c->n; i++) {
            size_t k = (size_t)l * c->n + i;
            out[k] = addmod(a[k], b[k], q);
        }
    }
}
OR_API void or_sub(const or_ctx *c, uint64_t *out, const uint64_t *a, const uint64_t *b,
                   const int32_t *mods, uint32_t L) {
    for (uint32_t l = 0; l < L; l++) {
        uint64_t q = c->q[mods[l]];
        for (uint32_t i = 0; i < c->n; i++) {
            size_t k = (size_t)l * c->n + i;
            out[k] = submod(a[k], b[k], q);
        }
    }
}
OR_API void or_mul(const or_ctx *c, uint64_t *out, const uint64_t *a, const uint64_t *b,
                   const int32_t *mods, uint32_t L) {
#pragma omp parallel for schedule(static)
    for (uint32_t l = 0; l < L; l++) {
        uint64_t q = c->q[mods[l]];
        for (uint32_t i = 0; i < c->n; i++) {
            size_t k = (size_t)l * c->n + i;
            out[k] = mulmod(a[k], b[k], q);
        }
    }
}
/* out = out + a*b (fused multiply-add, used by the MAC-heavy layers) */
OR_API void or_mac(const or_ctx *c, uint64_t *out, const uint64_t *a, const uint64_t *b,
                   const int32_t *mods, uint32_t L) {
#pragma omp parallel for schedule(static)
    for (uint32_t l = 0; l < L; l++) {
        uint64_t q = c->q[mods[l]];
        for (uint32_t i = 0; i < c->n; i++) {
            size_t k = (size_t)l * c->n + i;
            out[k] = addmod(out[k], mulmod(a[k], b[k], q), q);
        }
    }
}

/* Galois automorphism X -> X^(5^r) in slot order: cyclic shift of each half. */
OR_API void or_rotate_slots(const or_ctx *c, uint64_t *out, const uint64_t *in, uint32_t L, int64_t r) {
    const uint32_t n = c->n, half = n / 2;
    int64_t rr = half ? ((r % (int64_t)half) + half) % half : 0;
    for (uint32_t l = 0; l < L; l++)
        for (uint32_t side = 0; side < 2; side++)
            for (uint32_t j = 0; j < half; j++)
                out[(size_t)l * n + side * half + j] = in[(size_t)l * n + side * half + (j + rr) % half];
}

/* Coefficient-domain automorphism X -> X^g (g odd), for known-answer tests. */
OR_API void or_automorphism_coeff(const or_ctx *c, uint32_t m, const uint64_t *in, uint64_t *out, uint64_t g) {
    const uint64_t n = c->n, q = c->q[m];
    for (uint64_t i = 0; i < n; i++) {
        uint64_t e = (i * g) % (2 * n);
        if (e < n) out[e] = in[i];
        else out[e - n] = submod(0, in[i], q);
    }
}

/* signed coefficients -> residues of limbs mods[0..L) (no NTT) */
OR_API void or_from_signed(const or_ctx *c, uint64_t *out, const int64_t *coef, const int32_t *mods, uint32_t L) {
    for (uint32_t l = 0; l < L; l++)
        for (uint32_t i = 0; i < c->n; i++) out[(size_t)l * c->n + i] = from_signed(coef[i], c->q[mods[l]]);
}

/* -- rescale / ModUp / ModDown ---------------------------------------------- */
/* Divide by the top prime q_lev with centred rounding.  in: [lev+1][n] slot
 * order, moduli 0..lev; out: [lev][n], moduli 0..lev-1. */
OR_API void or_rescale(const or_ctx *c, uint64_t *out, const uint64_t *in, uint32_t lev) {
    const uint32_t n = c->n;
    const uint64_t ql = c->q[lev];
    uint64_t *top = (uint64_t *)malloc(sizeof(uint64_t) * n);
    memcpy(top, in + (size_t)lev * n, sizeof(uint64_t) * n);
    or_intt(c, lev, top);
#pragma omp parallel for schedule(static)
    for (uint32_t i = 0; i < lev; i++) {
        uint64_t q = c->q[i];
        uint64_t inv = invmod(ql % q, q);
        uint64_t *t = (uint64_t *)malloc(sizeof(uint64_t) * n);
        for (uint32_t k = 0; k < n; k++) t[k] = centred_to(top[k], ql, q);
        or_ntt(c, i, t);
        for (uint32_t k = 0; k < n; k++)
            out[(size_t)i * n + k] = mulmod(submod(in[(size_t)i * n + k], t[k], q), inv, q);
        free(t);
    }
    free(top);
}

/* ModUp of d (level lev, moduli 0..lev) into the QP basis, one digit per q_j.
 * out: [lev+1 digits][lev+2 limbs][n], limb order (q_0..q_lev, P), P being
 * modulus index `sp`. */
OR_API void or_modup(const or_ctx *c, uint64_t *out, const uint64_t *d, uint32_t lev, uint32_t sp) {
    const uint32_t n = c->n, L = lev + 1, LP = lev + 2;
#pragma omp parallel for schedule(dynamic)
    for (uint32_t j = 0; j < L; j++) {
        uint64_t qj = c->q[j];
        uint64_t *coef = (uint64_t *)malloc(sizeof(uint64_t) * n);
        memcpy(coef, d + (size_t)j * n, sizeof(uint64_t) * n);
        or_intt(c, j, coef);
        for (uint32_t k = 0; k < LP; k++) {
            uint64_t *dst = out + ((size_t)j * LP + k) * n;
            if (k == j) { memcpy(dst, d + (size_t)j * n, sizeof(uint64_t) * n); continue; }
            uint32_t mk = k < L ? k : sp;
            for (uint32_t i = 0; i < n; i++) dst[i] = centred_to(coef[i], qj, c->q[mk]);
            or_ntt(c, mk, dst);
        }
        free(coef);
    }
}

/* Key inner product.  D: modup output; key: [digits >= lev+1][2][key_limbs][n]
 * with limbs (q_0..q_{key_limbs-2}, P).  out: [2][lev+2][n] (QP basis). */
OR_API void or_key_inner(const or_ctx *c, uint64_t *out, const uint64_t *D, const uint64_t *key,
                         uint32_t key_limbs, uint32_t lev, uint32_t sp) {
    const uint32_t n = c->n, L = lev + 1, LP = lev + 2;
#pragma omp parallel for schedule(static) collapse(2)
    for (uint32_t comp = 0; comp < 2; comp++) {
        for (uint32_t k = 0; k < LP; k++) {
            uint32_t mk = k < L ? k : sp;
            uint32_t kk = k < L ? k : key_limbs - 1;
            uint64_t q = c->q[mk];
            uint64_t *dst = out + ((size_t)comp * LP + k) * n;
            for (uint32_t i = 0; i < n; i++) {
                u128 acc = 0;
                for (uint32_t j = 0; j < L; j++) {
                    acc += (u128)D[((size_t)j * LP + k) * n + i] *
                           key[(((size_t)j * 2 + comp) * key_limbs + kk) * n + i];  /* < 2^124 per 16 terms */
                    if ((j & 15) == 15) acc %= q;
                }
                dst[i] = (uint64_t)(acc % q);
            }
        }
    }
}

/* ModDown: [lev+2][n] (q_0..q_lev, P) -> [lev+1][n], divide by P with centred rounding. */
OR_API void or_moddown(const or_ctx *c, uint64_t *out, const uint64_t *in, uint32_t lev, uint32_t sp) {
    const uint32_t n = c->n, L = lev + 1;
    const uint64_t P = c->q[sp];
    uint64_t *top = (uint64_t *)malloc(sizeof(uint64_t) * n);
    memcpy(top, in + (size_t)L * n, sizeof(uint64_t) * n);
    or_intt(c, sp, top);
#pragma omp parallel for schedule(static)
    for (uint32_t i = 0; i < L; i++) {
        uint64_t q = c->q[i];
        uint64_t inv = invmod(P % q, q);
        uint64_t *t = (uint64_t *)malloc(sizeof(uint64_t) * n);
        for (uint32_t k = 0; k < n; k++) t[k] = centred_to(top[k], P, q);
        or_ntt(c, i, t);
        for (uint32_t k = 0; k < n; k++)
            out[(size_t)i * n + k] = mulmod(submod(in[(size_t)i * n + k], t[k], q), inv, q);
        free(t);
    }
    free(top);
}

/* Full key switch of d (level lev): out[2][lev+1][n] = ModDown(<ModUp(d), key>). */
OR_API void or_keyswitch(const or_ctx *c, uint64_t *out, const uint64_t *d, const uint64_t *key,
                         uint32_t key_limbs, uint32_t lev, uint32_t sp) {
    const uint32_t n = c->n, L = lev + 1, LP = lev + 2;
    uint64_t *D = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)L * LP * n);
    uint64_t *u = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)2 * LP * n);
    or_modup(c, D, d, lev, sp);
    or_key_inner(c, u, D, key, key_limbs, lev, sp);
    or_moddown(c, out, u, lev, sp);
    or_moddown(c, out + (size_t)L * n, u + (size_t)LP * n, lev, sp);
    free(D);
    free(u);
}

/* Rotation of a ciphertext ct[2][lev+1][n] by r slots with Galois key `key`. */
OR_API void or_rotate(const or_ctx *c, uint64_t *out, const uint64_t *ct, const uint64_t *key,
                      uint32_t key_limbs, uint32_t lev, uint32_t sp, int64_t r) {
    const uint32_t n = c->n, L = lev + 1;
    uint64_t *rot = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)2 * L * n);
    uint64_t *ks = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)2 * L * n);
    or_rotate_slots(c, rot, ct, 2 * L, r);
    or_keyswitch(c, ks, rot + (size_t)L * n, key, key_limbs, lev, sp);
    int32_t *mods = (int32_t *)malloc(sizeof(int32_t) * L);
    for (uint32_t i = 0; i < L; i++) mods[i] = (int32_t)i;
    or_add(c, out, rot, ks, mods, L);
    memcpy(out + (size_t)L * n, ks + (size_t)L * n, sizeof(uint64_t) * L * n);
    free(mods); free(rot); free(ks);
}

/* -- sampling (bit-identical definitions in csrc/rng.cuh) -------------------- */
/* Uniform residues, in evaluation form directly, for limbs with moduli mods[]. */
OR_API void or_sample_uniform(const or_ctx *c, uint64_t *out, uint64_t stream, const int32_t *mods, uint32_t L) {
    const uint32_t n = c->n;
    for (uint32_t l = 0; l < L; l++) {
        uint64_t q = c->q[mods[l]];
        for (uint32_t i = 0; i < n; i++) {
            uint64_t ctr = ((uint64_t)mods[l] * n + i) * 2;
            u128 v = ((u128)draw(stream, ctr) << 64) | draw(stream, ctr + 1);
            out[(size_t)l * n + i] = (uint64_t)(v % q);
        }
    }
}
/* Uniform ternary coefficients in {-1, 0, 1}. */
OR_API void or_sample_ternary(const or_ctx *c, int64_t *out, uint64_t stream) {
    for (uint32_t i = 0; i < c->n; i++) out[i] = (int64_t)(draw(stream, i) % 3) - 1;
}
/* Centred binomial noise, eta = 21 (sigma = 3.24). */
OR_API void or_sample_cbd(const or_ctx *c, int64_t *out, uint64_t stream) {
    for (uint32_t i = 0; i < c->n; i++) {
        uint64_t h = draw(stream, i);
        out[i] = (int64_t)__builtin_popcountll(h & 0x1FFFFFULL) - (int64_t)__builtin_popcountll((h >> 21) & 0x1FFFFFULL);
    }
}

/* Centred lift of one limb (coefficient form) to doubles. */
OR_API void or_to_double_centred(const or_ctx *c, double *out, const uint64_t *in, uint32_t m) {
    uint64_t q = c->q[m];
    for (uint32_t i = 0; i < c->n; i++) {
        uint64_t x = in[i];
        out[i] = x > (q - 1) / 2 ? -(double)(q - x) : (double)x;
    }
}

/* Forward / inverse NTT of L limbs (limb l modulo moduli[mods[l]]), OpenMP over limbs. */
OR_API void or_ntt_many(const or_ctx *c, uint64_t *a, const int32_t *mods, uint32_t L, int inverse) {
#pragma omp parallel for schedule(dynamic)
    for (uint32_t l = 0; l < L; l++) {
        if (inverse)
            or_intt(c, (uint32_t)mods[l], a + (size_t)l * c->n);
        else
            or_ntt(c, (uint32_t)mods[l], a + (size_t)l * c->n);
    }
}
