/*
 * CPU port of the engine's hoisted layer kernels -- TEST INFRASTRUCTURE AND CPU
 * BASELINE ONLY (loaded by tests/ and bench.py's cpu_baseline / reference arm).
 *
 * Same entry points, argument meaning and data layouts as the GPU C-ABI calls the
 * fused layer path (paper_2402_03060_b200/fused.py) issues -- uh_modup,
 * uh_hoisted_mac_bank, uh_divide_top, uh_divide_top2, uh_elementwise(_grouped),
 * uh_mul_relin_rescale_fused, uh_from_signed(_qp) -- so the unchanged fused.py
 * runs the SAME hoisted algorithm on the host (oracle/cpu_backend.py):
 *   ModUp once per input, every rotation's key switch + weight mask MAC in the QP
 *   basis, one fused ModDown + rescale per output.
 * Every result is a canonical residue fixed by its definition, so a GPU step and
 * this port agree residue for residue on the same inputs (tests/test_gpu_cpu_port.py).
 *
 * Parallelism: OpenMP over (polynomial, limb) for the NTT-based ops and over
 * (ciphertext, limb, coefficient block) for the MAC -- all host cores at any batch.
 * Arithmetic: the NTTs of ckks_oracle.c (Harvey/Shoup butterflies), 128-bit
 * products with 64-bit Barrett-free reductions (unsigned __int128 %), no SIMD.
 *
 * Reference semantics this restates (through the GPU kernels it mirrors):
 * layers.conv / avgpool / square / flatten / fc, pkg/src/slotcnn/layers.py:134-426,
 * over the operator interface he_backend.py:215-253.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;
#define HC_API __attribute__((visibility("default")))

#include "ckks_oracle.h"

/* allocation failure aborts: this is test / baseline infrastructure, a partial result would be wrong */
static void *xmalloc(size_t n) {
    void *p = malloc(n ? n : 1);
    if (!p) abort();
    return p;
}
static void *xcalloc(size_t n, size_t sz) {
    void *p = calloc(n ? n : 1, sz);
    if (!p) abort();
    return p;
}

static inline uint64_t addm(uint64_t a, uint64_t b, uint64_t q) {
    uint64_t s = a + b;
    return s >= q ? s - q : s;
}
static inline uint64_t subm(uint64_t a, uint64_t b, uint64_t q) { return a >= b ? a - b : a + q - b; }
static inline uint64_t mulm(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a * b) % q); }
static uint64_t powm(uint64_t b, uint64_t e, uint64_t q) {
    uint64_t r = 1;
    b %= q;
    while (e) {
        if (e & 1) r = mulm(r, b, q);
        b = mulm(b, b, q);
        e >>= 1;
    }
    return r;
}
static inline uint64_t invm(uint64_t a, uint64_t q) { return powm(a, q - 2, q); }
/* centred lift of x in [0, p) reduced into q */
static inline uint64_t centred(uint64_t x, uint64_t p, uint64_t q) {
    if (x > (p - 1) / 2) {
        uint64_t r = (p - x) % q;
        return r ? q - r : 0;
    }
    return x % q;
}
static inline int sp_of(const or_ctx *c) { return (int)c->count - 1; }
static inline uint64_t limb_q(const or_ctx *c, int k, int nq) { return c->q[k < nq ? k : sp_of(c)]; }
static inline uint32_t rot_idx(uint32_t n, uint32_t half, uint32_t r) {
    uint32_t h = n >= half ? half : 0, j = n - h + r;
    if (j >= half) j -= half;
    return h + j;
}

/* uh_elementwise(_grouped): out[p][k] = a[p][k] op b[(p / div) % bp][k], limb k mod q_k (k < nq) or P */
HC_API void hc_elementwise_grouped(const or_ctx *c, int op, uint64_t *out, const uint64_t *a, const uint64_t *b,
                                   int n_polys, int b_polys, int div, int nl, int nq, int out_ps, int a_ps, int b_ps) {
    const size_t N = c->n;
#pragma omp parallel for collapse(2) schedule(static)
    for (int p = 0; p < n_polys; p++)
        for (int k = 0; k < nl; k++) {
            const uint64_t q = limb_q(c, k, nq);
            uint64_t *o = out + ((size_t)p * out_ps + k) * N;
            const uint64_t *x = a + ((size_t)p * a_ps + k) * N;
            const uint64_t *y = (op == 4 || op == 5) ? NULL : b + ((size_t)((p / div) % b_polys) * b_ps + k) * N;
            for (size_t i = 0; i < N; i++) {
                uint64_t r;
                switch (op) {
                    case 0: r = addm(x[i], y[i], q); break;
                    case 1: r = subm(x[i], y[i], q); break;
                    case 2: r = mulm(x[i], y[i], q); break;
                    case 3: r = addm(o[i], mulm(x[i], y[i], q), q); break;
                    case 4: r = x[i] ? q - x[i] : 0; break;
                    default: r = x[i]; break;
                }
                o[i] = r;
            }
        }
}
HC_API void hc_elementwise(const or_ctx *c, int op, uint64_t *out, const uint64_t *a, const uint64_t *b, int n_polys,
                           int b_polys, int nl, int nq, int out_ps, int a_ps, int b_ps) {
    int div = 1;
    if (b_polys < 0) {  /* broadcast over the two components of each ciphertext */
        b_polys = -b_polys;
        div = 2;
    }
    hc_elementwise_grouped(c, op, out, a, b, n_polys, b_polys > 0 ? b_polys : 1, div, nl, nq, out_ps, a_ps, b_ps);
}

/* uh_from_signed / uh_from_signed_qp: signed coefficients -> evaluation form over nq q-limbs (+ P when qp) */
HC_API void hc_from_signed(const or_ctx *c, uint64_t *out, const int64_t *coef, int n_polys, int nq, int qp,
                           int out_ps) {
    const size_t N = c->n;
    const int nl = nq + (qp ? 1 : 0);
#pragma omp parallel for collapse(2) schedule(dynamic)
    for (int p = 0; p < n_polys; p++)
        for (int k = 0; k < nl; k++) {
            const int m = k < nq ? k : sp_of(c);
            const uint64_t q = c->q[m];
            uint64_t *o = out + ((size_t)p * out_ps + k) * N;
            const int64_t *x = coef + (size_t)p * N;
            for (size_t i = 0; i < N; i++) {
                const int64_t v = x[i];
                const uint64_t r = (uint64_t)(v < 0 ? -v : v) % q;
                o[i] = v < 0 ? (r ? q - r : 0) : r;
            }
            or_ntt(c, (uint32_t)m, o);
        }
}

/* uh_modup: in [n_polys][in_ps limbs][N] (limbs 0..level) -> D [n_polys][L][L+1][N] */
HC_API void hc_modup(const or_ctx *c, uint64_t *D, const uint64_t *in, int n_polys, int level, int in_ps) {
    const size_t N = c->n;
    const int L = level + 1, LP = level + 2;
#pragma omp parallel for collapse(2) schedule(dynamic)
    for (int p = 0; p < n_polys; p++)
        for (int j = 0; j < L; j++) {
            const uint64_t qj = c->q[j];
            const uint64_t *src = in + ((size_t)p * in_ps + j) * N;
            uint64_t *coef = (uint64_t *)xmalloc(sizeof(uint64_t) * N);
            memcpy(coef, src, sizeof(uint64_t) * N);
            or_intt(c, (uint32_t)j, coef);
            for (int k = 0; k < LP; k++) {
                uint64_t *dst = D + (((size_t)p * L + j) * LP + k) * N;
                if (k == j) {
                    memcpy(dst, src, sizeof(uint64_t) * N);
                    continue;
                }
                const int mk = k < L ? k : sp_of(c);
                const uint64_t q = c->q[mk];
                for (size_t i = 0; i < N; i++) dst[i] = centred(coef[i], qj, q);
                or_ntt(c, (uint32_t)mk, dst);
            }
            free(coef);
        }
}

/* uh_divide_top: in [n_polys][in_ps][N] limbs 0..nl-1 plus the top limb nl (modulus top_mod) ->
 * out [n_polys][out_ps][N], limb k = (in_k - centred(top) mod q_k) * q_top^-1 */
HC_API void hc_divide_top(const or_ctx *c, uint64_t *out, const uint64_t *in, int n_polys, int nl, int top_mod,
                          int out_ps, int in_ps) {
    const size_t N = c->n;
    const uint64_t qt = c->q[top_mod];
    uint64_t *tops = (uint64_t *)xmalloc(sizeof(uint64_t) * N * (size_t)(n_polys > 0 ? n_polys : 1));
#pragma omp parallel for schedule(dynamic)
    for (int p = 0; p < n_polys; p++) {
        memcpy(tops + (size_t)p * N, in + ((size_t)p * in_ps + nl) * N, sizeof(uint64_t) * N);
        or_intt(c, (uint32_t)top_mod, tops + (size_t)p * N);
    }
#pragma omp parallel for collapse(2) schedule(dynamic)
    for (int p = 0; p < n_polys; p++)
        for (int k = 0; k < nl; k++) {
            const uint64_t q = c->q[k], inv = invm(qt % q, q);
            const uint64_t *top = tops + (size_t)p * N;
            uint64_t *t = (uint64_t *)xmalloc(sizeof(uint64_t) * N);
            for (size_t i = 0; i < N; i++) t[i] = centred(top[i], qt, q);
            or_ntt(c, (uint32_t)k, t);
            const uint64_t *x = in + ((size_t)p * in_ps + k) * N;
            uint64_t *o = out + ((size_t)p * out_ps + k) * N;
            for (size_t i = 0; i < N; i++) o[i] = mulm(subm(x[i], t[i], q), inv, q);
            free(t);
        }
    free(tops);
}

/* uh_divide_top2: in [n_polys][in_ps][N] limbs (q_0..q_level, P) -> out limbs 0..level-1:
 * centred division by q_level * P.  x = CRT(x mod q_level, x mod P) in [0, q_level P), centred. */
HC_API void hc_divide_top2(const or_ctx *c, uint64_t *out, const uint64_t *in, int n_polys, int level, int out_ps,
                           int in_ps) {
    const size_t N = c->n;
    const int sp = sp_of(c);
    const uint64_t qt = c->q[level], P = c->q[sp];
    const uint64_t pinv = invm(P % qt, qt);
    const u128 M = (u128)qt * P, half = (M - 1) / 2;
    /* per coefficient: y = ((x_t - x_P) P^-1 mod q_t), x = x_P + P y; neg when x > (M - 1) / 2 */
    uint64_t *Y = (uint64_t *)xmalloc(sizeof(uint64_t) * N * (size_t)(n_polys > 0 ? n_polys : 1));
    uint64_t *XP = (uint64_t *)xmalloc(sizeof(uint64_t) * N * (size_t)(n_polys > 0 ? n_polys : 1));
    uint8_t *NEG = (uint8_t *)xmalloc(N * (size_t)(n_polys > 0 ? n_polys : 1));
#pragma omp parallel for schedule(dynamic)
    for (int p = 0; p < n_polys; p++) {
        uint64_t *yt = Y + (size_t)p * N, *xp = XP + (size_t)p * N;
        memcpy(yt, in + ((size_t)p * in_ps + level) * N, sizeof(uint64_t) * N);
        memcpy(xp, in + ((size_t)p * in_ps + level + 1) * N, sizeof(uint64_t) * N);
        or_intt(c, (uint32_t)level, yt);
        or_intt(c, (uint32_t)sp, xp);
        for (size_t i = 0; i < N; i++) {
            const uint64_t y = mulm(subm(yt[i], xp[i] % qt, qt), pinv, qt);
            const u128 x = (u128)xp[i] + (u128)P * y;
            yt[i] = y;
            NEG[(size_t)p * N + i] = x > half;
        }
    }
#pragma omp parallel for collapse(2) schedule(dynamic)
    for (int p = 0; p < n_polys; p++)
        for (int k = 0; k < level; k++) {
            const uint64_t q = c->q[k];
            const uint64_t inv = invm(mulm(qt % q, P % q, q), q);
            const uint64_t Mq = (uint64_t)(M % q), Pq = P % q;
            uint64_t *t = (uint64_t *)xmalloc(sizeof(uint64_t) * N);
            for (size_t i = 0; i < N; i++) {
                /* (x_P + P y) mod q, minus M when the centred value is negative */
                uint64_t v = addm(XP[(size_t)p * N + i] % q, mulm(Pq, Y[(size_t)p * N + i] % q, q), q);
                t[i] = NEG[(size_t)p * N + i] ? subm(v, Mq, q) : v;
            }
            or_ntt(c, (uint32_t)k, t);
            const uint64_t *x = in + ((size_t)p * in_ps + k) * N;
            uint64_t *o = out + ((size_t)p * out_ps + k) * N;
            for (size_t i = 0; i < N; i++) o[i] = mulm(subm(x[i], t[i], q), inv, q);
            free(t);
        }
    free(Y);
    free(XP);
    free(NEG);
}

/* key inner product of ModUp digits with a key [digits][2][key_limbs][N] (limbs q_0.., P last),
 * plus (P mod q_k) * add[b][comp][k] on the q-limbs when `add` is given:
 * u[p][comp][k] (QP basis, L + 1 limbs) */
static void key_inner_add(const or_ctx *c, uint64_t *u, const uint64_t *D, const uint64_t *key, int key_limbs,
                          int n_polys, int level, const uint64_t *add) {
    const size_t N = c->n;
    const int L = level + 1, LP = level + 2, sp = sp_of(c);
    const uint64_t P = c->q[sp];
#pragma omp parallel for collapse(3) schedule(dynamic)
    for (int p = 0; p < n_polys; p++)
        for (int comp = 0; comp < 2; comp++)
            for (int k = 0; k < LP; k++) {
                const int mk = k < L ? k : sp, kk = k < L ? k : key_limbs - 1;
                const uint64_t q = c->q[mk], Pk = P % q;
                uint64_t *dst = u + (((size_t)p * 2 + comp) * LP + k) * N;
                for (size_t i = 0; i < N; i++) {
                    u128 acc = 0;
                    for (int j = 0; j < L; j++)
                        acc += (u128)D[(((size_t)p * L + j) * LP + k) * N + i] *
                               key[(((size_t)j * 2 + comp) * key_limbs + kk) * N + i];
                    uint64_t r = (uint64_t)(acc % q);
                    if (add && k < L) r = addm(r, mulm(Pk, add[(((size_t)p * 2 + comp) * L + k) * N + i], q), q);
                    dst[i] = r;
                }
            }
}

/* uh_mul_relin_rescale_fused: tensor (d0, d1, d2) of a, b at `level`; u = <ModUp(d2), rk> + P (d0, d1)
 * in the QP basis; out = u / (q_level P) (hc_divide_top2) */
HC_API void hc_mul_relin_rescale_fused(const or_ctx *c, uint64_t *out, const uint64_t *a, const uint64_t *b, int B,
                                       int level, int out_ls, int a_ls, int b_ls, const uint64_t *rk, int rk_limbs) {
    const size_t N = c->n;
    const int L = level + 1, LP = level + 2;
    uint64_t *T = (uint64_t *)xmalloc(sizeof(uint64_t) * (size_t)B * 2 * L * N);
    uint64_t *D2 = (uint64_t *)xmalloc(sizeof(uint64_t) * (size_t)B * L * N);
#pragma omp parallel for collapse(2) schedule(static)
    for (int bb = 0; bb < B; bb++)
        for (int k = 0; k < L; k++) {
            const uint64_t q = c->q[k];
            const uint64_t *a0 = a + ((size_t)bb * 2 * a_ls + k) * N, *a1 = a0 + (size_t)a_ls * N;
            const uint64_t *b0 = b + ((size_t)bb * 2 * b_ls + k) * N, *b1 = b0 + (size_t)b_ls * N;
            uint64_t *t0 = T + ((size_t)bb * 2 * L + k) * N, *t1 = t0 + (size_t)L * N;
            uint64_t *d2 = D2 + ((size_t)bb * L + k) * N;
            for (size_t i = 0; i < N; i++) {
                t0[i] = mulm(a0[i], b0[i], q);
                t1[i] = (uint64_t)(((u128)a0[i] * b1[i] + (u128)a1[i] * b0[i]) % q);
                d2[i] = mulm(a1[i], b1[i], q);
            }
        }
    uint64_t *D = (uint64_t *)xmalloc(sizeof(uint64_t) * (size_t)B * L * LP * N);
    uint64_t *u = (uint64_t *)xmalloc(sizeof(uint64_t) * (size_t)B * 2 * LP * N);
    hc_modup(c, D, D2, B, level, L);
    key_inner_add(c, u, D, rk, rk_limbs, B, level, T);
    hc_divide_top2(c, out, u, 2 * B, level, out_ls, LP);
    free(T);
    free(D2);
    free(D);
    free(u);
}

/* uh_hoisted_mac_bank: acc[o][b][comp][k][n] (QP basis) = sum over terms q of
 *   masks[o][q][k][n] * (P rot_{s_t}(c0) + <rot_{s_t}(D), K_t>, <rot_{s_t}(D), K'_t>)
 * terms: diag 0: q = i T + t (key entry t); 1: q = i = t; 2: q = i T + t' (key entry q).
 * kbank [NT][L+1][2L][N]; masks NULL = all ones (every output the same sum).
 * Work split: (ciphertext, limb, block of 512 coefficients) per task; each task keeps its
 * outputs' 128-bit sums for the block and walks every term once. */
#define HC_NB 512
HC_API void hc_hoisted_mac_bank(const or_ctx *c, uint64_t *acc, const uint64_t *X, int xls, const uint64_t *D,
                                const uint64_t *masks, const uint64_t *kbank, const int32_t *shifts, int B, int I,
                                int T, int O, int diag, int level) {
    const size_t N = c->n;
    const uint32_t half = c->n / 2;
    const int L = level + 1, LP = level + 2, sp = sp_of(c);
    const int Q = diag == 1 ? I : I * T;
    const uint64_t P = c->q[sp];
    const int OM = masks ? O : 1;
    const int nblk = (int)((N + HC_NB - 1) / HC_NB);
#pragma omp parallel for collapse(3) schedule(dynamic)
    for (int b = 0; b < B; b++)
        for (int k = 0; k < LP; k++)
            for (int blk = 0; blk < nblk; blk++) {
                const int qlimb = k < L;
                const uint64_t q = c->q[qlimb ? k : sp], Pk = qlimb ? P % q : 0;
                const size_t n0 = (size_t)blk * HC_NB, nn = N - n0 < HC_NB ? N - n0 : HC_NB;
                u128 *s = (u128 *)xcalloc((size_t)OM * 2 * HC_NB, sizeof(u128));
                uint64_t v0[HC_NB], v1[HC_NB];
                int pending = 0;
                for (int qq = 0; qq < Q; qq++) {
                    int i, t;
                    if (diag == 1) {
                        i = t = qq;
                    } else {
                        i = qq / T;
                        t = diag == 2 ? qq : qq - i * T;
                    }
                    const uint32_t r = (uint32_t)shifts[t];
                    const uint64_t *c0 = X + (((size_t)i * B + b) * 2 * xls + k) * N;
                    const uint64_t *c1 = c0 + (size_t)xls * N;
                    if (r == 0) {
                        for (size_t e = 0; e < nn; e++) {
                            v0[e] = qlimb ? mulm(Pk, c0[n0 + e], q) : 0;
                            v1[e] = qlimb ? mulm(Pk, c1[n0 + e], q) : 0;
                        }
                    } else {
                        const uint64_t *Dd = D + (((size_t)i * B + b) * L * LP + k) * N;
                        const uint64_t *K = kbank + ((size_t)t * LP + k) * 2 * L * N;
                        for (size_t e = 0; e < nn; e++) {
                            const uint32_t n = (uint32_t)(n0 + e), src = rot_idx(n, half, r);
                            u128 a0 = 0, a1 = 0;
                            for (int j = 0; j < L; j++) {
                                const uint64_t d = Dd[(size_t)j * LP * N + src];
                                a0 += (u128)d * K[(size_t)(2 * j) * N + n];
                                a1 += (u128)d * K[(size_t)(2 * j + 1) * N + n];
                            }
                            if (qlimb) a0 += (u128)Pk * c0[src];
                            v0[e] = (uint64_t)(a0 % q);
                            v1[e] = (uint64_t)(a1 % q);
                        }
                    }
                    for (int o = 0; o < OM; o++) {
                        u128 *s0 = s + (size_t)o * 2 * HC_NB, *s1 = s0 + HC_NB;
                        if (masks) {
                            const uint64_t *mk = masks + (((size_t)o * Q + qq) * LP + k) * N + n0;
                            for (size_t e = 0; e < nn; e++) {
                                s0[e] += (u128)mk[e] * v0[e];
                                s1[e] += (u128)mk[e] * v1[e];
                            }
                        } else {
                            for (size_t e = 0; e < nn; e++) {
                                s0[e] += v0[e];
                                s1[e] += v1[e];
                            }
                        }
                    }
                    if (++pending == 64) {  /* 64 products < 2^126: fold before overflow */
                        pending = 0;
                        for (size_t x = 0; x < (size_t)OM * 2 * HC_NB; x++) s[x] %= q;
                    }
                }
                for (int o = 0; o < O; o++) {
                    const int so = masks ? o : 0;
                    for (int comp = 0; comp < 2; comp++) {
                        uint64_t *dst = acc + ((((size_t)o * B + b) * 2 + comp) * LP + k) * N + n0;
                        const u128 *sv = s + ((size_t)so * 2 + comp) * HC_NB;
                        for (size_t e = 0; e < nn; e++) dst[e] = (uint64_t)(sv[e] % q);
                    }
                }
                free(s);
            }
}
