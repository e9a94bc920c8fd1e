// Internal host-side launchers of the RNS-CKKS operations (ops.cu, keys.cu).
//
// Layout conventions.  A polynomial list is `n_polys` polynomials of `nl`
// limbs, poly p limb k at base + (p * pstride + k) * N, evaluation (slot)
// order unless stated.  A ciphertext batch of B ciphertexts at level l with
// `ls` stored limbs per polynomial is the list of 2B polys (c0, c1 of ct 0,
// c0, c1 of ct 1, ...) with pstride = ls >= l + 1.  Limb k < nq is modulus k,
// the optional extra limb is the special prime P.
#pragma once
#include "engine.cuh"

namespace uh {

Ctx *ctx_create(uint32_t n, const uint64_t *moduli, const uint64_t *psi, uint32_t count, int device);
void ctx_destroy(Ctx *c);

enum BinOp : int { OP_ADD = 0, OP_SUB = 1, OP_MUL = 2, OP_MAC = 3, OP_NEG = 4, OP_COPY = 5 };

// out[p] = op(a[p], b[p % b_polys]) over nl limbs, moduli 0..nq-1 (+P).
void elementwise(const Ctx &c, int op, uint64_t *out, const uint64_t *a, const uint64_t *b, int n_polys,
                 int b_polys, int nl, int nq, int out_ps, int a_ps, int b_ps, cudaStream_t s);
void elementwise_grouped(const Ctx &c, int op, uint64_t *out, const uint64_t *a, const uint64_t *b, int n_polys,
                         int b_polys, int group, int nl, int nq, int out_ps, int a_ps, int b_ps, cudaStream_t s);

// Divide by the top limb's modulus with centred rounding:
// in: n_polys x (nl + 1) limbs, limb nl has modulus `top_mod`, limbs 0..nl-1
// moduli 0..nl-1.  out: n_polys x nl limbs.  Used for rescale (top_mod = l)
// and ModDown (top_mod = P).
void divide_top(const Ctx &c, uint64_t *out, const uint64_t *in, int n_polys, int nl, int top_mod, int out_ps,
                int in_ps, cudaStream_t s);

// Fused ModDown + rescale: in n_polys x (level + 2) limbs (q_0..q_level, P) -> out n_polys x level limbs,
// the centred division by q_level * P (one inverse NTT pair, one forward NTT per output limb).
// bias (optional): plaintext rows bias[p / bias_group][level][N] added to the even polynomials (c0) in the
// forward NTT's epilogue -- the conv bias, without a pass of its own.
void divide_top2(const Ctx &c, uint64_t *out, const uint64_t *in, int n_polys, int level, int out_ps, int in_ps,
                 cudaStream_t s, const uint64_t *bias = nullptr, int bias_group = 1);

// ModUp of n_polys polys at level l (L = l + 1 limbs, strided in_ps) into
// D = [n_polys][L digits][L + 1 limbs (q_0..q_l, P)][N], compact.
void modup(const Ctx &c, uint64_t *D, const uint64_t *in, int n_polys, int level, int in_ps, cudaStream_t s,
           bool diag = true);  // diag = false: D[p][j][j] left unwritten (it is in[p][j])

// u[p][comp][k] = sum_j rot_r(D[p][j][k]) * key[j][comp][kk],  comp = 0, 1,
// k over (q_0..q_l, P); key limbs (q_0..q_{key_limbs-2}, P). u compact [n_polys][2][L+1][N].
void key_inner(const Ctx &c, uint64_t *u, const uint64_t *D, const uint64_t *key, int key_limbs, int n_polys,
               int level, int64_t r, cudaStream_t s);

// Key switch of n_polys polys d (level l): out[p][comp] (compact [n_polys][2][L][N]).
void keyswitch(const Ctx &c, uint64_t *out, const uint64_t *d, int n_polys, int level, int d_ps,
               const uint64_t *key, int key_limbs, int64_t r, cudaStream_t s);

// Ciphertext ops on batches (see layout above).
void ct_rotate(const Ctx &c, uint64_t *out, const uint64_t *in, int B, int level, int out_ls, int in_ls,
               const uint64_t *key, int key_limbs, int64_t r, cudaStream_t s);
void ct_rotate_hoisted(const Ctx &c, uint64_t *out, const uint64_t *in, const uint64_t *D, int B, int level,
                       int out_ls, int in_ls, const uint64_t *key, int key_limbs, int64_t r, cudaStream_t s);
void ct_rescale(const Ctx &c, uint64_t *out, const uint64_t *in, int B, int level, int out_ls, int in_ls,
                cudaStream_t s);
void ct_mul_relin_rescale(const Ctx &c, uint64_t *out, const uint64_t *a, const uint64_t *b, int B, int level,
                          int out_ls, int a_ls, int b_ls, const uint64_t *rk, int rk_limbs, cudaStream_t s);
// fused-path square/multiply: relinearise in the QP basis and divide once by q_level * P
void ct_mul_relin_rescale_fused(const Ctx &c, uint64_t *out, const uint64_t *a, const uint64_t *b, int B, int level,
                                int out_ls, int a_ls, int b_ls, const uint64_t *rk, int rk_limbs, cudaStream_t s);
void ct_mul_plain_rescale(const Ctx &c, uint64_t *out, const uint64_t *ct, const uint64_t *pt, int B, int level,
                          int out_ls, int ct_ls, int pt_ls, int pt_batched, cudaStream_t s);

// Randomness, keys, encryption.
void secret_gen(const Ctx &c, uint64_t *s_eval, uint64_t seed, cudaStream_t st);
void switch_keygen(const Ctx &c, uint64_t *key, const uint64_t *s_eval, const uint64_t *s_from_eval,
                   uint64_t seed, uint64_t key_id, int level, cudaStream_t st);
void galois_keygen(const Ctx &c, uint64_t *key, const uint64_t *s_eval, uint64_t seed, int64_t r, int level,
                   cudaStream_t st);
void relin_keygen(const Ctx &c, uint64_t *key, const uint64_t *s_eval, uint64_t seed, int level, cudaStream_t st);
void encrypt(const Ctx &c, uint64_t *out, const uint64_t *pt, const uint64_t *s_eval, int B, int level, int out_ls,
             int pt_ls, uint64_t seed, uint64_t ct_id0, cudaStream_t st);
void decrypt_coeffs(const Ctx &c, double *out, const uint64_t *ct, const uint64_t *s_eval, int B, int ct_ls,
                    cudaStream_t st);

// Encoding: signed int64 coefficients -> evaluation form over moduli 0..nq-1 (+ P if special).
void from_signed(const Ctx &c, uint64_t *out, const int64_t *coef, int n_polys, int nq, int special, int out_ps,
                 cudaStream_t s);

// hoist.cu -- generic hoisted rotation-MAC.  X: [n_in][B][2][xls][N] input ciphertexts; D:
// [n_in][B][L][L+1][N] ModUp of their c1; keys[t] (device array of device pointers; unused for
// shift 0); shifts[t] in [0, N/2).  acc[O][B][2][L+1][N] (QP) = sum over terms q of
// masks[o][q] * P * rot_{shifts[t]}(ct_i); terms dense (i, t) or diag (i == t); masks may be null (= 1).
void hoisted_mac(const Ctx &c, uint64_t *acc, const uint64_t *X, int xls, const uint64_t *D, const uint64_t *masks,
                 const uint64_t *const *keys, const int32_t *key_limbs, const int32_t *shifts, int B, int I, int T,
                 int O, int diag, int level, cudaStream_t s);
// hoist_bank.cu -- the same hoisted MAC (every term mode, masks optional) over a per-layer key bank
// kb[NT][L+1][2L][N] (limb-major, (digit, component) inner), compile-time strides (N = 2^15).
bool hoisted_bank_supported(const Ctx &c, int level, int O);
void hoisted_mac_bank(const Ctx &c, uint64_t *acc, const uint64_t *X, const uint64_t *D, const uint64_t *masks,
                      const uint64_t *kbank, const int32_t *shifts, int B, int I, int T, int O, int diag, int level,
                      cudaStream_t s);
// one masked output with the masks folded into the key bank: km[Q][L+1][2L+1][N] (km_bank: rows
// M_q K_{t(q)} and M_q P), 2L + 1 MACs per term and no per-term reduction; same residues as
// hoisted_mac_bank with O = 1
void km_bank(const Ctx &c, uint64_t *km, const uint64_t *masks, const uint64_t *kbank, const int32_t *shifts, int Q,
             int T, int diag, int level, cudaStream_t s);
void hoisted_mac_km(const Ctx &c, uint64_t *acc, const uint64_t *X, const uint64_t *D, const uint64_t *km,
                    const int32_t *shifts, int B, int I, int T, int diag, int level, cudaStream_t s);
// hoist_imma.cu: the weight-mask contraction of the dense 5..12-output layers on the tensor
// cores (u8 byte-split IMMA) for the 40-bit limbs; the 60-bit limbs stay on the IMAD kernel
bool hoisted_imma_supported(const Ctx &c, int level, int O, int Q);
size_t imma_bank_words(const Ctx &c, int level, int O, int Q);
void imma_mask_bank(const Ctx &c, uint32_t *ib, const uint64_t *masks, int O, int Q, int level, cudaStream_t s);
void hoisted_mac_imma(const Ctx &c, uint64_t *acc, const uint64_t *X, const uint64_t *D, const uint64_t *masks,
                      const uint32_t *ib, const uint64_t *kbank, const int32_t *shifts, int B, int I, int T, int O,
                      int level, cudaStream_t s);
// the same with phase A (the key switch of every term) on the tensor cores as well: digit bytes x
// byte-weighted key bytes, one m16n8k32 per (term, coefficient, component) for 16 ciphertexts
// (level + 1 <= 6, <= 128 terms).  `kt` is the per-layer key bank in B-fragment order (imma_ta_bank,
// imma_ta_bank_bytes bytes); residues identical to hoisted_mac_imma.
bool hoisted_imma_ta_supported(const Ctx &c, int level, int O, int Q);
size_t imma_ta_bank_bytes(const Ctx &c, int level, int T);
void imma_ta_bank(const Ctx &c, uint8_t *kt, const uint64_t *kbank, const int32_t *shifts, int T, int level,
                  cudaStream_t s);
void hoisted_mac_imma_ta(const Ctx &c, uint64_t *acc, const uint64_t *X, const uint64_t *D, const uint32_t *ib,
                         const uint8_t *kt, const uint64_t *kbank, const int32_t *shifts, int B, int I, int T, int O,
                         int level, cudaStream_t s);
// hoist_tc.cu: the weight-mask contraction of dense masked layers (1..12 outputs) on the
// 5th-generation tensor cores (tcgen05.mma kind::i8, TMEM accumulators), every limb: 5-byte
// operands on the 40-bit limbs, 8-byte operands on q_0 and P.  `bank` is the per-layer A-operand
// bank made by tc_mask_bank (tc_bank_bytes bytes).
bool hoisted_tc_supported(const Ctx &c, int level, int O, int Q);
size_t tc_bank_bytes(const Ctx &c, int level, int O, int Q);
void tc_mask_bank(const Ctx &c, uint8_t *bank, const uint64_t *masks, int O, int Q, int level, cudaStream_t s);
void hoisted_mac_tc(const Ctx &c, uint64_t *acc, const uint64_t *X, const uint64_t *D, const uint8_t *bank,
                    const uint64_t *kbank, const int32_t *shifts, int B, int I, int T, int O, int level,
                    cudaStream_t s);
// microbench.cu: rates[0] = IMAD/s, rates[1] = 128-bit MAC/s, rates[2] = reduced mulmod/s
void bench_peaks(const Ctx &c, double *rates);
// embed.cu -- canonical embedding (hand-written FP64 four-step FFT): slots [n_polys][N/2] <-> int64 / double
// coefficients [n_polys][N] at `scale`.
void encode_coeffs(const Ctx &c, int64_t *coef, const double *slots, int n_polys, double scale, cudaStream_t s);
void decode_coeffs(const Ctx &c, double *slots, const double *coef, int n_polys, double scale, cudaStream_t s);

}  // namespace uh
