/*
 * unihenn_b200.h -- C-ABI of the B200-native RNS-CKKS engine behind the
 * reference's operator boundary (pkg/src/slotcnn/he_backend.py:155-253).
 *
 * The reference has no native code and no FFI; its boundary is the Python
 * class `Backend` (encode / _plain / encrypt / decrypt / add / mul_plain /
 * mul_cipher / rotate).  Each entry point below is what a drop-in GPU
 * `Backend` binds through ctypes; the comment on each
 * names the reference interface it replaces.
 *
 * Conventions
 *  - Every uint64_t* / int64_t* / double* argument is a DEVICE pointer on the
 *    context's device, except the host arrays of uh_ctx_create.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *    asynchronous on that stream; scratch comes from the stream-ordered pool.
 *  - Polynomials are in evaluation ("slot") order: entry j < N/2 holds
 *    a(psi^(5^j)), entry N/2+j holds a(psi^(-5^j)); rotation by r slots is a
 *    cyclic shift of each half.  Residues are canonical, in [0, q).
 *  - A polynomial list is n_polys polys of nl limbs, poly p limb k at
 *    base + (p*pstride + k)*N; limb k < nq is modulus k, a further limb is the
 *    special prime P (modulus index count-1).  A batch of B ciphertexts with ls
 *    stored limbs is the list of 2B polys (c0,c1 of ct 0, c0,c1 of ct 1, ...)
 *    with pstride = ls.  Level l uses limbs 0..l.
 *  - Key-switching keys: [l+1 digits][2][key_limbs][N] with limbs
 *    (q_0..q_{key_limbs-2}, P); usable at every level <= key_limbs - 2.
 *  - Return value: 0 on success, nonzero on error; uh_last_error() gives the
 *    message (thread-local).  The Python wrapper raises
 *    LevelExhausted / SlotMismatch / OversizedInput itself before calling.
 */
#ifndef UNIHENN_B200_H
#define UNIHENN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct uh_ctx uh_ctx;

int uh_abi_version(void);
const char *uh_last_error(void);
/* Number of engine kernel launches so far in this process (bench evidence). */
unsigned long long uh_launch_count(void);
/* Integer-pipe peaks measured on the context's device (HOST array of >= 16):
 * IMAD/s, lazy 128-bit multiply-accumulate/s (engine form), reduced 64-bit
 * mulmod/s, 128-bit MAC/s in plain-C form, lazy Shoup products/s, exact FP64
 * modMAC/s, mixed IMAD+FP64 MAC/s, split-accumulator MAC/s, narrow-operand
 * (q < 2^41) MAC/s, u8 IMMA MAC/s (mma.sync m16n8k32), FP64 FMA/s, tcgen05
 * kind::i8 MAC/s: 12 entries
 * (the caller's buffer holds at least 16). */
int uh_bench_peaks(uh_ctx *ctx, double *rates);

/* Parameter set -> device context.  Replaces HEParams' role as the space
 * description (he_backend.py:34-77): moduli = q_0..q_depth, P; psi[i] a
 * primitive 2N-th root of unity mod moduli[i]. */
int uh_ctx_create(uh_ctx **out, uint32_t n, const uint64_t *moduli, const uint64_t *psi, uint32_t count,
                  int device);
int uh_ctx_destroy(uh_ctx *ctx);

/* Forward (coefficients -> slot order) or inverse NTT, in place.
 * Building block of encode (he_backend.py:176-190) and of every key switch. */
int uh_ntt(uh_ctx *ctx, uint64_t *data, int n_polys, int nl, int nq, int pstride, int inverse, void *stream);

/* Elementwise op over a polynomial list: 0 add, 1 sub, 2 mul, 3 out += a*b,
 * 4 negate, 5 copy.  b poly index = p % b_polys, or (p/2) % (-b_polys) when
 * b_polys < 0 (one plaintext per ciphertext).  add == Backend.add
 * (he_backend.py:215-224). */
int uh_elementwise(uh_ctx *ctx, int op, uint64_t *out, const uint64_t *a, const uint64_t *b, int n_polys,
                   int b_polys, int nl, int nq, int out_ps, int a_ps, int b_ps, void *stream);

/* uh_elementwise with grouped broadcast: b poly index = (p / group) % b_polys
 * (e.g. one bias plaintext per output channel over its B ciphertexts, one launch
 * for all channels: layers.conv's bias add, layers.py:193-195). */
int uh_elementwise_grouped(uh_ctx *ctx, int op, uint64_t *out, const uint64_t *a, const uint64_t *b, int n_polys,
                           int b_polys, int group, int nl, int nq, int out_ps, int a_ps, int b_ps, void *stream);

/* Divide by the modulus of the top limb with centred rounding (rescale when
 * top_mod = nl, ModDown when top_mod = P): in n_polys x (nl+1) -> out n_polys x nl. */
int uh_divide_top(uh_ctx *ctx, uint64_t *out, const uint64_t *in, int n_polys, int nl, int top_mod, int out_ps,
                  int in_ps, void *stream);

/* Fused ModDown + rescale of QP-basis accumulators: in n_polys x (level+2) limbs
 * (q_0..q_level, P) -> out n_polys x level limbs, centred division by q_level * P
 * (the single division the hoisted layers need per output; rounding differs
 * from ModDown-then-rescale by < 1 unit). */
int uh_divide_top2(uh_ctx *ctx, uint64_t *out, const uint64_t *in, int n_polys, int level, int out_ps, int in_ps,
                   void *stream);
/* uh_divide_top2 with the conv bias (layers.conv, layers.py:193-195) added in the same pass:
 * bias[n_polys / bias_group][level][N] (evaluation form at the output level), row set p / bias_group
 * added to the even polynomials (the c0 of each (c0, c1) pair); residues identical to
 * uh_divide_top2 followed by uh_elementwise_grouped.  Supported with the fast NTT
 * (uh_divide_top2_bias_supported: 2^13 <= N <= 2^15). */
int uh_divide_top2_bias_supported(uh_ctx *ctx);
int uh_divide_top2_bias(uh_ctx *ctx, uint64_t *out, const uint64_t *in, int n_polys, int level, int out_ps,
                        int in_ps, const uint64_t *bias, int bias_group, void *stream);

/* Rescale of a ciphertext batch at `level` (the level-1 of he_backend.py:226-247). */
int uh_rescale(uh_ctx *ctx, uint64_t *out, const uint64_t *in, int B, int level, int out_ls, int in_ls,
               void *stream);

/* Hybrid key switching pieces: ModUp (one digit per q_j, centred lift) into
 * D[n_polys][l+1][l+2][N]; inner product with a key, the Galois shift r folded
 * into the D reads -> u[n_polys][2][l+2][N]; full key switch -> [n_polys][2][l+1][N]. */
int uh_modup(uh_ctx *ctx, uint64_t *D, const uint64_t *in, int n_polys, int level, int in_ps, void *stream);
int uh_key_inner(uh_ctx *ctx, uint64_t *u, const uint64_t *D, const uint64_t *key, int key_limbs, int n_polys,
                 int level, int64_t r, void *stream);
int uh_keyswitch(uh_ctx *ctx, uint64_t *out, const uint64_t *d, int n_polys, int level, int d_ps,
                 const uint64_t *key, int key_limbs, void *stream);

/* Backend.rotate (he_backend.py:249-253): left rotation by r slots
 * (np.roll(v, -r)); r = 0 is a copy. */
int uh_rotate(uh_ctx *ctx, uint64_t *out, const uint64_t *in, int B, int level, int out_ls, int in_ls,
              const uint64_t *key, int key_limbs, int64_t r, void *stream);
/* uh_rotate given the ModUp digits D of in's c1 (uh_modup over the B c1 polys, in_ps = 2 * in_ls):
 * key product + ModDown + rot(c0) only, bit-identical to uh_rotate.  Backend.rotate
 * (he_backend.py:249-253) reuses D across consecutive rotations of one ciphertext, so the
 * reference's per-tap rotate calls (layers.py:165-196) are hoisted automatically. */
int uh_rotate_hoisted(uh_ctx *ctx, uint64_t *out, const uint64_t *in, const uint64_t *D, int B, int level,
                      int out_ls, int in_ls, const uint64_t *key, int key_limbs, int64_t r, void *stream);

/* Backend.mul_plain (he_backend.py:226-235): ct x pt then rescale; pt encoded
 * at scale q_level.  pt_batched: one plaintext per ciphertext instead of one shared. */
int uh_mul_plain_rescale(uh_ctx *ctx, uint64_t *out, const uint64_t *ct, const uint64_t *pt, int B, int level,
                         int out_ls, int ct_ls, int pt_ls, int pt_batched, void *stream);

/* Backend.mul_cipher (he_backend.py:237-247): tensor, relinearise with rk, rescale. */
int uh_mul_relin_rescale(uh_ctx *ctx, uint64_t *out, const uint64_t *a, const uint64_t *b, int B, int level,
                         int out_ls, int a_ls, int b_ls, const uint64_t *rk, int rk_limbs, void *stream);

/* Fused-path Backend.mul_cipher: relinearise in the QP basis (u + P*(d0, d1)) and
 * divide once by q_level * P (uh_divide_top2); used by the batched square layer. */
int uh_mul_relin_rescale_fused(uh_ctx *ctx, uint64_t *out, const uint64_t *a, const uint64_t *b, int B, int level,
                               int out_ls, int a_ls, int b_ls, const uint64_t *rk, int rk_limbs, void *stream);

/* Keys.  Secret: ternary, evaluation form over all `count` moduli, [count][N]. */
int uh_secret_gen(uh_ctx *ctx, uint64_t *s_eval, uint64_t seed, void *stream);
int uh_galois_keygen(uh_ctx *ctx, uint64_t *key, const uint64_t *s_eval, uint64_t seed, int64_t r, int level,
                     void *stream);
int uh_relin_keygen(uh_ctx *ctx, uint64_t *key, const uint64_t *s_eval, uint64_t seed, int level, void *stream);

/* Backend.encrypt (he_backend.py:202-204): secret-key encryption of B
 * plaintexts (pt_ls < 0: one plaintext for all) at `level`; ct b uses
 * randomness id ct_id0 + b. */
int uh_encrypt(uh_ctx *ctx, uint64_t *out, const uint64_t *pt, const uint64_t *s_eval, int B, int level,
               int out_ls, int pt_ls, uint64_t seed, uint64_t ct_id0, void *stream);

/* Backend.decrypt (he_backend.py:206-207), first half: c0 + c1*s on q_0,
 * inverse NTT, centred -> double coefficients [B][N]. */
int uh_decrypt_coeffs(uh_ctx *ctx, double *out, const uint64_t *ct, const uint64_t *s_eval, int B, int ct_ls,
                      void *stream);

/* Backend.encode (he_backend.py:176-190) on the device: canonical embedding
 * of real slot vectors [n_polys][N/2] at `scale` -> rounded int64 coefficients
 * [n_polys][N]; from_signed reduces them into nl limbs and NTTs. */
int uh_encode_coeffs(uh_ctx *ctx, int64_t *coef, const double *slots, int n_polys, double scale, void *stream);
int uh_from_signed(uh_ctx *ctx, uint64_t *out, const int64_t *coef, int n_polys, int nl, int out_ps, void *stream);
/* decrypt, second half: coefficients -> slot values [n_polys][N/2]. */
int uh_decode_coeffs(uh_ctx *ctx, double *slots, const double *coef, int n_polys, double scale, void *stream);
/* as uh_from_signed but into the QP basis (q_0..q_{nq-1}, P): plaintext weight masks for the hoisted layers. */
int uh_from_signed_qp(uh_ctx *ctx, uint64_t *out, const int64_t *coef, int n_polys, int nq, int out_ps,
                      void *stream);

/* Hoisted, fused convolution (replaces the op stream of layers.conv,
 * layers.py:165-196: K^2*ch_in rotations + ch_out*ch_in*K^2 masked products +
 * adds).  X: [I][B][2][xls][N] input ciphertexts at `level`; D: their c1 ModUp
 * (uh_modup over the I*B c1 polys); masks: [O][I][T][level+2][N] weight masks
 * in the QP basis encoded at scale q_level; keys: DEVICE array of T device
 * pointers to Galois keys (entry ignored when shifts[t] == 0) and key_limbs:
 * DEVICE int32 [T] their limb counts (each >= level + 2); shifts: DEVICE
 * int32 [T] in [0, N/2).  acc: [O][B][2][level+2][N], the QP-basis sum
 * sum_{i,t} masks[o][i][t] * P * rot_t(ct_i); ModDown (uh_divide_top with P)
 * then rescale give the layer output before the bias. */
int uh_conv_hoisted_mac(uh_ctx *ctx, uint64_t *acc, const uint64_t *X, int xls, const uint64_t *D,
                        const uint64_t *masks, const uint64_t *const *keys, const int32_t *key_limbs,
                        const int32_t *shifts, int B, int I, int T, int O, int level, void *stream);
/* Generic hoisted rotation-MAC behind every fused layer: acc[O][B][2][level+2][N]
 * = sum over terms q of masks[o][q] * P * rot_{shifts[t]}(ct_i), terms dense
 * (diag 0: q = i*T + t, T shared taps), diagonal (diag 1: q = i = t, I == T) or
 * block-diagonal (diag 2: q = i*T + t' with per-term taps t = q, i.e. shifts /
 * keys / key_limbs hold I*T entries; O <= 2); masks may be NULL (all ones, no
 * rescale needed).  Used for conv, pool, the flatten stages (masks pre-rotated:
 * rot(m .* x) = rot(m) .* rot(x)), the last flatten stage merged with the
 * channel packing (block-diagonal), and the FC diagonals / wrap fix / folds
 * (layers.py:263-426). */
int uh_hoisted_mac(uh_ctx *ctx, uint64_t *acc, const uint64_t *X, int xls, const uint64_t *D, const uint64_t *masks,
                   const uint64_t *const *keys, const int32_t *key_limbs, const int32_t *shifts, int B, int I, int T,
                   int O, int diag, int level, void *stream);
/* uh_hoisted_mac over a per-layer key bank instead of per-key pointers (every
 * term mode; masks may be NULL): kbank is [NT][level+2][2*(level+1)][N] with NT
 * = T (dense), I (diagonal) or I*T (block-diagonal) entries, one per entry of
 * `shifts` (limb-major; row (k, 2j + c) = component c of digit j of the Galois
 * key of that shift, limb k of q_0..q_level, P; any content for shift 0).
 * Same result as uh_hoisted_mac / uh_conv_hoisted_mac / uh_rot_sum_hoisted
 * (layers.conv / avgpool / flatten / fc, layers.py:134-426) bit for bit, with
 * compile-time strides.  Supported when uh_hoisted_bank_supported(ctx, level, O)
 * returns 1 (N = 2^15, level + 1 <= 10, 1 <= O <= 12); X must hold exactly
 * level + 1 limbs (xls == level + 1). */
int uh_hoisted_bank_supported(uh_ctx *ctx, int level, int O);
int uh_hoisted_mac_bank(uh_ctx *ctx, uint64_t *acc, const uint64_t *X, int xls, const uint64_t *D,
                        const uint64_t *masks, const uint64_t *kbank, const int32_t *shifts, int B, int I, int T,
                        int O, int diag, int level, void *stream);

/* One masked output (the flatten stages, layers.py:281-339) with the masks folded into the
 * key bank: uh_km_bank makes km[Q][level+2][2*(level+1)+1][N] from the mask bank
 * [Q][level+2][N] and the key bank (rows 2j + c of entry q = masks[q] (.) key row of the term's
 * shift, t = q mod T for dense terms and q otherwise; row 2*(level+1) = masks[q] * P on the
 * q-limbs), once per layer.  uh_hoisted_mac_km then needs 2*(level+1) + 1 multiply-accumulates
 * per term and no per-term reduction; acc[1][B][2][level+2][N] is residue-identical to
 * uh_hoisted_mac_bank with O = 1.  Supported when uh_hoisted_bank_supported(ctx, level, 1). */
int uh_km_supported(uh_ctx *ctx, int level);
int uh_km_bank(uh_ctx *ctx, uint64_t *km, const uint64_t *masks, const uint64_t *kbank, const int32_t *shifts, int Q,
               int T, int diag, int level, void *stream);
int uh_hoisted_mac_km(uh_ctx *ctx, uint64_t *acc, const uint64_t *X, int xls, const uint64_t *D, const uint64_t *km,
                      const int32_t *shifts, int B, int I, int T, int diag, int level, void *stream);

/* Tensor-core variant of uh_hoisted_mac_bank for dense masked layers with 5..48
 * outputs and <= 256 terms (LeNet conv2, the CIFAR-shape convs; layers.py:134-197):
 * the weight-mask contraction runs as byte-split u8 IMMA (exact; residues identical
 * to uh_hoisted_mac_bank) on the 40-bit limbs (5-byte operands), every output in
 * one pass; q_0 and P run 8-byte IMMA when both are below 2^60, else the IMAD
 * kernel from `masks` (<= 12 outputs per launch).  `ib` is the A-fragment mask bank
 * made once per layer by uh_imma_mask_bank from the uint64 mask bank
 * (uh_imma_bank_words uint32 words).  uh_imma_supported: 1 when the shape and the
 * chain (40-bit q_1..q_level, 60-bit q_0 and P) qualify. */
int uh_imma_supported(uh_ctx *ctx, int level, int O, int Q);
unsigned long long uh_imma_bank_words(uh_ctx *ctx, int level, int O, int Q);
int uh_imma_mask_bank(uh_ctx *ctx, uint32_t *ib, const uint64_t *masks, int O, int Q, int level, void *stream);
int uh_hoisted_mac_imma(uh_ctx *ctx, uint64_t *acc, const uint64_t *X, int xls, const uint64_t *D,
                        const uint64_t *masks, const uint32_t *ib, const uint64_t *kbank, const int32_t *shifts,
                        int B, int I, int T, int O, int level, void *stream);
/* uh_hoisted_mac_imma with the key switch of every term (phase A) on the tensor cores as well
 * (40-bit limbs; layers.conv's rotate + key switch, layers.py:165-196 via he_backend.rotate,
 * he_backend.py:249-253): the ModUp digits split into bytes, the byte weight 2^(8a) folded into
 * the Galois key (again 5 bytes), so one u8 m16n8k32 per (term, coefficient, component) forms the
 * key inner product of 16 ciphertexts; exact, residues identical to uh_hoisted_mac_imma.
 * `kt` is the per-layer key bank in fragment order made once by uh_imma_ta_bank from the key
 * bank (uh_imma_ta_bank_bytes bytes).  uh_imma_ta_supported: the uh_imma_supported shapes with
 * 5 * (level + 1) <= 32 and Q <= 128 (LeNet conv2). */
int uh_imma_ta_supported(uh_ctx *ctx, int level, int O, int Q);
unsigned long long uh_imma_ta_bank_bytes(uh_ctx *ctx, int level, int T);
int uh_imma_ta_bank(uh_ctx *ctx, uint8_t *kt, const uint64_t *kbank, const int32_t *shifts, int T, int level,
                    void *stream);
int uh_hoisted_mac_imma_ta(uh_ctx *ctx, uint64_t *acc, const uint64_t *X, int xls, const uint64_t *D,
                           const uint32_t *ib, const uint8_t *kt, const uint64_t *kbank, const int32_t *shifts,
                           int B, int I, int T, int O, int level, void *stream);
/* Same hoisted MAC (layers.conv, layers.py:165-196) with the weight-mask contraction of
 * every limb on the 5th-generation tensor cores: tcgen05.mma kind::i8 with TMEM
 * accumulators, byte-split operands (5 bytes on the 40-bit limbs, 8 on q_0 and P; exact,
 * residues identical to uh_hoisted_mac_bank).  `bank` is the A-operand bank made once
 * per layer by uh_tc_mask_bank from the uint64 mask bank [O][Q][level+2][N]
 * (uh_tc_bank_bytes bytes); uh_tc_supported: 1 when N = 2^15, the chain has 40-bit
 * q_1..q_level and 60-bit q_0, P, 1 <= O <= 12 and Q <= 128. */
int uh_tc_supported(uh_ctx *ctx, int level, int O, int Q);
unsigned long long uh_tc_bank_bytes(uh_ctx *ctx, int level, int O, int Q);
int uh_tc_mask_bank(uh_ctx *ctx, uint8_t *bank, const uint64_t *masks, int O, int Q, int level, void *stream);
int uh_hoisted_mac_tc(uh_ctx *ctx, uint64_t *acc, const uint64_t *X, int xls, const uint64_t *D,
                      const uint8_t *bank, const uint64_t *kbank, const int32_t *shifts, int B, int I, int T, int O,
                      int level, void *stream);
/* Hoisted rotation sum (layers.avgpool, layers.py:213-218): out[C][B][2][level+2][N]
 * = sum_t P * rot_t(ct_c) in the QP basis; ModDown gives the pooled ciphertexts. */
int uh_rot_sum_hoisted(uh_ctx *ctx, uint64_t *out, const uint64_t *X, int xls, const uint64_t *D,
                       const uint64_t *const *keys, const int32_t *key_limbs, const int32_t *shifts, int B, int C,
                       int T, int level, void *stream);

#ifdef __cplusplus
}
#endif
#endif
