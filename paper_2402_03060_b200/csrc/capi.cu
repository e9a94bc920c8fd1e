// extern "C" entry points (include/unihenn_b200.h): argument checks, error
// capture into a thread-local string, dispatch to the engine.
#include <cstdio>
#include <string>
#include "../../include/unihenn_b200.h"
#include "ntt_fast.cuh"
#include "ops.cuh"

struct uh_ctx {
    uh::Ctx *c;
};

namespace uh {
std::atomic<unsigned long long> g_launch_count{0};
}

namespace {
thread_local std::string g_err;

template <class F> int guard(F &&f) {
    try {
        f();
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) {
            g_err = std::string("CUDA: ") + cudaGetErrorString(e);
            return 2;
        }
        return 0;
    } catch (const std::exception &ex) {
        g_err = ex.what();
        return 1;
    } catch (...) {
        g_err = "unknown error";
        return 1;
    }
}
inline cudaStream_t S(void *s) { return reinterpret_cast<cudaStream_t>(s); }
inline const uh::Ctx &C(uh_ctx *x) {
    if (!x || !x->c) throw std::invalid_argument("null context");
    return *x->c;
}
void need(bool ok, const char *msg) {
    if (!ok) throw std::invalid_argument(msg);
}
void check_level(const uh::Ctx &c, int level) {
    need(level >= 0 && level <= (int)c.count - 2, "level out of range for this modulus chain");
}
}  // namespace

extern "C" {

__attribute__((visibility("default"))) int uh_abi_version(void) { return 1; }
__attribute__((visibility("default"))) unsigned long long uh_launch_count(void) {
    return uh::g_launch_count.load(std::memory_order_relaxed);
}
__attribute__((visibility("default"))) int uh_bench_peaks(uh_ctx *ctx, double *rates) {
    return guard([&] { uh::bench_peaks(C(ctx), rates); });
}
__attribute__((visibility("default"))) const char *uh_last_error(void) { return g_err.c_str(); }

__attribute__((visibility("default"))) int uh_ctx_create(uh_ctx **out, uint32_t n, const uint64_t *moduli,
                                                         const uint64_t *psi, uint32_t count, int device) {
    return guard([&] {
        need(out && moduli && psi, "null argument");
        uh_ctx *x = new uh_ctx;
        try {
            x->c = uh::ctx_create(n, moduli, psi, count, device);
        } catch (...) {
            delete x;
            throw;
        }
        *out = x;
    });
}

__attribute__((visibility("default"))) int uh_ctx_destroy(uh_ctx *ctx) {
    return guard([&] {
        if (!ctx) return;
        uh::ctx_destroy(ctx->c);
        delete ctx;
    });
}

__attribute__((visibility("default"))) int uh_ntt(uh_ctx *ctx, uint64_t *data, int n_polys, int nl, int nq,
                                                  int pstride, int inverse, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        need(nq >= 0 && nq <= nl && nq <= (int)c.count - 1 && nl - nq <= 1 && pstride >= nl, "bad basis");
        if (inverse)
            uh::ntt_inverse(c, data, n_polys, nl, nq, 0, pstride, S(stream));
        else
            uh::ntt_forward(c, data, n_polys, nl, nq, 0, pstride, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_elementwise(uh_ctx *ctx, int op, uint64_t *out, const uint64_t *a,
                                                          const uint64_t *b, int n_polys, int b_polys, int nl, int nq,
                                                          int out_ps, int a_ps, int b_ps, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        need(op >= 0 && op <= 5, "bad op");
        need(nq >= 0 && nq <= nl && nl - nq <= 1 && nq <= (int)c.count - 1, "bad basis");
        uh::elementwise(c, op, out, a, b, n_polys, b_polys, nl, nq, out_ps, a_ps, b_ps, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_elementwise_grouped(uh_ctx *ctx, int op, uint64_t *out, const uint64_t *a,
                                                                  const uint64_t *b, int n_polys, int b_polys,
                                                                  int group, int nl, int nq, int out_ps, int a_ps,
                                                                  int b_ps, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        need(op >= 0 && op <= 5, "bad op");
        need(b_polys >= 1 && group >= 1, "bad broadcast");
        need(nq >= 0 && nq <= nl && nl - nq <= 1 && nq <= (int)c.count - 1, "bad basis");
        uh::elementwise_grouped(c, op, out, a, b, n_polys, b_polys, group, nl, nq, out_ps, a_ps, b_ps, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_divide_top(uh_ctx *ctx, uint64_t *out, const uint64_t *in, int n_polys,
                                                         int nl, int top_mod, int out_ps, int in_ps, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        need(top_mod >= nl && top_mod < (int)c.count && nl >= 0, "bad top modulus");
        uh::divide_top(c, out, in, n_polys, nl, top_mod, out_ps, in_ps, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_divide_top2(uh_ctx *ctx, uint64_t *out, const uint64_t *in,
                                                          int n_polys, int level, int out_ps, int in_ps,
                                                          void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        need(level >= 1, "fused ModDown + rescale needs level >= 1");
        need(out != in, "out of place");
        uh::divide_top2(c, out, in, n_polys, level, out_ps, in_ps, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_divide_top2_bias_supported(uh_ctx *ctx) {
    return ctx && uh::ntt_fast_supported(C(ctx)) ? 1 : 0;
}

__attribute__((visibility("default"))) int uh_divide_top2_bias(uh_ctx *ctx, uint64_t *out, const uint64_t *in,
                                                               int n_polys, int level, int out_ps, int in_ps,
                                                               const uint64_t *bias, int bias_group, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        need(level >= 1, "fused ModDown + rescale needs level >= 1");
        need(out != in, "out of place");
        need(bias != nullptr && bias_group >= 2 && bias_group % 2 == 0 && n_polys % bias_group == 0,
             "bias rows cover whole (c0, c1) pairs: even bias_group dividing n_polys");
        uh::divide_top2(c, out, in, n_polys, level, out_ps, in_ps, S(stream), bias, bias_group);
    });
}

__attribute__((visibility("default"))) int uh_rescale(uh_ctx *ctx, uint64_t *out, const uint64_t *in, int B,
                                                      int level, int out_ls, int in_ls, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        need(level >= 1, "rescale needs level >= 1");
        uh::ct_rescale(c, out, in, B, level, out_ls, in_ls, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_modup(uh_ctx *ctx, uint64_t *D, const uint64_t *in, int n_polys,
                                                    int level, int in_ps, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        uh::modup(c, D, in, n_polys, level, in_ps, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_key_inner(uh_ctx *ctx, uint64_t *u, const uint64_t *D,
                                                        const uint64_t *key, int key_limbs, int n_polys, int level,
                                                        int64_t r, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        need(key_limbs >= level + 2, "key truncated below the requested level");
        uh::key_inner(c, u, D, key, key_limbs, n_polys, level, r, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_keyswitch(uh_ctx *ctx, uint64_t *out, const uint64_t *d, int n_polys,
                                                        int level, int d_ps, const uint64_t *key, int key_limbs,
                                                        void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        need(key_limbs >= level + 2, "key truncated below the requested level");
        uh::keyswitch(c, out, d, n_polys, level, d_ps, key, key_limbs, 0, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_rotate_hoisted(uh_ctx *ctx, uint64_t *out, const uint64_t *in,
                                                             const uint64_t *D, int B, int level, int out_ls,
                                                             int in_ls, const uint64_t *key, int key_limbs, int64_t r,
                                                             void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        need(out != in, "rotate is out of place");
        int64_t half = c.n / 2;
        bool zero = ((r % half) + half) % half == 0;
        need(zero || key_limbs >= level + 2, "key truncated below the requested level");
        uh::ct_rotate_hoisted(c, out, in, D, B, level, out_ls, in_ls, key, key_limbs, r, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_rotate(uh_ctx *ctx, uint64_t *out, const uint64_t *in, int B, int level,
                                                     int out_ls, int in_ls, const uint64_t *key, int key_limbs,
                                                     int64_t r, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        need(out != in, "rotate is out of place");
        int64_t half = c.n / 2;
        bool zero = ((r % half) + half) % half == 0;
        need(zero || key_limbs >= level + 2, "key truncated below the requested level");
        uh::ct_rotate(c, out, in, B, level, out_ls, in_ls, key, key_limbs, r, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_mul_plain_rescale(uh_ctx *ctx, uint64_t *out, const uint64_t *ct,
                                                                const uint64_t *pt, int B, int level, int out_ls,
                                                                int ct_ls, int pt_ls, int pt_batched, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        need(level >= 1, "no multiplication budget left");
        uh::ct_mul_plain_rescale(c, out, ct, pt, B, level, out_ls, ct_ls, pt_ls, pt_batched, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_mul_relin_rescale(uh_ctx *ctx, uint64_t *out, const uint64_t *a,
                                                                const uint64_t *b, int B, int level, int out_ls,
                                                                int a_ls, int b_ls, const uint64_t *rk, int rk_limbs,
                                                                void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        need(level >= 1, "no multiplication budget left");
        need(rk_limbs >= level + 2, "relinearisation key truncated below the requested level");
        uh::ct_mul_relin_rescale(c, out, a, b, B, level, out_ls, a_ls, b_ls, rk, rk_limbs, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_mul_relin_rescale_fused(uh_ctx *ctx, uint64_t *out, const uint64_t *a,
                                                                      const uint64_t *b, int B, int level, int out_ls,
                                                                      int a_ls, int b_ls, const uint64_t *rk,
                                                                      int rk_limbs, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        need(level >= 1, "no multiplication budget left");
        need(rk_limbs >= level + 2, "relinearisation key truncated below the requested level");
        uh::ct_mul_relin_rescale_fused(c, out, a, b, B, level, out_ls, a_ls, b_ls, rk, rk_limbs, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_secret_gen(uh_ctx *ctx, uint64_t *s_eval, uint64_t seed, void *stream) {
    return guard([&] { uh::secret_gen(C(ctx), s_eval, seed, S(stream)); });
}

__attribute__((visibility("default"))) int uh_galois_keygen(uh_ctx *ctx, uint64_t *key, const uint64_t *s_eval,
                                                            uint64_t seed, int64_t r, int level, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        uh::galois_keygen(c, key, s_eval, seed, r, level, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_relin_keygen(uh_ctx *ctx, uint64_t *key, const uint64_t *s_eval,
                                                           uint64_t seed, int level, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        uh::relin_keygen(c, key, s_eval, seed, level, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_encrypt(uh_ctx *ctx, uint64_t *out, const uint64_t *pt,
                                                      const uint64_t *s_eval, int B, int level, int out_ls, int pt_ls,
                                                      uint64_t seed, uint64_t ct_id0, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        uh::encrypt(c, out, pt, s_eval, B, level, out_ls, pt_ls, seed, ct_id0, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_decrypt_coeffs(uh_ctx *ctx, double *out, const uint64_t *ct,
                                                             const uint64_t *s_eval, int B, int ct_ls, void *stream) {
    return guard([&] { uh::decrypt_coeffs(C(ctx), out, ct, s_eval, B, ct_ls, S(stream)); });
}

__attribute__((visibility("default"))) int uh_encode_coeffs(uh_ctx *ctx, int64_t *coef, const double *slots,
                                                            int n_polys, double scale, void *stream) {
    return guard([&] { uh::encode_coeffs(C(ctx), coef, slots, n_polys, scale, S(stream)); });
}

__attribute__((visibility("default"))) int uh_from_signed(uh_ctx *ctx, uint64_t *out, const int64_t *coef,
                                                          int n_polys, int nl, int out_ps, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        need(nl >= 1 && nl <= (int)c.count - 1, "bad limb count");
        uh::from_signed(c, out, coef, n_polys, nl, 0, out_ps, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_from_signed_qp(uh_ctx *ctx, uint64_t *out, const int64_t *coef,
                                                             int n_polys, int nq, int out_ps, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        need(nq >= 1 && nq <= (int)c.count - 1, "bad limb count");
        uh::from_signed(c, out, coef, n_polys, nq, 1, out_ps, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_conv_hoisted_mac(uh_ctx *ctx, uint64_t *acc, const uint64_t *X, int xls,
                                                               const uint64_t *D, const uint64_t *masks,
                                                               const uint64_t *const *keys, const int32_t *key_limbs,
                                                               const int32_t *shifts, int B, int I, int T, int O,
                                                               int level, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        need(B > 0 && I > 0 && T > 0 && O > 0 && xls >= level + 1, "bad shape");
        uh::hoisted_mac(c, acc, X, xls, D, masks, keys, key_limbs, shifts, B, I, T, O, 0, level, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_rot_sum_hoisted(uh_ctx *ctx, uint64_t *out, const uint64_t *X, int xls,
                                                              const uint64_t *D, const uint64_t *const *keys,
                                                              const int32_t *key_limbs, const int32_t *shifts, int B,
                                                              int C_, int T, int level, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        need(B > 0 && C_ > 0 && T > 0 && xls >= level + 1, "bad shape");
        // channels ride the batch dimension, no masks: out[ch][b] = sum_t P * rot_t(ct[ch][b])
        uh::hoisted_mac(c, out, X, xls, D, nullptr, keys, key_limbs, shifts, C_ * B, 1, T, 1, 0, level, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_hoisted_mac(uh_ctx *ctx, uint64_t *acc, const uint64_t *X, int xls,
                                                          const uint64_t *D, const uint64_t *masks,
                                                          const uint64_t *const *keys, const int32_t *key_limbs,
                                                          const int32_t *shifts, int B, int I, int T, int O, int diag,
                                                          int level, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        need(B > 0 && I > 0 && T > 0 && O > 0 && xls >= level + 1, "bad shape");
        need(diag >= 0 && diag <= 2, "term mode must be 0 (dense), 1 (diagonal) or 2 (block-diagonal)");
        need(diag != 1 || I == T, "diagonal terms need I == T");
        uh::hoisted_mac(c, acc, X, xls, D, masks, keys, key_limbs, shifts, B, I, T, O, diag, level, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_hoisted_bank_supported(uh_ctx *ctx, int level, int O) {
    return ctx && uh::hoisted_bank_supported(C(ctx), level, O) ? 1 : 0;
}

__attribute__((visibility("default"))) int uh_hoisted_mac_bank(uh_ctx *ctx, uint64_t *acc, const uint64_t *X, int xls,
                                                               const uint64_t *D, const uint64_t *masks,
                                                               const uint64_t *kbank, const int32_t *shifts, int B,
                                                               int I, int T, int O, int diag, int level,
                                                               void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        need(B > 0 && I > 0 && T > 0 && O > 0 && xls == level + 1, "bad shape (xls must equal level + 1)");
        need(diag >= 0 && diag <= 2, "term mode must be 0 (dense), 1 (diagonal) or 2 (block-diagonal)");
        need(diag != 1 || I == T, "diagonal terms need I == T");
        need(diag != 2 || O <= 4, "block-diagonal terms are supported for up to 4 outputs");
        need(kbank != nullptr, "key bank is required");
        uh::hoisted_mac_bank(c, acc, X, D, masks, kbank, shifts, B, I, T, O, diag, level, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_km_supported(uh_ctx *ctx, int level) {
    return ctx && uh::hoisted_bank_supported(C(ctx), level, 1) ? 1 : 0;
}

__attribute__((visibility("default"))) int uh_km_bank(uh_ctx *ctx, uint64_t *km, const uint64_t *masks,
                                                      const uint64_t *kbank, const int32_t *shifts, int Q, int T,
                                                      int diag, int level, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        need(Q > 0 && T > 0 && diag >= 0 && diag <= 2, "bad shape");
        need(km && masks && kbank && shifts, "null operand");
        uh::km_bank(c, km, masks, kbank, shifts, Q, T, diag, level, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_hoisted_mac_km(uh_ctx *ctx, uint64_t *acc, const uint64_t *X, int xls,
                                                             const uint64_t *D, const uint64_t *km,
                                                             const int32_t *shifts, int B, int I, int T, int diag,
                                                             int level, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        need(B > 0 && I > 0 && T > 0 && xls == level + 1, "bad shape (xls must equal level + 1)");
        need(diag >= 0 && diag <= 2, "term mode must be 0 (dense), 1 (diagonal) or 2 (block-diagonal)");
        need(km != nullptr, "key-mask bank is required");
        uh::hoisted_mac_km(c, acc, X, D, km, shifts, B, I, T, diag, level, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_imma_supported(uh_ctx *ctx, int level, int O, int Q) {
    return ctx && uh::hoisted_imma_supported(C(ctx), level, O, Q) ? 1 : 0;
}

__attribute__((visibility("default"))) unsigned long long uh_imma_bank_words(uh_ctx *ctx, int level, int O, int Q) {
    return ctx && uh::hoisted_imma_supported(C(ctx), level, O, Q) ? uh::imma_bank_words(C(ctx), level, O, Q) : 0ull;
}

__attribute__((visibility("default"))) int uh_imma_mask_bank(uh_ctx *ctx, uint32_t *ib, const uint64_t *masks, int O,
                                                             int Q, int level, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        need(uh::hoisted_imma_supported(c, level, O, Q), "IMMA mask bank: unsupported shape");
        uh::imma_mask_bank(c, ib, masks, O, Q, level, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_hoisted_mac_imma(uh_ctx *ctx, uint64_t *acc, const uint64_t *X, int xls,
                                                               const uint64_t *D, const uint64_t *masks,
                                                               const uint32_t *ib, const uint64_t *kbank,
                                                               const int32_t *shifts, int B, int I, int T, int O,
                                                               int level, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        need(B > 0 && I > 0 && T > 0 && O > 0 && xls == level + 1, "bad shape (xls must equal level + 1)");
        need(kbank != nullptr && ib != nullptr && masks != nullptr, "key bank, IMMA mask bank and masks are required");
        uh::hoisted_mac_imma(c, acc, X, D, masks, ib, kbank, shifts, B, I, T, O, level, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_imma_ta_supported(uh_ctx *ctx, int level, int O, int Q) {
    return ctx && uh::hoisted_imma_ta_supported(C(ctx), level, O, Q) ? 1 : 0;
}

__attribute__((visibility("default"))) unsigned long long uh_imma_ta_bank_bytes(uh_ctx *ctx, int level, int T) {
    return ctx && level >= 1 && T >= 1 ? uh::imma_ta_bank_bytes(C(ctx), level, T) : 0ull;
}

__attribute__((visibility("default"))) int uh_imma_ta_bank(uh_ctx *ctx, uint8_t *kt, const uint64_t *kbank,
                                                           const int32_t *shifts, int T, int level, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        need(kt && kbank && shifts && T > 0, "null operand");
        need(5 * (level + 1) <= 32, "tensor-core phase A needs level + 1 <= 6");
        uh::imma_ta_bank(c, kt, kbank, shifts, T, level, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_hoisted_mac_imma_ta(uh_ctx *ctx, uint64_t *acc, const uint64_t *X,
                                                                  int xls, const uint64_t *D, const uint32_t *ib,
                                                                  const uint8_t *kt, const uint64_t *kbank,
                                                                  const int32_t *shifts, int B, int I, int T, int O,
                                                                  int level, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        need(B > 0 && I > 0 && T > 0 && O > 0 && xls == level + 1, "bad shape (xls must equal level + 1)");
        need(kbank != nullptr && ib != nullptr && kt != nullptr, "key bank, IMMA mask bank and tensor key bank are required");
        uh::hoisted_mac_imma_ta(c, acc, X, D, ib, kt, kbank, shifts, B, I, T, O, level, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_tc_supported(uh_ctx *ctx, int level, int O, int Q) {
    return ctx && uh::hoisted_tc_supported(C(ctx), level, O, Q) ? 1 : 0;
}

__attribute__((visibility("default"))) unsigned long long uh_tc_bank_bytes(uh_ctx *ctx, int level, int O, int Q) {
    return ctx && uh::hoisted_tc_supported(C(ctx), level, O, Q) ? uh::tc_bank_bytes(C(ctx), level, O, Q) : 0ull;
}

__attribute__((visibility("default"))) int uh_tc_mask_bank(uh_ctx *ctx, uint8_t *bank, const uint64_t *masks, int O,
                                                           int Q, int level, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        need(uh::hoisted_tc_supported(c, level, O, Q), "tensor-core mask bank: unsupported shape");
        uh::tc_mask_bank(c, bank, masks, O, Q, level, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_hoisted_mac_tc(uh_ctx *ctx, uint64_t *acc, const uint64_t *X, int xls,
                                                             const uint64_t *D, const uint8_t *bank,
                                                             const uint64_t *kbank, const int32_t *shifts, int B,
                                                             int I, int T, int O, int level, void *stream) {
    return guard([&] {
        const uh::Ctx &c = C(ctx);
        check_level(c, level);
        need(B > 0 && I > 0 && T > 0 && O > 0 && xls == level + 1, "bad shape (xls must equal level + 1)");
        need(kbank != nullptr && bank != nullptr, "key bank and tensor-core mask bank are required");
        uh::hoisted_mac_tc(c, acc, X, D, bank, kbank, shifts, B, I, T, O, level, S(stream));
    });
}

__attribute__((visibility("default"))) int uh_decode_coeffs(uh_ctx *ctx, double *slots, const double *coef,
                                                            int n_polys, double scale, void *stream) {
    return guard([&] { uh::decode_coeffs(C(ctx), slots, coef, n_polys, scale, S(stream)); });
}

}  // extern "C"
