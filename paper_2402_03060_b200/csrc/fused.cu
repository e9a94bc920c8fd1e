// Fused layer entry points on top of the generic hoisted rotation-MAC kernel
// (hoist.cu).
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
//      basis on the fly and immediately multiply-accumulates it with every
//      output channel's plaintext weight mask (lazily, in 128 bits),
//   3. leaves one ModDown (and one rescale) per output channel to the caller.
// Nothing per-rotation ever touches HBM.
#include "ops.cuh"

namespace uh {

void conv_hoisted_mac(const Ctx &c, uint64_t *acc, const uint64_t *X, int xls, const uint64_t *D,
                      const uint64_t *masks, const uint64_t *const *keys, const int32_t *key_limbs,
                      const int32_t *shifts, int B, int I, int T, int O, int level, cudaStream_t s) {
    hoisted_mac(c, acc, X, xls, D, masks, keys, key_limbs, shifts, B, I, T, O, 0, level, s);
}

// average pooling: every channel independently (channels ride the batch
// dimension), no masks: out[ch][b] = sum_t P * rot_t(ct[ch][b]).
void rot_sum_hoisted(const Ctx &c, uint64_t *out, const uint64_t *X, int xls, const uint64_t *D,
                     const uint64_t *const *keys, const int32_t *key_limbs, const int32_t *shifts, int B, int C,
                     int T, int level, cudaStream_t s) {
    hoisted_mac(c, out, X, xls, D, nullptr, keys, key_limbs, shifts, C * B, 1, T, 1, 0, level, s);
}

}  // namespace uh
