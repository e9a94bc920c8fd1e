// Shared device primitives of the B200 RNS-CKKS engine (sm_100a).
//
// 64-bit modular arithmetic built from 32-bit IMAD: every prime is < 2^62,
// residues are canonical in [0, q) in memory, products are formed as 128-bit
// values (IMAD.WIDE.U32 partial products) and reduced with
//   * Shoup multiplication when one operand is a precomputed constant
//     (NTT twiddles, q_l^-1, P^-1, 2^64 mod q), and
//   * a 128-bit -> [0,q) reduction (`reduce128`) for variable x variable
//     products, which also closes lazily accumulated multiply-add chains
//     (key-switching inner products, plaintext-weight MACs).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace uh {

typedef unsigned __int128 u128;

// Per-modulus constants (device resident, one entry per RNS prime).
struct Mod {
    uint64_t q;      // the prime, q < 2^62
    uint64_t bar;    // floor(2^64 / q)
    uint64_t r64;    // 2^64 mod q
    uint64_t r64s;   // Shoup companion of r64: floor(r64 * 2^64 / q)
    uint64_t ninv;   // N^-1 mod q
    uint64_t ninvs;  // Shoup companion
    uint64_t pad0, pad1;
};

// high 64 bits of a 64x64 product as an explicit 32-bit carry chain (ptxas turns
// it into IMAD.WIDE.U32 with carry-in/out; ~1.5x the throughput of __umul64hi
// in the microbenchmarks of microbench.cu)
__device__ __forceinline__ uint64_t mulhi(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("{\n\t.reg .u32 a0,a1,b0,b1,t0,t1,t2;\n\t"
        "mov.b64 {a0,a1}, %1;\n\tmov.b64 {b0,b1}, %2;\n\t"
        "mul.hi.u32 t0, a0, b0;\n\t"
        "mad.lo.cc.u32 t0, a0, b1, t0;\n\tmadc.hi.u32 t1, a0, b1, 0;\n\t"
        "mad.lo.cc.u32 t0, a1, b0, t0;\n\tmadc.hi.cc.u32 t1, a1, b0, t1;\n\taddc.u32 t2, 0, 0;\n\t"
        "mad.lo.cc.u32 t1, a1, b1, t1;\n\tmadc.hi.u32 t2, a1, b1, t2;\n\t"
        "mov.b64 %0, {t1,t2};\n\t}"
        : "=l"(r)
        : "l"(a), "l"(b));
    return r;
}

// Shoup: x * w mod q for any x < 2^64, given ws = floor(w * 2^64 / q); result in [0, 2q).
__device__ __forceinline__ uint64_t shoup_lazy(uint64_t x, uint64_t w, uint64_t ws, uint64_t q) {
    uint64_t qh = mulhi(x, ws);
    return x * w - qh * q;
}
__device__ __forceinline__ uint64_t csub(uint64_t x, uint64_t q) { return x >= q ? x - q : x; }
__device__ __forceinline__ uint64_t shoup(uint64_t x, uint64_t w, uint64_t ws, uint64_t q) {
    return csub(shoup_lazy(x, w, ws, q), q);
}
// x mod q within [0, 2q) for any x < 2^64.
__device__ __forceinline__ uint64_t barrett_lite(uint64_t x, const Mod &m) {
    return x - mulhi(x, m.bar) * m.q;
}
// (hi * 2^64 + lo) mod q, canonical.
__device__ __forceinline__ uint64_t reduce128(uint64_t hi, uint64_t lo, const Mod &m) {
    uint64_t s = shoup_lazy(hi, m.r64, m.r64s, m.q) + barrett_lite(lo, m);  // < 4q < 2^64
    s = s >= 2 * m.q ? s - 2 * m.q : s;
    return csub(s, m.q);
}
__device__ __forceinline__ uint64_t mulmod(uint64_t a, uint64_t b, const Mod &m) {
    return reduce128(mulhi(a, b), a * b, m);
}
__device__ __forceinline__ uint64_t addmod(uint64_t a, uint64_t b, uint64_t q) { return csub(a + b, q); }
__device__ __forceinline__ uint64_t submod(uint64_t a, uint64_t b, uint64_t q) { return a >= b ? a - b : a + q - b; }

// (hi:lo) += x * y  (mod 2^128) as a 32-bit multi-precision carry chain;
// ptxas fuses it into four IMAD.WIDE.U32 with carry-in/out.
__device__ __forceinline__ void mac128(uint64_t &lo, uint64_t &hi, uint64_t x, uint64_t y) {
    asm("{\n\t.reg .u32 x0,x1,y0,y1,a0,a1,a2,a3;\n\t"
        "mov.b64 {x0,x1}, %2;\n\tmov.b64 {y0,y1}, %3;\n\t"
        "mov.b64 {a0,a1}, %0;\n\tmov.b64 {a2,a3}, %1;\n\t"
        "mad.lo.cc.u32 a0, x0, y0, a0;\n\tmadc.hi.cc.u32 a1, x0, y0, a1;\n\t"
        "madc.lo.cc.u32 a2, x1, y1, a2;\n\tmadc.hi.u32 a3, x1, y1, a3;\n\t"
        "mad.lo.cc.u32 a1, x0, y1, a1;\n\tmadc.hi.cc.u32 a2, x0, y1, a2;\n\taddc.u32 a3, a3, 0;\n\t"
        "mad.lo.cc.u32 a1, x1, y0, a1;\n\tmadc.hi.cc.u32 a2, x1, y0, a2;\n\taddc.u32 a3, a3, 0;\n\t"
        "mov.b64 %0, {a0,a1};\n\tmov.b64 %1, {a2,a3};\n\t}"
        : "+l"(lo), "+l"(hi)
        : "l"(x), "l"(y));
}

// (a3:a2:a1:a0) += x * y on four 32-bit registers.  Ordered so every 64-bit
// IMAD.WIDE works on an aligned register pair (a0:a1, a2:a3, t0:t1): the two
// "diagonal" partial products accumulate in place, the cross products are
// summed separately and added with one carry chain -- no register shuffles.
__device__ __forceinline__ void mac128x4(uint32_t &a0, uint32_t &a1, uint32_t &a2, uint32_t &a3, uint64_t x,
                                         uint64_t y) {
    asm("{\n\t.reg .u32 x0,x1,y0,y1,t0,t1,t2;\n\t"
        "mov.b64 {x0,x1}, %4;\n\tmov.b64 {y0,y1}, %5;\n\t"
        "mad.lo.cc.u32 %0, x0, y0, %0;\n\tmadc.hi.cc.u32 %1, x0, y0, %1;\n\t"
        "madc.lo.cc.u32 %2, x1, y1, %2;\n\tmadc.hi.u32 %3, x1, y1, %3;\n\t"
        "mul.lo.u32 t0, x0, y1;\n\tmul.hi.u32 t1, x0, y1;\n\t"
        "mad.lo.cc.u32 t0, x1, y0, t0;\n\tmadc.hi.cc.u32 t1, x1, y0, t1;\n\taddc.u32 t2, 0, 0;\n\t"
        "add.cc.u32 %1, %1, t0;\n\taddc.cc.u32 %2, %2, t1;\n\taddc.u32 %3, %3, t2;\n\t}"
        : "+r"(a0), "+r"(a1), "+r"(a2), "+r"(a3)
        : "l"(x), "l"(y));
}

// Narrow-operand accumulator for limbs with q < 2^41: both factors below 2^42,
// so their high 32-bit words x1, y1 are below 2^10.  The 128-bit sum is kept in
// two 64-bit words, value = a + b * 2^32:
//   a = sum x0*y0 mod 2^64,
//   b = sum (x0*y1 + x1*y0) + 2^32 * sum (x1*y1 + carry out of a)
//     (< 2^43 + 2^52 + 2^32 per term: exact for up to 2^11 terms between folds).
// One multiply-accumulate is three IMAD.WIDE.U32 (one with carry-out) and one
// IMAD.X into b's high word -- against four IMAD.WIDE.U32 plus a carry chain for
// full 64-bit operands -- in the same four registers.
struct AccN {
    uint64_t a, b;
    __device__ __forceinline__ void zero() { a = b = 0; }
    __device__ __forceinline__ void mac(uint64_t x, uint64_t y) {
        asm("{\n\t.reg .u32 x0,x1,y0,y1,a0,a1,b0,b1;\n\t"
            "mov.b64 {x0,x1}, %2;\n\tmov.b64 {y0,y1}, %3;\n\tmov.b64 {a0,a1}, %0;\n\tmov.b64 {b0,b1}, %1;\n\t"
            "mad.lo.cc.u32 a0, x0, y0, a0;\n\tmadc.hi.cc.u32 a1, x0, y0, a1;\n\tmadc.lo.u32 b1, x1, y1, b1;\n\t"
            "mov.b64 %0, {a0,a1};\n\tmov.b64 %1, {b0,b1};\n\t"
            "mad.wide.u32 %1, x0, y1, %1;\n\tmad.wide.u32 %1, x1, y0, %1;\n\t}"
            : "+l"(a), "+l"(b)
            : "l"(x), "l"(y));
    }
    __device__ __forceinline__ void add(uint64_t x) {  // any 64-bit addend
        asm("{\n\t.reg .u32 x0,x1,a0,a1,b0,b1;\n\t"
            "mov.b64 {x0,x1}, %2;\n\tmov.b64 {a0,a1}, %0;\n\tmov.b64 {b0,b1}, %1;\n\t"
            "add.cc.u32 a0, a0, x0;\n\taddc.cc.u32 a1, a1, x1;\n\taddc.u32 b1, b1, 0;\n\t"
            "mov.b64 %0, {a0,a1};\n\tmov.b64 %1, {b0,b1};\n\t}"
            : "+l"(a), "+l"(b)
            : "l"(x));
    }
    // the 128-bit value as (hi, lo)
    __device__ __forceinline__ void value(uint64_t &hi, uint64_t &lo) const {
        lo = a + (b << 32);
        hi = (b >> 32) + (lo < a);
    }
    __device__ __forceinline__ uint64_t lo64() const { return a + (b << 32); }
    __device__ __forceinline__ uint64_t hi64() const {
        uint64_t h, l;
        value(h, l);
        return h;
    }
    __device__ __forceinline__ void set(uint64_t l, uint64_t h) {  // callers only set values below 2^96
        a = l;
        b = h << 32;
    }
    __device__ __forceinline__ uint64_t reduce(const Mod &m) const {
        uint64_t h, l;
        value(h, l);
        return reduce128(h, l, m);
    }
};

// Split accumulator: A = sum x0*y0 + (x1*y1 << 64) (a0..a3) and C = sum of the
// cross products x0*y1 + x1*y0 (c0:c1, carries counted in c2); value = A + (C << 32).
// Every IMAD.WIDE accumulates into an aligned register pair in place (no moves).
struct AccS {
    uint32_t a0, a1, a2, a3, c0, c1, c2;
    __device__ __forceinline__ void zero() { a0 = a1 = a2 = a3 = c0 = c1 = c2 = 0; }
    __device__ __forceinline__ void mac(uint64_t x, uint64_t y) {
        asm("{\n\t.reg .u32 x0,x1,y0,y1;\n\t"
            "mov.b64 {x0,x1}, %7;\n\tmov.b64 {y0,y1}, %8;\n\t"
            "mad.lo.cc.u32 %0, x0, y0, %0;\n\tmadc.hi.cc.u32 %1, x0, y0, %1;\n\t"
            "madc.lo.cc.u32 %2, x1, y1, %2;\n\tmadc.hi.u32 %3, x1, y1, %3;\n\t"
            "mad.lo.cc.u32 %4, x0, y1, %4;\n\tmadc.hi.cc.u32 %5, x0, y1, %5;\n\taddc.u32 %6, %6, 0;\n\t"
            "mad.lo.cc.u32 %4, x1, y0, %4;\n\tmadc.hi.cc.u32 %5, x1, y0, %5;\n\taddc.u32 %6, %6, 0;\n\t}"
            : "+r"(a0), "+r"(a1), "+r"(a2), "+r"(a3), "+r"(c0), "+r"(c1), "+r"(c2)
            : "l"(x), "l"(y));
    }
    __device__ __forceinline__ void add(uint64_t x) {
        asm("add.cc.u32 %0, %0, %4;\n\taddc.cc.u32 %1, %1, %5;\n\taddc.cc.u32 %2, %2, 0;\n\taddc.u32 %3, %3, 0;"
            : "+r"(a0), "+r"(a1), "+r"(a2), "+r"(a3)
            : "r"((uint32_t)x), "r"((uint32_t)(x >> 32)));
    }
    // fold C into A: (a3:a2:a1:a0) += (c2:c1:c0) << 32
    __device__ __forceinline__ void fold() {
        asm("add.cc.u32 %0, %0, %3;\n\taddc.cc.u32 %1, %1, %4;\n\taddc.u32 %2, %2, %5;"
            : "+r"(a1), "+r"(a2), "+r"(a3)
            : "r"(c0), "r"(c1), "r"(c2));
        c0 = c1 = c2 = 0;
    }
    __device__ __forceinline__ uint64_t lo64() { fold(); return ((uint64_t)a1 << 32) | a0; }
    __device__ __forceinline__ uint64_t hi64() { fold(); return ((uint64_t)a3 << 32) | a2; }
    __device__ __forceinline__ void set(uint64_t lo, uint64_t hi) {
        a0 = (uint32_t)lo; a1 = (uint32_t)(lo >> 32); a2 = (uint32_t)hi; a3 = (uint32_t)(hi >> 32);
        c0 = c1 = c2 = 0;
    }
};

// 128-bit accumulator for lazy multiply-add chains.
#ifndef UH_ACC32
// Two 64-bit halves: the register allocator keeps each half in an aligned register
// pair, so the in-place IMAD.WIDE.U32 accumulations need no register shuffles.
__device__ __forceinline__ void mac128p(uint64_t &lo, uint64_t &hi, uint64_t x, uint64_t y) {
    asm("{\n\t.reg .u32 x0,x1,y0,y1,l0,l1,h0,h1,t0,t1,t2;\n\t"
        "mov.b64 {x0,x1}, %2;\n\tmov.b64 {y0,y1}, %3;\n\t"
        "mov.b64 {l0,l1}, %0;\n\tmov.b64 {h0,h1}, %1;\n\t"
        "mad.lo.cc.u32 l0, x0, y0, l0;\n\tmadc.hi.cc.u32 l1, x0, y0, l1;\n\t"
        "madc.lo.cc.u32 h0, x1, y1, h0;\n\tmadc.hi.u32 h1, x1, y1, h1;\n\t"
        "mul.lo.u32 t0, x0, y1;\n\tmul.hi.u32 t1, x0, y1;\n\t"
        "mad.lo.cc.u32 t0, x1, y0, t0;\n\tmadc.hi.cc.u32 t1, x1, y0, t1;\n\taddc.u32 t2, 0, 0;\n\t"
        "add.cc.u32 l1, l1, t0;\n\taddc.cc.u32 h0, h0, t1;\n\taddc.u32 h1, h1, t2;\n\t"
        "mov.b64 %0, {l0,l1};\n\tmov.b64 %1, {h0,h1};\n\t}"
        : "+l"(lo), "+l"(hi)
        : "l"(x), "l"(y));
}
struct Acc {
    uint64_t lo, hi;
    __device__ __forceinline__ void zero() { lo = hi = 0; }
    __device__ __forceinline__ void mac(uint64_t a, uint64_t b) { mac128p(lo, hi, a, b); }
    __device__ __forceinline__ uint64_t lo64() const { return lo; }
    __device__ __forceinline__ uint64_t hi64() const { return hi; }
    __device__ __forceinline__ uint32_t hi32lo() const { return (uint32_t)hi; }  // bits 64..95
    __device__ __forceinline__ void set(uint64_t l, uint64_t h) { lo = l; hi = h; }
    __device__ __forceinline__ void mac_c(uint64_t a, uint64_t b) {  // plain-C reference form
        uint64_t pl = a * b, ph = mulhi(a, b);
        lo += pl;
        hi += ph + (lo < pl);
    }
    __device__ __forceinline__ void add(uint64_t a) {
        asm("{\n\t.reg .u32 a0,a1,l0,l1,h0,h1;\n\t"
            "mov.b64 {a0,a1}, %2;\n\tmov.b64 {l0,l1}, %0;\n\tmov.b64 {h0,h1}, %1;\n\t"
            "add.cc.u32 l0, l0, a0;\n\taddc.cc.u32 l1, l1, a1;\n\taddc.cc.u32 h0, h0, 0;\n\taddc.u32 h1, h1, 0;\n\t"
            "mov.b64 %0, {l0,l1};\n\tmov.b64 %1, {h0,h1};\n\t}"
            : "+l"(lo), "+l"(hi)
            : "l"(a));
    }
    __device__ __forceinline__ uint64_t reduce(const Mod &m) const { return reduce128(hi, lo, m); }
    __device__ __forceinline__ void value(uint64_t &h, uint64_t &l) const { h = hi; l = lo; }
};
#else
// four 32-bit words (previous form, UH_ACC32)
struct Acc {
    uint32_t w0, w1, w2, w3;
    __device__ __forceinline__ void zero() { w0 = w1 = w2 = w3 = 0; }
    __device__ __forceinline__ void mac(uint64_t a, uint64_t b) { mac128x4(w0, w1, w2, w3, a, b); }
    __device__ __forceinline__ uint64_t lo64() const { return ((uint64_t)w1 << 32) | w0; }
    __device__ __forceinline__ uint64_t hi64() const { return ((uint64_t)w3 << 32) | w2; }
    __device__ __forceinline__ uint32_t hi32lo() const { return w2; }
    __device__ __forceinline__ void set(uint64_t lo, uint64_t hi) {
        w0 = (uint32_t)lo; w1 = (uint32_t)(lo >> 32); w2 = (uint32_t)hi; w3 = (uint32_t)(hi >> 32);
    }
    __device__ __forceinline__ void mac_c(uint64_t a, uint64_t b) {  // plain-C reference form
        uint64_t lo = lo64(), hi = hi64();
        uint64_t pl = a * b, ph = mulhi(a, b);
        lo += pl;
        hi += ph + (lo < pl);
        set(lo, hi);
    }
    __device__ __forceinline__ void add(uint64_t a) {
        asm("add.cc.u32 %0, %0, %4;\n\taddc.cc.u32 %1, %1, %5;\n\taddc.cc.u32 %2, %2, 0;\n\taddc.u32 %3, %3, 0;"
            : "+r"(w0), "+r"(w1), "+r"(w2), "+r"(w3)
            : "r"((uint32_t)a), "r"((uint32_t)(a >> 32)));
    }
    __device__ __forceinline__ uint64_t reduce(const Mod &m) const { return reduce128(hi64(), lo64(), m); }
};
#endif

// Centred lift of x in [0, p) reduced into q: x > (p-1)/2 represents x - p.
__device__ __forceinline__ uint64_t centred_to(uint64_t x, uint64_t p, const Mod &mq) {
    if (x > (p - 1) / 2) {
        uint64_t neg = p - x;  // in (0, p/2]
        uint64_t r = neg < mq.q ? neg : csub(barrett_lite(neg, mq), mq.q);
        return r == 0 ? 0 : mq.q - r;
    }
    return x < mq.q ? x : csub(barrett_lite(x, mq), mq.q);
}

// -- counter-based RNG (bit-identical to oracle/ckks_oracle.c) ---------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t rng_stream(uint64_t seed, uint64_t tag, uint64_t a, uint64_t b) {
    return mix64(mix64(mix64(mix64(seed) ^ tag) ^ a) ^ b);
}
__device__ __forceinline__ uint64_t rng_draw(uint64_t stream, uint64_t i) { return mix64(stream ^ mix64(i)); }

enum : uint64_t { TAG_SECRET = 1, TAG_ENC_A = 2, TAG_ENC_E = 3, TAG_KSK_A = 4, TAG_KSK_E = 5 };

// limb index -> modulus index for a basis of `nq` q-limbs (moduli base..base+nq-1)
// optionally followed by P (modulus index sp).
__device__ __forceinline__ int limb_mod(int k, int nq, int base, int sp) { return k < nq ? base + k : sp; }

}  // namespace uh
