// Register-tiled two-pass negacyclic NTT for N >= 2^13 (sm_100a).
//
// N = N1 * N2 viewed as an N1 x N2 row-major matrix.
//   pass 1: a CTA owns 32 columns (lane <-> column: every global access is a
//           256-byte coalesced row segment); the first log2(N1) Cooley-Tukey
//           stages run as two register-resident radix-2^a sub-networks with one
//           shared-memory exchange in between.
//   pass 2: a CTA owns 4096/N2 contiguous N2-blocks; the remaining log2(N2)
//           stages again run as two register radix sub-networks around one
//           (bank-conflict-padded) shared-memory exchange; the epilogue
//           reduces to [0, q) and scatters to slot order.
// Butterflies are Harvey's lazy ones (values in [0, 4q) forward, [0, 2q)
// inverse; every prime is < 2^62) with Shoup twiddles read as interleaved
// (w, w') 16-byte pairs.  The inverse mirrors both passes (Gentleman-Sande).
//
// Load / store transforms are fused into the passes, so no extra HBM round
// trip is needed for:
//   mode PLAIN  -- strided limbs in, strided limbs out (in place allowed);
//   mode MODUP  -- ModUp: limb (p, j, k) loads centred(C[p][j], q_j) mod q_k;
//   mode DIVIDE -- rescale / ModDown: limb (p, k) loads centred(top[p], q_top)
//                  mod q_k and the epilogue writes (in[p][k] - y) * q_top^-1.
#include "ntt_fast.cuh"

#ifndef UH_NTT_P1_LOADS_FIRST
#define UH_NTT_P1_LOADS_FIRST 1
#endif
#ifndef UH_NTT_P2_WARPSYNC
#define UH_NTT_P2_WARPSYNC 1  // N2 = 256: the pass-2 exchange is warp-local (0.306 vs 0.310 us/limb forward)
#endif
#ifndef UH_NTT_KP
#define UH_NTT_KP 0
#endif
#ifndef UH_NTT_MINB
#define UH_NTT_MINB 4  // min resident CTAs per SM requested from ptxas (register cap: 64)
#endif
#ifndef UH_NTT_P2_MINB
#define UH_NTT_P2_MINB UH_NTT_MINB  // the same for pass 2 (forward) / pass A (inverse)
#endif

namespace uh {
namespace {

constexpr int kThreads = 256;

struct LimbInfo {
    int mod;
    int mode;
    const uint64_t *src;
    uint64_t qsrc;  // 0: plain load, else centred lift from modulus qsrc
    uint64_t *dst;
    const uint64_t *in;  // DIVIDE / DIVIDE2
    uint64_t w, ws;      // DIVIDE: q_top^-1 mod q_k (Shoup pair)
    // DIVIDE2
    const uint64_t *src2;
    uint64_t w2, ws2;     // P^-1 mod q_k
    uint64_t P, qpk;      // P, (q_top * P) mod q_k
    ulonglong2 pinv;      // P^-1 mod q_top (Shoup pair)
    ulonglong2 pk;        // P mod q_k (Shoup pair)
    Mod mt;               // the top modulus
    const uint64_t *bias; // DIVIDE2: row added to the result (c0 polynomials), or null
};

__device__ __forceinline__ int job_limb(const NttJob &J, int i) { return i; }

__device__ __forceinline__ LimbInfo limb_info(const NttJob &J, int f, int logn, const Mod *__restrict__ mods) {
    LimbInfo li;
    li.mode = J.mode;
    li.qsrc = 0;
    li.in = nullptr;
    li.bias = nullptr;
    li.w = li.ws = 0;
    if (J.mode == NTT_DIVIDE2) {
        const int p = f / J.nl, k = f - p * J.nl;
        const int t = J.top_mod, sp = J.sp, cnt = J.count;
        const Mod m = mods[k];
        li.mod = k;
        li.src = J.src + ((size_t)(2 * p) << logn);
        li.src2 = li.src + ((size_t)1 << logn);
        li.qsrc = 1;
        li.dst = J.dst + (((size_t)p * J.dst_ps + k) << logn);
        li.in = J.in + (((size_t)p * J.in_ps + k) << logn);
        li.bias = J.bias && !(p & 1) ? J.bias + (((size_t)(p / J.bias_group) * J.nl + k) << logn) : nullptr;
        li.w = J.inv2[(size_t)k * cnt + t];  // (q_t P)^-1 mod q_k
        li.ws = J.inv2s[(size_t)k * cnt + t];
        li.mt = mods[t];
        li.P = mods[sp].q;
        li.pk = J.pmod[k];
        const uint64_t qtk = li.mt.q < m.q ? li.mt.q : csub(barrett_lite(li.mt.q, m), m.q);
        li.qpk = mulmod(qtk, li.pk.x, m);
        return li;
    }
    if (J.mode == NTT_MODUP) {
        // limbs (p, j, k) with k != j (the diagonal limb D_j[j] is the input limb itself: copied, not transformed)
        const int LP = J.L + 1;
        const int kk = f % J.L, pj = f / J.L, j = pj % J.L;
        const int k = kk + (kk >= j);
        li.mod = limb_mod(k, J.L, 0, J.sp);
        li.src = J.src + ((size_t)pj << logn);
        li.qsrc = mods[j].q;
        li.dst = J.dst + (((size_t)pj * LP + k) << logn);
    } else {
        const int p = f / J.nl, k = f - p * J.nl;
        li.mod = limb_mod(k, J.nq, J.base, J.sp);
        li.dst = J.dst + (((size_t)p * J.dst_ps + k) << logn);
        if (J.mode == NTT_DIVIDE) {
            li.src = J.src + ((size_t)p << logn);
            li.qsrc = mods[J.top_mod].q;
            li.in = J.in + (((size_t)p * J.in_ps + k) << logn);
            li.w = J.inv[(size_t)k * J.count + J.top_mod];
            li.ws = J.invs[(size_t)k * J.count + J.top_mod];
        } else {
            li.src = J.src + (((size_t)p * J.src_ps + k) << logn);
        }
    }
    return li;
}

// centred CRT lift reduced into q_k: a = y | neg << 63 (x = b + P y, y in [0, q_t), prepared
// once per coefficient by ops.cu k_crt2_pre), b = x mod P
__device__ __forceinline__ uint64_t crt2_to(uint64_t a, uint64_t b, const LimbInfo &li, const Mod &m) {
    const bool neg = a >> 63;
    const uint64_t y = a & 0x7FFFFFFFFFFFFFFFull;
    const uint64_t yk = y < m.q ? y : csub(barrett_lite(y, m), m.q);
    const uint64_t bk = b < m.q ? b : csub(barrett_lite(b, m), m.q);
    const uint64_t t = addmod(bk, shoup(yk, li.pk.x, li.pk.y, m.q), m.q);
    return neg ? submod(t, li.qpk, m.q) : t;
}

// Compile-time load transform of pass 1: 0 plain, 1 centred lift (ModUp / ModDown / rescale),
// 2 CRT pair (fused ModDown + rescale).  The centred lift is branch-free; the magnitude
// needs a reduction only when the source modulus exceeds twice the target (a 60-bit
// digit into a 40-bit limb), which is uniform per limb (`red`).
template <int LM>
__device__ __forceinline__ uint64_t load_t(const LimbInfo &li, size_t idx, const Mod &m, bool red) {
    if (LM == 2) return crt2_to(li.src[idx], li.src2[idx], li, m);
    const uint64_t x = li.src[idx];
    if (LM == 0) return x;
    const uint64_t p = li.qsrc;
    const bool neg = x > ((p - 1) >> 1);
    uint64_t v = neg ? p - x : x;
    if (red) v = csub(barrett_lite(v, m), m.q);
    const uint64_t nv = v ? m.q - v : 0;
    return neg ? nv : v;
}

// the transform of load_t on an already loaded word (LM 0 / 1)
template <int LM>
__device__ __forceinline__ uint64_t lift_t(uint64_t x, const LimbInfo &li, const Mod &m, bool red) {
    if (LM == 0) return x;
    const uint64_t p = li.qsrc;
    const bool neg = x > ((p - 1) >> 1);
    uint64_t v = neg ? p - x : x;
    if (red) v = csub(barrett_lite(v, m), m.q);
    const uint64_t nv = v ? m.q - v : 0;
    return neg ? nv : v;
}

// Harvey CT butterfly: x, y in [0, 4q) -> [0, 4q)
__device__ __forceinline__ void bf_ct(uint64_t &x, uint64_t &y, ulonglong2 w, uint64_t q) {
    uint64_t q2 = 2 * q;
    uint64_t u = x >= q2 ? x - q2 : x;
    uint64_t t = shoup_lazy(y, w.x, w.y, q);
    x = u + t;
    y = u - t + q2;
}
// Harvey GS butterfly: x, y in [0, 2q) -> [0, 2q)
__device__ __forceinline__ void bf_gs(uint64_t &x, uint64_t &y, ulonglong2 w, uint64_t q) {
    uint64_t q2 = 2 * q;
    uint64_t s = x + y;
    uint64_t d = x - y + q2;
    x = s >= q2 ? s - q2 : s;
    y = shoup_lazy(d, w.x, w.y, q);
}

// ---- FP64-pipe arithmetic for limbs with q < 2^42 ----
// Values are signed integers held exactly in doubles (|v| < 2^50).  Twiddles are
// (w, w / q) pairs.  y * w mod q (centred, |r| <= 0.51 q) is exact:
//   p = fl(y w), e = y w - p (one fma, exact), k = rint(y * (w / q)) (|k q - y w| <= 0.51 q),
//   r = (p - k q) + e, where p - k q is an integer below 2^53 (one fma, exact).
// A CT butterfly is 8 FP64 operations and no integer work; the 64-bit Shoup
// butterfly costs ~14 IMAD-pipe slots.  Magnitudes: forward 15 stages from [0, q)
// stay below 9q; inverse butterflies double the sum output, so the inverse reduces
// once between its passes (<= 2^8 q, then <= 2^7 q / 2).
constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52: fma(x, y, kMagic) - kMagic = rint(x * y)
constexpr double kTwo52 = 4503599627370496.0;
__device__ __forceinline__ double fmm(double y, double2 w, double q) {
    const double p = y * w.x;
    const double e = fma(y, w.x, -p);
#if UH_NTT_KP == 1   // quotient from the rounded product: no w / q operand (experiment)
    const double k = fma(p, 1.0 / q, kMagic) - kMagic;
#elif UH_NTT_KP == 2  // rint instruction instead of the magic-number pair
    const double k = rint(y * w.y);
#else
    const double k = fma(y, w.y, kMagic) - kMagic;
#endif
    return fma(-k, q, p) + e;
}
__device__ __forceinline__ void bf_ct(double &x, double &y, double2 w, double q) {
    const double t = fmm(y, w, q);
    const double u = x;
    x = u + t;
    y = u - t;
}
__device__ __forceinline__ void bf_gs(double &x, double &y, double2 w, double q) {
    const double s = x + y, d = x - y;
    x = s;
    y = fmm(d, w, q);
}
__device__ __forceinline__ double u2d(uint64_t x) {  // exact for x < 2^52
    return __longlong_as_double((long long)(x | 0x4330000000000000ull)) - kTwo52;
}
__device__ __forceinline__ double fred(double v, double q, double qinv) {  // centred: |result| <= q / 2 (+ tiny)
    const double k = fma(v, qinv, kMagic) - kMagic;
    return fma(-k, q, v);
}
__device__ __forceinline__ uint64_t d2u_canon(double v, double q, double qinv) {  // -> [0, q)
    double r = fred(v, q, qinv);
    r = r < 0 ? r + q : r;
    return (uint64_t)__double_as_longlong(r + kTwo52) ^ 0x4330000000000000ull;
}
__device__ __forceinline__ uint64_t reduce4q(uint64_t x, uint64_t q) {
    x = x >= 2 * q ? x - 2 * q : x;
    return x >= q ? x - q : x;
}
__device__ __forceinline__ ulonglong2 tw(const ulonglong2 *__restrict__ t, int i) { return __ldg(t + i); }
__device__ __forceinline__ double2 tw(const double2 *__restrict__ t, int i) { return __ldg(t + i); }

// value type of a limb's arithmetic: 64-bit integers (Shoup) or FP64
template <bool FP> struct Arith;
template <> struct Arith<false> {
    using V = uint64_t;
    using W = ulonglong2;
    uint64_t q;
    __device__ Arith(uint64_t q_) : q(q_) {}
    __device__ static V in(uint64_t x) { return x; }           // canonical residue -> V
    __device__ static V raw_in(uint64_t x) { return x; }       // stored word -> V
    __device__ static uint64_t raw(V v) { return v; }          // V -> stored word
    __device__ uint64_t canon(V v) const { return reduce4q(v, q); }
    __device__ uint64_t qv() const { return q; }
};
template <> struct Arith<true> {
    using V = double;
    using W = double2;
    double q, qinv;
    __device__ Arith(uint64_t q_) : q((double)q_), qinv(1.0 / (double)q_) {}
    __device__ static V in(uint64_t x) { return u2d(x); }
    __device__ static V raw_in(uint64_t x) { return __longlong_as_double((long long)x); }
    __device__ static uint64_t raw(V v) { return (uint64_t)__double_as_longlong(v); }
    __device__ uint64_t canon(V v) const { return d2u_canon(v, q, qinv); }
    __device__ double qv() const { return q; }
};
__device__ __forceinline__ bool fp_limb(uint64_t q) { return (q >> 42) == 0; }

// Twiddle accessors: (local stage m', index j) -> twiddle of global index m' * f + j.
template <typename W>
struct TwG {  // global table (read-only path)
    const W *__restrict__ T;
    int f;
    __device__ W operator()(int m, int j) const { return tw(T, m * f + j); }
};

// Composite pass-2 twiddles (FP64 limbs).  With m = 2^s, the pass-2 twiddle of global index
// m (n1 + blk) + j is psi^e, e = 2^(B-1-s) (1 + 2 brv_A(blk)) + 2^(logn-s) brv_s(j), which factors as
//   F[blk][s] * R[s][j]                          (first network, s < 4, j < 2^s)
//   F[blk][s] * U[s-4][u] * R[s-4][v]            (second network, j = u 2^(s-4) + v, u < 16)
// (context.cu builds F, U, R).  A thread holds its network's per-stage head H[s] (F, or F U: one
// product) in registers; the stage-s twiddles are H[s] (v = 0) and H[s] R[s'][v] -- one exact FP64
// product each -- instead of one N-word table read per twiddle (the L1 wavefronts and L2 latency
// that bounded pass 2).
struct TwC {
    const double2 *R;  // this modulus' 16 (R, R / q) pairs at (1 << s') - 1 + v, staged in shared memory
    double q, qinv;
};
__device__ __forceinline__ double2 tw_c(double h, int idx, const TwC &t) {  // h R[idx] (idx > 0)
    const double c = fmm(h, t.R[idx], t.q);
    return make_double2(c, c * t.qinv);
}
// one stage s of a forward / inverse network of R = 2^LR register values: distance R / 2^(s+1),
// butterfly x uses twiddle H[s] R[s][x / 2dx]
template <int LR, int S>
__device__ __forceinline__ void fwd_stage_c(double (&v)[1 << LR], double h, const TwC &t) {
    constexpr int R = 1 << LR, dx = R >> (S + 1);
#pragma unroll
    for (int jv = 0; jv < (1 << S); jv++) {  // one twiddle live at a time (register budget)
        const double2 w = jv ? tw_c(h, (1 << S) - 1 + jv, t) : make_double2(h, h * t.qinv);
#pragma unroll
        for (int k = 0; k < dx; k++) bf_ct(v[jv * 2 * dx + k], v[jv * 2 * dx + k + dx], w, t.q);
    }
}
template <int LR, int S>
__device__ __forceinline__ void inv_stage_c(double (&v)[1 << LR], double h, const TwC &t) {
    constexpr int R = 1 << LR, dx = R >> (S + 1);
#pragma unroll
    for (int jv = 0; jv < (1 << S); jv++) {
        const double2 w = jv ? tw_c(h, (1 << S) - 1 + jv, t) : make_double2(h, h * t.qinv);
#pragma unroll
        for (int k = 0; k < dx; k++) bf_gs(v[jv * 2 * dx + k], v[jv * 2 * dx + k + dx], w, t.q);
    }
}
// H(s): the stage-s head, formed right before the stage (one live double: register budget)
template <int LR, class HF>  // stages s = 0 .. LR-1 (LR <= 4)
__device__ __forceinline__ void fwd_net_c(double (&v)[1 << LR], const HF &H, const TwC &t) {
    fwd_stage_c<LR, 0>(v, H(0), t);
    if constexpr (LR > 1) fwd_stage_c<LR, 1>(v, H(1), t);
    if constexpr (LR > 2) fwd_stage_c<LR, 2>(v, H(2), t);
    if constexpr (LR > 3) fwd_stage_c<LR, 3>(v, H(3), t);
}
template <int LR, class HF>  // mirror: stages s = LR-1 .. 0
__device__ __forceinline__ void inv_net_c(double (&v)[1 << LR], const HF &H, const TwC &t) {
    if constexpr (LR > 3) inv_stage_c<LR, 3>(v, H(3), t);
    if constexpr (LR > 2) inv_stage_c<LR, 2>(v, H(2), t);
    if constexpr (LR > 1) inv_stage_c<LR, 1>(v, H(1), t);
    inv_stage_c<LR, 0>(v, H(0), t);
}
// per-thread stage heads: first network F[blk][s]; second network F[blk][4 + s] U[s][u]
struct Heads1 {
    const double *__restrict__ f;  // F + blk * 8
    __device__ double operator()(int s) const { return __ldg(f + s); }
};
struct Heads2 {
    const double *__restrict__ f;   // F + blk * 8 + 4
    const double2 *__restrict__ u;  // U + u
    double q;
    __device__ double operator()(int s) const { return fmm(__ldg(f + s), __ldg(u + s * 16), q); }
};

struct TwP2 {  // one FP64 limb's composite pass-2 tables (context.cu)
    const double *__restrict__ F;   // [n1][8]
    const double2 *__restrict__ U;  // [4][16]
    const double2 *__restrict__ R;  // [16]
};
struct TwTabs {  // every modulus' tables (Ctx::d_tfF / d_tfU / d_tfR, or the inverse ones)
    const double *F;
    const double2 *U, *R;
    __device__ TwP2 at(int mod, int n1) const {
        return TwP2{F + (size_t)mod * n1 * 8, U + (size_t)mod * 64, R + (size_t)mod * 16};
    }
};

// forward radix network on R register values (elements base + S*x), stages with
// distance dx = R/2 .. 1; twiddle (m, off(s) + x / (2 dx)), m = m0 * (1 << s)
template <int R, typename V, typename TA, typename Q>
__device__ __forceinline__ void fwd_strided(V (&v)[R], const TA &ta, int m0, int moff, Q q) {
    int m = m0, off = moff;
#pragma unroll
    for (int dx = R / 2; dx >= 1; dx >>= 1) {
#pragma unroll
        for (int x = 0; x < R; x++) {
            if (x & dx) continue;
            bf_ct(v[x], v[x + dx], ta(m, off + x / (2 * dx)), q);
        }
        m <<= 1;
        off <<= 1;
    }
}
template <int R, typename V, typename TA, typename Q>
__device__ __forceinline__ void inv_strided(V (&v)[R], const TA &ta, int mlast, int offlast, Q q) {
    // mirror of fwd_strided: distances 1 .. R/2, m halves each stage
    int m = mlast, off = offlast;
#pragma unroll
    for (int dx = 1; dx <= R / 2; dx <<= 1) {
#pragma unroll
        for (int x = 0; x < R; x++) {
            if (x & dx) continue;
            bf_gs(v[x], v[x + dx], ta(m, off + x / (2 * dx)), q);
        }
        m >>= 1;
        off >>= 1;
    }
}

struct Tw {  // both twiddle tables of one limb's modulus
    const ulonglong2 *i;
    const double2 *f;
};
template <bool FP> __device__ __forceinline__ const typename Arith<FP>::W *pick(const Tw &t);
template <> __device__ __forceinline__ const ulonglong2 *pick<false>(const Tw &t) { return t.i; }
template <> __device__ __forceinline__ const double2 *pick<true>(const Tw &t) { return t.f; }

// ---------------- pass 1 (columns), N1 = 2^A ----------------
template <int A>
struct P1 {
    static constexpr int N1 = 1 << A, A1 = (A + 1) / 2, A2 = A - A1;
    static constexpr int R1 = 1 << A1, S1 = 1 << A2, R2 = 1 << A2;
    static constexpr int GS = S1 * 32 / kThreads;  // strided groups per thread
    static constexpr int GC = R1 * 32 / kThreads;  // contiguous groups per thread
};

template <int A, int LM, bool FP>
__device__ __forceinline__ void fwd_p1_body(uint64_t *sm, const LimbInfo &li, const Mod &m, bool red,
                                            const Tw &tws, uint64_t *out, int n2, int col, int lane, int wq) {
    using C = P1<A>;
    using AR = Arith<FP>;
    using V = typename AR::V;
    const AR ar(m.q);
    const auto *T = pick<FP>(tws);
#pragma unroll
    for (int g = 0; g < C::GS; g++) {
        const int r0 = wq + 8 * g;  // < S1
        V v[C::R1];
#if UH_NTT_P1_LOADS_FIRST
        if constexpr (LM != 2) {
            // every row of the column is requested before the first lift / butterfly (left to itself the
            // compiler sinks the later loads between the butterflies, where each waits out its own latency)
            uint64_t raw[C::R1];
#pragma unroll
            for (int x = 0; x < C::R1; x++) raw[x] = li.src[(size_t)(r0 + C::S1 * x) * n2 + col];
            asm volatile("" ::: "memory");
#pragma unroll
            for (int x = 0; x < C::R1; x++) v[x] = AR::in(lift_t<LM>(raw[x], li, m, red));
        } else
#endif
        {
#pragma unroll
            for (int x = 0; x < C::R1; x++)
                v[x] = AR::in(load_t<LM>(li, (size_t)(r0 + C::S1 * x) * n2 + col, m, red));
        }
        fwd_strided<C::R1>(v, TwG<typename AR::W>{T, 1}, 1, 0, ar.qv());
#pragma unroll
        for (int x = 0; x < C::R1; x++) sm[(r0 + C::S1 * x) * 32 + lane] = AR::raw(v[x]);
    }
    __syncthreads();
#pragma unroll
    for (int g = 0; g < C::GC; g++) {
        const int grp = wq + 8 * g;  // < R1
        const int r0 = grp * C::R2;
        V v[C::R2];
#pragma unroll
        for (int z = 0; z < C::R2; z++) v[z] = AR::raw_in(sm[(r0 + z) * 32 + lane]);
        // stages m = R1 .. N1/2 on contiguous rows r0 + z: twiddle m + (r0 + z) / (2t)
        fwd_strided<C::R2>(v, TwG<typename AR::W>{T, 1}, C::R1, grp, ar.qv());
#pragma unroll
        for (int z = 0; z < C::R2; z++) out[(size_t)(r0 + z) * n2 + col] = AR::raw(v[z]);
    }
}

template <int A, int LM>
__global__ void __launch_bounds__(kThreads, UH_NTT_MINB) k_fwd_p1(NttJob J, uint64_t *__restrict__ tmp, int logn,
                                                    const Mod *__restrict__ mods,
                                                    const ulonglong2 *__restrict__ twd,
                                                    const double2 *__restrict__ twf) {
    __shared__ uint64_t sm[P1<A>::N1 * 32];
    const int f = job_limb(J, J.f0 + blockIdx.y), lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const int n2 = 1 << (logn - A);
    const int col = blockIdx.x * 32 + lane;
    const LimbInfo li = limb_info(J, f, logn, mods);
    const Mod m = mods[li.mod];
    const bool red = LM == 1 && ((li.qsrc - 1) >> 1) >= m.q;
    const Tw tws{twd + ((size_t)li.mod << logn), twf + ((size_t)li.mod << logn)};
    uint64_t *out = tmp + ((size_t)blockIdx.y << logn);
    if (fp_limb(m.q))
        fwd_p1_body<A, LM, true>(sm, li, m, red, tws, out, n2, col, lane, wq);
    else
        fwd_p1_body<A, LM, false>(sm, li, m, red, tws, out, n2, col, lane, wq);
}

template <int A, bool FP>
__device__ __forceinline__ void inv_pb_body(uint64_t *sm, const LimbInfo &li, const Mod &m, const Tw &tws,
                                            const uint64_t *in, int n2, int col, int lane, int wq) {
    using C = P1<A>;
    using AR = Arith<FP>;
    using V = typename AR::V;
    const AR ar(m.q);
    const auto *T = pick<FP>(tws);
#pragma unroll
    for (int g = 0; g < C::GC; g++) {
        const int grp = wq + 8 * g;
        const int r0 = grp * C::R2;
        V v[C::R2];
#pragma unroll
        for (int z = 0; z < C::R2; z++) v[z] = AR::raw_in(in[(size_t)(r0 + z) * n2 + col]);
        // mirror of the forward contiguous stages: last stage m = N1/2 with offset grp * (R2/2)
        inv_strided<C::R2>(v, TwG<typename AR::W>{T, 1}, C::N1 / 2, grp * (C::R2 / 2), ar.qv());
#pragma unroll
        for (int z = 0; z < C::R2; z++) sm[(r0 + z) * 32 + lane] = AR::raw(v[z]);
    }
    __syncthreads();
    double2 nf;
    if (FP) nf = make_double2((double)m.ninv, (double)m.ninv / (double)m.q);
#pragma unroll
    for (int g = 0; g < C::GS; g++) {
        const int r0 = wq + 8 * g;
        V v[C::R1];
#pragma unroll
        for (int x = 0; x < C::R1; x++) v[x] = AR::raw_in(sm[(r0 + C::S1 * x) * 32 + lane]);
        inv_strided<C::R1>(v, TwG<typename AR::W>{T, 1}, C::R1 / 2, 0, ar.qv());
#pragma unroll
        for (int x = 0; x < C::R1; x++) {
            uint64_t r;
            if constexpr (FP)
                r = ar.canon(fmm(v[x], nf, ar.q));
            else
                r = csub(shoup_lazy(v[x], m.ninv, m.ninvs, m.q), m.q);
            li.dst[(size_t)(r0 + C::S1 * x) * n2 + col] = r;
        }
    }
}


template <int A>
__global__ void __launch_bounds__(kThreads, UH_NTT_MINB) k_inv_pb(NttJob J, const uint64_t *__restrict__ tmp, int logn,
                                                    const Mod *__restrict__ mods,
                                                    const ulonglong2 *__restrict__ itwd,
                                                    const double2 *__restrict__ itwf) {
    __shared__ uint64_t sm[P1<A>::N1 * 32];
    const int f = job_limb(J, J.f0 + blockIdx.y), lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const int n2 = 1 << (logn - A);
    const int col = blockIdx.x * 32 + lane;
    const LimbInfo li = limb_info(J, f, logn, mods);
    const Mod m = mods[li.mod];
    const Tw tws{itwd + ((size_t)li.mod << logn), itwf + ((size_t)li.mod << logn)};
    const uint64_t *in = tmp + ((size_t)blockIdx.y << logn);
    if (fp_limb(m.q))
        inv_pb_body<A, true>(sm, li, m, tws, in, n2, col, lane, wq);
    else
        inv_pb_body<A, false>(sm, li, m, tws, in, n2, col, lane, wq);
}

// ---------------- pass 2 (contiguous blocks), N2 = 2^B ----------------
template <int B>
struct P2 {
    static constexpr int N2 = 1 << B, B2 = B - 4;
    static constexpr int R1 = 16, S = N2 / 16, R2 = 1 << B2;
    static constexpr int G = 4096 / N2;                  // blocks per CTA
    static constexpr int GC = (4096 / R2) / kThreads;    // contiguous groups per thread
    static constexpr int PAD = N2 + N2 / 16;             // padded block stride in shared memory
    __device__ static int at(int g, int c) { return g * PAD + c + (c >> 4); }
};

// Slot-order I/O of pass 2.  Block blk of the N1 x N2 view evaluates at the
// coset e0 * {x = 1 mod 2N/N2... }: its N2 outputs land on slots
// {h * N/2 + j0 + (N1/2) * v : v < N2} (one half h, one residue j0 mod N1/2).
// CTA x takes the G blocks with half h = x / (N1/(2G)) and residues
// j0 = (x mod N1/(2G)) * G + g, so its 4096 slots are G-long contiguous runs
// at stride N1/2: slot i of the CTA (i < 4096, increasing) is
//   h * N/2 + j_start + (i mod G) + (N1/2) * (i / G),
// and reading/writing them in that order is coalesced.  csl[slot] is the
// element index c of the slot inside its block (host table).
template <int B>
__device__ __forceinline__ size_t cta_slot(int i, int logn) {
    using C = P2<B>;
    const int n1 = 1 << (logn - B);
    const int per_half = (n1 / 2) / C::G;
    const int h = blockIdx.x / per_half, js = (blockIdx.x % per_half) * C::G;
    return ((size_t)h << (logn - 1)) + js + (i % C::G) + (size_t)(n1 / 2) * (i / C::G);
}


// pass-2 input: the pass-1 intermediate in global memory (two-pass NTT)
template <int B>
struct InGlobal {
    const uint64_t *in;
    __device__ uint64_t operator()(int blk, int c) const { return in[(size_t)blk * P2<B>::N2 + c]; }
};
template <int B, int EM>
__device__ __forceinline__ void fwd_p2_epilogue(const uint64_t *sm, const LimbInfo &li, uint64_t q,
                                                const uint8_t *__restrict__ csl, int logn, int tid);

// pass 2 forward stages: tmp (pass-1 output) -> canonical residues in shared memory
// FP64 limbs form their twiddles from the composite tables (TwC); the 60-bit limbs read
// interleaved Shoup pairs from the N-word table.
template <int B, bool FP>
__device__ __forceinline__ void fwd_p2_body(uint64_t *sm, const double2 *s_R, const TwP2 &tc, const Mod &m, const Tw &tw2,
                                            const InGlobal<B> &in, const int *sel, int n1, int tid) {
    using C = P2<B>;
    using AR = Arith<FP>;
    using V = typename AR::V;
    const AR ar(m.q);
    const auto *T = pick<FP>(tw2);
    auto acc = [&](int blk) { return TwG<typename AR::W>{T, n1 + blk}; };
    {
        const int g = tid / C::S, c0 = tid % C::S, blk = sel[g];
        V v[C::R1];
#pragma unroll
        for (int x = 0; x < C::R1; x++) v[x] = AR::raw_in(in(blk, c0 + C::S * x));
        // local stages m' = 1..8: global twiddle index m' * (n1 + blk) + x / (2 dx)
        if constexpr (FP) {
            fwd_net_c<4>(v, Heads1{tc.F + blk * 8}, TwC{s_R, ar.q, ar.qinv});
        } else {
            fwd_strided<C::R1>(v, acc(blk), 1, 0, ar.qv());
        }
#pragma unroll
        for (int x = 0; x < C::R1; x++) sm[C::at(g, c0 + C::S * x)] = AR::raw(v[x]);
    }
    // N2 = 256: both networks of a block run on the same 16 threads (tid / 16 == block), so the
    // exchange only needs the warp to agree
    if (UH_NTT_P2_WARPSYNC && B == 8)
        __syncwarp();
    else
        __syncthreads();
#pragma unroll
    for (int gi = 0; gi < C::GC; gi++) {
        const int grp = tid + kThreads * gi;
        const int per = C::N2 / C::R2;
        const int g = grp / per, c = (grp % per) * C::R2, blk = sel[g];
        V v[C::R2];
#pragma unroll
        for (int z = 0; z < C::R2; z++) v[z] = AR::raw_in(sm[C::at(g, c + z)]);
        // local stages m' = 16 .. N2/2 on contiguous c + z
        if constexpr (FP) {
            fwd_net_c<B - 4>(v, Heads2{tc.F + blk * 8 + 4, tc.U + c / C::R2, ar.q}, TwC{s_R, ar.q, ar.qinv});
        } else {
            fwd_strided<C::R2>(v, acc(blk), 16, (c / C::R2), ar.qv());
        }
#pragma unroll
        for (int z = 0; z < C::R2; z++) sm[C::at(g, c + z)] = ar.canon(v[z]);
    }
    __syncthreads();
}


template <int B>
constexpr size_t p2_smem() {  // the G padded block tiles
    return (size_t)P2<B>::G * P2<B>::PAD * 8;
}

template <int B, int EM>
__global__ void __launch_bounds__(kThreads, UH_NTT_P2_MINB) k_fwd_p2(NttJob J, const uint64_t *__restrict__ tmp, int logn,
                                                    const Mod *__restrict__ mods,
                                                    const ulonglong2 *__restrict__ twd,
                                                    const TwTabs tt,
                                                    const double2 *__restrict__ twf,
                                                    const int32_t *__restrict__ bsel,
                                                    const uint8_t *__restrict__ csl) {
    using C = P2<B>;
    extern __shared__ uint64_t dsm[];
    uint64_t *sm = dsm;
    const int f = job_limb(J, J.f0 + blockIdx.y), tid = threadIdx.x;
    const int n1 = 1 << (logn - B);
    const int *sel = bsel + blockIdx.x * C::G;
    const LimbInfo li = limb_info(J, f, logn, mods);
    const Mod m = mods[li.mod];
    const uint64_t q = m.q;
    const Tw tw2{twd + ((size_t)li.mod << logn), twf + ((size_t)li.mod << logn)};
    const InGlobal<B> in{tmp + ((size_t)blockIdx.y << logn)};
    __shared__ double2 s_R[16];  // the composite-twiddle roots of this limb's modulus
    if (fp_limb(q)) {
        const TwP2 tc = tt.at(li.mod, n1);
        if (tid < 16) s_R[tid] = __ldg(tc.R + tid);
        __syncthreads();
        fwd_p2_body<B, true>(sm, s_R, tc, m, tw2, in, sel, n1, tid);
    } else {
        fwd_p2_body<B, false>(sm, s_R, TwP2{}, m, tw2, in, sel, n1, tid);
    }
    fwd_p2_epilogue<B, EM>(sm, li, q, csl, logn, tid);
}

// coalesced slot-order epilogue: a thread's 16 slot-table (and DIVIDE input) loads are
// issued together, then the shared-memory gathers and the stores
template <int B, int EM>
__device__ __forceinline__ void fwd_p2_epilogue(const uint64_t *sm, const LimbInfo &li, uint64_t q,
                                                const uint8_t *__restrict__ csl, int logn, int tid) {
    using C = P2<B>;
    constexpr int E = EM ? 8 : 16;  // loads in flight per round (register budget)
#pragma unroll
    for (int e0 = 0; e0 < 4096 / kThreads; e0 += E) {
        int cs[E];
        uint64_t a[E];
#pragma unroll
        for (int e = 0; e < E; e++) {
            const size_t s = cta_slot<B>(tid + kThreads * (e0 + e), logn);
            cs[e] = __ldg(csl + s);
            if (EM != 0) a[e] = li.in[s];
        }
#pragma unroll
        for (int e = 0; e < E; e++) {
            const int i = tid + kThreads * (e0 + e);
            const size_t s = cta_slot<B>(i, logn);
            const uint64_t y = sm[C::at(i % C::G, cs[e])];
            if (EM == 1)
                li.dst[s] = csub(shoup_lazy(submod(a[e], y, q), li.w, li.ws, q), q);
            else if (EM == 2) {
                uint64_t r = shoup(submod(a[e], y, q), li.w, li.ws, q);
                if (li.bias) r = addmod(r, __ldg(li.bias + s), q);  // CTA-uniform
                li.dst[s] = r;
            }
            else
                li.dst[s] = y;
        }
    }
}


// inverse pass A stages: canonical residues in shared memory -> tmp (pass-B input)
template <int B, bool FP>
__device__ __forceinline__ void inv_pa_body(uint64_t *sm, const double2 *s_R, const TwP2 &tc, const Mod &m, const Tw &tw2,
                                            uint64_t *out, const int *sel, int n1, int tid) {
    using C = P2<B>;
    using AR = Arith<FP>;
    using V = typename AR::V;
    const AR ar(m.q);
    const auto *T = pick<FP>(tw2);
    auto acc = [&](int blk) { return TwG<typename AR::W>{T, n1 + blk}; };
#pragma unroll
    for (int gi = 0; gi < C::GC; gi++) {
        const int grp = tid + kThreads * gi;
        const int per = C::N2 / C::R2;
        const int g = grp / per, c = (grp % per) * C::R2, blk = sel[g];
        V v[C::R2];
#pragma unroll
        for (int z = 0; z < C::R2; z++) v[z] = AR::in(sm[C::at(g, c + z)]);
        // mirror of the forward contiguous stages: last local stage m' = N2/2
        if constexpr (FP) {
            inv_net_c<B - 4>(v, Heads2{tc.F + blk * 8 + 4, tc.U + c / C::R2, ar.q}, TwC{s_R, ar.q, ar.qinv});
        } else {
            inv_strided<C::R2>(v, acc(blk), C::N2 / 2, (c / C::R2) * (C::R2 / 2), ar.qv());
        }
#pragma unroll
        for (int z = 0; z < C::R2; z++) sm[C::at(g, c + z)] = AR::raw(v[z]);
    }
    if (UH_NTT_P2_WARPSYNC && B == 8)
        __syncwarp();
    else
        __syncthreads();
    {
        const int g = tid / C::S, c0 = tid % C::S, blk = sel[g];
        V v[C::R1];
#pragma unroll
        for (int x = 0; x < C::R1; x++) v[x] = AR::raw_in(sm[C::at(g, c0 + C::S * x)]);
        if constexpr (FP) {
            inv_net_c<4>(v, Heads1{tc.F + blk * 8}, TwC{s_R, ar.q, ar.qinv});
        } else {
            inv_strided<C::R1>(v, acc(blk), 8, 0, ar.qv());
        }
#pragma unroll
        for (int x = 0; x < C::R1; x++) {
            V r = v[x];
            if constexpr (FP) r = fred(r, ar.q, ar.qinv);  // bound the growth before pass B
            out[(size_t)blk * C::N2 + c0 + C::S * x] = AR::raw(r);
        }
    }
}


template <int B>
__global__ void __launch_bounds__(kThreads, UH_NTT_P2_MINB) k_inv_pa(NttJob J, uint64_t *__restrict__ tmp, int logn,
                                                    const Mod *__restrict__ mods,
                                                    const ulonglong2 *__restrict__ itwd,
                                                    const TwTabs tt,
                                                    const double2 *__restrict__ itwf,
                                                    const int32_t *__restrict__ bsel,
                                                    const uint8_t *__restrict__ csl) {
    using C = P2<B>;
    extern __shared__ uint64_t dsm[];
    uint64_t *sm = dsm;
    const int f = job_limb(J, J.f0 + blockIdx.y), tid = threadIdx.x;
    const int n1 = 1 << (logn - B);
    const int *sel = bsel + blockIdx.x * C::G;
    const LimbInfo li = limb_info(J, f, logn, mods);
    const Mod m = mods[li.mod];
    const Tw tw2{itwd + ((size_t)li.mod << logn), itwf + ((size_t)li.mod << logn)};
    const bool fp = fp_limb(m.q);
    __shared__ double2 s_R[16];  // the composite-twiddle roots of this limb's modulus
    if (fp && tid < 16) s_R[tid] = __ldg(tt.R + (size_t)li.mod * 16 + tid);
    // coalesced slot-order gather into the blocks' shared-memory tiles (plain limbs: the only
    // inverse mode); all of a thread's loads are issued before the shared-memory stores
    {
        constexpr int E = 4096 / kThreads;
        int cs[E];
        uint64_t a[E];
        uint64_t *dg = nullptr;  // ModUp diagonal D[p][k][k] (CTA-uniform)
        if (J.diag) {
            const int p = f / J.nl, k = f - p * J.nl;
            dg = J.diag + (((size_t)(p * J.nl + k) * (J.nl + 1) + k) << logn);
        }
#pragma unroll
        for (int e = 0; e < E; e++) {
            const size_t s = cta_slot<B>(tid + kThreads * e, logn);
            cs[e] = __ldg(csl + s);
            a[e] = li.src[s];
        }
        if (dg) {  // after every load is in flight (a store in the loop would wait for its load)
#pragma unroll
            for (int e = 0; e < E; e++) dg[cta_slot<B>(tid + kThreads * e, logn)] = a[e];
        }
#pragma unroll
        for (int e = 0; e < E; e++) sm[C::at((tid + kThreads * e) % C::G, cs[e])] = a[e];
    }
    __syncthreads();
    uint64_t *out = tmp + ((size_t)blockIdx.y << logn);
    if (fp)
        inv_pa_body<B, true>(sm, s_R, tt.at(li.mod, n1), m, tw2, out, sel, n1, tid);
    else
        inv_pa_body<B, false>(sm, s_R, TwP2{}, m, tw2, out, sel, n1, tid);
}

constexpr int kMaxGridY = 65535;

template <int A, int B>
void run_fwd(const Ctx &c, const NttJob &J0, int limbs, cudaStream_t s) {
    const int ch = std::min(limbs, kMaxGridY);
    Scratch tmp((size_t)ch * c.n * 8, s);
    uint64_t *t = tmp.as<uint64_t>();
    const int ln = (int)c.logn;
    constexpr size_t sm2 = p2_smem<B>();
    for (int f0 = 0; f0 < limbs; f0 += ch) {
        NttJob J = J0;
        J.f0 = f0;
        const int nl = std::min(ch, limbs - f0);
        dim3 g1((1u << B) / 32, nl), g2((1u << A) / P2<B>::G, nl);
        if (J.mode == NTT_PLAIN)
            k_fwd_p1<A, 0><<<g1, kThreads, 0, s>>>(J, t, ln, c.d_mods, c.d_tw2, c.d_twf);
        else if (J.mode == NTT_DIVIDE2)
            k_fwd_p1<A, 2><<<g1, kThreads, 0, s>>>(J, t, ln, c.d_mods, c.d_tw2, c.d_twf);
        else
            k_fwd_p1<A, 1><<<g1, kThreads, 0, s>>>(J, t, ln, c.d_mods, c.d_tw2, c.d_twf);
        UH_LAUNCH_CHECK();
        if (J.mode == NTT_DIVIDE) {
            smem_optin(k_fwd_p2<B, 1>, sm2);
            k_fwd_p2<B, 1><<<g2, kThreads, sm2, s>>>(J, t, ln, c.d_mods, c.d_tw2, TwTabs{c.d_tfF, c.d_tfU, c.d_tfR}, c.d_twf, c.d_bsel, c.d_csl);
        } else if (J.mode == NTT_DIVIDE2) {
            smem_optin(k_fwd_p2<B, 2>, sm2);
            k_fwd_p2<B, 2><<<g2, kThreads, sm2, s>>>(J, t, ln, c.d_mods, c.d_tw2, TwTabs{c.d_tfF, c.d_tfU, c.d_tfR}, c.d_twf, c.d_bsel, c.d_csl);
        } else {
            smem_optin(k_fwd_p2<B, 0>, sm2);
            k_fwd_p2<B, 0><<<g2, kThreads, sm2, s>>>(J, t, ln, c.d_mods, c.d_tw2, TwTabs{c.d_tfF, c.d_tfU, c.d_tfR}, c.d_twf, c.d_bsel, c.d_csl);
        }
        UH_LAUNCH_CHECK();
    }
}

template <int A, int B>
void run_inv(const Ctx &c, const NttJob &J0, int limbs, cudaStream_t s) {
    if (J0.mode != NTT_PLAIN) throw std::invalid_argument("inverse NTT: plain limbs only");
    const int ch = std::min(limbs, kMaxGridY);
    Scratch tmp((size_t)ch * c.n * 8, s);
    constexpr size_t sm2 = p2_smem<B>();
    smem_optin(k_inv_pa<B>, sm2);
    for (int f0 = 0; f0 < limbs; f0 += ch) {
        NttJob J = J0;
        J.f0 = f0;
        const int nl = std::min(ch, limbs - f0);
        dim3 g1((1u << B) / 32, nl), g2((1u << A) / P2<B>::G, nl);
        k_inv_pa<B><<<g2, kThreads, sm2, s>>>(J, tmp.as<uint64_t>(), (int)c.logn, c.d_mods, c.d_itw2,
                                              TwTabs{c.d_itfF, c.d_itfU, c.d_itfR}, c.d_itwf, c.d_bsel, c.d_csl);
        UH_LAUNCH_CHECK();
        k_inv_pb<A><<<g1, kThreads, 0, s>>>(J, tmp.as<uint64_t>(), (int)c.logn, c.d_mods, c.d_itw2, c.d_itwf);
        UH_LAUNCH_CHECK();
    }
}

}  // namespace

bool ntt_fast_supported(const Ctx &c) { return c.logn >= 13 && c.logn <= 15; }

void ntt_fast_forward(const Ctx &c, const NttJob &J, int limbs, cudaStream_t s) {
    if (limbs <= 0) return;
    switch (c.logn) {
        case 13: run_fwd<6, 7>(c, J, limbs, s); break;
        case 14: run_fwd<7, 7>(c, J, limbs, s); break;
        case 15: run_fwd<7, 8>(c, J, limbs, s); break;
        default: throw std::invalid_argument("fast NTT supports 2^13 <= N <= 2^15");
    }
}

void ntt_fast_inverse(const Ctx &c, const NttJob &J, int limbs, cudaStream_t s) {
    if (limbs <= 0) return;
    switch (c.logn) {
        case 13: run_inv<6, 7>(c, J, limbs, s); break;
        case 14: run_inv<7, 7>(c, J, limbs, s); break;
        case 15: run_inv<7, 8>(c, J, limbs, s); break;
        default: throw std::invalid_argument("fast NTT supports 2^13 <= N <= 2^15");
    }
}

}  // namespace uh
