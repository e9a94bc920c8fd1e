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

#ifndef UH_NTT_STAGE
#define UH_NTT_STAGE 0  // 1: pass-2 FP64 twiddles staged in shared memory (measured slower at 4 CTAs/SM)
#endif
#ifndef UH_NTT_TW8
#define UH_NTT_TW8 1  // pass-2 FP64 twiddles read as w only (8 B), w / q formed with one multiply
#endif
#ifndef UH_NTT_TWIST
#define UH_NTT_TWIST 0  // (opt-in, measured slower: 0.343 vs 0.313 us/limb) FP64 limbs: pass-2 blocks twisted by beta^c, shared twiddles W[0, N2/2) in shared memory
#endif
#ifndef UH_NTT_MINB
#define UH_NTT_MINB 4  // min resident CTAs per SM requested from ptxas (register cap: 64)
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
};

__device__ __forceinline__ int job_limb(const NttJob &J, int i) {
    if (!J.sel) return i;
    const int p = i / J.sel_cnt;
    return p * J.sel_T + (int)__ldg(J.sel + (i - p * J.sel_cnt));
}

__device__ __forceinline__ LimbInfo limb_info(const NttJob &J, int f, int logn, const Mod *__restrict__ mods) {
    LimbInfo li;
    li.mode = J.mode;
    li.qsrc = 0;
    li.in = nullptr;
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
    const double k = fma(y, w.y, kMagic) - kMagic;
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
struct TwGd {  // FP64 limbs, w-only global table: (w, w / q) with one multiply, half the bytes of TwG<double2>
    const double *__restrict__ T;
    int f;
    double qinv;
    __device__ double2 operator()(int m, int j) const {
        const double w = __ldg(T + m * f + j);
        return make_double2(w, w * qinv);
    }
};
#if UH_NTT_STAGE
struct TwS {  // FP64 limbs: w staged in shared memory at [m' + j] (m' + j < 256), w / q formed on the fly
    const double *t;
    double qinv;
    __device__ double2 operator()(int m, int j) const {
        const double w = t[m + j];
        return make_double2(w, w * qinv);
    }
};
#else
struct TwS {  // unused unless UH_NTT_STAGE
    const double *t;
    double qinv;
};
#endif

struct TwSh {  // twisted pass 2: every block uses the shared twiddles W[j] (staged as (w, w / q))
    const double2 *t;
    __device__ double2 operator()(int, int j) const { return t[j]; }
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

// centred lift of a canonical residue x mod p into q (as load_t<1>, from a register)
__device__ __forceinline__ uint64_t lift_reg(uint64_t x, uint64_t p, const Mod &m, bool red) {
    const bool neg = x > ((p - 1) >> 1);
    uint64_t v = neg ? p - x : x;
    if (red) v = csub(barrett_lite(v, m), m.q);
    const uint64_t nv = v ? m.q - v : 0;
    return neg ? nv : v;
}

template <int A, int LM, bool FP, bool OUT_SM = false>
__device__ __forceinline__ void fwd_p1_body(uint64_t *sm, const LimbInfo &li, const Mod &m, bool red,
                                            const Tw &tws, uint64_t *out, int n2, int col, int lane, int wq,
                                            const uint64_t *tile = nullptr) {
    using C = P1<A>;
    using AR = Arith<FP>;
    using V = typename AR::V;
    const AR ar(m.q);
    const auto *T = pick<FP>(tws);
#pragma unroll
    for (int g = 0; g < C::GS; g++) {
        const int r0 = wq + 8 * g;  // < S1
        V v[C::R1];
#pragma unroll
        for (int x = 0; x < C::R1; x++)
            v[x] = AR::in(tile ? lift_reg(tile[(r0 + C::S1 * x) * 32 + lane], li.qsrc, m, red)  // ModUp from a
                                                                                                // coefficient tile
                               : load_t<LM>(li, (size_t)(r0 + C::S1 * x) * n2 + col, m, red));
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
        for (int z = 0; z < C::R2; z++) {
            if constexpr (OUT_SM)  // cluster-fused NTT: the column tile stays in this CTA's shared memory
                sm[(r0 + z) * 32 + lane] = AR::raw(v[z]);
            else
                out[(size_t)(r0 + z) * n2 + col] = AR::raw(v[z]);
        }
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
                                            const uint64_t *in, int n2, int col, int lane, int wq,
                                            uint64_t *tile = nullptr) {
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
            if (tile)
                tile[(r0 + C::S1 * x) * 32 + lane] = r;
            else
                li.dst[(size_t)(r0 + C::S1 * x) * n2 + col] = r;
        }
    }
}

#ifndef UH_MODUP_MINB
#define UH_MODUP_MINB 3
#endif
// ModUp with the inverse NTT's last pass and the forward NTTs' first pass fused: CTA (column
// block, poly p x digit j) finishes the inverse transform of digit j into a coefficient tile in
// shared memory and runs forward pass 1 of every target limb k != j from that tile (centred
// lift of q_j into q_k in the load) -- the coefficient-form digits never go through HBM, and
// the L forward pass-1 loads of a digit become shared-memory reads.
template <int A>
__global__ void __launch_bounds__(kThreads, UH_MODUP_MINB) k_modup_pbp1(NttJob Ji, NttJob Jf, const uint64_t *__restrict__ ti,
                                                       uint64_t *__restrict__ tf, int logn,
                                                       const Mod *__restrict__ mods,
                                                       const ulonglong2 *__restrict__ itwd,
                                                       const double2 *__restrict__ itwf,
                                                       const ulonglong2 *__restrict__ twd,
                                                       const double2 *__restrict__ twf) {
    extern __shared__ uint64_t msm[];
    uint64_t *sm = msm, *tile = msm + P1<A>::N1 * 32;
    const int pj = blockIdx.y, lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const int n2 = 1 << (logn - A);
    const int col = blockIdx.x * 32 + lane;
    {
        const LimbInfo li = limb_info(Ji, pj, logn, mods);
        const Mod m = mods[li.mod];
        const Tw tws{itwd + ((size_t)li.mod << logn), itwf + ((size_t)li.mod << logn)};
        const uint64_t *in = ti + ((size_t)pj << logn);
        if (fp_limb(m.q))
            inv_pb_body<A, true>(sm, li, m, tws, in, n2, col, lane, wq, tile);
        else
            inv_pb_body<A, false>(sm, li, m, tws, in, n2, col, lane, wq, tile);
    }
    const int L = Jf.L;
#pragma unroll 1
    for (int kk = 0; kk < L; kk++) {
        __syncthreads();  // tile complete / previous target done with the exchange buffer
        const int f = pj * L + kk;
        const LimbInfo li = limb_info(Jf, f, logn, mods);
        const Mod m = mods[li.mod];
        const bool red = ((li.qsrc - 1) >> 1) >= m.q;
        const Tw tws{twd + ((size_t)li.mod << logn), twf + ((size_t)li.mod << logn)};
        uint64_t *out = tf + ((size_t)f << logn);
        if (fp_limb(m.q))
            fwd_p1_body<A, 1, true>(sm, li, m, red, tws, out, n2, col, lane, wq, tile);
        else
            fwd_p1_body<A, 1, false>(sm, li, m, red, tws, out, n2, col, lane, wq, tile);
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

// FP64 limbs: stage the pass-2 twiddles of the CTA's G blocks in shared memory (w only,
// coalesced runs: stage m' of block blk uses T[m' (n1 + blk) + j], j < m'), so the
// butterflies read them at shared-memory latency instead of L2 latency.
template <int B>
__device__ __forceinline__ void stage_twiddles(double *tws, const double *__restrict__ Tw, const int *sel, int n1,
                                               int tid) {
    using C = P2<B>;
    static_assert(kThreads % C::N2 == 0, "a thread keeps one in-block index r");
    const int r = tid & (C::N2 - 1);  // the same for all of this thread's entries
    if (r == 0) return;
    const int mp = 1 << (31 - __clz(r)), j = r - mp;
    const double *src = Tw + j;
#pragma unroll
    for (int g = tid >> B; g < C::G; g += kThreads / C::N2) tws[(g << B) + r] = __ldg(src + (size_t)mp * (n1 + sel[g]));
}

// pass-2 input: the pass-1 intermediate in global memory (two-pass NTT)
template <int B>
struct InGlobal {
    const uint64_t *in;
    __device__ uint64_t operator()(int blk, int c) const { return in[(size_t)blk * P2<B>::N2 + c]; }
    __device__ void done() const {}
};
template <int B, int EM>
__device__ __forceinline__ void fwd_p2_epilogue(const uint64_t *sm, const LimbInfo &li, uint64_t q,
                                                const int32_t *__restrict__ csl, int logn, int tid);

// pass 2 forward stages: tmp (pass-1 output) -> canonical residues in shared memory
template <int B, bool FP, class IN, bool STAGED = true>
__device__ __forceinline__ void fwd_p2_body(uint64_t *sm, const double *tws, const Mod &m, const Tw &tw2,
                                            const IN &in, const int *sel, int n1, int tid) {
    using C = P2<B>;
    using AR = Arith<FP>;
    using V = typename AR::V;
    const AR ar(m.q);
    const auto *T = pick<FP>(tw2);
    auto acc = [&](int g, int blk) {
        if constexpr (FP && STAGED)
            return TwS{tws + g * C::N2, ar.qinv};
        else if constexpr (FP && UH_NTT_TW8)
            return TwGd{tws, n1 + blk, ar.qinv};  // tws: the limb's w-only global table here
        else
            return TwG<typename AR::W>{T, n1 + blk};
    };
    {
        const int g = tid / C::S, c0 = tid % C::S, blk = sel[g];
        V v[C::R1];
#pragma unroll
        for (int x = 0; x < C::R1; x++) v[x] = AR::raw_in(in(blk, c0 + C::S * x));
        in.done();
        // local stages m' = 1..8: global twiddle index m' * (n1 + blk) + x / (2 dx)
        fwd_strided<C::R1>(v, acc(g, blk), 1, 0, ar.qv());
#pragma unroll
        for (int x = 0; x < C::R1; x++) sm[C::at(g, c0 + C::S * x)] = AR::raw(v[x]);
    }
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
        fwd_strided<C::R2>(v, acc(g, blk), 16, (c / C::R2), ar.qv());
#pragma unroll
        for (int z = 0; z < C::R2; z++) sm[C::at(g, c + z)] = ar.canon(v[z]);
    }
    __syncthreads();
}

// Twisted pass 2 (FP64 limbs): block blk's CT network with twiddles W[(X << s) + g]
// (X = N1 + blk) equals the same network with the shared twiddles W[g] applied to the
// input scaled elementwise by beta_X^c (context.cu builds the twist table): one
// coalesced twist load and one exact FP64 product per element replace the per-block
// twiddle loads (the dominant L1 traffic of the untwisted pass), and the twist resets
// the magnitudes to |v| <= 0.51 q.
template <int B, class IN>
__device__ __forceinline__ void fwd_p2_twist(uint64_t *sm, const double2 *sw, const double *__restrict__ twist,
                                             const Mod &m, const IN &in, const int *sel, int tid) {
    using C = P2<B>;
    using AR = Arith<true>;
    const AR ar(m.q);
    const TwSh ta{sw};
    {
        const int g = tid / C::S, c0 = tid % C::S, blk = sel[g];
        double v[C::R1];
        const double *tb = twist + (size_t)blk * C::N2 + c0;
#pragma unroll
        for (int x = 0; x < C::R1; x++) v[x] = AR::raw_in(in(blk, c0 + C::S * x));
        in.done();
#pragma unroll
        for (int x = 0; x < C::R1; x++) {
            const double t = __ldg(tb + C::S * x);
            v[x] = fmm(v[x], make_double2(t, t * ar.qinv), ar.q);
        }
        fwd_strided<C::R1>(v, ta, 1, 0, ar.qv());
#pragma unroll
        for (int x = 0; x < C::R1; x++) sm[C::at(g, c0 + C::S * x)] = AR::raw(v[x]);
    }
    __syncthreads();
#pragma unroll
    for (int gi = 0; gi < C::GC; gi++) {
        const int grp = tid + kThreads * gi;
        const int per = C::N2 / C::R2;
        const int g = grp / per, c = (grp % per) * C::R2;
        double v[C::R2];
#pragma unroll
        for (int z = 0; z < C::R2; z++) v[z] = AR::raw_in(sm[C::at(g, c + z)]);
        fwd_strided<C::R2>(v, ta, 16, (c / C::R2), ar.qv());
#pragma unroll
        for (int z = 0; z < C::R2; z++) sm[C::at(g, c + z)] = ar.canon(v[z]);
    }
    __syncthreads();
}
// shared twiddles W[0, N2/2) of the limb's prime as (w, w / q) in shared memory
template <int B>
__device__ __forceinline__ void stage_shared_tw(double2 *sw, const double *__restrict__ T, double qinv, int tid) {
    for (int j = tid; j < P2<B>::N2 / 2; j += kThreads) {
        const double w = __ldg(T + j);
        sw[j] = make_double2(w, w * qinv);
    }
}

template <int B>
constexpr size_t p2_smem() {  // data tiles + FP64 twiddle stage (per-block staged twiddles or the shared ones)
    return (size_t)(P2<B>::G * P2<B>::PAD +
                    (UH_NTT_STAGE ? P2<B>::G * P2<B>::N2 : (UH_NTT_TWIST ? P2<B>::N2 : 0))) * 8;
}

template <int B, int EM>
__global__ void __launch_bounds__(kThreads, UH_NTT_MINB) k_fwd_p2(NttJob J, const uint64_t *__restrict__ tmp, int logn,
                                                    const Mod *__restrict__ mods,
                                                    const ulonglong2 *__restrict__ twd,
                                                    const double *__restrict__ twdd,
                                                    const double2 *__restrict__ twf,
                                                    const int32_t *__restrict__ bsel,
                                                    const int32_t *__restrict__ csl,
                                                    const double *__restrict__ twist) {
    using C = P2<B>;
    extern __shared__ uint64_t dsm[];
    uint64_t *sm = dsm;
    double *tws = reinterpret_cast<double *>(dsm + C::G * C::PAD);
    const int f = job_limb(J, J.f0 + blockIdx.y), tid = threadIdx.x;
    const int n1 = 1 << (logn - B);
    const int *sel = bsel + blockIdx.x * C::G;
    const LimbInfo li = limb_info(J, f, logn, mods);
    const Mod m = mods[li.mod];
    const uint64_t q = m.q;
    const Tw tw2{twd + ((size_t)li.mod << logn), twf + ((size_t)li.mod << logn)};
    const InGlobal<B> in{tmp + ((size_t)blockIdx.y << logn)};
    if (fp_limb(q)) {
        if constexpr (UH_NTT_TWIST && !UH_NTT_STAGE) {
            double2 *sw = reinterpret_cast<double2 *>(tws);
            stage_shared_tw<B>(sw, twdd + ((size_t)li.mod << logn), 1.0 / (double)q, tid);
            __syncthreads();
            fwd_p2_twist<B>(sm, sw, twist + ((size_t)li.mod << logn), m, in, sel, tid);
            fwd_p2_epilogue<B, EM>(sm, li, q, csl, logn, tid);
            return;
        }
        if constexpr (UH_NTT_STAGE) {
            stage_twiddles<B>(tws, twdd + ((size_t)li.mod << logn), sel, n1, tid);
            __syncthreads();
        }
        fwd_p2_body<B, true, InGlobal<B>, UH_NTT_STAGE>(
            sm, UH_NTT_STAGE ? tws : twdd + ((size_t)li.mod << logn), m, tw2, in, sel, n1, tid);
    } else {
        fwd_p2_body<B, false>(sm, tws, m, tw2, in, sel, n1, tid);
    }
    fwd_p2_epilogue<B, EM>(sm, li, q, csl, logn, tid);
}

// coalesced slot-order epilogue: a thread's 16 slot-table (and DIVIDE input) loads are
// issued together, then the shared-memory gathers and the stores
template <int B, int EM>
__device__ __forceinline__ void fwd_p2_epilogue(const uint64_t *sm, const LimbInfo &li, uint64_t q,
                                                const int32_t *__restrict__ csl, int logn, int tid) {
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
            else if (EM == 2)
                li.dst[s] = shoup(submod(a[e], y, q), li.w, li.ws, q);
            else
                li.dst[s] = y;
        }
    }
}

// ---------------- cluster-fused forward NTT (one kernel, no global intermediate) ----------------
// A thread-block cluster of NC = N2 / 32 CTAs owns one limb.  CTA `rank` runs pass 1 on the
// 32 columns [32 rank, 32 rank + 32) and keeps its N1 x 32 tile in shared memory; after a
// cluster barrier, pass 2 of CTA `rank` (blocks bsel[rank * G ..]) gathers each of its rows
// from the NC tiles through distributed shared memory (DSMEM) -- the N1 x N2 transpose
// happens on-chip, so the limb is read from HBM once and written once.
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::); }
__device__ __forceinline__ void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::);
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::); }
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
// 64-bit load from the shared memory of CTA `rank` of the cluster at the same offset as `local`
__device__ __forceinline__ uint64_t dsmem_ld(const uint64_t *local, uint32_t rank) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(local), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(a), "r"(rank));
    uint64_t v;
    asm volatile("ld.shared::cluster.u64 %0, [%1];\n" : "=l"(v) : "r"(ra) : "memory");
    return v;
}
template <int B>
struct InCluster {  // row blk, column c of the limb -> CTA c / 32 of the cluster, tile row blk
    const uint64_t *tile;
    __device__ uint64_t operator()(int blk, int c) const { return dsmem_ld(tile + blk * 32 + (c & 31), c >> 5); }
    // this CTA's remote reads are consumed (values in registers): no ordering to release
    __device__ void done() const { cluster_arrive_relaxed(); }
};

template <int A, int B>
constexpr size_t fused_smem() {  // column tile + pass-2 tiles (twiddles from L2: 3 CTAs / SM)
    return (size_t)(P1<A>::N1 * 32 + P2<B>::G * P2<B>::PAD) * 8;
}

template <int A, int B, int LM, int EM>
__global__ void __launch_bounds__(kThreads, UH_NTT_MINB) k_fwd_fused(NttJob J, int logn, const Mod *__restrict__ mods,
                                                       const ulonglong2 *__restrict__ twd,
                                                       const double2 *__restrict__ twf,
                                                       const double *__restrict__ twdd,
                                                       const int32_t *__restrict__ bsel,
                                                       const int32_t *__restrict__ csl) {
    using C2 = P2<B>;
    static_assert((1 << B) / 32 == (1 << A) / C2::G, "pass-1 and pass-2 CTA counts per limb must agree");
    extern __shared__ uint64_t dsm[];
    uint64_t *tile = dsm;                                   // [N1][32]
    uint64_t *sm2 = dsm + P1<A>::N1 * 32;                   // [G][PAD]
    const uint32_t rank = cluster_rank();
    const int f = job_limb(J, J.f0 + blockIdx.y), tid = threadIdx.x, lane = tid & 31, wq = tid >> 5;
    const int n2 = 1 << (logn - A), n1 = 1 << (logn - B);
    const LimbInfo li = limb_info(J, f, logn, mods);
    const Mod m = mods[li.mod];
    const uint64_t q = m.q;
    const bool red = LM == 1 && ((li.qsrc - 1) >> 1) >= q;
    const Tw tw1{twd + ((size_t)li.mod << logn), twf + ((size_t)li.mod << logn)};
    const int *sel = bsel + rank * C2::G;
    const bool fp = fp_limb(q);
    // pass 1 on this CTA's 32 columns, result left in `tile`
    if (fp)
        fwd_p1_body<A, LM, true, true>(tile, li, m, red, tw1, nullptr, n2, rank * 32 + lane, lane, wq);
    else
        fwd_p1_body<A, LM, false, true>(tile, li, m, red, tw1, nullptr, n2, rank * 32 + lane, lane, wq);
    // every tile of the cluster complete and visible (also orders the twiddle stage)
    cluster_arrive();
    cluster_wait();
    const InCluster<B> in{tile};
    if (fp)
        fwd_p2_body<B, true, InCluster<B>, false>(sm2, twdd + ((size_t)li.mod << logn), m, tw1, in, sel, n1, tid);
    else
        fwd_p2_body<B, false, InCluster<B>, false>(sm2, nullptr, m, tw1, in, sel, n1, tid);
    fwd_p2_epilogue<B, EM>(sm2, li, q, csl, logn, tid);
    cluster_wait();  // no CTA leaves while others may still read its tile
}

// inverse pass A stages: canonical residues in shared memory -> tmp (pass-B input)
template <int B, bool FP, bool STAGED = true>
__device__ __forceinline__ void inv_pa_body(uint64_t *sm, const double *tws, const Mod &m, const Tw &tw2,
                                            uint64_t *out, const int *sel, int n1, int tid) {
    using C = P2<B>;
    using AR = Arith<FP>;
    using V = typename AR::V;
    const AR ar(m.q);
    const auto *T = pick<FP>(tw2);
    auto acc = [&](int g, int blk) {
        if constexpr (FP && STAGED)
            return TwS{tws + g * C::N2, ar.qinv};
        else if constexpr (FP && UH_NTT_TW8)
            return TwGd{tws, n1 + blk, ar.qinv};  // tws: the limb's w-only global table here
        else
            return TwG<typename AR::W>{T, n1 + blk};
    };
#pragma unroll
    for (int gi = 0; gi < C::GC; gi++) {
        const int grp = tid + kThreads * gi;
        const int per = C::N2 / C::R2;
        const int g = grp / per, c = (grp % per) * C::R2, blk = sel[g];
        V v[C::R2];
#pragma unroll
        for (int z = 0; z < C::R2; z++) v[z] = AR::in(sm[C::at(g, c + z)]);
        // mirror of the forward contiguous stages: last local stage m' = N2/2
        inv_strided<C::R2>(v, acc(g, blk), C::N2 / 2, (c / C::R2) * (C::R2 / 2), ar.qv());
#pragma unroll
        for (int z = 0; z < C::R2; z++) sm[C::at(g, c + z)] = AR::raw(v[z]);
    }
    __syncthreads();
    {
        const int g = tid / C::S, c0 = tid % C::S, blk = sel[g];
        V v[C::R1];
#pragma unroll
        for (int x = 0; x < C::R1; x++) v[x] = AR::raw_in(sm[C::at(g, c0 + C::S * x)]);
        inv_strided<C::R1>(v, acc(g, blk), 8, 0, ar.qv());
#pragma unroll
        for (int x = 0; x < C::R1; x++) {
            V r = v[x];
            if constexpr (FP) r = fred(r, ar.q, ar.qinv);  // bound the growth before pass B
            out[(size_t)blk * C::N2 + c0 + C::S * x] = AR::raw(r);
        }
    }
}

// twisted inverse pass A (FP64 limbs): the GS network with the shared inverse twiddles,
// then element c of block blk scaled by beta_X^-c (exact FP64 product, centred result)
template <int B>
__device__ __forceinline__ void inv_pa_twist(uint64_t *sm, const double2 *sw, const double *__restrict__ itwist,
                                             const Mod &m, uint64_t *out, const int *sel, int tid) {
    using C = P2<B>;
    using AR = Arith<true>;
    const AR ar(m.q);
    const TwSh ta{sw};
#pragma unroll
    for (int gi = 0; gi < C::GC; gi++) {
        const int grp = tid + kThreads * gi;
        const int per = C::N2 / C::R2;
        const int g = grp / per, c = (grp % per) * C::R2;
        double v[C::R2];
#pragma unroll
        for (int z = 0; z < C::R2; z++) v[z] = AR::in(sm[C::at(g, c + z)]);
        inv_strided<C::R2>(v, ta, C::N2 / 2, (c / C::R2) * (C::R2 / 2), ar.qv());
#pragma unroll
        for (int z = 0; z < C::R2; z++) sm[C::at(g, c + z)] = AR::raw(v[z]);
    }
    __syncthreads();
    {
        const int g = tid / C::S, c0 = tid % C::S, blk = sel[g];
        double v[C::R1];
        const double *tb = itwist + (size_t)blk * C::N2 + c0;
#pragma unroll
        for (int x = 0; x < C::R1; x++) v[x] = AR::raw_in(sm[C::at(g, c0 + C::S * x)]);
        inv_strided<C::R1>(v, ta, 8, 0, ar.qv());
#pragma unroll
        for (int x = 0; x < C::R1; x++) {
            const double t = __ldg(tb + C::S * x);
            out[(size_t)blk * C::N2 + c0 + C::S * x] = AR::raw(fmm(v[x], make_double2(t, t * ar.qinv), ar.q));
        }
    }
}

template <int B>
__global__ void __launch_bounds__(kThreads, UH_NTT_MINB) k_inv_pa(NttJob J, uint64_t *__restrict__ tmp, int logn,
                                                    const Mod *__restrict__ mods,
                                                    const ulonglong2 *__restrict__ itwd,
                                                    const double *__restrict__ itwdd,
                                                    const double2 *__restrict__ itwf,
                                                    const int32_t *__restrict__ bsel,
                                                    const int32_t *__restrict__ csl,
                                                    const double *__restrict__ itwist) {
    using C = P2<B>;
    extern __shared__ uint64_t dsm[];
    uint64_t *sm = dsm;
    double *tws = reinterpret_cast<double *>(dsm + C::G * C::PAD);
    const int f = job_limb(J, J.f0 + blockIdx.y), tid = threadIdx.x;
    const int n1 = 1 << (logn - B);
    const int *sel = bsel + blockIdx.x * C::G;
    const LimbInfo li = limb_info(J, f, logn, mods);
    const Mod m = mods[li.mod];
    const Tw tw2{itwd + ((size_t)li.mod << logn), itwf + ((size_t)li.mod << logn)};
    const bool fp = fp_limb(m.q);
    if (UH_NTT_STAGE && fp) stage_twiddles<B>(tws, itwdd + ((size_t)li.mod << logn), sel, n1, tid);
    if (UH_NTT_TWIST && !UH_NTT_STAGE && fp)
        stage_shared_tw<B>(reinterpret_cast<double2 *>(tws), itwdd + ((size_t)li.mod << logn), 1.0 / (double)m.q, tid);
    // coalesced slot-order gather into the blocks' shared-memory tiles (plain limbs: the only
    // inverse mode); all of a thread's loads are issued before the shared-memory stores
    {
        constexpr int E = 4096 / kThreads;
        int cs[E];
        uint64_t a[E];
#pragma unroll
        for (int e = 0; e < E; e++) {
            const size_t s = cta_slot<B>(tid + kThreads * e, logn);
            cs[e] = __ldg(csl + s);
            a[e] = li.src[s];
        }
#pragma unroll
        for (int e = 0; e < E; e++) sm[C::at((tid + kThreads * e) % C::G, cs[e])] = a[e];
    }
    __syncthreads();
    uint64_t *out = tmp + ((size_t)blockIdx.y << logn);
    if (UH_NTT_TWIST && !UH_NTT_STAGE && fp)
        inv_pa_twist<B>(sm, reinterpret_cast<const double2 *>(tws), itwist + ((size_t)li.mod << logn), m, out, sel, tid);
    else if (fp)
        inv_pa_body<B, true, UH_NTT_STAGE>(sm, UH_NTT_STAGE ? tws : itwdd + ((size_t)li.mod << logn), m, tw2, out,
                                           sel, n1, tid);
    else
        inv_pa_body<B, false>(sm, tws, m, tw2, out, sel, n1, tid);
}

template <auto K>
void p2_attr(size_t smem) {  // opt in to > 48 KB dynamic shared memory, once per kernel instance
    static bool done = false;
    if (!done) {
        UH_CHECK(cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        done = true;
    }
}

// Limbs are transformed in chunks whose pass-1 -> pass-2 intermediate (one reused
// scratch buffer) stays resident in the 126 MB L2, so the intermediate never
// round-trips through HBM.
inline int ntt_chunk(const Ctx &c, int limbs) {
    static const int env = [] {
        const char *e = getenv("UH_NTT_CHUNK_MB");
        return e ? atoi(e) : 0;  // measured: chunking starves the grid (B200), off by default
    }();
    if (env <= 0) return std::min(limbs, 65535);  // grid.y limit
    const int ch = (int)(((size_t)env << 20) / (c.n * 8));
    return std::max(1, std::min(std::min(limbs, ch), 65535));
}

template <auto K>
void fused_attr(size_t smem) {
    static bool done = false;
    if (!done) {
        UH_CHECK(cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        UH_CHECK(cudaFuncSetAttribute(K, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        done = true;
    }
}

template <int A, int B, int LM, int EM>
void launch_fused(const Ctx &c, const NttJob &J, int nl, cudaStream_t s) {
    constexpr size_t smem = fused_smem<A, B>();
    constexpr unsigned ncta = (1u << B) / 32;
    fused_attr<k_fwd_fused<A, B, LM, EM>>(smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ncta, nl, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = ncta;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    UH_CHECK(cudaLaunchKernelEx(&cfg, k_fwd_fused<A, B, LM, EM>, J, (int)c.logn, (const Mod *)c.d_mods,
                                (const ulonglong2 *)c.d_tw2, (const double2 *)c.d_twf, (const double *)c.d_twd,
                                (const int32_t *)c.d_bsel, (const int32_t *)c.d_csl));
    UH_LAUNCH_CHECK();
}

// Opt-in (UH_NTT_FUSED=1): measured slower than the two passes on B200 at N = 2^15
// (0.41 vs 0.35 us per limb, 512 limbs): with one limb per 8-CTA cluster, the cluster
// barriers and DSMEM gather latency are exposed, while the two-pass grids keep ~4k
// independent CTAs in flight and the intermediate largely stays in L2.
inline bool fused_ntt_on() {
    static const bool on = [] {
        const char *e = getenv("UH_NTT_FUSED");
        return e && std::string(e) == "1";
    }();
    return on;
}

// ---------------- persistent cluster-pair forward NTT (N = 2^15, FP64 limbs, one HBM pass) ----------------
// A 2-CTA cluster (one CTA per SM, 512 threads, 224 KB shared memory) walks a strided list of
// limbs.  CTA h owns output half h (slots [h N/2, (h+1) N/2): output index k and its slot lie
// in the same half, context.cu checks it) and stages the raw input half h with TMA bulk copies
// (cp.async.bulk + mbarrier) -- the next limb's copy is in flight while this limb's last 10
// stages run, so the load latency is off the critical path.
//   phase B : CTA h takes columns [512 h, 512 h + 512) of the 2^15 = 32 x 1024 view; it reads
//             x[e] (half 0) and x[e + N/2] (half 1) from the two CTAs' staging buffers (one of
//             them over DSMEM), forms the first CT stage for both halves, runs local stages
//             0..3 of each half (radix 16) and writes half 0's values into CTA 0's and half 1's
//             into CTA 1's shared data area (again one of them over DSMEM);
//   rounds 2, 3 : local stages 4..8 and 9..13 (radix 32) in this CTA's data area;
//   output  : canonical residues gathered in slot order, coalesced stores (+ the DIVIDE epilogue).
// The data area keeps 48-bit two's-complement integers (lo32 + hi16; FP64 values stay below
// 9q < 2^44, no reduction between rounds) under an XOR swizzle e ^ ((e >> 5) & 31), which
// makes all three access patterns bank-conflict free without padding.
constexpr int kPT = 512;
constexpr int kPH = 1 << 14;
constexpr size_t kPStage = (size_t)kPH * 8, kPLo = (size_t)kPH * 4, kPHi = (size_t)kPH * 2;
constexpr size_t kPSmem = kPStage + kPLo + kPHi + 16;
__device__ __forceinline__ int psw(int e) { return e ^ ((e >> 5) & 31); }
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cl_map(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint64_t ld_cl64(uint32_t a) {
    uint64_t v;
    asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(a));
    return v;
}
// store one FP64 value (|v| < 2^47, integer) as lo32 + hi16 at swizzled element e of a data area
__device__ __forceinline__ void pput(uint32_t lo_a, uint32_t hi_a, bool remote, int e, double v) {
    const long long b = __double_as_longlong(v + kMagic);
    const int se = psw(e);
    const uint32_t l = (uint32_t)b;
    const uint16_t hh = (uint16_t)(b >> 32);
    if (remote) {
        asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(lo_a + 4 * se), "r"(l));
        asm volatile("st.shared::cluster.u16 [%0], %1;" ::"r"(hi_a + 2 * se), "h"(hh));
    } else {
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(lo_a + 4 * se), "r"(l));
        asm volatile("st.shared.u16 [%0], %1;" ::"r"(hi_a + 2 * se), "h"(hh));
    }
}
__device__ __forceinline__ double pget(const uint32_t *lo, const uint16_t *hi, int e) {
    const int se = psw(e);
    const long long b = ((long long)(int16_t)hi[se] << 32) | (long long)lo[se];
    return __longlong_as_double(b + 0x4338000000000000LL) - kMagic;
}
__device__ __forceinline__ void pputl(uint32_t *lo, uint16_t *hi, int e, double v) {
    const long long b = __double_as_longlong(v + kMagic);
    const int se = psw(e);
    lo[se] = (uint32_t)b;
    hi[se] = (uint16_t)(b >> 32);
}
// load transform on a staged word: 0 plain, 1 centred lift (as load_t)
template <int LM>
__device__ __forceinline__ uint64_t xform(uint64_t x, uint64_t p, const Mod &m, bool red) {
    if (LM == 0) return x;
    const bool neg = x > ((p - 1) >> 1);
    uint64_t v = neg ? p - x : x;
    if (red) v = csub(barrett_lite(v, m), m.q);
    const uint64_t nv = v ? m.q - v : 0;
    return neg ? nv : v;
}

template <int LM, int EM>
__global__ void __launch_bounds__(kPT, 1) k_fwd_pair(NttJob J, const Mod *__restrict__ mods,
                                                     const double *__restrict__ twdd,
                                                     const uint16_t *__restrict__ hpos, int nl) {
    constexpr int LOGN = 15;
    extern __shared__ __align__(128) unsigned char psm[];
    uint64_t *stg = reinterpret_cast<uint64_t *>(psm);
    uint32_t *lo = reinterpret_cast<uint32_t *>(psm + kPStage);
    uint16_t *hi = reinterpret_cast<uint16_t *>(psm + kPStage + kPLo);
    uint64_t *bar = reinterpret_cast<uint64_t *>(psm + kPStage + kPLo + kPHi);
    const int h = blockIdx.x, tid = threadIdx.x;
    const uint32_t stg_l = su32(stg), lo_l = su32(lo), hi_l = su32(hi), bar_l = su32(bar);
    const uint32_t stg_r = cl_map(stg_l, h ^ 1), lo_r = cl_map(lo_l, h ^ 1), hi_r = cl_map(hi_l, h ^ 1);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(bar_l));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int i) {  // thread 0: TMA bulk copy of raw input half h of launch limb i
        const LimbInfo li = limb_info(J, job_limb(J, J.f0 + i), LOGN, mods);
        const uint64_t *src = li.src + (size_t)h * kPH;
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar_l), "r"((uint32_t)kPStage)
                     : "memory");
#pragma unroll
        for (int k = 0; k < 4; k++)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 32768, [%2];" ::"r"(
                    stg_l + 32768u * k),
                "l"(src + 4096 * k), "r"(bar_l)
                : "memory");
    };
    const int ncl = gridDim.y;
    uint32_t parity = 0;
    if (tid == 0 && (int)blockIdx.y < nl) issue(blockIdx.y);
#pragma unroll 1
    for (int i = blockIdx.y; i < nl; i += ncl) {
        const LimbInfo li = limb_info(J, job_limb(J, J.f0 + i), LOGN, mods);
        const Mod m = mods[li.mod];
        const bool red = LM == 1 && ((li.qsrc - 1) >> 1) >= m.q;
        const double q = (double)m.q, qinv = 1.0 / q;
        const double *T = twdd + ((size_t)li.mod << LOGN);
        {  // wait for this CTA's staging, then for the partner's (and for its previous output phase)
            uint32_t ok = 0;
            while (!ok)
                asm volatile(
                    "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                    : "=r"(ok)
                    : "r"(bar_l), "r"(parity)
                    : "memory");
            parity ^= 1;
        }
        cl_sync();
        // ---- phase B: first stage (both halves) + local stages 0..3 of each half on column c ----
        {
            const int c = 512 * h + tid;
            const double w1 = __ldg(T + 1);
            const double2 W1 = make_double2(w1, w1 * qinv);
            // half 0 input lives in CTA 0's staging, half 1 in CTA 1's
            double v0[16], v1[16];
#pragma unroll
            for (int t0 = 0; t0 < 16; t0 += 8) {
                uint64_t r0[8], r1[8];
#pragma unroll
                for (int t = 0; t < 8; t++) {
                    const int e = (t0 + t) * 1024 + c;
                    const uint64_t mine = stg[e], other = ld_cl64(stg_r + 8u * e);
                    r0[t] = h == 0 ? mine : other;
                    r1[t] = h == 0 ? other : mine;
                }
#pragma unroll
                for (int t = 0; t < 8; t++) {
                    const double x = u2d(xform<LM>(r0[t], li.qsrc, m, red));
                    const double y = fmm(u2d(xform<LM>(r1[t], li.qsrc, m, red)), W1, q);
                    v0[t0 + t] = x + y;
                    v1[t0 + t] = x - y;
                }
            }
            fwd_strided<16>(v0, TwGd{T, 2, qinv}, 1, 0, q);
#pragma unroll
            for (int t = 0; t < 16; t++) pput(h == 0 ? lo_l : lo_r, h == 0 ? hi_l : hi_r, h != 0, t * 1024 + c, v0[t]);
            fwd_strided<16>(v1, TwGd{T, 3, qinv}, 1, 0, q);
#pragma unroll
            for (int t = 0; t < 16; t++) pput(h == 1 ? lo_l : lo_r, h == 1 ? hi_l : hi_r, h != 1, t * 1024 + c, v1[t]);
        }
        cl_sync();  // both data areas complete; both staging buffers consumed
        if (tid == 0 && i + ncl < nl) issue(i + ncl);
        const TwGd ta{T, 2 + h, qinv};
        {  // ---- round 2: local stages 4..8 on (t, c0) = (tid / 32, tid % 32) ----
            const int t = tid >> 5, c0 = tid & 31;
            double v[32];
#pragma unroll
            for (int u = 0; u < 32; u++) v[u] = pget(lo, hi, t * 1024 + u * 32 + c0);
            fwd_strided<32>(v, ta, 16, t, q);
#pragma unroll
            for (int u = 0; u < 32; u++) pputl(lo, hi, t * 1024 + u * 32 + c0, v[u]);
        }
        __syncthreads();
        {  // ---- round 3: local stages 9..13 on 32 contiguous elements; canonical residues ----
            const int grp = tid;
            double v[32];
#pragma unroll
            for (int z = 0; z < 32; z++) v[z] = pget(lo, hi, grp * 32 + z);
            fwd_strided<32>(v, ta, 512, grp, q);
#pragma unroll
            for (int z = 0; z < 32; z++) {
                const uint64_t r = d2u_canon(v[z], q, qinv);
                const int se = psw(grp * 32 + z);
                lo[se] = (uint32_t)r;
                hi[se] = (uint16_t)(r >> 32);
            }
        }
        __syncthreads();
        {  // ---- output: slots h N/2 + j in order (coalesced), gathered from the bit-reversed half ----
            const size_t sbase = (size_t)h << (LOGN - 1);
            const uint16_t *hp = hpos + sbase;
            const uint64_t qq = m.q;
#pragma unroll 1
            for (int i0 = 0; i0 < kPH / kPT; i0 += 16) {
                int e[16];
                uint64_t a[16];
#pragma unroll
                for (int k = 0; k < 16; k++) {
                    const int j = tid + kPT * (i0 + k);
                    e[k] = __ldg(hp + j);
                    if (EM != 0) a[k] = li.in[sbase + j];
                }
#pragma unroll
                for (int k = 0; k < 16; k++) {
                    const int j = tid + kPT * (i0 + k);
                    const int se = psw(e[k]);
                    const uint64_t y = (uint64_t)lo[se] | ((uint64_t)hi[se] << 32);
                    uint64_t r;
                    if (EM == 1)
                        r = csub(shoup_lazy(submod(a[k], y, qq), li.w, li.ws, qq), qq);
                    else
                        r = y;
                    li.dst[sbase + j] = r;
                }
            }
        }
        // the next iteration's cluster barrier orders this output phase before the partner's
        // phase-B writes into this data area
    }
}

template <int LM, int EM>
void launch_pair(const Ctx &c, const NttJob &J, int nl, cudaStream_t s) {
    static bool done = false;
    if (!done) {
        UH_CHECK(cudaFuncSetAttribute(k_fwd_pair<LM, EM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPSmem));
        done = true;
    }
    static int sms = 0;
    if (!sms) UH_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
    const int ncl = std::max(1, std::min(nl, sms / 2));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2, ncl, 1);
    cfg.blockDim = dim3(kPT, 1, 1);
    cfg.dynamicSmemBytes = kPSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    UH_CHECK(cudaLaunchKernelEx(&cfg, k_fwd_pair<LM, EM>, J, (const Mod *)c.d_mods, (const double *)c.d_twd,
                                (const uint16_t *)c.d_hpos, nl));
    UH_LAUNCH_CHECK();
}

// Opt-in (UH_NTT_PAIR=1): measured slower than the two passes on B200 (forward, 512 limbs at
// N = 2^15: 0.48 vs 0.31 us per limb; ModUp 0.39 vs 0.30).  ncu: FP64 pipe 31% active, issue
// 30%, stalls on DSMEM / round-3 twiddle (L2) latency with 16 warps per SM and 128-register
// threads; the two-pass grids keep 32 warps per SM with 16-value register tiles.  An earlier
// non-persistent variant (two 99 KB CTAs per SM, each loading both input halves) measured
// 0.40 us per limb.  Both are bit-exact (tests/test_gpu_primitives.py runs the NTT parity
// cases with UH_NTT_PAIR=1 in a subprocess).
inline bool pair_ntt_on() {
    static const bool on = [] {
        const char *e = getenv("UH_NTT_PAIR");
        return e && std::string(e) == "1";
    }();
    return on;
}

// Limb selection of a forward job: FP64 limbs (half-limb kernel) and the rest (two-pass),
// one period of the job's limb pattern each, cached per job shape in the context.
struct LimbSplit {
    const int16_t *d = nullptr;  // [nfp offsets][nint offsets]
    int T = 0, nfp = 0, nint = 0;
};
inline LimbSplit limb_split(const Ctx &c, const NttJob &J) {
    LimbSplit r;
    std::vector<int> mod_of;
    if (J.mode == NTT_MODUP) {
        r.T = J.L * J.L;
        for (int j = 0; j < J.L; j++)
            for (int kk = 0; kk < J.L; kk++) {
                const int k = kk + (kk >= j);
                mod_of.push_back(k < J.L ? k : J.sp);
            }
    } else if (J.mode == NTT_PLAIN) {
        r.T = J.nl;
        for (int k = 0; k < J.nl; k++) mod_of.push_back(k < J.nq ? J.base + k : J.sp);
    } else {
        r.T = J.nl;
        for (int k = 0; k < J.nl; k++) mod_of.push_back(k);
    }
    if (r.T <= 0 || r.T > 4096) return LimbSplit{};
    std::vector<int16_t> fp, in;
    for (int o = 0; o < r.T; o++) ((c.h_q[mod_of[o]] >> 42) == 0 ? fp : in).push_back((int16_t)o);
    r.nfp = (int)fp.size();
    r.nint = (int)in.size();
    const uint64_t key = ((uint64_t)J.mode << 56) ^ ((uint64_t)J.L << 48) ^ ((uint64_t)J.nl << 32) ^
                         ((uint64_t)J.nq << 16) ^ ((uint64_t)J.base << 8) ^ (uint64_t)J.sp;
    auto &cache = const_cast<Ctx &>(c).ntt_sel;
    for (auto &e : cache)
        if (e.first == key) {
            r.d = e.second;
            return r;
        }
    std::vector<int16_t> all(fp);
    all.insert(all.end(), in.begin(), in.end());
    int16_t *d = nullptr;
    UH_CHECK(cudaMalloc(&d, all.size() * sizeof(int16_t)));
    UH_CHECK(cudaMemcpy(d, all.data(), all.size() * sizeof(int16_t), cudaMemcpyHostToDevice));
    cache.emplace_back(key, d);
    r.d = d;
    return r;
}

template <int A, int B>
void run_fwd_two_pass(const Ctx &c, const NttJob &J0, int limbs, cudaStream_t s);

template <int A, int B>
void run_fwd(const Ctx &c, const NttJob &J0, int limbs, cudaStream_t s) {
    if (c.logn == 15 && c.d_hpos && pair_ntt_on() && !fused_ntt_on() && J0.mode != NTT_DIVIDE2) {
        const LimbSplit sp = limb_split(c, J0);
        if (sp.T > 0 && limbs % sp.T == 0) {
            const int periods = limbs / sp.T;
            if (sp.nfp) {
                NttJob J = J0;
                J.sel = sp.d;
                J.sel_T = sp.T;
                J.sel_cnt = sp.nfp;
                const int n = periods * sp.nfp;
                for (int f0 = 0; f0 < n; f0 += 65535) {
                    J.f0 = f0;
                    const int nl = std::min(65535, n - f0);
                    if (J.mode == NTT_PLAIN) launch_pair<0, 0>(c, J, nl, s);
                    else if (J.mode == NTT_DIVIDE) launch_pair<1, 1>(c, J, nl, s);
                    else launch_pair<1, 0>(c, J, nl, s);
                }
            }
            if (sp.nint) {
                NttJob J = J0;
                J.sel = sp.d + sp.nfp;
                J.sel_T = sp.T;
                J.sel_cnt = sp.nint;
                run_fwd_two_pass<A, B>(c, J, periods * sp.nint, s);
            }
            return;
        }
    }
    run_fwd_two_pass<A, B>(c, J0, limbs, s);
}

template <int A, int B>
void run_fwd_two_pass(const Ctx &c, const NttJob &J0, int limbs, cudaStream_t s) {
    if constexpr ((1 << B) / 32 == (1 << A) / P2<B>::G) {
        if (fused_ntt_on()) {
            for (int f0 = 0; f0 < limbs; f0 += 65535) {
                NttJob J = J0;
                J.f0 = f0;
                const int nl = std::min(65535, limbs - f0);
                const int lm = J.mode == NTT_PLAIN ? 0 : J.mode == NTT_DIVIDE2 ? 2 : 1;
                const int em = J.mode == NTT_DIVIDE ? 1 : J.mode == NTT_DIVIDE2 ? 2 : 0;
                if (lm == 0) launch_fused<A, B, 0, 0>(c, J, nl, s);
                else if (lm == 2) launch_fused<A, B, 2, 2>(c, J, nl, s);
                else if (em == 1) launch_fused<A, B, 1, 1>(c, J, nl, s);
                else launch_fused<A, B, 1, 0>(c, J, nl, s);
            }
            return;
        }
    }
    const int ch = ntt_chunk(c, limbs);
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
            p2_attr<k_fwd_p2<B, 1>>(sm2);
            k_fwd_p2<B, 1><<<g2, kThreads, sm2, s>>>(J, t, ln, c.d_mods, c.d_tw2, c.d_twd, c.d_twf, c.d_bsel, c.d_csl, c.d_twist);
        } else if (J.mode == NTT_DIVIDE2) {
            p2_attr<k_fwd_p2<B, 2>>(sm2);
            k_fwd_p2<B, 2><<<g2, kThreads, sm2, s>>>(J, t, ln, c.d_mods, c.d_tw2, c.d_twd, c.d_twf, c.d_bsel, c.d_csl, c.d_twist);
        } else {
            p2_attr<k_fwd_p2<B, 0>>(sm2);
            k_fwd_p2<B, 0><<<g2, kThreads, sm2, s>>>(J, t, ln, c.d_mods, c.d_tw2, c.d_twd, c.d_twf, c.d_bsel, c.d_csl, c.d_twist);
        }
        UH_LAUNCH_CHECK();
    }
}

template <int A, int B>
void run_inv(const Ctx &c, const NttJob &J0, int limbs, cudaStream_t s) {
    if (J0.mode != NTT_PLAIN) throw std::invalid_argument("inverse NTT: plain limbs only");
    const int ch = ntt_chunk(c, limbs);
    Scratch tmp((size_t)ch * c.n * 8, s);
    constexpr size_t sm2 = p2_smem<B>();
    p2_attr<k_inv_pa<B>>(sm2);
    for (int f0 = 0; f0 < limbs; f0 += ch) {
        NttJob J = J0;
        J.f0 = f0;
        const int nl = std::min(ch, limbs - f0);
        dim3 g1((1u << B) / 32, nl), g2((1u << A) / P2<B>::G, nl);
        k_inv_pa<B><<<g2, kThreads, sm2, s>>>(J, tmp.as<uint64_t>(), (int)c.logn, c.d_mods, c.d_itw2, c.d_itwd,
                                              c.d_itwf, c.d_bsel, c.d_csl, c.d_itwist);
        UH_LAUNCH_CHECK();
        k_inv_pb<A><<<g1, kThreads, 0, s>>>(J, tmp.as<uint64_t>(), (int)c.logn, c.d_mods, c.d_itw2, c.d_itwf);
        UH_LAUNCH_CHECK();
    }
}

}  // namespace

bool ntt_fast_supported(const Ctx &c) { return c.logn >= 13 && c.logn <= 15; }

#ifndef UH_MODUP_FUSED
#define UH_MODUP_FUSED 0  // opt-in: bit-exact, measured slower (ModUp 0.310 vs 0.302 us/limb, step 124.3 vs 123.3 ms)
#endif
// ModUp of n_polys polys of L limbs (strided rows `in`, pstride in_ps) into D [p][j][L+1][N]
// except the diagonal limbs: inverse pass A -> fused inverse pass B + forward pass 1 -> forward
// pass 2.  Returns false (nothing launched) where the fused path does not apply.
bool ntt_fast_modup(const Ctx &c, uint64_t *D, const uint64_t *in, int n_polys, int L, int in_ps, cudaStream_t s) {
    if (!UH_MODUP_FUSED || c.logn != 15 || pair_ntt_on() || fused_ntt_on()) return false;
    constexpr int A = 7, B = 8;
    const long long npj = (long long)n_polys * L, nf = npj * L;
    if (nf > 65535 || L < 2) return false;
    NttJob Ji;
    Ji.nl = L;
    Ji.nq = L;
    Ji.sp = c.sp();
    Ji.src = in;
    Ji.src_ps = in_ps;
    NttJob Jf;
    Jf.mode = NTT_MODUP;
    Jf.L = L;
    Jf.sp = c.sp();
    Jf.dst = D;
    Scratch ti((size_t)npj * c.n * 8, s), tf((size_t)nf * c.n * 8, s);
    constexpr size_t sm2 = p2_smem<B>();
    p2_attr<k_inv_pa<B>>(sm2);
    k_inv_pa<B><<<dim3((1u << A) / P2<B>::G, (unsigned)npj), kThreads, sm2, s>>>(
        Ji, ti.as<uint64_t>(), (int)c.logn, c.d_mods, c.d_itw2, c.d_itwd, c.d_itwf, c.d_bsel, c.d_csl, c.d_itwist);
    UH_LAUNCH_CHECK();
    constexpr size_t sm1 = (size_t)2 * P1<A>::N1 * 32 * 8;
    p2_attr<k_modup_pbp1<A>>(sm1);
    k_modup_pbp1<A><<<dim3((1u << B) / 32, (unsigned)npj), kThreads, sm1, s>>>(
        Ji, Jf, ti.as<uint64_t>(), tf.as<uint64_t>(), (int)c.logn, c.d_mods, c.d_itw2, c.d_itwf, c.d_tw2, c.d_twf);
    UH_LAUNCH_CHECK();
    p2_attr<k_fwd_p2<B, 0>>(sm2);
    k_fwd_p2<B, 0><<<dim3((1u << A) / P2<B>::G, (unsigned)nf), kThreads, sm2, s>>>(
        Jf, tf.as<uint64_t>(), (int)c.logn, c.d_mods, c.d_tw2, c.d_twd, c.d_twf, c.d_bsel, c.d_csl, c.d_twist);
    UH_LAUNCH_CHECK();
    return true;
}

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
