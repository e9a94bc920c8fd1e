// Canonical embedding (CKKS encode / decode) as a hand-written FP64 FFT.
//
// Reference semantics: he_backend.py:176-207 (encode zero-fills a real slot
// vector; decrypt returns every slot).  Slot j of the engine's slot order sits
// at the odd exponent e_j = 5^j mod 2N (psi = e^(i pi / N)); e_j = 1 mod 4, so
// l_j = (e_j - 1) / 4 is a permutation of [0, M), M = N / 2.  With
// Omega = e^(2 pi i / M):
//
//   decode  z_j = Re sum_{n<N} m_n psi^(e_j n)
//               = Re sum_{n<M} u_n Omega^(l_j n),  u_n = (m_n + i m_{n+M}) psi^n
//   encode  w_n = sum_j z_j psi^(-e_j n) = psi^-n sum_j z_j Omega^(-l_j n)   (n < M)
//           m_n = rint(2 Delta / N Re w_n),  m_{n+M} = rint(2 Delta / N Im w_n)
//           (psi^(-e_j M) = -i turns the upper half into the imaginary part)
//
// so both directions are one M-point complex DFT (16384 points at N = 2^15)
// plus an elementwise twist and the slot permutation.  The DFT runs as a
// four-step FFT, M = M1 * M2 (n = M2 a + b, k = k1 + M1 k2):
//   pass 1: for every column b, the M1-point DFT over a, times W^(b k1)
//           -> T[k1][b] (the twist / slot gather fused into the loads);
//   pass 2: for every row k1, the M2-point DFT over b -> X[k1 + M1 k2]
//           (the slot scatter / psi^-n twist + rounding fused into the stores).
// Each CTA runs radix-2 stages in shared memory over a block of sequences
// (coalesced column / row blocks); twiddles come from sincospi (FP64, ~1 ulp),
// so the coefficients agree with the oracle's numpy FFT up to rounding (the
// rounded encode coefficients to within one unit at .5 ties).
#include "ops.cuh"

namespace uh {
namespace {

constexpr int kET = 256;       // threads per CTA
constexpr int kEElems = 2048;  // complex elements per CTA (32 KB of shared memory)

struct Geo {
    int m, M, m1, M1, M2;
};
Geo geo(uint32_t n) {
    Geo g;
    int logn = 0;
    while ((1u << logn) < n) logn++;
    g.m = logn - 1;
    g.M = 1 << g.m;
    g.m1 = (g.m + 1) / 2;
    g.M1 = 1 << g.m1;
    g.M2 = g.M / g.M1;
    return g;
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// e^(i pi x)
__device__ __forceinline__ double2 cis_pi(double x) {
    double s, c;
    sincospi(x, &s, &c);
    return make_double2(c, s);
}
__device__ __forceinline__ uint32_t brv(uint32_t x, int bits) { return bits ? __brev(x) >> (32 - bits) : 0; }

// In-place radix-2 DIT over `nseq` sequences of length P = 2^bits stored at buf[c * P + i]
// (loaded in bit-reversed order); sign +1: Omega^(+kn), -1: Omega^(-kn).
__device__ void smem_fft(double2 *buf, int nseq, int bits, double sign) {
    const int P = 1 << bits, halfP = P >> 1;
    for (int s = 1; s <= bits; s++) {
        __syncthreads();
        const int h = 1 << (s - 1);
        for (int t = threadIdx.x; t < nseq * halfP; t += blockDim.x) {
            const int c = t / halfP, r = t - c * halfP;
            const int grp = r >> (s - 1), pos = r & (h - 1);
            const int i = c * P + grp * 2 * h + pos, j = i + h;
            const double2 w = cis_pi(sign * (double)pos / (double)h);
            const double2 x = buf[i], y = cmul(buf[j], w);
            buf[i] = make_double2(x.x + y.x, x.y + y.y);
            buf[j] = make_double2(x.x - y.x, x.y - y.y);
        }
    }
    __syncthreads();
}

// pass 1.  DEC: input the centred coefficients m (double) -> u_n = (m_n + i m_{n+M}) psi^n;
// ENC: input the slots z (double) -> x_n = z_{jof[n]}.  Output T[p][k1][b] (times W^(b k1)).
template <bool ENC>
__global__ void __launch_bounds__(kET) k_embed_p1(double2 *__restrict__ T, const double *__restrict__ in, int m,
                                                  int m1, int cb, const int32_t *__restrict__ jof) {
    extern __shared__ double2 ebuf[];
    const int M = 1 << m, M1 = 1 << m1, M2 = M >> m1;
    const int p = blockIdx.y, b0 = blockIdx.x * cb;
    const int nb = min(cb, M2 - b0);
    const double sign = ENC ? -1.0 : 1.0;
    const double invN = 1.0 / (double)(2 * M);
    for (int t = threadIdx.x; t < nb * M1; t += blockDim.x) {
        const int c = t % nb, a = t / nb;
        const int n = M2 * a + b0 + c;
        double2 v;
        if (ENC) {
            v = make_double2(in[(size_t)p * M + jof[n]], 0.0);
        } else {
            const double lo = in[(size_t)p * 2 * M + n], hi = in[(size_t)p * 2 * M + M + n];
            v = cmul(make_double2(lo, hi), cis_pi((double)n * invN));  // psi^n, psi = e^(i pi / N)
        }
        ebuf[c * M1 + brv(a, m1)] = v;
    }
    smem_fft(ebuf, nb, m1, sign);
    for (int t = threadIdx.x; t < nb * M1; t += blockDim.x) {
        const int c = t % nb, k1 = t / nb;
        const int b = b0 + c;
        // W^(b k1) = e^(sign 2 pi i b k1 / M) = cis_pi(sign * 2 b k1 / M); b k1 < 2^30, exact
        const double2 w = cis_pi(sign * 2.0 * (double)(b * k1) / (double)M);
        T[((size_t)p * M1 + k1) * M2 + b] = cmul(ebuf[c * M1 + k1], w);
    }
}

// pass 2: rows k1 of T -> X[k1 + M1 k2].  DEC: slots[p][jof[l]] = Re X_l / scale.
// ENC: w_n = psi^-n X_n, coef[p][n] = rint(f Re w_n), coef[p][n + M] = rint(f Im w_n).
template <bool ENC>
__global__ void __launch_bounds__(kET) k_embed_p2(const double2 *__restrict__ T, double *__restrict__ slots,
                                                  int64_t *__restrict__ coef, int m, int m1, int ck, double f,
                                                  const int32_t *__restrict__ jof) {
    extern __shared__ double2 ebuf[];
    const int M = 1 << m, M1 = 1 << m1, m2 = m - m1, M2 = 1 << m2;
    const int p = blockIdx.y, k10 = blockIdx.x * ck;
    const int nk = min(ck, M1 - k10);
    const double sign = ENC ? -1.0 : 1.0;
    for (int t = threadIdx.x; t < nk * M2; t += blockDim.x) {
        const int c = t / M2, b = t - c * M2;
        ebuf[c * M2 + brv(b, m2)] = T[((size_t)p * M1 + k10 + c) * M2 + b];
    }
    smem_fft(ebuf, nk, m2, sign);
    for (int t = threadIdx.x; t < nk * M2; t += blockDim.x) {
        const int k2 = t / nk, c = t - k2 * nk;  // consecutive threads: consecutive k1
        const int l = k10 + c + M1 * k2;
        const double2 x = ebuf[c * M2 + k2];
        if (ENC) {
            const double2 w = cmul(x, cis_pi(-(double)l / (double)(2 * M)));
            coef[(size_t)p * 2 * M + l] = __double2ll_rn(w.x * f);
            coef[(size_t)p * 2 * M + M + l] = __double2ll_rn(w.y * f);
        } else {
            slots[(size_t)p * M + jof[l]] = x.x * f;
        }
    }
}

void embed_run(const Ctx &c, bool enc, double *slots, int64_t *coef, const double *coef_in, int n_polys,
               double f, cudaStream_t s) {
    const Geo g = geo(c.n);
    Scratch T((size_t)n_polys * g.M * sizeof(double2), s);
    const int cb = std::max(1, std::min(g.M2, kEElems / g.M1));
    const int ck = std::max(1, std::min(g.M1, kEElems / g.M2));
    for (int p0 = 0; p0 < n_polys; p0 += 65535) {
        const int np = std::min(65535, n_polys - p0);
        dim3 g1((unsigned)((g.M2 + cb - 1) / cb), (unsigned)np), g2((unsigned)((g.M1 + ck - 1) / ck), (unsigned)np);
        const size_t sm1 = (size_t)cb * g.M1 * sizeof(double2), sm2 = (size_t)ck * g.M2 * sizeof(double2);
        double2 *t = T.as<double2>() + (size_t)p0 * g.M;
        if (enc) {
            k_embed_p1<true><<<g1, kET, sm1, s>>>(t, slots + (size_t)p0 * g.M, g.m, g.m1, cb, c.d_jof);
            UH_LAUNCH_CHECK();
            k_embed_p2<true><<<g2, kET, sm2, s>>>(t, nullptr, coef + (size_t)p0 * 2 * g.M, g.m, g.m1, ck, f, c.d_jof);
        } else {
            k_embed_p1<false><<<g1, kET, sm1, s>>>(t, coef_in + (size_t)p0 * 2 * g.M, g.m, g.m1, cb, c.d_jof);
            UH_LAUNCH_CHECK();
            k_embed_p2<false><<<g2, kET, sm2, s>>>(t, slots + (size_t)p0 * g.M, nullptr, g.m, g.m1, ck, f, c.d_jof);
        }
        UH_LAUNCH_CHECK();
    }
}

}  // namespace

void encode_coeffs(const Ctx &c, int64_t *coef, const double *slots, int n_polys, double scale, cudaStream_t s) {
    if (n_polys <= 0) return;
    embed_run(c, true, const_cast<double *>(slots), coef, nullptr, n_polys, 2.0 * scale / (double)c.n, s);
}

void decode_coeffs(const Ctx &c, double *slots, const double *coef, int n_polys, double scale, cudaStream_t s) {
    if (n_polys <= 0) return;
    embed_run(c, false, slots, nullptr, coef, n_polys, 1.0 / scale, s);
}

}  // namespace uh
