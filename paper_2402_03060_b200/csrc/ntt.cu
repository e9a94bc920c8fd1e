// Negacyclic NTT over the RNS primes, slot-order output (sm_100a).
//
// Forward transform = the merged Cooley-Tukey negacyclic NTT (psi folded
// into bit-reversed twiddles) followed by the permutation that puts entry k
// (the evaluation at psi^(2*brv(k)+1)) at its slot-order index, so that every
// Galois rotation X -> X^(5^r) becomes a cyclic shift of each half of the
// evaluation vector (see params.slot_tables).  The inverse gathers from slot
// order, runs Gentleman-Sande stages and scales by N^-1.
//
// Large N (>= 2^13) is split N = N1 * N2 into two passes so each CTA works
// on a shared-memory tile: pass 1 runs the first log2(N1) stages on
// C-column tiles of the N1 x N2 row-major view (stride-N2 butterflies,
// coalesced 128-byte rows), pass 2 runs the remaining stages on contiguous
// N2-blocks and scatters to slot order.  Small N runs in one pass per limb.
// Butterflies use Shoup twiddle products (precomputed companions).
#include "engine.cuh"
#include "ntt_fast.cuh"

namespace uh {

namespace {

constexpr int kCols = 16;     // columns per pass-1 tile (16 x 8 B = one 128 B row segment)
constexpr int kThreads = 256;

__device__ __forceinline__ const uint64_t *limb_ptr(const uint64_t *base, int f, int nl, int pstride, int n) {
    int p = f / nl, k = f - p * nl;
    return base + ((size_t)p * pstride + k) * n;
}

__device__ __forceinline__ void ct_bfly(uint64_t &x, uint64_t &y, uint64_t w, uint64_t ws, uint64_t q) {
    uint64_t u = x, v = shoup(y, w, ws, q);
    x = addmod(u, v, q);
    y = submod(u, v, q);
}
__device__ __forceinline__ void gs_bfly(uint64_t &x, uint64_t &y, uint64_t w, uint64_t ws, uint64_t q) {
    uint64_t u = x, v = y;
    x = addmod(u, v, q);
    y = shoup(submod(u, v, q), w, ws, q);
}

// ---- one pass (small N): one CTA per limb --------------------------------
__global__ void k_ntt_fwd_small(uint64_t *data, int nl, int nq, int base, int sp, int pstride, int n,
                                const Mod *__restrict__ mods, const uint64_t *__restrict__ psi,
                                const uint64_t *__restrict__ psis, const int32_t *__restrict__ sob) {
    extern __shared__ uint64_t sm[];
    int f = blockIdx.x;
    int k = f % nl;
    int mi = limb_mod(k, nq, base, sp);
    uint64_t q = mods[mi].q;
    uint64_t *x = const_cast<uint64_t *>(limb_ptr(data, f, nl, pstride, n));
    const uint64_t *w = psi + (size_t)mi * n, *ws = psis + (size_t)mi * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = x[i];
    __syncthreads();
    for (int len = 1, t = n >> 1; len < n; len <<= 1, t >>= 1) {
        for (int b = threadIdx.x; b < (n >> 1); b += blockDim.x) {
            int i = b / t, j = 2 * i * t + (b - i * t);
            ct_bfly(sm[j], sm[j + t], w[len + i], ws[len + i], q);
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) x[sob[i]] = sm[i];
}

__global__ void k_ntt_inv_small(uint64_t *data, int nl, int nq, int base, int sp, int pstride, int n,
                                const Mod *__restrict__ mods, const uint64_t *__restrict__ ipsi,
                                const uint64_t *__restrict__ ipsis, const int32_t *__restrict__ sob) {
    extern __shared__ uint64_t sm[];
    int f = blockIdx.x;
    int k = f % nl;
    int mi = limb_mod(k, nq, base, sp);
    const Mod m = mods[mi];
    uint64_t q = m.q;
    uint64_t *x = const_cast<uint64_t *>(limb_ptr(data, f, nl, pstride, n));
    const uint64_t *w = ipsi + (size_t)mi * n, *ws = ipsis + (size_t)mi * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = x[sob[i]];
    __syncthreads();
    for (int len = n >> 1, t = 1; len >= 1; len >>= 1, t <<= 1) {
        for (int b = threadIdx.x; b < (n >> 1); b += blockDim.x) {
            int i = b / t, j = 2 * i * t + (b - i * t);
            gs_bfly(sm[j], sm[j + t], w[len + i], ws[len + i], q);
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = shoup(sm[i], m.ninv, m.ninvs, q);
}

// ---- two-pass (large N) ----------------------------------------------------
// pass 1 forward: src (strided limbs) -> dst (compact), first log2(n1) stages.
__global__ void k_ntt_fwd_p1(const uint64_t *src, uint64_t *dst, int nl, int nq, int base, int sp, int pstride,
                             int n, int n1, int n2, const Mod *__restrict__ mods,
                             const uint64_t *__restrict__ psi, const uint64_t *__restrict__ psis) {
    extern __shared__ uint64_t sm[];  // [n1][kCols]
    int f = blockIdx.y;
    int mi = limb_mod(f % nl, nq, base, sp);
    uint64_t q = mods[mi].q;
    const uint64_t *x = limb_ptr(src, f, nl, pstride, n);
    uint64_t *y = dst + (size_t)f * n;
    const uint64_t *w = psi + (size_t)mi * n, *ws = psis + (size_t)mi * n;
    int c0 = blockIdx.x * kCols;
    for (int idx = threadIdx.x; idx < n1 * kCols; idx += blockDim.x) {
        int r = idx / kCols, c = idx % kCols;
        sm[idx] = x[(size_t)r * n2 + c0 + c];
    }
    __syncthreads();
    for (int m = 1, t = n1 >> 1; m < n1; m <<= 1, t >>= 1) {
        for (int bf = threadIdx.x; bf < (n1 >> 1) * kCols; bf += blockDim.x) {
            int c = bf % kCols, b = bf / kCols;
            int i = b / t, r = 2 * i * t + (b - i * t);
            ct_bfly(sm[r * kCols + c], sm[(r + t) * kCols + c], w[m + i], ws[m + i], q);
        }
        __syncthreads();
    }
    for (int idx = threadIdx.x; idx < n1 * kCols; idx += blockDim.x) {
        int r = idx / kCols, c = idx % kCols;
        y[(size_t)r * n2 + c0 + c] = sm[idx];
    }
}

// pass 2 forward: src (compact) -> dst (strided limbs, slot order), stages m = n1..n/2.
__global__ void k_ntt_fwd_p2(const uint64_t *src, uint64_t *dst, int nl, int nq, int base, int sp, int pstride,
                             int n, int n1, int n2, int g, const Mod *__restrict__ mods,
                             const uint64_t *__restrict__ psi, const uint64_t *__restrict__ psis,
                             const int32_t *__restrict__ sob) {
    extern __shared__ uint64_t sm[];  // [g][n2]
    int f = blockIdx.y;
    int mi = limb_mod(f % nl, nq, base, sp);
    uint64_t q = mods[mi].q;
    const uint64_t *x = src + (size_t)f * n;
    uint64_t *y = const_cast<uint64_t *>(limb_ptr(dst, f, nl, pstride, n));
    const uint64_t *w = psi + (size_t)mi * n, *ws = psis + (size_t)mi * n;
    int b0 = blockIdx.x * g;
    for (int idx = threadIdx.x; idx < g * n2; idx += blockDim.x) sm[idx] = x[(size_t)b0 * n2 + idx];
    __syncthreads();
    int half2 = n2 >> 1;
    for (int m = n1, t = half2; m < n; m <<= 1, t >>= 1) {
        int per = m / n1;  // twiddles per block at this stage
        for (int bf = threadIdx.x; bf < g * half2; bf += blockDim.x) {
            int gg = bf / half2, wq = bf - gg * half2;
            int i = wq / t, c = 2 * i * t + (wq - i * t);
            int ti = m + (b0 + gg) * per + i;
            ct_bfly(sm[gg * n2 + c], sm[gg * n2 + c + t], w[ti], ws[ti], q);
        }
        __syncthreads();
    }
    for (int idx = threadIdx.x; idx < g * n2; idx += blockDim.x) y[sob[(size_t)b0 * n2 + idx]] = sm[idx];
}

// inverse pass A: src (strided limbs, slot order) -> dst (compact), GS stages m = n/2 .. n1.
__global__ void k_ntt_inv_pa(const uint64_t *src, uint64_t *dst, int nl, int nq, int base, int sp, int pstride,
                             int n, int n1, int n2, int g, const Mod *__restrict__ mods,
                             const uint64_t *__restrict__ ipsi, const uint64_t *__restrict__ ipsis,
                             const int32_t *__restrict__ sob) {
    extern __shared__ uint64_t sm[];
    int f = blockIdx.y;
    int mi = limb_mod(f % nl, nq, base, sp);
    uint64_t q = mods[mi].q;
    const uint64_t *x = limb_ptr(src, f, nl, pstride, n);
    uint64_t *y = dst + (size_t)f * n;
    const uint64_t *w = ipsi + (size_t)mi * n, *ws = ipsis + (size_t)mi * n;
    int b0 = blockIdx.x * g;
    for (int idx = threadIdx.x; idx < g * n2; idx += blockDim.x) sm[idx] = x[sob[(size_t)b0 * n2 + idx]];
    __syncthreads();
    int half2 = n2 >> 1;
    for (int m = n >> 1, t = 1; m >= n1; m >>= 1, t <<= 1) {
        int per = m / n1;
        for (int bf = threadIdx.x; bf < g * half2; bf += blockDim.x) {
            int gg = bf / half2, wq = bf - gg * half2;
            int i = wq / t, c = 2 * i * t + (wq - i * t);
            int ti = m + (b0 + gg) * per + i;
            gs_bfly(sm[gg * n2 + c], sm[gg * n2 + c + t], w[ti], ws[ti], q);
        }
        __syncthreads();
    }
    for (int idx = threadIdx.x; idx < g * n2; idx += blockDim.x) y[(size_t)b0 * n2 + idx] = sm[idx];
}

// inverse pass B: src (compact) -> dst (strided limbs, natural order), GS stages m = n1/2 .. 1, x N^-1.
__global__ void k_ntt_inv_pb(const uint64_t *src, uint64_t *dst, int nl, int nq, int base, int sp, int pstride,
                             int n, int n1, int n2, const Mod *__restrict__ mods,
                             const uint64_t *__restrict__ ipsi, const uint64_t *__restrict__ ipsis) {
    extern __shared__ uint64_t sm[];
    int f = blockIdx.y;
    int mi = limb_mod(f % nl, nq, base, sp);
    const Mod md = mods[mi];
    uint64_t q = md.q;
    const uint64_t *x = src + (size_t)f * n;
    uint64_t *y = const_cast<uint64_t *>(limb_ptr(dst, f, nl, pstride, n));
    const uint64_t *w = ipsi + (size_t)mi * n, *ws = ipsis + (size_t)mi * n;
    int c0 = blockIdx.x * kCols;
    for (int idx = threadIdx.x; idx < n1 * kCols; idx += blockDim.x) {
        int r = idx / kCols, c = idx % kCols;
        sm[idx] = x[(size_t)r * n2 + c0 + c];
    }
    __syncthreads();
    for (int m = n1 >> 1, t = 1; m >= 1; m >>= 1, t <<= 1) {
        for (int bf = threadIdx.x; bf < (n1 >> 1) * kCols; bf += blockDim.x) {
            int c = bf % kCols, b = bf / kCols;
            int i = b / t, r = 2 * i * t + (b - i * t);
            gs_bfly(sm[r * kCols + c], sm[(r + t) * kCols + c], w[m + i], ws[m + i], q);
        }
        __syncthreads();
    }
    for (int idx = threadIdx.x; idx < n1 * kCols; idx += blockDim.x) {
        int r = idx / kCols, c = idx % kCols;
        y[(size_t)r * n2 + c0 + c] = shoup(sm[idx], md.ninv, md.ninvs, q);
    }
}

int pass2_group(const Ctx &c) {
    int g = 2048 / (int)c.n2;
    if (g < 1) g = 1;
    if (g > (int)c.n1) g = (int)c.n1;
    return g;
}

}  // namespace

void ntt_forward(const Ctx &c, uint64_t *data, int n_polys, int nl, int nq, int base, int pstride, cudaStream_t s) {
    int limbs = n_polys * nl;
    if (limbs == 0) return;
    int n = (int)c.n;
    if (c.n1 == 0) {
        k_ntt_fwd_small<<<limbs, kThreads, n * sizeof(uint64_t), s>>>(data, nl, nq, base, c.sp(), pstride, n, c.d_mods,
                                                                    c.d_psi, c.d_psis, c.d_sob);
        UH_LAUNCH_CHECK();
        return;
    }
    if (ntt_fast_supported(c)) {
        NttJob J;
        J.nl = nl;
        J.nq = nq;
        J.base = base;
        J.sp = c.sp();
        J.src = data;
        J.src_ps = pstride;
        J.dst = data;
        J.dst_ps = pstride;
        ntt_fast_forward(c, J, limbs, s);
        return;
    }
    if (limbs > 65535) throw std::invalid_argument("NTT: more than 65535 limbs in one call at this ring degree");
    Scratch tmp((size_t)limbs * n * sizeof(uint64_t), s);
    int n1 = (int)c.n1, n2 = (int)c.n2, g = pass2_group(c);
    dim3 g1(n2 / kCols, limbs), g2(n1 / g, limbs);
    k_ntt_fwd_p1<<<g1, kThreads, n1 * kCols * sizeof(uint64_t), s>>>(data, tmp.as<uint64_t>(), nl, nq, base, c.sp(),
                                                                      pstride, n, n1, n2, c.d_mods, c.d_psi, c.d_psis);
    UH_LAUNCH_CHECK();
    k_ntt_fwd_p2<<<g2, kThreads, g * n2 * sizeof(uint64_t), s>>>(tmp.as<uint64_t>(), data, nl, nq, base, c.sp(), pstride,
                                                                  n, n1, n2, g, c.d_mods, c.d_psi, c.d_psis, c.d_sob);
    UH_LAUNCH_CHECK();
}

void ntt_inverse(const Ctx &c, uint64_t *data, int n_polys, int nl, int nq, int base, int pstride, cudaStream_t s) {
    int limbs = n_polys * nl;
    if (limbs == 0) return;
    int n = (int)c.n;
    if (c.n1 == 0) {
        k_ntt_inv_small<<<limbs, kThreads, n * sizeof(uint64_t), s>>>(data, nl, nq, base, c.sp(), pstride, n, c.d_mods,
                                                                    c.d_ipsi, c.d_ipsis, c.d_sob);
        UH_LAUNCH_CHECK();
        return;
    }
    if (ntt_fast_supported(c)) {
        NttJob J;
        J.nl = nl;
        J.nq = nq;
        J.base = base;
        J.sp = c.sp();
        J.src = data;
        J.src_ps = pstride;
        J.dst = data;
        J.dst_ps = pstride;
        ntt_fast_inverse(c, J, limbs, s);
        return;
    }
    if (limbs > 65535) throw std::invalid_argument("NTT: more than 65535 limbs in one call at this ring degree");
    Scratch tmp((size_t)limbs * n * sizeof(uint64_t), s);
    int n1 = (int)c.n1, n2 = (int)c.n2, g = pass2_group(c);
    dim3 g1(n2 / kCols, limbs), g2(n1 / g, limbs);
    k_ntt_inv_pa<<<g2, kThreads, g * n2 * sizeof(uint64_t), s>>>(data, tmp.as<uint64_t>(), nl, nq, base, c.sp(), pstride,
                                                                  n, n1, n2, g, c.d_mods, c.d_ipsi, c.d_ipsis, c.d_sob);
    UH_LAUNCH_CHECK();
    k_ntt_inv_pb<<<g1, kThreads, n1 * kCols * sizeof(uint64_t), s>>>(tmp.as<uint64_t>(), data, nl, nq, base, c.sp(),
                                                                      pstride, n, n1, n2, c.d_mods, c.d_ipsi, c.d_ipsis);
    UH_LAUNCH_CHECK();
}

}  // namespace uh
