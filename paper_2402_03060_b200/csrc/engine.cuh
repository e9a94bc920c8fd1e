// Internal host-side interface of the engine (not part of the C-ABI).
#pragma once
#include <atomic>
#include <utility>
#include <cstdint>
#include <string>
#include <vector>
#include <stdexcept>
#include <cuda_runtime.h>
#include "common.cuh"

namespace uh {

struct Ctx {
    int device = 0;
    uint32_t n = 0, logn = 0, count = 0;  // count = depth + 2 moduli (q_0..q_depth, P)
    uint32_t n1 = 0, n2 = 0;              // two-pass NTT split, n = n1 * n2 (n1 = 0: one pass)
    std::vector<uint64_t> h_q;
    std::vector<Mod> h_mods;                     // host copies of d_mods / d_inv / d_invs
    std::vector<uint64_t> h_inv, h_invs;
    Mod *d_mods = nullptr;               // [count]
    uint64_t *d_psi = nullptr, *d_psis = nullptr;    // [count][n] psi^brv(i), Shoup companions
    uint64_t *d_ipsi = nullptr, *d_ipsis = nullptr;  // [count][n] psi^-brv(i)
    ulonglong2 *d_tw2 = nullptr, *d_itw2 = nullptr;  // [count][n] interleaved (w, w') pairs of the above
    double2 *d_twf = nullptr, *d_itwf = nullptr;     // [count][n] (w, w / q) for FP64-pipe limbs (q < 2^42), else 0
    // pass-2 composite twiddles of the FP64-pipe limbs (ntt_fast.cu, TwC): the twiddle of global
    // index m (n1 + blk) + j factors as F[blk][s] * U[s - 4][u] * R[s'][v] (m = 2^s), so pass 2
    // reads 8 per-block heads + 16 roots instead of the N-word table (forward / inverse)
    double *d_tfF = nullptr, *d_itfF = nullptr;     // [count][n1][8] heads F[blk][s]
    double2 *d_tfU = nullptr, *d_itfU = nullptr;    // [count][4][16] (U, U / q)
    double2 *d_tfR = nullptr, *d_itfR = nullptr;    // [count][16] (R, R / q) at (1 << s') - 1 + v
    int32_t *d_sob = nullptr;            // [n] slot-order index of bit-reversed NTT output k
    int32_t *d_bsel = nullptr;           // [n1] pass-2 block of CTA x, position g (ntt_fast.cu)
    uint8_t *d_csl = nullptr;            // [n] element index (< 256) inside its pass-2 block, per slot: 32 KB, L1-resident
    uint64_t *d_inv = nullptr, *d_invs = nullptr;  // [count][count]: q_j^-1 mod q_i at [i*count+j]
    uint64_t *d_inv2 = nullptr, *d_inv2s = nullptr;  // [count][count]: (q_j * P)^-1 mod q_i at [i*count+j]
    ulonglong2 *d_pmod = nullptr;        // [count] (P mod q_i, Shoup companion)
    int32_t *d_pos = nullptr;            // [n/2] index (5^j mod 2N - 1)/2 : slot j -> odd exponent slot
    int32_t *d_neg = nullptr;            // [n/2] index (2N - 5^j - 1)/2
    int32_t *d_jof = nullptr;            // [n/2] slot j of the DFT index l = (5^j mod 2N - 1)/4 (embed.cu)
    int sp() const { return (int)count - 1; }
};

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define UH_CHECK(x)                                                                            \
    do {                                                                                       \
        cudaError_t e__ = (x);                                                                 \
        if (e__ != cudaSuccess)                                                                \
            throw ::uh::CudaError(std::string(#x) + ": " + cudaGetErrorString(e__));           \
    } while (0)
// every kernel launch of the engine is followed by UH_LAUNCH_CHECK, which also
// counts it (uh_launch_count(): the bench's gpu_launches evidence)
extern std::atomic<unsigned long long> g_launch_count;
#define UH_LAUNCH_CHECK()                                          \
    do {                                                           \
        ::uh::g_launch_count.fetch_add(1, std::memory_order_relaxed); \
        UH_CHECK(cudaGetLastError());                              \
    } while (0)

// Switch to `device` for a scope and restore the caller's current device afterwards.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int device) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != device) UH_CHECK(cudaSetDevice(device));
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard &) = delete;
    DeviceGuard &operator=(const DeviceGuard &) = delete;
};

// Opt a kernel in to > 48 KB of dynamic shared memory on the current device.  The
// attribute is per (kernel, device): the record is a set of both, under a mutex.
void smem_optin_raw(const void *kernel, size_t smem);
template <class K>
void smem_optin(K *kernel, size_t smem) {
    smem_optin_raw(reinterpret_cast<const void *>(kernel), smem);
}

// stream-ordered scratch buffer
struct Scratch {
    void *p = nullptr;
    cudaStream_t s;
    Scratch(size_t bytes, cudaStream_t st) : s(st) {
        if (bytes) UH_CHECK(cudaMallocAsync(&p, bytes, s));
    }
    ~Scratch() {
        if (p) cudaFreeAsync(p, s);
    }
    template <class T> T *as() { return static_cast<T *>(p); }
    Scratch(const Scratch &) = delete;
    Scratch &operator=(const Scratch &) = delete;
};

// ---- ntt.cu ----
// In-place forward (coefficients -> slot order) / inverse NTT of n_polys
// polynomials of nl limbs each, limb k reduced modulo limb_mod(k, nq, sp).
// Poly p, limb k lives at data + (p * pstride + k) * n; limb k < nq uses
// modulus base + k, limbs >= nq use the special prime.
void ntt_forward(const Ctx &c, uint64_t *data, int n_polys, int nl, int nq, int base, int pstride, cudaStream_t s);
void ntt_inverse(const Ctx &c, uint64_t *data, int n_polys, int nl, int nq, int base, int pstride, cudaStream_t s);

}  // namespace uh
