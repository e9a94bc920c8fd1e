// Context creation: per-prime constants, twiddle tables and slot-order tables,
// computed once on the host (exact 128-bit arithmetic) and kept in HBM.
#include <mutex>
#include <map>
#include <set>

#include "engine.cuh"
#include "ops.cuh"

namespace uh {

namespace {
typedef unsigned __int128 hu128;

uint64_t h_mulmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((hu128)a * b) % q); }
uint64_t h_pow(uint64_t b, uint64_t e, uint64_t q) {
    uint64_t r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = h_mulmod(r, b, q);
        b = h_mulmod(b, b, q);
        e >>= 1;
    }
    return r;
}
uint64_t h_inv(uint64_t a, uint64_t q) { return h_pow(a % q, q - 2, q); }
uint64_t h_shoup(uint64_t w, uint64_t q) { return (uint64_t)(((hu128)w << 64) / q); }
uint32_t h_brv(uint32_t x, uint32_t bits) {
    uint32_t r = 0;
    for (uint32_t i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}
template <class T> T *upload(const std::vector<T> &v) {
    T *d = nullptr;
    UH_CHECK(cudaMalloc(&d, v.size() * sizeof(T)));
    UH_CHECK(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return d;
}
}  // namespace

void smem_optin_raw(const void *kernel, size_t smem) {
    static std::mutex mu;
    // the largest opt-in granted so far per (kernel, device): a later launch of the same kernel
    // with a bigger tile (e.g. more terms) raises it
    static std::map<std::pair<const void *, int>, size_t> done;
    int dev = 0;
    UH_CHECK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    auto it = done.find({kernel, dev});
    if (it != done.end() && it->second >= smem) return;
    UH_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    done[{kernel, dev}] = smem;
}

Ctx *ctx_create(uint32_t n, const uint64_t *moduli, const uint64_t *psi, uint32_t count, int device) {
    if (n < 4 || (n & (n - 1))) throw std::invalid_argument("n must be a power of two >= 4");
    if (count < 2) throw std::invalid_argument("need at least one q prime and the special prime");
    for (uint32_t i = 0; i < count; i++) {
        if (moduli[i] >= (1ULL << 62) || moduli[i] % (2ULL * n) != 1)
            throw std::invalid_argument("every modulus must be < 2^62 and congruent to 1 mod 2N");
    }
    // the caller's current device is restored on return (torch keeps its own notion of it)
    DeviceGuard guard(device);
    // Scratch comes from the device's default stream-ordered pool; keep freed
    // blocks cached across synchronisations instead of returning them to the
    // driver (the default threshold 0 would re-map pages every step).
    cudaMemPool_t pool;
    UH_CHECK(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = ~0ull;
    UH_CHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    Ctx *c = new Ctx();
    c->device = device;
    c->n = n;
    c->count = count;
    while ((1u << c->logn) < n) c->logn++;
    if (n >= 8192) {
        c->n1 = 1u << (c->logn / 2);
        c->n2 = n / c->n1;
    }
    c->h_q.assign(moduli, moduli + count);

    std::vector<Mod> mods(count);
    std::vector<uint64_t> tw((size_t)count * n), tws((size_t)count * n), itw((size_t)count * n),
        itws((size_t)count * n);
    std::vector<double> tfF, itfF;
    std::vector<double2> tfU, itfU, tfR, itfR;
    if (c->n1) {
        tfF.assign((size_t)count * c->n1 * 8, 0.0);
        itfF.assign(tfF.size(), 0.0);
        tfU.assign((size_t)count * 4 * 16, make_double2(0, 0));
        itfU.assign(tfU.size(), make_double2(0, 0));
        tfR.assign((size_t)count * 16, make_double2(0, 0));
        itfR.assign(tfR.size(), make_double2(0, 0));
    }
    for (uint32_t m = 0; m < count; m++) {
        uint64_t q = moduli[m];
        if (h_pow(psi[m], n, q) != q - 1) throw std::invalid_argument("psi is not a primitive 2N-th root of unity");
        Mod &md = mods[m];
        md.q = q;
        md.bar = (uint64_t)((((hu128)1) << 64) / q);
        md.r64 = (uint64_t)((((hu128)1) << 64) % q);
        md.r64s = h_shoup(md.r64, q);
        md.ninv = h_inv(n, q);
        md.ninvs = h_shoup(md.ninv, q);
        std::vector<uint64_t> pw(n), ipw(n);
        uint64_t ip = h_inv(psi[m], q);
        pw[0] = 1;
        ipw[0] = 1;
        for (uint32_t i = 1; i < n; i++) {
            pw[i] = h_mulmod(pw[i - 1], psi[m], q);
            ipw[i] = h_mulmod(ipw[i - 1], ip, q);
        }
        if (c->n1 && (q >> 42) == 0) {  // composite pass-2 twiddles (FP64-pipe limbs only)
            const uint32_t logn = c->logn;
            uint32_t la = 0;  // log2 n1
            while ((1u << la) < c->n1) la++;
            const uint32_t B = logn - la;
            for (uint32_t blk = 0; blk < c->n1; blk++)
                for (uint32_t st = 0; st < B; st++) {
                    const uint32_t e = (1u << (B - 1 - st)) * (1 + 2 * h_brv(blk, la));
                    tfF[((size_t)m * c->n1 + blk) * 8 + st] = (double)pw[e];
                    itfF[((size_t)m * c->n1 + blk) * 8 + st] = (double)ipw[e];
                }
            for (uint32_t sp_ = 0; sp_ + 4 < B; sp_++)
                for (uint32_t u = 0; u < 16; u++) {
                    const uint32_t e = (1u << (logn - 4 - sp_)) * h_brv(u, 4);
                    tfU[((size_t)m * 4 + sp_) * 16 + u] = make_double2((double)pw[e], (double)pw[e] / (double)q);
                    itfU[((size_t)m * 4 + sp_) * 16 + u] = make_double2((double)ipw[e], (double)ipw[e] / (double)q);
                }
            for (uint32_t sp_ = 0; sp_ < 4; sp_++)
                for (uint32_t v = 0; v < (1u << sp_); v++) {
                    const uint32_t e = sp_ ? (1u << (logn - sp_)) * h_brv(v, sp_) : 0;
                    tfR[(size_t)m * 16 + (1u << sp_) - 1 + v] = make_double2((double)pw[e], (double)pw[e] / (double)q);
                    itfR[(size_t)m * 16 + (1u << sp_) - 1 + v] =
                        make_double2((double)ipw[e], (double)ipw[e] / (double)q);
                }
        }
        for (uint32_t i = 0; i < n; i++) {
            uint32_t e = h_brv(i, c->logn);
            size_t at = (size_t)m * n + i;
            tw[at] = pw[e];
            tws[at] = h_shoup(pw[e], q);
            itw[at] = ipw[e];
            itws[at] = h_shoup(ipw[e], q);
        }
    }
    // slot tables
    uint32_t half = n / 2, two_n = 2 * n;
    std::vector<int32_t> dlog(two_n, -1), pos(half), neg(half), sob(n), jof(half, -1);
    uint64_t e = 1;
    for (uint32_t j = 0; j < half; j++) {
        dlog[e] = (int32_t)j;
        jof[(e - 1) / 4] = (int32_t)j;  // e = 1 mod 4 for every power of 5
        dlog[two_n - e] = (int32_t)(half + j);
        pos[j] = (int32_t)((e - 1) / 2);
        neg[j] = (int32_t)((two_n - e - 1) / 2);
        e = e * 5 % two_n;
    }
    for (uint32_t k = 0; k < n; k++) sob[k] = dlog[2 * h_brv(k, c->logn) + 1];
    // pass-2 block selection and per-slot element index for the coalesced
    // slot-order I/O of the fast NTT (see ntt_fast.cu, cta_slot)
    std::vector<int32_t> bsel;
    std::vector<uint8_t> csl;
    if (c->n1) {
        const uint32_t n1 = c->n1, n2 = c->n2, G = 4096 / n2, per_half = (n1 / 2) / G;
        bsel.assign(n1, -1);
        csl.assign(n, 0);
        std::vector<int32_t> k_of(n);
        for (uint32_t k = 0; k < n; k++) {
            csl[sob[k]] = (uint8_t)(k % n2);  // n2 <= 256
            k_of[sob[k]] = (int32_t)k;
        }
        for (uint32_t blk = 0; blk < n1; blk++) {
            uint32_t s0 = (uint32_t)sob[(size_t)blk * n2];
            uint32_t h = s0 / half, j0 = (s0 % half) % (n1 / 2);
            bsel[(size_t)(h * per_half + j0 / G) * G + j0 % G] = (int32_t)blk;
        }
        for (uint32_t x = 0; x < n1 / G; x++)
            for (uint32_t i = 0; i < 4096; i++) {
                uint32_t h = x / per_half, js = (x % per_half) * G;
                uint32_t s = h * half + js + i % G + (n1 / 2) * (i / G);
                if (bsel[(size_t)x * G + i % G] != k_of[s] / (int32_t)n2)
                    throw std::logic_error("NTT pass-2 slot layout invariant violated");
            }
    }
    // cross-modulus inverses
    std::vector<uint64_t> inv((size_t)count * count, 0), invs((size_t)count * count, 0);
    for (uint32_t i = 0; i < count; i++)
        for (uint32_t j = 0; j < count; j++) {
            if (i == j) continue;
            uint64_t v = h_inv(moduli[j] % moduli[i], moduli[i]);
            inv[(size_t)i * count + j] = v;
            invs[(size_t)i * count + j] = h_shoup(v, moduli[i]);
        }
    std::vector<ulonglong2> tw2((size_t)count * n), itw2((size_t)count * n);
    std::vector<double2> twf((size_t)count * n, make_double2(0, 0)), itwf((size_t)count * n, make_double2(0, 0));
    for (size_t i = 0; i < tw2.size(); i++) {
        tw2[i] = make_ulonglong2(tw[i], tws[i]);
        itw2[i] = make_ulonglong2(itw[i], itws[i]);
        const uint64_t q = moduli[i / n];
        if ((q >> 42) == 0) {  // FP64-pipe NTT limbs (ntt_fast.cu, fp_limb)
            twf[i] = make_double2((double)tw[i], (double)tw[i] / (double)q);
            itwf[i] = make_double2((double)itw[i], (double)itw[i] / (double)q);
        }
    }
    if (c->n1) {
        c->d_bsel = upload(bsel);
        c->d_csl = upload(csl);
        c->d_tfF = upload(tfF);
        c->d_itfF = upload(itfF);
        c->d_tfU = upload(tfU);
        c->d_itfU = upload(itfU);
        c->d_tfR = upload(tfR);
        c->d_itfR = upload(itfR);
    }
    // (q_t * P)^-1 mod q_k: the fused ModDown + rescale epilogue (one Shoup product)
    std::vector<uint64_t> inv2((size_t)count * count, 0), inv2s((size_t)count * count, 0);
    for (uint32_t k = 0; k + 1 < count; k++)
        for (uint32_t t = 0; t + 1 < count; t++) {
            if (t == k) continue;
            const uint64_t qk = moduli[k];
            const uint64_t v = h_mulmod(h_inv(moduli[t] % qk, qk), h_inv(moduli[count - 1] % qk, qk), qk);
            inv2[(size_t)k * count + t] = v;
            inv2s[(size_t)k * count + t] = h_shoup(v, qk);
        }
    c->d_inv2 = upload(inv2);
    c->d_inv2s = upload(inv2s);
    std::vector<ulonglong2> pmod(count);
    for (uint32_t i = 0; i < count; i++) {
        uint64_t pm = moduli[count - 1] % moduli[i];
        pmod[i] = make_ulonglong2(pm, h_shoup(pm, moduli[i]));
    }
    c->d_pmod = upload(pmod);
    c->d_tw2 = upload(tw2);
    c->d_itw2 = upload(itw2);
    c->d_twf = upload(twf);
    c->d_itwf = upload(itwf);
    c->d_mods = upload(mods);
    c->h_mods = mods;
    c->h_inv = inv;
    c->h_invs = invs;
    c->d_psi = upload(tw);
    c->d_psis = upload(tws);
    c->d_ipsi = upload(itw);
    c->d_ipsis = upload(itws);
    c->d_sob = upload(sob);
    c->d_inv = upload(inv);
    c->d_invs = upload(invs);
    c->d_pos = upload(pos);
    c->d_neg = upload(neg);
    for (int32_t v : jof)
        if (v < 0) throw std::logic_error("canonical-embedding slot permutation invariant violated");
    c->d_jof = upload(jof);
    return c;
}

void ctx_destroy(Ctx *c) {
    if (!c) return;
    DeviceGuard guard(c->device);
    for (void *p : {(void *)c->d_pmod, (void *)c->d_tfF, (void *)c->d_itfF, (void *)c->d_tfU, (void *)c->d_itfU, (void *)c->d_tfR, (void *)c->d_itfR, (void *)c->d_bsel, (void *)c->d_csl, (void *)c->d_tw2, (void *)c->d_itw2, (void *)c->d_twf, (void *)c->d_itwf, (void *)c->d_mods, (void *)c->d_psi, (void *)c->d_psis,
                    (void *)c->d_ipsi, (void *)c->d_ipsis,
                    (void *)c->d_sob, (void *)c->d_inv, (void *)c->d_invs, (void *)c->d_inv2, (void *)c->d_inv2s, (void *)c->d_pos, (void *)c->d_neg, (void *)c->d_jof})
        if (p) cudaFree(p);
    delete c;
}

}  // namespace uh
