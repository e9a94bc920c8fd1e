"""The engine's hoisted layer path on the host -- TEST INFRASTRUCTURE AND CPU BASELINE ONLY.

``CpuHoistedBackend`` runs the UNCHANGED fused layer code (``paper_2402_03060_b200.fused``:
ModUp once per input, every rotation's key switch and weight-mask MAC in the QP basis,
one fused ModDown + rescale per output) on CPU tensors: each C-ABI call the fused path
issues (``backend._call("uh_...", ...)``, same arguments and layouts) is served by the
OpenMP C port in ``oracle/ckks_hoisted.c`` instead of a CUDA kernel.  Keys come from the
oracle's key generation (bit-identical to the GPU's), so on the same ciphertexts and mask
banks a GPU step and this port produce identical residues (tests/test_gpu_cpu_port.py).

Used as (1) the hoisted CPU baseline of bench.py (``cpu_baseline.kind = "port-hoisted"``,
the survey's "same algorithm on all host cores"), and (2) a whole-network residue pin of
the GPU fused path.  Never imported by the product package.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from oracle import ckks_oracle as oc
from paper_2402_03060_b200.counter import OpCounter
from paper_2402_03060_b200.he_backend import CipherVector, GpuBackend
from paper_2402_03060_b200.params import HEParams, rns_chain

_I, _D, _P = ctypes.c_int, ctypes.c_double, ctypes.c_void_p
_SIGS = {
    "hc_elementwise": [_P, _I, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I],
    "hc_elementwise_grouped": [_P, _I, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I],
    "hc_from_signed": [_P, _P, _P, _I, _I, _I, _I],
    "hc_modup": [_P, _P, _P, _I, _I, _I],
    "hc_divide_top": [_P, _P, _P, _I, _I, _I, _I, _I],
    "hc_divide_top2": [_P, _P, _P, _I, _I, _I, _I],
    "hc_mul_relin_rescale_fused": [_P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _I],
    "hc_hoisted_mac_bank": [_P, _P, _P, _I, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I],
}


def _clib():
    lib = oc.lib()
    if not getattr(lib, "_hc_typed", False):
        for name, args in _SIGS.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = None
        lib._hc_typed = True
    return lib


def _addr(p) -> int:
    return p.value if isinstance(p, ctypes.c_void_p) else int(p)


def _view(p, dtype, count: int) -> np.ndarray:
    ct = {np.float64: ctypes.c_double, np.int64: ctypes.c_int64}[dtype]
    return np.ctypeslib.as_array((ct * count).from_address(_addr(p)))


class CpuHoistedBackend(GpuBackend):
    """GpuBackend's interface on CPU tensors, every engine call served by ckks_hoisted.c."""

    def __init__(self, params: HEParams):  # noqa: D107 (no CUDA init); threads: OMP_NUM_THREADS at process start
        if params.seed is None:
            raise ValueError("the CPU port derives its keys from the oracle: give HEParams an explicit seed")
        self.params = params
        self._secret_seed = self._enc_seed = params.seed
        self.counter = OpCounter()
        self.chain = rns_chain(params)
        self.n = params.poly_degree
        self.depth = params.depth
        self.count = len(self.chain.moduli)
        self.sp = self.count - 1
        self.device = torch.device("cpu")
        self.scale0 = float(2 ** params.scale_bits)
        self.o = oc.Oracle(params)
        self._ctx = ctypes.c_void_p(self.o._ctx)
        self._s = self.o.secret()
        self.secret = torch.from_numpy(self._s.view(np.int64))
        self._gk, self._rk, self._ct_id = {}, None, 0
        self._lib = _clib()

    def __del__(self):
        pass

    # -- plumbing --------------------------------------------------------------
    def _stream(self):
        return ctypes.c_void_p(0)

    def _empty(self, *shape) -> torch.Tensor:
        return torch.empty(shape, dtype=torch.int64)

    def kernel_supported(self, name: str, *args) -> bool:
        return name == "uh_hoisted_bank_supported"  # the generic key-bank MAC; no tensor-core kernels

    def _call(self, name, *args):
        L, c = self._lib, self._ctx
        a = list(args)
        if name == "uh_modup":  # D, in, n_polys, level, in_ps, stream
            L.hc_modup(c, *a[:5])
        elif name == "uh_hoisted_mac_bank":  # acc, X, xls, D, masks, kbank, shifts, B, I, T, O, diag, level, st
            L.hc_hoisted_mac_bank(c, *a[:13])
        elif name == "uh_divide_top":  # out, in, n_polys, nl, top_mod, out_ps, in_ps, st
            L.hc_divide_top(c, *a[:7])
        elif name == "uh_rescale":  # out, in, B, level, out_ls, in_ls, st (both components)
            L.hc_divide_top(c, a[0], a[1], 2 * int(a[2]), int(a[3]), int(a[3]), a[4], a[5])
        elif name == "uh_divide_top2":  # out, in, n_polys, level, out_ps, in_ps, st
            L.hc_divide_top2(c, *a[:6])
        elif name == "uh_elementwise":  # op, out, a, b, n_polys, b_polys, nl, nq, out_ps, a_ps, b_ps, st
            L.hc_elementwise(c, *a[:11])
        elif name == "uh_elementwise_grouped":  # op, out, a, b, n_polys, b_polys, group, nl, nq, ..., st
            L.hc_elementwise_grouped(c, *a[:12])
        elif name == "uh_mul_relin_rescale_fused":  # out, a, b, B, level, out_ls, a_ls, b_ls, rk, rk_limbs, st
            L.hc_mul_relin_rescale_fused(c, *a[:10])
        elif name == "uh_from_signed_qp":  # out, coef, n_polys, nq, out_ps, st
            L.hc_from_signed(c, a[0], a[1], a[2], a[3], 1, a[4])
        elif name == "uh_from_signed":  # out, coef, n_polys, nl, out_ps, st
            L.hc_from_signed(c, a[0], a[1], a[2], a[3], 0, a[4])
        elif name == "uh_encode_coeffs":  # coef, slots, n_polys, scale, st
            rows, half = int(a[2]), self.params.num_slots
            coef = _view(a[0], np.int64, rows * self.n).reshape(rows, self.n)
            vals = _view(a[1], np.float64, rows * half).reshape(rows, half)
            for r in range(rows):
                coef[r] = oc.encode_coeffs(vals[r], float(a[3]), self.n)
        else:
            raise NotImplementedError(f"the CPU port has no {name}")

    # -- keys (the oracle's key generation: bit-identical to uh_galois_keygen / uh_relin_keygen) --
    def galois_key(self, r: int, level: int) -> torch.Tensor:
        r %= self.params.num_slots
        key = self._gk.get(r)
        if key is None or key.shape[0] < level + 1:
            key = torch.from_numpy(self.o.galois_key(self._s, r, level).view(np.int64))
            self._gk[r] = key
        return key

    def relin_key(self, level: int) -> torch.Tensor:
        if self._rk is None or self._rk.shape[0] < level + 1:
            self._rk = torch.from_numpy(self.o.relin_key(self._s, level).view(np.int64))
        return self._rk

    # -- client side (encrypt / decrypt) -------------------------------------------
    def _encrypt_encoded(self, pt: torch.Tensor) -> CipherVector:
        lev = self.depth
        m = pt.numpy().view(np.uint64)
        cts = [self.o.encrypt_eval(m[b], self._s, lev, self._ct_id + b) for b in range(m.shape[0])]
        self._ct_id += m.shape[0]
        return CipherVector(torch.from_numpy(np.stack(cts).view(np.int64)), lev, self.scale0, self)

    def decrypt_device(self, c: CipherVector) -> torch.Tensor:
        c = self._ready(c)
        data = c.data.numpy().view(np.uint64)
        rows = [oc.decode_coeffs(self.o.decrypt_coeffs(data[b], self._s), c.scale, self.n)
                for b in range(data.shape[0])]
        return torch.from_numpy(np.stack(rows))
