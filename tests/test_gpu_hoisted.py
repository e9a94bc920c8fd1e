"""Residue-level parity of the hoisted rotation-MAC kernels (hoist.cu) against the CPU oracle.

uh_hoisted_mac forms, in the QP basis and without ModDown,

    acc[o][b] = sum_{i, t} M[o][i*T + t] (.) P * rot_{s_t}(ct_i[b])

where P * rot_s(ct) is the hoisted key-switched rotation (ModUp digits of c1
read at the rotated slots, inner product with the Galois key, plus P * rot(c0)).
The reference restates that sum term by term with the oracle's own ModUp, key
inner product, slot rotation and modular products, and the GPU accumulators
must match it on every residue.  Output counts and mask/no-mask cases are chosen
so every kernel the dispatcher picks runs: the register-only direct kernel
(1-2 outputs, 3-4 outputs), the shared-memory tiled kernel (5, 6, 12 outputs)
and unmasked rotation sums.  The chain is the BASELINE shape (60-bit q_0 and P,
40-bit middle primes), so both the narrow-operand (q < 2^41) and the full
128-bit accumulator paths are exercised; masks are uniform residues up to q - 1
(worst-case operand sizes).
"""

import numpy as np
import pytest
import torch

from oracle.ckks_oracle import Oracle
from paper_2402_03060_b200 import fused
from paper_2402_03060_b200.he_backend import GpuBackend
from paper_2402_03060_b200.params import HEParams

pytestmark = pytest.mark.gpu

PARAMS = HEParams(poly_degree=1 << 12, depth=5, scale_bits=40, seed=4)
_CACHE = {}


def _pair():
    if "p" not in _CACHE:
        _CACHE["p"] = (GpuBackend(PARAMS), Oracle(PARAMS))
    return _CACHE["p"]


def _reference(o, s, X, level, shifts, masks, O, B):
    """acc [O][B][2][L+1][N] restated with oracle primitives (one term at a time)."""
    L, n, half = level + 1, o.n, o.n // 2
    qp = o.qp_mods(level)
    P = int(o.moduli[o.sp])
    pvec = np.stack([np.full(n, P % int(o.moduli[m]), dtype=np.uint64) for m in qp])
    I, T = X.shape[0], len(shifts)
    keys = {r % half: o.galois_key(s, r % half, level) for r in shifts if r % half}
    acc = np.zeros((O, B, 2, L + 1, n), dtype=np.uint64)
    for i in range(I):
        for b in range(B):
            c0, c1 = X[i, b, 0, :L], X[i, b, 1, :L]
            D = o.modup(c1, level)  # [L digits][L + 1][N]
            for t, r in enumerate(shifts):
                r %= half
                u = np.zeros((2, L + 1, n), dtype=np.uint64)
                if r == 0:
                    u[0, :L] = o.mul(c0, pvec[:L], qp[:L])
                    u[1, :L] = o.mul(c1, pvec[:L], qp[:L])
                else:
                    Dr = o.rotate_slots(D.reshape(-1, n), r).reshape(D.shape)
                    u = o.key_inner(Dr, keys[r], level)
                    pc0 = o.mul(o.rotate_slots(c0, r), pvec[:L], qp[:L])
                    u[0, :L] = o.add(u[0, :L], pc0, qp[:L])
                for out in range(O):
                    for c in range(2):
                        term = u[c] if masks is None else o.mul(masks[out, i * T + t], u[c], qp)
                        acc[out, b, c] = o.add(acc[out, b, c], term, qp)
    return acc


@pytest.mark.parametrize("O,with_masks", [(1, True), (2, True), (3, True), (4, True), (5, True), (6, True),
                                          (12, True), (1, False), (3, False)])
def test_hoisted_mac_bit_exact_vs_oracle(O, with_masks):
    be, o = _pair()
    s = o.secret()
    level, B, I = 4, 3, 2
    shifts = [0, 1, -3, 7, 64]
    rng = np.random.default_rng(10 + O)
    cts = [be.encrypt(be.encode_batch(rng.uniform(-1, 1, size=(B, PARAMS.num_slots)))) for _ in range(I)]
    X = fused.stack_cts(be, cts, level)  # [I][B][2][L][N]
    qp = o.qp_mods(level)
    masks = None
    mdev = None
    if with_masks:
        masks = np.zeros((O, I * len(shifts), level + 2, o.n), dtype=np.uint64)
        for k, m in enumerate(qp):
            masks[:, :, k] = rng.integers(0, int(o.moduli[m]), size=(O, I * len(shifts), o.n), dtype=np.uint64)
        mdev = torch.from_numpy(masks.view(np.int64)).to(be.device)
    got = fused._hoist(be, X, level, shifts, mdev, O, False, B)
    torch.cuda.synchronize()
    want = _reference(o, s, X.cpu().numpy().view(np.uint64), level, shifts, masks, O, B)
    assert np.array_equal(got.cpu().numpy().view(np.uint64), want)


def test_hoisted_diag_bit_exact_vs_oracle():
    """Term mode 1 (input i with its own shift i), the pooling / flatten rotation sum."""
    be, o = _pair()
    s = o.secret()
    level, B = 3, 2
    shifts = [0, 5, -11]
    rng = np.random.default_rng(3)
    cts = [be.encrypt(be.encode_batch(rng.uniform(-1, 1, size=(B, PARAMS.num_slots)))) for _ in shifts]
    X = fused.stack_cts(be, cts, level)
    got = fused._hoist(be, X, level, shifts, None, 1, True, B).cpu().numpy().view(np.uint64)
    Xh = X.cpu().numpy().view(np.uint64)
    qp = o.qp_mods(level)
    want = _reference(o, s, Xh[0:1], level, [shifts[0]], None, 1, B)
    for i in range(1, len(shifts)):
        part = _reference(o, s, Xh[i:i + 1], level, [shifts[i]], None, 1, B)
        for b in range(B):
            for c in range(2):
                want[0, b, c] = o.add(want[0, b, c], part[0, b, c], qp)
    assert np.array_equal(got, want)


C2 = HEParams(poly_degree=1 << 15, depth=9, scale_bits=40, seed=6)  # BASELINE config-2 chain


def _c2():
    if "c2" not in _CACHE:
        _CACHE["c2"] = (GpuBackend(C2), Oracle(C2))
    return _CACHE["c2"]


def _rand_masks(o, rng, O, Q, level):
    masks = np.zeros((O, Q, level + 2, o.n), dtype=np.uint64)
    for k, m in enumerate(o.qp_mods(level)):
        masks[:, :, k] = rng.integers(0, int(o.moduli[m]), size=(O, Q, o.n), dtype=np.uint64)
    return masks


@pytest.mark.parametrize("O,level", [(12, 5), (5, 2), (1, 7)])
def test_key_bank_kernel_bit_exact_vs_oracle(O, level, monkeypatch):
    """The key-bank kernel (hoist_bank.cu, N = 2^15 only) on the BASELINE chain, residue for residue."""
    monkeypatch.setenv("UH_KEY_BANK", "1")
    be, o = _c2()
    assert fused._key_bank_ok(be, level, O)
    s = o.secret()
    B, I = 3, 2
    shifts = [0, 1, 28, -29, 16383]
    rng = np.random.default_rng(20 + O)
    cts = [be.encrypt(be.encode_batch(rng.uniform(-1, 1, size=(B, C2.num_slots)))) for _ in range(I)]
    X = fused.stack_cts(be, cts, level)
    masks = _rand_masks(o, rng, O, I * len(shifts), level)
    got = fused._hoist(be, X, level, shifts, torch.from_numpy(masks.view(np.int64)).to(be.device), O, False, B)
    want = _reference(o, s, X.cpu().numpy().view(np.uint64), level, shifts, masks, O, B)
    assert np.array_equal(got.cpu().numpy().view(np.uint64), want)


def test_key_bank_kernel_equals_generic_at_lenet_conv2_shape(monkeypatch):
    """LeNet conv2 shape (4 inputs x 25 taps, 12 outputs, level 5): bank kernel == generic kernel, bit for bit."""
    be, o = _c2()
    level, B, I, O = 5, 5, 4, 12
    shifts = [a + 28 * b for b in range(5) for a in range(5)]
    rng = np.random.default_rng(9)
    cts = [be.encrypt(be.encode_batch(rng.uniform(-1, 1, size=(B, C2.num_slots)))) for _ in range(I)]
    X = fused.stack_cts(be, cts, level)
    mdev = torch.from_numpy(_rand_masks(o, rng, O, I * len(shifts), level).view(np.int64)).to(be.device)
    monkeypatch.setenv("UH_KEY_BANK", "1")
    got = fused._hoist(be, X, level, shifts, mdev, O, False, B)
    monkeypatch.setenv("UH_KEY_BANK", "0")
    want = fused._hoist(be, X, level, shifts, mdev, O, False, B)
    assert torch.equal(got, want)


@pytest.mark.parametrize("O,with_masks,diag", [(1, True, 0), (2, True, 0), (3, True, 0), (4, True, 0),
                                               (1, False, 0), (3, False, 0), (1, False, 1), (2, True, 2)])
def test_key_bank_kernels_equal_generic_every_mode(O, with_masks, diag, monkeypatch):
    """Register-only key-bank kernel (narrow layers, rotation sums, diagonal / block-diagonal terms) ==
    the generic kernel (oracle-pinned above), bit for bit, at N = 2^15 on the BASELINE chain."""
    be, o = _c2()
    level, B = 3, 9  # B not a multiple of the 8-ciphertext CTA tile
    if diag == 1:
        I, shifts, taps, Q = 3, [0, 5, -11], None, 3
    elif diag == 2:
        I, shifts, taps = 2, [1, 29, -3, 0], 2
        Q = 4
    else:
        I, shifts, taps = 2, [0, 1, 28, -29, 16383], None
        Q = I * len(shifts)
    rng = np.random.default_rng(40 + O + diag)
    cts = [be.encrypt(be.encode_batch(rng.uniform(-1, 1, size=(B, C2.num_slots)))) for _ in range(I)]
    X = fused.stack_cts(be, cts, level)
    mdev = None
    if with_masks:
        mdev = torch.from_numpy(_rand_masks(o, rng, O, Q, level).view(np.int64)).to(be.device)
    mode = 2 if diag == 2 else bool(diag)
    monkeypatch.setenv("UH_KEY_BANK", "1")
    got = fused._hoist(be, X, level, shifts, mdev, O, mode, B, taps=taps)
    monkeypatch.setenv("UH_KEY_BANK", "0")
    want = fused._hoist(be, X, level, shifts, mdev, O, mode, B, taps=taps)
    assert torch.equal(got, want)


@pytest.mark.parametrize("diag,I,T", [(0, 2, 35), (2, 3, 12), (1, 3, 3), (0, 1, 4)])
def test_key_mask_bank_kernel_equals_masked_kernel(diag, I, T, monkeypatch):
    """One masked output over the key-mask bank (masks folded into the key rows, hoist_bank.cu
    k_km_bank / k_direct_bank<PRE>) == the masked register-only kernel (oracle-pinned above), bit
    for bit, in every term mode; enough terms that the running sums fold (wide limbs: 240 MACs)."""
    be, o = _c2()
    level, B = 3, 9
    rng = np.random.default_rng(70 + diag + T)
    if diag == 1:
        shifts, taps, Q = [0, 5, -11], None, 3
    elif diag == 2:
        shifts = [int(x) for x in rng.choice(np.arange(1, 400), size=I * T, replace=False)]
        shifts[5] = 0
        taps, Q = T, I * T
    else:
        shifts = [0] + [int(x) for x in rng.choice(np.arange(1, 400), size=T - 1, replace=False)]
        taps, Q = None, I * T
    cts = [be.encrypt(be.encode_batch(rng.uniform(-1, 1, size=(B, C2.num_slots)))) for _ in range(I)]
    X = fused.stack_cts(be, cts, level)
    mdev = torch.from_numpy(_rand_masks(o, rng, 1, Q, level).view(np.int64)).to(be.device)
    mode = 2 if diag == 2 else bool(diag)
    monkeypatch.setenv("UH_KM_BANK", "1")
    assert fused._km_ok(be, level)
    from paper_2402_03060_b200 import _lib

    launches = _lib.launch_count()
    got = fused._hoist(be, X, level, shifts, mdev, 1, mode, B, taps=taps)
    monkeypatch.setenv("UH_KM_BANK", "0")
    want = fused._hoist(be, X, level, shifts, mdev, 1, mode, B, taps=taps)
    assert torch.equal(got, want)
    assert _lib.launch_count() > launches


def test_long_unmasked_rotation_sum_folds(monkeypatch):
    """An unmasked rotation sum long enough that the register-only kernel folds its running sums
    (60 terms x 9 MACs > the 240-MAC budget of the 60-bit limbs) == the generic kernel."""
    be, o = _c2()
    level, B, I = 3, 3, 1
    rng = np.random.default_rng(81)
    shifts = [0] + [int(x) for x in rng.choice(np.arange(1, 300), size=59, replace=False)]
    cts = [be.encrypt(be.encode_batch(rng.uniform(-1, 1, size=(B, C2.num_slots)))) for _ in range(I)]
    X = fused.stack_cts(be, cts, level)
    monkeypatch.setenv("UH_KEY_BANK", "1")
    got = fused._hoist(be, X, level, shifts, None, 1, False, B)
    monkeypatch.setenv("UH_KEY_BANK", "0")
    want = fused._hoist(be, X, level, shifts, None, 1, False, B)
    assert torch.equal(got, want)


@pytest.mark.parametrize("O,level,I,shifts,B", [
    (12, 5, 4, [a + 28 * b for b in range(5) for a in range(5)], 5),   # LeNet conv2 shape, partial ct tile
    (7, 3, 3, [0, 1, 28, -29, 16383, 57, -2, 3, 700], 4),              # partial m-tile, Q = 27 (not / 4)
    (5, 2, 2, [0, 1, 28, -29, 16383], 3),                              # one k-step, 2 m-tiles
    (9, 8, 1, [3, 0, -5], 9),                                          # high level, 3 terms, 3 ct tiles
    (6, 2, 16, [a + 32 * b for b in range(4) for a in range(4)], 5),   # CIFAR conv2 terms: Q = 256, 8 k-steps
    (5, 3, 5, [a + 28 * b for b in range(5) for a in range(5)], 4),    # Q = 125: 4 k-steps, one short
    (7, 2, 6, [a + 28 * b for b in range(5) for a in range(5)], 6),    # Q = 150: 5 k-steps (wide tile)
    (32, 2, 4, [a + 32 * b for b in range(4) for a in range(4)], 5),   # CIFAR conv2 outputs: 11 m-tiles, 3 q_0/P groups
    (16, 3, 3, [0, 1, 2, 32, 33, 34, 64, 65, 66], 4),                  # CIFAR conv1 shape: 6 m-tiles, 12 + 4 on q_0/P
])
def test_imma_kernel_equals_key_bank_kernel(O, level, I, shifts, B, monkeypatch):
    """Tensor-core mask contraction (hoist_imma.cu: byte-split u8 IMMA on the 40-bit limbs, the IMAD
    kernel on q_0 and P) == the key-bank IMAD kernel (oracle-pinned above), residue for residue, with
    worst-case (uniform up to q - 1) masks."""
    be, o = _c2()
    monkeypatch.setenv("UH_TC", "0")  # the mma.sync kernel, not the tcgen05 one
    monkeypatch.setenv("UH_IMMA_TA", "0")  # IMAD phase A (the tensor-core phase A has its own test below)
    rng = np.random.default_rng(70 + O + level)
    cts = [be.encrypt(be.encode_batch(rng.uniform(-1, 1, size=(B, C2.num_slots)))) for _ in range(I)]
    X = fused.stack_cts(be, cts, level)
    mdev = torch.from_numpy(_rand_masks(o, rng, O, I * len(shifts), level).view(np.int64)).to(be.device)
    monkeypatch.setenv("UH_IMMA", "1")
    assert fused._imma_ok(be, level, O, I * len(shifts))
    got = fused._hoist(be, X, level, shifts, mdev, O, False, B)
    monkeypatch.setenv("UH_IMMA", "0")
    want = fused._hoist(be, X, level, shifts, mdev, O, False, B)
    assert torch.equal(got, want)


@pytest.mark.parametrize("O,level,I,shifts,B", [
    (12, 5, 4, [a + 28 * b for b in range(5) for a in range(5)], 21),  # LeNet conv2 shape, 16 + 5 ciphertexts
    (12, 5, 4, [a + 28 * b for b in range(5) for a in range(5)], 16),  # one full 16-ciphertext tile
    (7, 3, 3, [0, 1, 28, -29, 16383, 57, -2, 3, 700], 4),              # partial m-tile, Q = 27, zero shift
    (5, 2, 2, [0, 1, 28, -29, 16383], 3),                              # one k-step, 15 digit bytes
    (5, 3, 5, [a + 28 * b for b in range(5) for a in range(5)], 9),    # Q = 125: 4 k-steps, one short; rows 8.. empty but one
    (48, 4, 2, [0, 5, -7, 64], 33),                                    # 16 m-tiles, three ciphertext tiles
])
def test_imma_tensor_phase_a_equals_key_bank_kernel(O, level, I, shifts, B, monkeypatch):
    """Key switch on the tensor cores (hoist_imma.cu k_hoisted_imma_ta: digit bytes x byte-weighted key
    bytes, quad recombination, P c0 pre-multiplied) + IMMA mask contraction == the key-bank IMAD kernel
    (oracle-pinned above), residue for residue, with worst-case masks."""
    be, o = _c2()
    monkeypatch.setenv("UH_TC", "0")
    monkeypatch.setenv("UH_IMMA_TA", "1")
    rng = np.random.default_rng(170 + O + level)
    cts = [be.encrypt(be.encode_batch(rng.uniform(-1, 1, size=(B, C2.num_slots)))) for _ in range(I)]
    X = fused.stack_cts(be, cts, level)
    mdev = torch.from_numpy(_rand_masks(o, rng, O, I * len(shifts), level).view(np.int64)).to(be.device)
    monkeypatch.setenv("UH_IMMA", "1")
    assert fused._imma_ok(be, level, O, I * len(shifts)) and fused._imma_ta_ok(be, level, O, I * len(shifts), B)
    got = fused._hoist(be, X, level, shifts, mdev, O, False, B)
    monkeypatch.setenv("UH_IMMA", "0")
    want = fused._hoist(be, X, level, shifts, mdev, O, False, B)
    assert torch.equal(got, want)


def test_tensor_phase_a_selection(monkeypatch):
    """The tensor-core phase A serves the shapes it is compiled for (level + 1 <= 6, <= 128 terms) and
    only batches that fill its 16-ciphertext tiles; everything else keeps the IMAD phase A."""
    be, _ = _c2()
    monkeypatch.delenv("UH_IMMA_TA", raising=False)
    assert fused._imma_ta_ok(be, 5, 12, 100, 128) and fused._imma_ta_ok(be, 5, 12, 100, 13)
    assert not fused._imma_ta_ok(be, 5, 12, 100, 1) and not fused._imma_ta_ok(be, 5, 12, 100, 17)
    assert not fused._imma_ta_ok(be, 6, 12, 100, 128)   # 7 digits: 35 bytes > one k-step
    assert not fused._imma_ta_ok(be, 5, 12, 150, 128)   # > 128 terms
    monkeypatch.setenv("UH_IMMA_TA", "0")
    assert not fused._imma_ta_ok(be, 5, 12, 100, 128)


@pytest.mark.parametrize("O,level,I,shifts,B", [
    (12, 5, 4, [a + 28 * b for b in range(5) for a in range(5)], 13),  # LeNet conv2 shape, partial ct tiles
    (4, 7, 1, [a + 28 * b for b in range(5) for a in range(5)], 9),    # LeNet conv1 shape (O <= 8: M = 64 on q_0 / P)
    (9, 3, 3, [0, 1, 28, -29, 16383, 57, -2, 3, 700], 4),              # Q = 27 (not / 4), 8 < O: M = 128
    (1, 2, 2, [0, 1, 28, -29, 16383], 3),                              # one output, one K-step
    (7, 8, 1, [3, 0, -5], 5),                                          # high level, 3 terms
])
def test_tcgen05_kernel_equals_key_bank_kernel(O, level, I, shifts, B, monkeypatch):
    """The tcgen05 kernel (hoist_tc.cu: byte-split u8 tcgen05.mma kind::i8 with TMEM accumulators on
    every limb -- 5-byte operands on the 40-bit limbs, 8-byte on q_0 and P) == the key-bank IMAD
    kernel (oracle-pinned above), residue for residue, with worst-case (uniform up to q - 1) masks."""
    be, o = _c2()
    rng = np.random.default_rng(90 + O + level)
    cts = [be.encrypt(be.encode_batch(rng.uniform(-1, 1, size=(B, C2.num_slots)))) for _ in range(I)]
    X = fused.stack_cts(be, cts, level)
    mdev = torch.from_numpy(_rand_masks(o, rng, O, I * len(shifts), level).view(np.int64)).to(be.device)
    monkeypatch.setenv("UH_TC", "1")
    assert fused._tc_ok(be, level, O, I * len(shifts))
    got = fused._hoist(be, X, level, shifts, mdev, O, False, B)
    monkeypatch.setenv("UH_TC", "0")
    monkeypatch.setenv("UH_IMMA", "0")
    want = fused._hoist(be, X, level, shifts, mdev, O, False, B)
    assert torch.equal(got, want)


def test_tcgen05_kernel_vs_oracle(monkeypatch):
    """The tcgen05 kernel directly against the CPU oracle (no transitive pin): 2 inputs x 5 shifts,
    12 outputs, level 5 on the BASELINE chain."""
    monkeypatch.setenv("UH_TC", "1")  # opt-in path
    be, o = _c2()
    s = o.secret()
    B, I, O, level = 2, 2, 12, 5
    shifts = [0, 1, 28, -29, 16383]
    rng = np.random.default_rng(99)
    cts = [be.encrypt(be.encode_batch(rng.uniform(-1, 1, size=(B, C2.num_slots)))) for _ in range(I)]
    X = fused.stack_cts(be, cts, level)
    masks = _rand_masks(o, rng, O, I * len(shifts), level)
    assert fused._tc_ok(be, level, O, I * len(shifts))
    got = fused._hoist(be, X, level, shifts, torch.from_numpy(masks.view(np.int64)).to(be.device), O, False, B)
    want = _reference(o, s, X.cpu().numpy().view(np.uint64), level, shifts, masks, O, B)
    assert np.array_equal(got.cpu().numpy().view(np.uint64), want)
