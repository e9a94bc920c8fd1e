"""The reference engine's own operator stream replayed through GpuBackend.

tests/golden/opstream_m2_n4096.npz was recorded in the build container by running the
unmodified reference ``slotcnn.run_inference`` (engine.py:196-208) over builtin M2 at
N = 2^12 with a recording subclass of the reference ``Backend`` (tests/golden/make_opstream.py).
Here every recorded call -- encode / encrypt / add / mul_plain / mul_cipher / rotate / decrypt,
with the reference's own plaintext masks -- is issued, in order, against GpuBackend (real
RNS-CKKS on the B200).  That is the drop-in claim of INTEGRATION.md section 1 exercised on
hardware: the reference's layer constructions (layers.py) driving the B200 backend op for op.

Checks: decrypted outputs vs the reference simulator's decrypted vectors and its logits vs the
plaintext forward pass (CKKS tolerance), and the GPU backend's op census identical to the
reference's (kind, level) histogram.
"""

import os

import numpy as np
import pytest

from paper_2402_03060_b200.he_backend import GpuBackend, PlainVector
from paper_2402_03060_b200.params import HEParams

FIX = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "opstream_m2_n4096.npz")
ENCRYPT, ADD_CT, ADD_PT, MUL_PLAIN, MUL_CIPHER, ROTATE, DECRYPT = range(7)


def _plaintexts(z, slots):
    out = []
    for i, kind in enumerate(z["p_kind"]):
        v = np.zeros(slots)
        if kind == 0:
            p = z["p_pat"][i]
            v[z["pat_idx"][z["pat_off"][p]:z["pat_off"][p + 1]]] = z["p_scalar"][i]
        elif kind == 1:
            a, b = z["p_sp_off"][i], z["p_sp_off"][i + 1]
            v[z["p_sp_idx"][a:b]] = z["p_sp_val"][a:b]
        out.append(PlainVector(v))
    return out


def replay(be, z):
    """Issue the recorded calls against backend ``be``; returns {decrypt index: slots}."""
    plains = _plaintexts(z, be.params.num_slots)
    if not isinstance(be, GpuBackend):  # the slot restatement has its own plaintext type
        plains = [be._plain(p.values) for p in plains]
    ops = z["ops"]

    def ct_operands(code, a, b):
        if code in (ADD_CT, MUL_CIPHER):
            return (a, b)
        if code in (ADD_PT, MUL_PLAIN, ROTATE, DECRYPT):
            return (a,)
        return ()

    last = {}
    for k, (code, out, a, b, r) in enumerate(ops):
        for h in ct_operands(code, a, b):
            last[h] = k
    cts, got = {}, {}
    for k, (code, out, a, b, r) in enumerate(ops):
        if code == ENCRYPT:
            cts[out] = be.encrypt(plains[a])
        elif code == ADD_CT:
            cts[out] = be.add(cts[a], cts[b])
        elif code == ADD_PT:
            cts[out] = be.add(cts[a], plains[b])
        elif code == MUL_PLAIN:
            cts[out] = be.mul_plain(cts[a], plains[b])
        elif code == MUL_CIPHER:
            cts[out] = be.mul_cipher(cts[a], cts[b])
        elif code == ROTATE:
            cts[out] = be.rotate(cts[a], int(r))
        elif code == DECRYPT:
            got[int(r)] = np.asarray(be.decrypt(cts[a]))
        for h in set(ct_operands(code, a, b)):  # free ciphertexts after their last use
            if last[h] == k:
                cts.pop(h, None)
    return got


def _hist(z):
    return {(str(k), int(lv)): int(c) for k, lv, c in zip(z["hist_kind"], z["hist_level"], z["hist_count"])}


def test_reference_opstream_replays_on_slot_restatement():
    """CPU check of the fixture and the replay loop: through the slot restatement the recorded
    stream reproduces the reference's decrypted vectors bit for bit and its census."""
    from oracle.slot_sim import SimBackend

    z = np.load(FIX)
    n, depth, sb = (int(x) for x in z["params"])
    be = SimBackend(HEParams(poly_degree=n, depth=depth, scale_bits=sb))
    got = replay(be, z)
    for i in range(z["decrypted"].shape[0]):
        assert np.array_equal(got[i], z["decrypted"][i])
    assert be.counter.by_level == _hist(z)


@pytest.mark.gpu
def test_reference_opstream_replays_on_gpu():
    z = np.load(FIX)
    n, depth, sb = (int(x) for x in z["params"])
    be = GpuBackend(HEParams(poly_degree=n, depth=depth, scale_bits=sb))
    got = replay(be, z)
    dec = z["decrypted"]
    assert len(got) == dec.shape[0]
    for i in range(dec.shape[0]):
        scale = max(1.0, float(np.max(np.abs(dec[i]))))
        assert np.max(np.abs(got[i] - dec[i])) / scale < 1e-5
    assert np.max(np.abs(z["outputs"] - z["refs"])) < 1e-9  # the recorded reference run itself
    assert be.counter.by_level == _hist(z)
