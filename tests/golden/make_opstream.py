"""Record the reference engine's own operator stream (build container only).

Runs the UNMODIFIED reference ``slotcnn.run_inference`` (pkg/src/slotcnn/engine.py:196-208)
on builtin M2 (LeNet-1, model.py:663-675) at N = 2^12 with a recording subclass of the
reference ``Backend`` (he_backend.py:155-253): every encode / _plain / encrypt / add /
mul_plain / mul_cipher / rotate / decrypt the reference's layers.py issues is logged with
handle ids, together with the plaintext values it passes, the reference's decrypted outputs
and its op census.  tests/test_gpu_opstream.py replays the stream through GpuBackend on the
GPU box (where the reference is absent): that is the reference's own engine driving the
B200 backend through the operator boundary, op for op.

Plaintexts are stored compactly: a mask that is one scalar times a 0/1 position pattern
(every conv / pool / bias mask, layers.py:183-195) as (pattern id, scalar), anything else as
sparse (index, value) pairs.

    python tests/golden/make_opstream.py      # writes tests/golden/opstream_m2_n4096.npz
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"

OPS = {"encrypt": 0, "add_ct": 1, "add_pt": 2, "mul_plain": 3, "mul_cipher": 4, "rotate": 5, "decrypt": 6}


def record(n_log: int = 12, depth: int = 7, seed: int = 5):
    sys.path.insert(0, REF)
    import slotcnn
    from slotcnn import he_backend as hb

    ops, plains, decrypted = [], [], []
    handles = {}  # id(obj) -> handle; objects kept alive in `keep` so ids are never reused
    keep = []

    def hid(obj, kind):
        key = id(obj)
        if key not in handles:
            handles[key] = (kind, len(plains) if kind == "p" else sum(1 for v in handles.values() if v[0] == "c"))
            keep.append(obj)
            if kind == "p":
                plains.append(np.array(obj.values, dtype=np.float64))
        return handles[key][1]

    class Rec(hb.Backend):
        def encode(self, data):
            p = super().encode(data)
            hid(p, "p")
            return p

        def _plain(self, arr):
            p = super()._plain(arr)
            hid(p, "p")
            return p

        def encrypt(self, plain):
            c = super().encrypt(plain)
            ops.append((OPS["encrypt"], hid(c, "c"), hid(plain, "p"), -1, 0))
            return c

        def add(self, a, b):
            c = super().add(a, b)
            if isinstance(b, hb.PlainVector):
                ops.append((OPS["add_pt"], hid(c, "c"), hid(a, "c"), hid(b, "p"), 0))
            else:
                ops.append((OPS["add_ct"], hid(c, "c"), hid(a, "c"), hid(b, "c"), 0))
            return c

        def mul_plain(self, cipher, plain):
            c = super().mul_plain(cipher, plain)
            ops.append((OPS["mul_plain"], hid(c, "c"), hid(cipher, "c"), hid(plain, "p"), 0))
            return c

        def mul_cipher(self, a, b):
            c = super().mul_cipher(a, b)
            ops.append((OPS["mul_cipher"], hid(c, "c"), hid(a, "c"), hid(b, "c"), 0))
            return c

        def rotate(self, cipher, r):
            c = super().rotate(cipher, r)
            ops.append((OPS["rotate"], hid(c, "c"), hid(cipher, "c"), -1, int(r)))
            return c

        def decrypt(self, cipher):
            v = super().decrypt(cipher)
            ops.append((OPS["decrypt"], -1, hid(cipher, "c"), -1, len(decrypted)))
            decrypted.append(np.array(v))
            return v

    params = slotcnn.HEParams(poly_degree=1 << n_log, depth=depth, scale_bits=40)
    m = slotcnn.builtin("M2")
    rng = np.random.default_rng(seed)
    plan = slotcnn.footprint(m, params)
    samples = list(rng.uniform(0.0, 1.0, size=(plan.capacity, m.channels, m.height, m.width)))
    be = Rec(params)
    outputs, metrics, plan = slotcnn.run_inference(m, samples, params, plan=plan, backend=be)
    refs = [slotcnn.reference_infer(m, s) for s in samples]
    return params, be.counter, ops, plains, decrypted, outputs, refs, metrics


def pack(plains):
    """Plaintext table: kind 0 = scalar x pattern, kind 1 = sparse values, kind 2 = all zero."""
    pat_index, patterns = {}, []
    kind, pat_id, scal, sp_off, sp_idx, sp_val = [], [], [], [0], [], []
    for v in plains:
        nz = np.flatnonzero(v)
        if nz.size == 0:
            kind.append(2), pat_id.append(-1), scal.append(0.0)
        elif np.all(v[nz] == v[nz[0]]):
            key = nz.tobytes()
            if key not in pat_index:
                pat_index[key] = len(patterns)
                patterns.append(nz.astype(np.int32))
            kind.append(0), pat_id.append(pat_index[key]), scal.append(float(v[nz[0]]))
        else:
            kind.append(1), pat_id.append(-1), scal.append(0.0)
            sp_idx.append(nz.astype(np.int32))
            sp_val.append(v[nz])
        if kind[-1] == 1:
            sp_off.append(sp_off[-1] + nz.size)
        else:
            sp_off.append(sp_off[-1])
    pat_off = np.cumsum([0] + [p.size for p in patterns]).astype(np.int64)
    cat = lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dt)  # noqa: E731
    return {"p_kind": np.array(kind, np.int8), "p_pat": np.array(pat_id, np.int32), "p_scalar": np.array(scal),
            "p_sp_off": np.array(sp_off, np.int64), "p_sp_idx": cat(sp_idx, np.int32),
            "p_sp_val": cat(sp_val, np.float64), "pat_off": pat_off, "pat_idx": cat(patterns, np.int32)}


def main():
    params, counter, ops, plains, decrypted, outputs, refs, metrics = record()
    table = pack(plains)
    hist = sorted(counter.by_level.items())
    out = os.path.join(HERE, "opstream_m2_n4096.npz")
    np.savez_compressed(
        out, ops=np.array(ops, dtype=np.int64), **table,
        params=np.array([params.poly_degree, params.depth, params.scale_bits]),
        decrypted=np.stack(decrypted), outputs=np.stack(outputs), refs=np.stack(refs),
        hist_kind=np.array([k for (k, _), _ in hist]), hist_level=np.array([lv for (_, lv), _ in hist]),
        hist_count=np.array([c for _, c in hist]),
        level_trace=np.array([r.level_after for r in metrics.per_layer]))
    print(f"{out}: {len(ops)} ops, {len(plains)} plaintexts, {os.path.getsize(out) / 1e3:.0f} kB")


if __name__ == "__main__":
    main()
