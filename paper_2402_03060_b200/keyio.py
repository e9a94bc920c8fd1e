"""Evaluation-key container: the on-disk / wire format for Galois and
relinearisation keys (the reference has no key material at
all -- its backend simulates encryption in the clear, ``he_backend.py:155-253``).

A server that evaluates the network needs the parameter set and the evaluation
keys, never the secret key.  Keys are written exactly as the engine consumes
them (``he_backend.GpuBackend.galois_key`` / ``relin_key``): residues
``uint64[level+1 digits][2 components][level+2 limbs][N]`` in the NTT (slot
order) domain, truncated to the highest level the key is used at.

Layout (all integers little-endian)::

    offset 0   8 bytes   magic  b"UHEVK\\0" + uint16 format version (1)
    offset 8   8 bytes   uint64 header length H
    offset 16  H bytes   UTF-8 JSON header (see below), zero-padded to 64 B
    ...        each key's residues, 64-byte aligned, at the offsets the header lists

Header::

    {"format": 2, "poly_degree": N, "moduli": [q_0, .., q_depth, P],
     "scale_bits": s, "depth": d,
     "keys": [{"kind": "galois", "rotation": r, "galois_elt": 5^r mod 2N,
               "level": l, "shape": [l+1, 2, l+2, N], "offset": o,
               "nbytes": b, "crc32": c}, ...,
              {"kind": "relin", "level": l, ...}]}

The container never holds the secret key or anything it can be derived from:
in particular not the secret seed (``HEParams.seed``; format 1 wrote it, and
format-1 files are refused).

Every failure to read a file (bad magic, unknown version, truncated data,
checksum mismatch, parameters that do not match the reader's) raises the
reference's :class:`~paper_2402_03060_b200.errors.ParseError`.
"""

from __future__ import annotations

import json
import struct
import zlib
from dataclasses import dataclass, field

import numpy as np

from .errors import ParseError

MAGIC = b"UHEVK\0"
VERSION = 2
ALIGN = 64


def _pad(n: int) -> int:
    return (-n) % ALIGN


@dataclass
class EvalKeys:
    """Evaluation keys in host memory (uint64 residue arrays)."""

    poly_degree: int
    moduli: list
    scale_bits: int
    depth: int
    galois: dict = field(default_factory=dict)  # rotation r (mod N/2) -> uint64[l+1][2][l+2][N]
    relin: np.ndarray | None = None            # uint64[l+1][2][l+2][N]

    def check_params(self, poly_degree: int, moduli) -> None:
        if int(poly_degree) != self.poly_degree or [int(q) for q in moduli] != [int(q) for q in self.moduli]:
            raise ParseError(f"evaluation keys were made for N={self.poly_degree} and moduli {self.moduli}, "
                             f"not N={poly_degree} and {list(moduli)}")


def _check_key(arr: np.ndarray, n: int, count: int, what: str) -> int:
    if arr.ndim != 4 or arr.shape[1] != 2 or arr.shape[3] != n or arr.shape[2] != arr.shape[0] + 1:
        raise ParseError(f"{what}: shape {arr.shape} is not [l+1, 2, l+2, {n}]")
    level = arr.shape[0] - 1
    if level + 2 > count:
        raise ParseError(f"{what}: level {level} exceeds the chain (depth {count - 2})")
    return level


def save_eval_keys(path: str, keys: EvalKeys) -> None:
    """Write ``keys`` to ``path`` in the container format above."""
    n, count = keys.poly_degree, len(keys.moduli)
    entries, blobs = [], []
    items = [("galois", r % (n // 2), a) for r, a in sorted(keys.galois.items())]
    if keys.relin is not None:
        items.append(("relin", None, keys.relin))
    for kind, r, arr in items:
        a = np.ascontiguousarray(np.asarray(arr).astype(np.uint64, copy=False))
        level = _check_key(a, n, count, f"{kind} key" + (f" r={r}" if r is not None else ""))
        raw = a.astype("<u8", copy=False).tobytes()
        e = {"kind": kind, "level": level, "shape": list(a.shape), "nbytes": len(raw), "crc32": zlib.crc32(raw)}
        if kind == "galois":
            e["rotation"] = int(r)
            e["galois_elt"] = pow(5, int(r), 2 * n)
        entries.append(e)
        blobs.append(raw)
    header = {"format": VERSION, "poly_degree": n, "moduli": [int(q) for q in keys.moduli],
              "scale_bits": int(keys.scale_bits), "depth": int(keys.depth), "keys": entries}
    # offsets depend on the header length, which depends on the offsets' digits: iterate to a fixed point
    hlen = 0
    while True:
        pos = 16 + hlen + _pad(16 + hlen)
        for e, raw in zip(entries, blobs):
            e["offset"] = pos
            pos += len(raw) + _pad(len(raw))
        hb = json.dumps(header, sort_keys=True).encode()
        if len(hb) == hlen:
            break
        hlen = len(hb)
    with open(path, "wb") as f:
        f.write(MAGIC + struct.pack("<H", VERSION) + struct.pack("<Q", len(hb)) + hb)
        f.write(b"\0" * _pad(16 + len(hb)))
        for raw in blobs:
            f.write(raw)
            f.write(b"\0" * _pad(len(raw)))


def load_eval_keys(path: str, poly_degree: int | None = None, moduli=None) -> EvalKeys:
    """Read a key container; with ``poly_degree``/``moduli`` given, refuse keys made for other parameters."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise ParseError(f"cannot read evaluation keys: {e}") from e
    if len(data) < 16 or data[:6] != MAGIC:
        raise ParseError("not an evaluation-key container (bad magic)")
    (version,) = struct.unpack("<H", data[6:8])
    if version != VERSION:
        raise ParseError(f"unsupported evaluation-key format version {version}")
    (hlen,) = struct.unpack("<Q", data[8:16])
    if 16 + hlen > len(data):
        raise ParseError("truncated evaluation-key header")
    try:
        header = json.loads(data[16:16 + hlen].decode())
        n, mods = int(header["poly_degree"]), [int(q) for q in header["moduli"]]
        if "seed" in header:
            raise ParseError("evaluation-key header carries a seed (secret material): refusing it")
        out = EvalKeys(n, mods, int(header["scale_bits"]), int(header["depth"]))
        entries = list(header["keys"])
    except (ValueError, KeyError, TypeError) as e:
        raise ParseError(f"malformed evaluation-key header: {e}") from e
    if poly_degree is not None or moduli is not None:
        out.check_params(poly_degree if poly_degree is not None else n, moduli if moduli is not None else mods)
    for e in entries:
        try:
            off, nb, shape = int(e["offset"]), int(e["nbytes"]), tuple(int(x) for x in e["shape"])
            kind = e["kind"]
        except (ValueError, KeyError, TypeError) as ex:
            raise ParseError(f"malformed key entry {e}: {ex}") from ex
        if off + nb > len(data) or nb != 8 * int(np.prod(shape)):
            raise ParseError(f"truncated or inconsistent {kind} key data")
        raw = data[off:off + nb]
        if zlib.crc32(raw) != int(e.get("crc32", -1)):
            raise ParseError(f"checksum mismatch in {kind} key" + (f" r={e.get('rotation')}" if kind == "galois" else ""))
        arr = np.frombuffer(raw, dtype="<u8").reshape(shape).copy()
        _check_key(arr, n, len(mods), f"{kind} key")
        if kind == "galois":
            r = int(e["rotation"])
            if pow(5, r, 2 * n) != int(e.get("galois_elt", -1)):
                raise ParseError(f"galois key r={r}: element does not match 5^r mod 2N")
            out.galois[r] = arr
        elif kind == "relin":
            out.relin = arr
        else:
            raise ParseError(f"unknown key kind {kind!r}")
    return out
