"""Operation census of the operator boundary.

Same contract as the reference's ``OpCounter``/``diff_snapshots``
(``pkg/src/slotcnn/he_backend.py:104-152``): per-kind totals plus a
``(kind, level)`` histogram, level = operand level at call time (result
level for rotations and additions).  The GPU engine records exactly the
census the reference's schedule produces -- also on the fused layer paths,
which execute fewer, larger kernels for the same logical operations.
"""

from __future__ import annotations

from dataclasses import dataclass, field

__all__ = ["OpCounter", "diff_snapshots"]

_KINDS = {"rotation": "rotations", "pt_mult": "pt_mults", "ct_mult": "ct_mults", "add": "adds"}


@dataclass
class OpCounter:
    rotations: int = 0
    pt_mults: int = 0
    ct_mults: int = 0
    adds: int = 0
    by_level: dict = field(default_factory=dict)

    def record(self, kind: str, level: int, count: int = 1) -> None:
        attr = _KINDS[kind]
        setattr(self, attr, getattr(self, attr) + count)
        key = (kind, level)
        self.by_level[key] = self.by_level.get(key, 0) + count

    def totals(self) -> dict:
        return {"rotations": self.rotations, "pt_mults": self.pt_mults,
                "ct_mults": self.ct_mults, "adds": self.adds}

    def snapshot(self) -> tuple:
        return (self.rotations, self.pt_mults, self.ct_mults, self.adds, dict(self.by_level))


def diff_snapshots(before: tuple, after: tuple) -> tuple:
    names = ("rotations", "pt_mults", "ct_mults", "adds")
    totals = {name: after[i] - before[i] for i, name in enumerate(names)}
    hist = {}
    for key, count in after[4].items():
        delta = count - before[4].get(key, 0)
        if delta:
            hist[key] = delta
    return totals, hist
