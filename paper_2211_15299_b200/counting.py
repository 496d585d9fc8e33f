"""Complex-operation tally with the reference's interface (counting.py:15-79).

The device transform does not count at run time: a Hi-DFT's counts are
analytic (A/2 multiplications and A additions per stage, hidft.py:165-167),
so the host wrappers record them here under the same phase names.  Any
object with add(n, phase) / mul(n, phase) (e.g. structfft.OpCounter) works
as a `counter=` argument too.
"""

from __future__ import annotations

from collections import defaultdict


class OpCounter:
    def __init__(self) -> None:
        self._tally = defaultdict(lambda: [0, 0])  # phase -> [adds, mults]
        self.bit_ops = 0

    def _bump(self, phase: str, slot: int, n: int) -> None:
        if n < 0:
            raise ValueError("op counts are monotone")
        self._tally[phase][slot] += int(n)

    def add(self, n: int = 1, phase: str = "default") -> None:
        self._bump(phase, 0, n)

    def mul(self, n: int = 1, phase: str = "default") -> None:
        self._bump(phase, 1, n)

    def count_bit_ops(self, n: int) -> None:
        self.bit_ops += int(n)

    complex_adds = property(lambda self: sum(v[0] for v in self._tally.values()))
    complex_mults = property(lambda self: sum(v[1] for v in self._tally.values()))
    total = property(lambda self: self.complex_adds + self.complex_mults)

    def phase(self, name: str) -> tuple[int, int]:
        v = self._tally.get(name, (0, 0))
        return int(v[0]), int(v[1])

    def phase_total(self, name: str) -> int:
        return sum(self.phase(name))

    @property
    def phases(self) -> dict[str, tuple[int, int]]:
        return {k: (v[0], v[1]) for k, v in self._tally.items()}

    def reset(self) -> None:
        self._tally.clear()
        self.bit_ops = 0

    def __repr__(self) -> str:
        return f"OpCounter(adds={self.complex_adds}, mults={self.complex_mults})"
