"""Host-side arithmetic of the pr x pc Sparse-SUMMA grid (generalised
to non-square grids with s = lcm(pr, pc) inner panels).  Mirrors the
formulas in csrc/capi.cu (mcl_summa_iterate); no arithmetic of the method lives here."""
from __future__ import annotations

from dataclasses import dataclass
from math import gcd


def cut(n: int, parts: int, k: int) -> int:
    """Boundary k of [0, n) cut into `parts` near-equal ranges (floor(k n / parts))."""
    return (k * n) // parts


@dataclass(frozen=True)
class Grid:
    pr: int
    pc: int
    rank: int

    @property
    def i(self) -> int:
        return self.rank // self.pc

    @property
    def j(self) -> int:
        return self.rank % self.pc

    @property
    def s(self) -> int:
        return self.pr * self.pc // gcd(self.pr, self.pc)

    def rows(self, n: int, i: int | None = None):
        i = self.i if i is None else i
        return cut(n, self.pr, i), cut(n, self.pr, i + 1)

    def cols(self, n: int, j: int | None = None):
        j = self.j if j is None else j
        return cut(n, self.pc, j), cut(n, self.pc, j + 1)

    def panel(self, n: int, q: int):
        return cut(n, self.s, q), cut(n, self.s, q + 1)

    def a_owner_col(self, q: int) -> int:
        """Column index of the rank in my row that broadcasts A[rows_i, K_q] at stage q."""
        return q * self.pc // self.s

    def b_owner_row(self, q: int) -> int:
        """Row index of the rank in my column that broadcasts A[K_q, cols_j] at stage q."""
        return q * self.pr // self.s


def binary_merge_schedule(nstages: int):
    """Alg. 2: after pushing list i (1-based) merge nmerges+1 lists, where
    nmerges counts the halvings of i while even.  Returns [(i, nmerges)]."""
    out = []
    for i in range(1, nstages + 1):
        j, nm = i, 0
        while j % 2 == 0 and j != 0:
            nm += 1
            j //= 2
        out.append((i, nm))
    return out
