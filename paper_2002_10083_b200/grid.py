"""The pr x pc Sparse-SUMMA grid (generalised to non-square grids with
s = lcm(pr, pc) inner panels) as the library runs it: every quantity
comes from libmclx.so's mcl_summa_schedule (the same functions mcl_summa_iterate uses), so
the multi-process CPU test exercises the product's schedule, not a mirror of it."""
from __future__ import annotations

from dataclasses import dataclass

from . import summa_schedule


@dataclass(frozen=True)
class Grid:
    pr: int
    pc: int
    rank: int
    stage_mult: int = 1

    def _sched(self, n: int, rank: int | None = None) -> dict:
        return summa_schedule(self.pr, self.pc, self.rank if rank is None else rank, n,
                              self.stage_mult)

    @property
    def i(self) -> int:
        return self.rank // self.pc

    @property
    def j(self) -> int:
        return self.rank % self.pc

    @property
    def s(self) -> int:
        return self._sched(0)["s"]

    def rows(self, n: int, i: int | None = None):
        i = self.i if i is None else i
        return tuple(self._sched(n, i * self.pc)["rows"])

    def cols(self, n: int, j: int | None = None):
        j = self.j if j is None else j
        return tuple(self._sched(n, j)["cols"])

    def panel(self, n: int, q: int):
        st = self._sched(n)["stages"][q]
        return st["k0"], st["k1"]

    def a_owner_col(self, q: int) -> int:
        """Column index of the rank in my row that broadcasts A[rows_i, K_q] at stage q."""
        return self._sched(0)["stages"][q]["a_owner_col"]

    def b_owner_row(self, q: int) -> int:
        """Row index of the rank in my column that broadcasts A[K_q, cols_j] at stage q."""
        return self._sched(0)["stages"][q]["b_owner_row"]

    def nmerges(self, q: int) -> int:
        """Alg. 2: lists merged after pushing stage q's partial (0-based q)."""
        return self._sched(0)["stages"][q]["nmerges"]
