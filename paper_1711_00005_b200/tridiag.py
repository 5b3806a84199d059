"""Batched complex tridiagonal solves on the GPU, with the reference's types.

Mirrors ``pkg/src/pe3d/tridiag.py``: ``TriDiagSystem`` (:36-79),
``SolveBatch`` (:82-142), ``solve_batch`` (:248-281), ``solve_thomas``
(:223-234) and ``solve_cyclic`` (:237-245).  The solve runs in the
thread-per-system CUDA kernel ``k_solve_batch`` through
``pe3d_solve_batch_host``; the result layout (member, row), the
1e-300 pivot floor, the Sherman-Morrison corner convention and the
lowest-failing-member error rule are the reference's.
``dense_oracle_solve`` (a CPU test oracle in the reference) is not part of
the product; the checker keeps it in ``oracle/pe3d_oracle.py``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import DomainError, InvariantError, ShapeError

OPEN = "open"
CYCLIC = "cyclic"
PIVOT_FLOOR = 1e-300
TILE = 64   # the reference's fixed member tile; kept for its error rule (tridiag.py:32)


@dataclass(eq=False)
class TriDiagSystem:
    sub: np.ndarray
    main: np.ndarray
    sup: np.ndarray
    rhs: np.ndarray
    topology: str = OPEN

    def __post_init__(self):
        for name in ("sub", "main", "sup", "rhs"):
            setattr(self, name, np.asarray(getattr(self, name), dtype=np.complex128))
        if self.topology not in (OPEN, CYCLIC):
            raise InvariantError(f"topology in ({OPEN}, {CYCLIC})")
        if any(a.ndim != 1 for a in (self.sub, self.main, self.sup, self.rhs)):
            raise ShapeError("diagonals and rhs must be vectors")
        n = self.main.shape[0]
        if self.rhs.shape[0] != n:
            raise ShapeError(f"rhs length {self.rhs.shape[0]} != n {n}")
        if self.topology == OPEN:
            if n < 1:
                raise InvariantError("n >= 1 for open systems")
            want = n - 1
        else:
            if n < 3:
                raise InvariantError("n >= 3 for cyclic systems")
            want = n
        if self.sub.shape[0] != want or self.sup.shape[0] != want:
            raise ShapeError(f"{self.topology} system of size {n} needs off-diagonals of "
                             f"length {want}, got {self.sub.shape[0]}/{self.sup.shape[0]}")

    @property
    def n(self) -> int:
        return self.main.shape[0]


@dataclass(eq=False)
class SolveBatch:
    """(row, member) structure-of-arrays; arrays may be broadcast views."""

    sub: np.ndarray
    main: np.ndarray
    sup: np.ndarray
    rhs: np.ndarray
    topology: str = OPEN

    def __post_init__(self):
        if self.topology not in (OPEN, CYCLIC):
            raise InvariantError(f"topology in ({OPEN}, {CYCLIC})")
        if any(np.ndim(a) != 2 for a in (self.sub, self.main, self.sup, self.rhs)):
            raise ShapeError("batch arrays must be 2-D (row x member)")
        n, w = self.main.shape
        if self.rhs.shape != (n, w):
            raise ShapeError(f"rhs shape {self.rhs.shape} != {(n, w)}")
        want = n if self.topology == CYCLIC else n - 1
        if self.sub.shape != (want, w) or self.sup.shape != (want, w):
            raise ShapeError("off-diagonal batch shapes inconsistent with topology")
        if self.topology == CYCLIC and n < 3:
            raise InvariantError("n >= 3 for cyclic systems")

    @property
    def n(self) -> int:
        return self.main.shape[0]

    @property
    def n_systems(self) -> int:
        return self.main.shape[1]

    @classmethod
    def from_systems(cls, systems) -> "SolveBatch":
        systems = list(systems)
        if not systems:
            raise InvariantError("batch nonempty")
        n, topo = systems[0].n, systems[0].topology
        if any(s.n != n or s.topology != topo for s in systems[1:]):
            raise InvariantError("all batch members share one n and topology")
        stack = lambda name: np.stack([getattr(s, name) for s in systems], axis=1)  # noqa: E731
        return cls(stack("sub"), stack("main"), stack("sup"), stack("rhs"), topo)

    def system(self, i: int) -> TriDiagSystem:
        return TriDiagSystem(self.sub[:, i].copy(), self.main[:, i].copy(), self.sup[:, i].copy(),
                             self.rhs[:, i].copy(), self.topology)


def _strided(a: np.ndarray, keep_alive: list) -> _native.Strided:
    a = np.asarray(a, dtype=np.complex128)
    if a.size and (min(a.strides) < 0 or any(s % 16 for s in a.strides)):
        a = np.ascontiguousarray(a)
    keep_alive.append(a)
    if a.ndim != 2:
        raise ShapeError("batch arrays must be 2-D (row x member)")
    rs, ms = (s // 16 for s in a.strides)
    rs = rs if a.shape[0] > 1 else 0
    ms = ms if a.shape[1] > 1 else 0
    return _native.Strided(a.ctypes.data if a.size else None, rs, ms)


def solve_batch(batch: SolveBatch, parallel_hint: int = 1, device: int = 0) -> np.ndarray:
    """Solve every member on the GPU; returns (n_systems, n).  A singular
    member aborts the batch with SingularSystemError naming the lowest
    failing member (ref tridiag.py:274-280).  ``parallel_hint`` is accepted
    for signature compatibility; the CUDA grid replaces the thread pool."""
    if parallel_hint < 1:
        raise InvariantError("parallel_hint >= 1")
    w = batch.n_systems
    if w == 0:
        raise InvariantError("batch nonempty")
    n = batch.n
    out = np.empty((w, n), dtype=np.complex128)
    keep: list = []
    cyclic = batch.topology == CYCLIC
    if not cyclic and n == 1:
        # off-diagonals have no rows; pass a dummy 1x1 so the ABI sees valid pointers
        dummy = np.zeros((1, w), dtype=np.complex128)
        sub = sup = _strided(dummy, keep)
    else:
        sub, sup = _strided(batch.sub, keep), _strided(batch.sup, keep)
    _native.call("pe3d_solve_batch_host", _native.handle(device), n, w, int(cyclic), sub,
                 _strided(batch.main, keep), sup, _strided(batch.rhs, keep), _native.ptr(out))
    return out


def solve_thomas(system: TriDiagSystem) -> np.ndarray:
    if system.topology != OPEN:
        raise DomainError("solve_thomas requires open topology")
    return solve_batch(SolveBatch(system.sub[:, None], system.main[:, None], system.sup[:, None],
                                  system.rhs[:, None], OPEN))[0]


def solve_cyclic(system: TriDiagSystem) -> np.ndarray:
    if system.topology != CYCLIC:
        raise DomainError("solve_cyclic requires cyclic topology")
    return solve_batch(SolveBatch(system.sub[:, None], system.main[:, None], system.sup[:, None],
                                  system.rhs[:, None], CYCLIC))[0]
