"""Step coefficients of Eq. (4); ref ``pkg/src/pe3d/operators.py:31-62``.

    [1 + cx_lhs X(n_{j+1})] [1 + cy_lhs Y(r_{j+1})] u_{j+1}
        = [1 + cx_rhs X(n_j)] [1 + cy_rhs Y(r_j)] u_j,     d = i k0 dr

with cx = 1/4 -/+ d/4 and cy = -/+ d/4.  The matrix-free operators and
the per-system assembly of the reference (``operators.py:90-272``) live
inside the CUDA kernels (``csrc/pe3d_depth.cu``, ``csrc/pe3d_ring.cu``) and, as the checker,
in ``oracle/pe3d_oracle.py``.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import InvariantError


@dataclass(frozen=True)
class StepCoefficients:
    delta: complex
    cx_lhs: complex
    cx_rhs: complex
    cy_lhs: complex
    cy_rhs: complex

    def __post_init__(self):
        # Exact for purely imaginary delta (ref operators.py:46-50).
        if self.cx_lhs + self.cx_rhs != 0.5 + 0.0j:
            raise InvariantError("cx_lhs + cx_rhs == 1/2 exactly")
        if self.cy_lhs + self.cy_rhs != 0.0 + 0.0j:
            raise InvariantError("cy_lhs + cy_rhs == 0 exactly")

    @classmethod
    def for_step(cls, k0: float, delta_r: float) -> "StepCoefficients":
        d = 1j * (k0 * delta_r)
        q = d / 4.0
        return cls(delta=d, cx_lhs=0.25 - q, cx_rhs=0.25 + q, cy_lhs=-q, cy_rhs=+q)

