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

from .errors import DomainError, InvariantError


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


def depth_scale(k0: float, delta_z: float) -> float:
    """s_z = 1/(k0 dz)^2 (ref ``operators.py:90-94``)."""
    if k0 <= 0 or delta_z <= 0:
        raise DomainError("k0 and delta_z must be > 0")
    return 1.0 / (k0 * delta_z) ** 2


def azimuth_scale(k0: float, r: float, delta_theta: float) -> float:
    """s_theta = 1/(k0 r dtheta)^2 (ref ``operators.py:97-102``)."""
    if r <= 0:
        raise DomainError(f"range must be > 0, got {r}")
    if k0 <= 0 or delta_theta <= 0:
        raise DomainError("k0 and delta_theta must be > 0")
    return 1.0 / (k0 * r * delta_theta) ** 2
