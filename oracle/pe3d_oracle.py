"""CPU oracle: a numpy restatement of the reference's range-marching path.

TEST INFRASTRUCTURE.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may use it,
and only as the checker or the timed CPU baseline -- never on the product
path.

It restates, in numpy and with the same operation order, the algorithm of
the reference package ``pe3d`` (``/root/reference/pkg/src/pe3d``): Thomas
elimination and the Sherman-Morrison cyclic solve (``tridiag.py``), the
Eq. (4) operators and system assembly (``operators.py``), and the range
step / frequency march (``marching.py``).  Each function names the
reference lines it follows.  Differences from the reference that do not
change values: members are processed in one vectorised block instead of
64-wide tiles (``tridiag.py:32``), and no thread pool is used.

Pinning: ``tests/test_oracle_golden.py`` checks this module against
fixtures produced by running the reference itself
(``tests/golden/make_golden.py``); on this container's host the results
agree to the last bit or within 1e-15 relative.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

PIVOT_FLOOR = 1e-300          # tridiag.py:31
TL_FLOOR_DB = 300.0           # environment.py:29
MAX_OUTPUT_SAMPLES = 512      # marching.py:45


class OracleSingular(Exception):
    def __init__(self, pivot, member, rank1=False):
        self.pivot, self.member, self.rank1 = pivot, member, rank1
        super().__init__(f"singular: pivot {pivot}, member {member}")


class OracleStepError(Exception):
    def __init__(self, range_index, sweep, member):
        self.range_index, self.sweep, self.member = range_index, sweep, member
        super().__init__(f"step {range_index} failed in {sweep} sweep at {member}")


# ----------------------------------------------------------------- solvers

def _pivot_check(denom: np.ndarray, row: int) -> None:
    """tridiag.py:145-148 -- lowest member index of the smallest pivot."""
    mags = np.abs(denom)
    if mags.min() < PIVOT_FLOOR:
        raise OracleSingular(row, int(np.argmin(mags)))


def factor_open(sub, main, sup):
    """Forward elimination, tridiag.py:151-167.  Arrays are (row, member)."""
    n, w = main.shape
    inv = np.empty((n, w), dtype=np.complex128)
    cp = np.empty((max(n - 1, 0), w), dtype=np.complex128)
    _pivot_check(main[0], 0)
    inv[0] = 1.0 / main[0]
    if n > 1:
        cp[0] = sup[0] * inv[0]
    for k in range(1, n):
        denom = main[k] - sub[k - 1] * cp[k - 1]
        _pivot_check(denom, k)
        inv[k] = 1.0 / denom
        if k < n - 1:
            cp[k] = sup[k] * inv[k]
    return cp, inv


def substitute_open(cp, inv, sub, rhs):
    """Forward/back substitution, tridiag.py:170-178."""
    n = rhs.shape[0]
    x = np.empty_like(rhs)
    x[0] = rhs[0] * inv[0]
    for k in range(1, n):
        x[k] = (rhs[k] - sub[k - 1] * x[k - 1]) * inv[k]
    for k in range(n - 2, -1, -1):
        x[k] -= cp[k] * x[k + 1]
    return x


def solve_open(sub, main, sup, rhs):
    cp, inv = factor_open(sub, main, sup)
    return substitute_open(cp, inv, sub, rhs)


def solve_cyclic(sub, main, sup, rhs):
    """Sherman-Morrison cyclic solve, tridiag.py:186-212.  Corner storage:
    sub[0] = A[0, n-1], sup[n-1] = A[n-1, 0] (tridiag.py:13-16)."""
    n = main.shape[0]
    alpha, beta = sub[0], sup[n - 1]
    gamma = np.where(np.abs(main[0]) > 0, -main[0], np.complex128(1.0))
    mod = np.array(main, dtype=np.complex128)
    mod[0] = main[0] - gamma
    mod[n - 1] = main[n - 1] - alpha * beta / gamma
    cp, inv = factor_open(sub[1:], mod, sup[: n - 1])
    y = substitute_open(cp, inv, sub[1:], rhs)
    spike = np.zeros_like(rhs)
    spike[0] = gamma
    spike[n - 1] = beta
    q = substitute_open(cp, inv, sub[1:], spike)
    weight = alpha / gamma
    denom = 1.0 + q[0] + weight * q[n - 1]
    mags = np.abs(denom)
    if mags.min() < PIVOT_FLOOR:
        raise OracleSingular(n, int(np.argmin(mags)), rank1=True)
    return y - q * ((y[0] + weight * y[n - 1]) / denom)


def solve_batch(sub, main, sup, rhs, cyclic: bool) -> np.ndarray:
    """solve_batch, tridiag.py:248-281: (row, member) SoA in, (member, row)
    out; a singular member aborts the batch naming the lowest member."""
    main = np.asarray(main, dtype=np.complex128)
    w = main.shape[1]
    shape_off = (main.shape[0] if cyclic else main.shape[0] - 1, w)
    sub = np.broadcast_to(np.asarray(sub, dtype=np.complex128), shape_off)
    sup = np.broadcast_to(np.asarray(sup, dtype=np.complex128), shape_off)
    rhs = np.asarray(rhs, dtype=np.complex128)
    fn = solve_cyclic if cyclic else solve_open
    return np.ascontiguousarray(fn(sub, main, sup, rhs).T)


def dense_solve(sub, main, sup, rhs, cyclic: bool) -> np.ndarray:
    """Partial-pivoting Gaussian elimination on the full matrix
    (tridiag.py:284-326), for one system given as 1-D arrays."""
    n = len(main)
    a = np.zeros((n, n), dtype=np.complex128)
    idx = np.arange(n)
    a[idx, idx] = main
    if cyclic:
        a[idx[1:], idx[:-1]] = sub[1:]
        a[idx[:-1], idx[1:]] = sup[:-1]
        a[0, n - 1] = sub[0]
        a[n - 1, 0] = sup[n - 1]
    elif n > 1:
        a[idx[1:], idx[:-1]] = sub
        a[idx[:-1], idx[1:]] = sup
    b = np.array(rhs, dtype=np.complex128)
    for k in range(n):
        p = k + int(np.argmax(np.abs(a[k:, k])))
        if abs(a[p, k]) < PIVOT_FLOOR:
            raise OracleSingular(k, 0)
        if p != k:
            a[[k, p]] = a[[p, k]]
            b[[k, p]] = b[[p, k]]
        if k + 1 < n:
            mult = a[k + 1:, k] / a[k, k]
            a[k + 1:, k + 1:] -= np.outer(mult, a[k, k + 1:])
            a[k + 1:, k] = 0.0
            b[k + 1:] -= mult * b[k]
    x = np.empty(n, dtype=np.complex128)
    for k in range(n - 1, -1, -1):
        x[k] = (b[k] - a[k, k + 1:] @ x[k + 1:]) / a[k, k]
    return x


def random_system(rng, n: int, cyclic: bool):
    """Seeded diagonally dominant complex system, the fixture of
    selftest.py:58-72: returns (sub, main, sup, rhs)."""
    n_off = n if cyclic else n - 1
    sub = rng.standard_normal(n_off) + 1j * rng.standard_normal(n_off)
    sup = rng.standard_normal(n_off) + 1j * rng.standard_normal(n_off)
    row_sum = np.zeros(n)
    if cyclic:
        row_sum += np.abs(sub) + np.abs(sup)
    else:
        row_sum[1:] += np.abs(sub)
        row_sum[:-1] += np.abs(sup)
    phase = np.exp(1j * rng.uniform(0, 2 * math.pi, n))
    main = (row_sum + 1.0 + rng.uniform(0.1, 2.0, n)) * phase
    rhs = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    return sub, main, sup, rhs


# --------------------------------------------------------------- operators

def second_difference(u: np.ndarray, axis: int, periodic: bool) -> np.ndarray:
    """operators.py:105-122 (zero exterior unless periodic)."""
    if periodic:
        return np.roll(u, -1, axis=axis) + np.roll(u, 1, axis=axis) - 2.0 * u
    d2 = np.empty_like(u)
    axis = axis % u.ndim
    sl = lambda s: tuple(s if a == axis else slice(None) for a in range(u.ndim))  # noqa: E731
    d2[sl(slice(1, -1))] = u[sl(slice(2, None))] - 2.0 * u[sl(slice(1, -1))] + u[sl(slice(None, -2))]
    d2[sl(0)] = u[sl(1)] - 2.0 * u[sl(0)]
    d2[sl(-1)] = u[sl(-2)] - 2.0 * u[sl(-1)]
    return d2


@dataclass(frozen=True)
class StepGeometry:
    n_theta: int
    n_depth: int
    delta_theta: float
    delta_z: float
    periodic: bool = True


def compute_rhs(u, local_now, k0, r_now, geo: StepGeometry, cx_rhs, cy_rhs):
    """[1 + cx_rhs X][1 + cy_rhs Y] u, operators.py:197-210 (Y first, at
    the slab's range; X with the local term n^2-1, operators.py:125-153)."""
    s_theta = 1.0 / (k0 * r_now * geo.delta_theta) ** 2
    s_z = 1.0 / (k0 * geo.delta_z) ** 2
    yu = s_theta * second_difference(u, 0, geo.periodic)
    temp = u + cy_rhs * yu
    xt = local_now * temp + s_z * second_difference(temp, -1, False)
    return temp + cx_rhs * xt


def apply_boundary(u: np.ndarray, periodic: bool) -> np.ndarray:
    """marching.py:80-90: surface row, and sector edges, set to zero."""
    u[:, 0] = 0.0
    if not periodic:
        u[0, :] = 0.0
        u[-1, :] = 0.0
    return u


def depth_solve(rhs, local_new, k0, geo: StepGeometry, cx_lhs):
    """assemble_depth_batch (operators.py:213-241) + open solve_batch:
    one system per azimuth, surface row imposed as v = 0."""
    s = 1.0 / (k0 * geo.delta_z) ** 2
    local = np.broadcast_to(np.asarray(local_new), rhs.shape)
    main = np.ascontiguousarray((1.0 + cx_lhs * (local - 2.0 * s)).T)
    off = np.complex128(cx_lhs * s)
    n_az, n_dep = rhs.shape
    sub = np.broadcast_to(off, (n_dep - 1, n_az))
    sup = np.full((n_dep - 1, n_az), off)
    b = np.ascontiguousarray(rhs.T)
    main[0] = 1.0
    sup[0] = 0.0
    b[0] = 0.0
    return solve_batch(sub, main, sup, b, cyclic=False)          # (n_az, n_dep)


def azimuth_solve(v, k0, r_new, geo: StepGeometry, cy_lhs):
    """assemble_azimuth_batch (operators.py:244-272) + solve_batch: one
    system per depth; periodic -> cyclic constants, sector -> identity
    edge rows.  Returns (n_dep, n_az)."""
    s = 1.0 / (k0 * r_new * geo.delta_theta) ** 2
    diag = np.complex128(1.0 - 2.0 * cy_lhs * s)
    off = np.complex128(cy_lhs * s)
    n_az, n_dep = v.shape
    rhs = np.ascontiguousarray(v)
    if geo.periodic:
        main = np.broadcast_to(diag, (n_az, n_dep))
        offs = np.broadcast_to(off, (n_az, n_dep))
        return solve_batch(offs, main, offs, rhs, cyclic=True)
    main = np.full((n_az, n_dep), diag)
    sub = np.full((n_az - 1, n_dep), off)
    sup = np.full((n_az - 1, n_dep), off)
    main[0] = main[-1] = 1.0
    sup[0] = 0.0
    sub[-1] = 0.0
    rhs = rhs.copy()
    rhs[0] = 0.0
    rhs[-1] = 0.0
    return solve_batch(sub, main, sup, rhs, cyclic=False)


def range_step(u, j: int, r_now: float, r_new: float, k0: float, coeffs,
               local_now, local_new, geo: StepGeometry):
    """marching.py:93-136.  ``coeffs`` = (delta, cx_lhs, cx_rhs, cy_lhs,
    cy_rhs).  Mutates ``u``'s boundary rows in place like the reference;
    returns (new u, new range)."""
    delta, cx_lhs, cx_rhs, cy_lhs, cy_rhs = coeffs
    apply_boundary(u, geo.periodic)
    if delta == 0:
        return u, r_now
    rhs = compute_rhs(u, local_now, k0, r_now, geo, cx_rhs, cy_rhs)
    apply_boundary(rhs, geo.periodic)
    try:
        v = depth_solve(rhs, local_new, k0, geo, cx_lhs)
    except OracleSingular as exc:
        raise OracleStepError(j + 1, "depth", exc.member) from exc
    try:
        w = azimuth_solve(v, k0, r_new, geo, cy_lhs)
    except OracleSingular as exc:
        raise OracleStepError(j + 1, "azimuth", exc.member) from exc
    new = np.ascontiguousarray(w.T)
    apply_boundary(new, geo.periodic)
    return new, r_new


# ----------------------------------------------------------- the march

def hankel_abs(k0: float, r: float) -> float:
    """|w(r)| with w = (cos k0 r + i sin k0 r)/sqrt(r), environment.py:287-294."""
    return abs(complex(math.cos(k0 * r), math.sin(k0 * r)) / math.sqrt(r))


def transmission_loss(values, w_abs):
    """environment.py:308-315."""
    mag = np.abs(values) * w_abs
    zero = mag == 0.0
    with np.errstate(divide="ignore"):
        tl = np.where(zero, TL_FLOOR_DB, -20.0 * np.log10(np.where(zero, 1.0, mag)))
    return tl, int(np.count_nonzero(zero))


def default_output_stride(n_steps: int) -> int:
    """marching.py:139-141."""
    return max(1, (n_steps + 1 + MAX_OUTPUT_SAMPLES - 1) // MAX_OUTPUT_SAMPLES)


@dataclass
class OracleResult:
    ranges: np.ndarray
    tl_field: np.ndarray          # (S, n_theta, n_depth)
    clamped: int
    final: np.ndarray             # (n_theta, n_depth)
    snapshots: Optional[np.ndarray]


def march(u0: np.ndarray, k0: float, coeffs, geo: StepGeometry, r_start: float,
          delta_r: float, n_steps: int, stride: int,
          local_at: Callable[[float], np.ndarray],
          max_range: Optional[float] = None, keep_snapshots: bool = False) -> OracleResult:
    """run_frequency's range loop, marching.py:159-193, from a given
    starter slab: TL of the starter and of every ``stride``-th step, the
    ``max_range`` cut with 1e-12 slack (marching.py:177-179)."""
    u = apply_boundary(np.array(u0, dtype=np.complex128), geo.periodic)
    r = r_start
    ranges, tls, snaps, clamped = [r], [], [], 0

    def record(field, rr):
        nonlocal clamped
        tl, n = transmission_loss(field, hankel_abs(k0, rr))
        tls.append(tl)
        clamped += n
        if keep_snapshots:
            snaps.append(field.copy())

    record(u, r)
    for j in range(1, n_steps + 1):
        r_j = r_start + j * delta_r
        if max_range is not None and r_j > max_range * (1.0 + 1e-12):
            break
        u, r = range_step(u, j - 1, r, r_j, k0, coeffs, local_at(r), local_at(r_j), geo)
        if j % stride == 0:
            ranges.append(r)
            record(u, r)
    return OracleResult(np.asarray(ranges), np.stack(tls), clamped, u,
                        np.stack(snaps) if keep_snapshots else None)


def run_frequency(config, frequency: float, keep_snapshots: bool = False,
                  n_steps: Optional[int] = None) -> OracleResult:
    """run_frequency (marching.py:144-193) for a ``Config`` of either the
    reference or the B200 package.  The medium comes from the product's
    shared medium definition (``environment.local_term_grid``)."""
    from paper_1711_00005_b200.environment import gaussian_starter, local_term_grid, wavenumber
    grid, env, source, options = config
    k0 = wavenumber(frequency, env.c0)
    d = 1j * (k0 * grid.delta_r)
    q = d / 4.0
    coeffs = (d, 0.25 - q, 0.25 + q, -q, +q)
    geo = StepGeometry(grid.n_azimuth, grid.n_depth, grid.delta_theta, grid.delta_z,
                       grid.azimuth_topology == "periodic")
    u0 = gaussian_starter(grid, source, k0).values
    steps = grid.n_range if n_steps is None else n_steps
    stride = options.output_stride or default_output_stride(grid.n_range)
    return march(u0, k0, coeffs, geo, grid.r_start, grid.delta_r, steps, stride,
                 lambda r: local_term_grid(env, grid, r, k0), options.max_range,
                 keep_snapshots)
