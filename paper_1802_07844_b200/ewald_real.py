"""Short-range (real-space) component: drop-in for hsewald.ewald_real.

The cell list (ewald_real.py:192-251) and the screened pair sums with image
and wall-correction terms (ewald_real.py:258-455) run on the GPU
(csrc/cell_list.cu, csrc/sort.cu, csrc/pair.cu).  Small single-point helpers
(``f_derivs``, ``self_interaction``) are host utilities kept for API parity.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._plan import get_evaluator
from .errors import GeometryError, ParameterError
from .system import HALF_SPACE, ROTLET, STOKESLET, STRESSLET, VelocityResult
from .point_kernels import correction_phi_real, harmonic_real_derivs, kernel_real  # noqa: E402,F401  (ref:ewald_real.py:115-190)

_SQRT_PI = math.sqrt(math.pi)


@dataclass
class RealSpaceParams:
    """Screening parameter and cutoff (ewald_real.py:61-72)."""

    xi: float
    rc: float

    def __post_init__(self):
        if self.xi <= 0:
            raise ParameterError(f"xi must be positive, got {self.xi}")
        if self.rc < 0:
            raise ParameterError(f"rc must be nonnegative, got {self.rc}")


def f_derivs(r, xi):
    """erf(xi r)/r and its first three derivatives (ewald_real.py:79-98); host helper."""
    from scipy.special import erf
    r = np.asarray(r, dtype=float)
    if np.any(r <= 0):
        raise ParameterError("f_derivs requires r > 0")
    if xi <= 0:
        raise ParameterError("f_derivs requires xi > 0")
    e = (2.0 * xi / _SQRT_PI) * np.exp(-(xi * r) ** 2)
    f = erf(xi * r) / r
    f1 = (e - f) / r
    e1 = -2.0 * xi**2 * r * e
    f2 = (e1 - 2.0 * f1) / r
    e2 = -2.0 * xi**2 * e * (1.0 - 2.0 * xi**2 * r**2)
    f3 = (e2 - 3.0 * f2) / r
    return f, f1, f2, f3


def self_interaction(kind, xi):
    """Zero-displacement limit of the screened kernel (ewald_real.py:101-112)."""
    if xi <= 0:
        raise ParameterError("self_interaction requires xi > 0")
    if kind == STOKESLET:
        return -(4.0 * xi / _SQRT_PI) * np.eye(3)
    if kind in (STRESSLET, ROTLET):
        return np.zeros((3, 3))
    raise ValueError(f"unknown kind {kind!r}")


@dataclass
class CellList:
    """Non-periodic cell list (ewald_real.py:192-225)."""

    positions: np.ndarray
    rc: float
    origin: np.ndarray
    edge: np.ndarray
    dims: np.ndarray
    order: np.ndarray
    start: np.ndarray

    def cell_of(self, x):
        c = np.floor((np.asarray(x, float) - self.origin) / self.edge).astype(np.int64)
        return np.clip(c, 0, self.dims - 1)

    def query(self, x):
        cx, cy, cz = self.cell_of(x)
        out = []
        nx, ny, nz = self.dims
        for ix in range(max(cx - 1, 0), min(cx + 2, nx)):
            for iy in range(max(cy - 1, 0), min(cy + 2, ny)):
                for iz in range(max(cz - 1, 0), min(cz + 2, nz)):
                    flat = (ix * ny + iy) * nz + iz
                    out.append(self.order[self.start[flat]:self.start[flat + 1]])
        return np.concatenate(out) if out else np.empty(0, dtype=np.int64)

    def neighbors_within(self, x):
        cand = self.query(x)
        d = self.positions[cand] - np.asarray(x, float)
        return cand[np.sum(d * d, axis=1) <= self.rc**2]


def build_cell_list(points, rc, bounds) -> CellList:
    """GPU cell list, bit-exact with the reference (ewald_real.py:228-251)."""
    points = np.ascontiguousarray(np.atleast_2d(np.asarray(points, float)))
    lo = np.ascontiguousarray(np.asarray(bounds[0], float))
    hi = np.ascontiguousarray(np.asarray(bounds[1], float))
    if rc <= 0:
        raise ParameterError("build_cell_list requires rc > 0")
    lib = _lib.load_library()
    dims = np.zeros(3, np.int64)
    edge = np.zeros(3)
    _lib.check(lib.hs_cell_dims(float(rc), _lib.dptr(lo), _lib.dptr(hi), _lib.i64ptr(dims), _lib.dptr(edge)))
    n = points.shape[0]
    order = np.empty(n, np.int64)
    start = np.empty(int(np.prod(dims)) + 1, np.int64)
    ctx = _lib.Context.get()
    ctx.bind_stream(None)
    _lib.check(lib.hs_cell_list(ctx.handle, points.ctypes.data_as(C.c_void_p), n, float(rc), _lib.dptr(lo),
                                _lib.dptr(hi), order.ctypes.data_as(C.c_void_p), start.ctypes.data_as(C.c_void_p),
                                _lib.HS_MEM_HOST))
    return CellList(positions=points, rc=rc, origin=lo, edge=edge, dims=dims, order=order, start=start)


class _RealOnlyGrid:
    """Grid descriptor of a real-space-only plan: M = 0 tells hs_plan_create to allocate no grids,
    transforms or tables (include/hsewald_b200.h), so any (xi, rc) works, e.g. the xi -> 0
    screening limits of the reference's tests (ref tests/test_ewald_real.py:33-51)."""

    M, P, h, eta = 0, 0, 0.0, 1.0
    origin = (0.0, 0.0, 0.0)
    dims = padded_dims = (0, 0, 0)


def _real_grid(system, xi):
    return _RealOnlyGrid()


def real_space_sum(system, params: RealSpaceParams, targets=None, target_indices=None) -> VelocityResult:
    """Truncated screened sum plus self term (ewald_real.py:381-455), on the GPU."""
    if targets is None:
        tas, tg, tc, nt = True, None, None, system.n
    else:
        tas = False
        tg = np.atleast_2d(np.asarray(targets, float))
        nt = tg.shape[0]
        tc = None if target_indices is None else np.asarray(target_indices, dtype=np.int64)
    grid = _real_grid(system, params.xi)
    ev = get_evaluator(system.kind, system.geometry, system.box_length, params.xi, params.rc, grid, system.n, nt, tas)
    sa, sb = (system.f, None) if system.kind == STOKESLET else (system.g, system.q)
    _, ur, _, _ = ev.execute(system.positions, sa, sb, targets=tg, tcols=tc, what=1)
    uk = np.empty((nt, 3))
    uc = np.empty((nt, 3))
    _lib.check(ev.lib.hs_plan_real_parts(ev.handle, uk.ctypes.data_as(C.c_void_p), uc.ctypes.data_as(C.c_void_p),
                                         _lib.HS_MEM_HOST))
    return VelocityResult(velocities=ur, parts={"kernel": uk, "correction": uc},
                          meta={"kind": system.kind, "geometry": system.geometry, "xi": params.xi, "rc": params.rc})
