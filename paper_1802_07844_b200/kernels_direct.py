"""Exact O(N Nt) direct sums on the GPU (reference: kernels_direct.py:211-371).

The direct sum is the reference's correctness oracle for the fast method; here
it runs as a shared-memory tiled FP64 kernel (csrc/pair.cu:k_direct) reusing
the pair machinery with the unscreened coefficients.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .errors import GeometryError
from .system import HALF_SPACE, STOKESLET, VelocityResult
from .point_kernels import (HarmonicDerivs, correction_phi, gfam_coeffs, harmonic_derivs,  # noqa: F401
                            phi_and_grad, phi_channels, rotlet_apply, stokeslet, stresslet_apply)


def _direct(system, geometry, targets, target_indices):
    if system.kind == "mixed":   # ewald.MixedSystem: the two kinds' sums
        return (_direct(system.stokeslet, geometry, targets, target_indices)
                + _direct(system.stresslet, geometry, targets, target_indices))
    if targets is None:
        targets = system.positions
        target_indices = np.arange(system.n)
    tg = np.ascontiguousarray(np.atleast_2d(np.asarray(targets, float)))
    tc = None if target_indices is None else np.ascontiguousarray(np.asarray(target_indices, np.int64))
    sa, sb = (system.f, None) if system.kind == STOKESLET else (system.g, system.q)
    pos = np.ascontiguousarray(system.positions, float)
    sa = np.ascontiguousarray(sa, float)
    sb = None if sb is None else np.ascontiguousarray(sb, float)
    u = np.empty((tg.shape[0], 3))
    ctx = _lib.Context.get()
    ctx.bind_stream(None)
    vp = lambda x: x.ctypes.data_as(C.c_void_p) if x is not None else None  # noqa: E731
    _lib.check(ctx.lib.hs_direct_sum(ctx.handle, _lib.KIND_ID[system.kind], _lib.GEOM_ID[geometry], system.n,
                                     vp(pos), vp(sa), vp(sb), tg.shape[0], vp(tg), vp(tc), vp(u), _lib.HS_MEM_HOST))
    return u


def direct_sum_free(system, targets=None, target_indices=None) -> VelocityResult:
    u = _direct(system, "free", targets, target_indices)
    return VelocityResult(velocities=u, meta={"kind": system.kind, "geometry": "free", "n": system.n})


def direct_sum_half(system, targets=None, target_indices=None) -> VelocityResult:
    if system.geometry != HALF_SPACE:
        raise GeometryError("direct_sum_half requires a half-space system")
    if targets is not None and np.any(np.atleast_2d(np.asarray(targets, float))[:, 2] < 0):
        raise GeometryError("half-space targets must have x3 >= 0")
    u = _direct(system, "half", targets, target_indices)
    return VelocityResult(velocities=u, meta={"kind": system.kind, "geometry": "half", "n": system.n})
