"""Single-point kernel helpers of the reference's public API (host NumPy; not on the hot path).

The reference exports, next to its sums, the closed-form kernels for one displacement
(ref:kernels_direct.py:36-92,93-197; ref:ewald_real.py:79-98,115-150).  The GPU path
evaluates the same expressions inside csrc/pair.cu; these host versions keep
`hsewald.stokeslet(...)`-style calls working for callers that switch packages.  Same
names, arguments, conventions and errors as the reference; the algebra is written
out here independently.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import SingularityError
from .system import ROTLET, STOKESLET, STRESSLET

_PI4 = 4.0 * math.pi
_PI8 = 8.0 * math.pi
_MIRROR = np.array([1.0, 1.0, -1.0])


def _disp(r, what="kernel evaluated at zero displacement"):
    r = np.asarray(r, dtype=float)
    n = float(np.linalg.norm(r))
    if n == 0.0:
        raise SingularityError(what)
    return r, n


def stokeslet(r) -> np.ndarray:
    """S(r) = (I/|r| + r r^T/|r|^3) / (8 pi)   (ref:kernels_direct.py:44-47)."""
    r, n = _disp(r)
    return (np.eye(3) + np.outer(r, r) / (n * n)) / (_PI8 * n)


def stresslet_apply(r, g, q) -> np.ndarray:
    """T(r) : (g q^T) = -6 r (r.g)(r.q) / |r|^5 / (8 pi)   (ref:kernels_direct.py:50-55)."""
    r, n = _disp(r)
    rg, rq = float(r @ np.asarray(g, float)), float(r @ np.asarray(q, float))
    return r * (-6.0 * rg * rq / (_PI8 * n ** 5))


def rotlet_apply(r, g, q) -> np.ndarray:
    """2 W(r) (g x q) = 2 (g x q) x r / |r|^3 / (4 pi)   (ref:kernels_direct.py:58-62)."""
    r, n = _disp(r)
    w = np.cross(np.asarray(g, float), np.asarray(q, float))
    return np.cross(w, r) * (2.0 / (_PI4 * n ** 3))


@dataclass
class HarmonicDerivs:
    """G = 1/(4 pi |r|) and its first three derivative tensors (ref:kernels_direct.py:65-72)."""

    G: float
    gradG: np.ndarray
    hessG: np.ndarray
    thirdG: np.ndarray


def harmonic_derivs(r) -> HarmonicDerivs:
    """Derivatives of 1/(4 pi |r|) (ref:kernels_direct.py:75-90)."""
    r, n = _disp(r)
    u = r / n
    I = np.eye(3)
    sym = np.einsum("ij,k->ijk", I, u) + np.einsum("ik,j->ijk", I, u) + np.einsum("jk,i->ijk", I, u)
    return HarmonicDerivs(
        G=1.0 / (_PI4 * n),
        gradG=-u / (_PI4 * n * n),
        hessG=(3.0 * np.outer(u, u) - I) / (_PI4 * n ** 3),
        thirdG=(3.0 * sym - 15.0 * np.einsum("i,j,k->ijk", u, u, u)) / (_PI4 * n ** 4))


def phi_channels(kind, y, f=None, g=None, q=None):
    """Wall-correction channels (s, v, M) per source, phi = s G + v.grad G + M:hess G with G
    centred at the image (ref:kernels_direct.py:93-127).  Inputs (n, 3)."""
    y = np.atleast_2d(np.asarray(y, float))
    n = y.shape[0]
    h = y[:, 2]
    s, v, M = np.zeros(n), np.zeros((n, 3)), np.zeros((n, 3, 3))
    if kind == STOKESLET:
        f = np.atleast_2d(np.asarray(f, float))
        s = -f[:, 2]
        v = -(h[:, None] * (f * _MIRROR))
    elif kind == STRESSLET:
        gm = np.atleast_2d(np.asarray(g, float)) * _MIRROR
        qm = np.atleast_2d(np.asarray(q, float)) * _MIRROR
        v[:, 2] = 2.0 * np.einsum("ij,ij->i", gm, qm)
        gq = gm[:, :, None] * qm[:, None, :]
        M = -(h[:, None, None] * (gq + np.swapaxes(gq, 1, 2)))
    elif kind == ROTLET:
        g = np.atleast_2d(np.asarray(g, float))
        q = np.atleast_2d(np.asarray(q, float))
        v = 4.0 * (q[:, 2:3] * (g * _MIRROR) - g[:, 2:3] * (q * _MIRROR))
    else:
        raise ValueError(f"unknown kind {kind!r}")
    return s, v, M


def gfam_coeffs(r, screen=None):
    """Radial coefficients (c0..c3) with G = c0, grad G = -c1 r, hess G = -c1 I + c2 r r, ...
    (ref:kernels_direct.py:130-151); screen = (f, f1, f2, f3) of erf(xi r)/r subtracts the
    smooth part (the screened real-space family)."""
    r = np.asarray(r, float)
    a = 1.0 / r
    a2 = a * a
    c = [a, a2 * a, 3.0 * a2 * a2 * a, -15.0 * a2 * a2 * a2 * a]
    if screen is None:
        return tuple(c)
    f, f1, f2, f3 = screen
    return (c[0] - f, c[1] + f1 * a, c[2] + f1 * a2 * a - f2 * a2,
            c[3] - 3.0 * f1 * a2 * a2 * a + 3.0 * f2 * a2 * a2 - f3 * a2 * a)


def phi_and_grad(d, coeffs, s, v, M):
    """(phi, grad phi) of the correction potential in the 4 pi G convention (ref:kernels_direct.py:154-172)."""
    c0, c1, c2, c3 = coeffs
    dv = np.einsum("...i,...i->...", d, v)
    tr = np.trace(M, axis1=-2, axis2=-1)
    Md = np.einsum("...ij,...j->...i", M, d)
    dM = np.einsum("...j,...ji->...i", d, M)
    dMd = np.einsum("...i,...i->...", Md, d)
    phi = s * c0 - c1 * (dv + tr) + c2 * dMd
    coef_d = -c1 * s + c2 * dv + c2 * tr + c3 * dMd
    grad = coef_d[..., None] * d - c1[..., None] * v + c2[..., None] * (Md + dM)
    return phi, grad


def correction_phi(kind, y, x, f=None, g=None, q=None):
    """(phi, grad phi) / (4 pi) of one source's wall correction at x (ref:kernels_direct.py:175-197)."""
    y = np.asarray(y, float)
    d = np.asarray(x, float) - y * _MIRROR
    rn = float(np.linalg.norm(d))
    if rn == 0.0:
        raise SingularityError("evaluation point coincides with an image")
    one = lambda a: None if a is None else np.asarray(a, float)[None, :]  # noqa: E731
    s, v, M = phi_channels(kind, y[None, :], f=one(f), g=one(g), q=one(q))
    phi, grad = phi_and_grad(d[None, :], gfam_coeffs(np.array([rn])), s, v, M)
    return phi[0] / _PI4, grad[0] / _PI4


def kernel_real(kind, r, xi):
    """Screened (erfc) kernel tensor at displacement r, raw convention (ref:ewald_real.py:115-150):
    3x3 for the stokeslet / rotlet, 3x3x3 for the stresslet."""
    from scipy.special import erfc
    r, n = _disp(r, "kernel_real evaluated at zero displacement")
    u = r / n
    x = xi * n
    E = math.exp(-x * x)
    C = float(erfc(x))
    k = 2.0 * xi / math.sqrt(math.pi)
    I = np.eye(3)
    if kind == STOKESLET:
        a = k * E + C / n
        return a * (I + np.outer(u, u)) - 2.0 * k * E * I
    if kind == STRESSLET:
        c1 = -(2.0 / n) * (3.0 * C / n + k * (3.0 + 2.0 * x * x) * E)
        c2 = 2.0 * k * xi * xi * E
        T = c1 * np.einsum("j,l,m->jlm", u, u, u)
        T = T + c2 * (np.einsum("jl,m->jlm", I, r) + np.einsum("lm,j->jlm", I, r) + np.einsum("mj,l->jlm", I, r))
        return T
    if kind == ROTLET:
        dd = C / (n * n) + k * E / n
        # epsilon_{jlm} u_m
        W = np.array([[0.0, u[2], -u[1]], [-u[2], 0.0, u[0]], [u[1], -u[0], 0.0]])
        return 2.0 * dd * W
    raise ValueError(f"unknown kind {kind!r}")


def harmonic_real_derivs(r, xi) -> HarmonicDerivs:
    """Screened harmonic family G, grad G, hess G, third G at displacement r, raw 4 pi G = 1/r
    convention (ref:ewald_real.py:152-168): the radial coefficients with the erf(xi r)/r part
    removed, assembled into the tensors of the closed forms above."""
    from .ewald_real import f_derivs
    r = np.asarray(r, dtype=float)
    rn = float(np.linalg.norm(r))
    if rn == 0.0:
        raise SingularityError("harmonic_real_derivs at zero displacement")
    c0, c1, c2, c3 = (float(c[0]) for c in gfam_coeffs(np.array([rn]), screen=f_derivs(np.array([rn]), xi)))
    I = np.eye(3)
    sym = np.einsum("ij,k->ijk", I, r) + np.einsum("ik,j->ijk", I, r) + np.einsum("jk,i->ijk", I, r)
    return HarmonicDerivs(G=c0, gradG=-c1 * r, hessG=-c1 * I + c2 * np.outer(r, r),
                          thirdG=c2 * sym + c3 * np.einsum("i,j,k->ijk", r, r, r))


def correction_phi_real(kind, y, x, xi, f=None, g=None, q=None):
    """Screened wall correction (phi_R, grad phi_R) of one source at x, raw 4 pi convention
    (ref:ewald_real.py:171-190); the pair kernel evaluates the same per image pair."""
    from .ewald_real import f_derivs
    y = np.asarray(y, float)
    d = np.asarray(x, float) - y * _MIRROR
    rn = float(np.linalg.norm(d))
    if rn == 0.0:
        raise SingularityError("evaluation point coincides with an image")
    one = lambda a: None if a is None else np.asarray(a, float)[None, :]  # noqa: E731
    s, v, M = phi_channels(kind, y[None, :], f=one(f), g=one(g), q=one(q))
    phi, grad = phi_and_grad(d[None, :], gfam_coeffs(np.array([rn]), screen=f_derivs(np.array([rn]), xi)), s, v, M)
    return float(phi[0]), grad[0]
