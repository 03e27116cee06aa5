"""Seeded synthetic workloads of BASELINE.json.

The reference measures on no public dataset; these generators stand in with the
shapes and distributions BASELINE.json states.  Generator: numpy PCG64
``default_rng(1000 + cfg)`` (the headline HL case uses seed 1000); draw order:
x, y, z of sources; strengths; normals/torques; separate targets.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .system import PointSystem


@dataclass(frozen=True)
class Workload:
    name: str
    kind: str
    n: int
    L: float
    xi: float
    rc: float
    M: int
    P: int
    seed: int
    zdist: str = "uniform01"      # uniform01 | uniform0 | wall_exp
    separate_targets: bool = False


WORKLOADS = {
    # BASELINE configs[0]: the reference's CPU-runnable case
    "cfg1": Workload("cfg1", "stokeslet", 1000, 1.0, 12.0, 0.35, 64, 24, 1001),
    # SURVEY App. B balanced rule xi = 0.26 M / L; rc = estimates.select_rc(kind, 1e-10 * rms(u), xi, L, Q)
    # (reference estimator, ref:estimates.py:105-125; rms(u) from SURVEY App. B)
    "cfg2": Workload("cfg2", "stokeslet", 100_000, 1.0, 33.28, 0.151, 128, 24, 1002),
    "cfg3": Workload("cfg3", "stresslet", 100_000, 1.0, 33.28, 0.163, 128, 24, 1003, zdist="uniform0"),
    "cfg4": Workload("cfg4", "rotlet", 1_000_000, 1.0, 83.2, 0.0555, 320, 24, 1004, zdist="wall_exp"),
    # the metric's configuration: half-space stokeslet, N = 1e6
    "HL": Workload("HL", "stokeslet", 1_000_000, 1.0, 49.92, 0.101, 192, 24, 1000),
    # BASELINE configs[4]: stokeslet + stresslet sources at the same 4e6 points, 4e6 separate targets,
    # L = 2 (the multi-GPU scaling case); one mixed plan (ewald.ewald_sum_mixed)
    "cfg5": Workload("cfg5", "mixed", 4_000_000, 2.0, 49.92, 0.10, 384, 24, 1005, separate_targets=True),
}


def _unit(v):
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def make_system(w: Workload | str, n: int | None = None):
    """Return (PointSystem, targets or None) for a workload (optionally with fewer points);
    kind "mixed" returns an ewald.MixedSystem (stokeslet f, stresslet g / q at the same points)."""
    if isinstance(w, str):
        w = WORKLOADS[w]
    n = w.n if n is None else int(n)
    rng = np.random.default_rng(w.seed)
    L = w.L
    top = np.nextafter(1.0, 0.0)
    x = rng.uniform(0.0, L, n)
    y = rng.uniform(0.0, L, n)
    if w.zdist == "uniform01":
        z = rng.uniform(0.01, 1.0, n)
    elif w.zdist == "uniform0":
        z = rng.uniform(0.0, 1.0, n)
        while np.any(z == 0.0):
            z[z == 0.0] = rng.uniform(0.0, 1.0, int(np.sum(z == 0.0)))
    elif w.zdist == "wall_exp":
        z = np.minimum(0.005 + rng.exponential(0.1, n), top)
    else:
        raise ValueError(w.zdist)
    pos = np.column_stack([x, y, z])
    if w.kind == "mixed":
        from .ewald import MixedSystem
        f = rng.normal(size=(n, 3))
        g = rng.normal(size=(n, 3))
        q = _unit(rng.normal(size=(n, 3)))
        sysm = MixedSystem(
            PointSystem(kind="stokeslet", geometry="half", box_length=L, positions=pos, f=f, seed=w.seed),
            PointSystem(kind="stresslet", geometry="half", box_length=L, positions=pos, g=g, q=q, seed=w.seed))
    elif w.kind == "stokeslet":
        sysm = PointSystem(kind="stokeslet", geometry="half", box_length=L, positions=pos,
                           f=rng.normal(size=(n, 3)), seed=w.seed)
    elif w.kind == "stresslet":
        g = rng.normal(size=(n, 3))
        q = _unit(rng.normal(size=(n, 3)))
        sysm = PointSystem(kind="stresslet", geometry="half", box_length=L, positions=pos, g=g, q=q, seed=w.seed)
    else:
        tau = rng.normal(size=(n, 3))
        e = np.zeros((n, 3))
        use_y = np.abs(tau[:, 0]) > 0.9 * np.linalg.norm(tau, axis=1)
        e[~use_y, 0] = 1.0
        e[use_y, 1] = 1.0
        g = _unit(np.cross(tau, e))
        q = np.cross(tau, g)          # g x q = tau
        sysm = PointSystem(kind="rotlet", geometry="half", box_length=L, positions=pos, g=g, q=q, seed=w.seed)
    targets = None
    if w.separate_targets:
        targets = np.column_stack([rng.uniform(0.0, L, n), rng.uniform(0.0, L, n), rng.uniform(0.01, 1.0, n)])
    return sysm, targets
