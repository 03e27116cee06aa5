"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container (the reference is not present on GPU boxes):
    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_golden \
        python tests/golden/make_golden.py
Outputs tests/golden/*.npz (inputs + reference outputs).  These pin both the
CPU oracle (oracle/hsoracle.py) and the CUDA path.
"""

import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))

import hsewald  # noqa: E402  (the reference, from PYTHONPATH)
from hsewald import ewald_fourier as ref_f  # noqa: E402
from hsewald import ewald_real as ref_r  # noqa: E402
from hsewald.ewald import EwaldParams, ewald_sum  # noqa: E402
from hsewald.kernels_direct import direct_sum_free, direct_sum_half  # noqa: E402
from hsewald.system import PointSystem  # noqa: E402

from paper_1802_07844_b200.configs import make_system  # noqa: E402  (seeded generators only)

KINDS = ("stokeslet", "stresslet", "rotlet")


def sys_arrays(s):
    d = {"pos": s.positions}
    if s.kind == "stokeslet":
        d["f"] = s.f
    else:
        d["g"], d["q"] = s.g, s.q
    return d


def cell_lists():
    out = {}
    rng = np.random.default_rng(7)
    cases = {}
    cases["rand"] = (rng.uniform(0.0, 1.0, (500, 3)), 0.17, np.zeros(3), np.ones(3))
    s = hsewald.generate_system(300, 1.5, "stokeslet", "half", seed=4)
    img = hsewald.reflect(s)
    cases["half"] = (img.combined_positions, 0.15, np.array([0.0, 0.0, -1.5]), np.array([1.5, 1.5, 1.5]))
    edge = 0.125
    grid = np.stack(np.meshgrid(*[np.arange(9) * edge] * 3, indexing="ij"), -1).reshape(-1, 3)
    extra = np.array([[0.0, 0.0, 0.0], [1.0, 1.0, 1.0], [1.0 + 5e-13, 0.5, -5e-13], [0.375, 0.625, 0.999999999999]])
    cases["faces"] = (np.vstack([grid, extra]), 0.125, np.zeros(3), np.ones(3))
    z = np.minimum(0.005 + rng.exponential(0.05, 400), np.nextafter(1.0, 0))
    cl = np.column_stack([rng.uniform(0, 1, 400), rng.uniform(0, 1, 400), z])
    cases["cluster"] = (np.vstack([cl, cl * [1, 1, -1]]), 0.05, np.array([0.0, 0.0, -1.0]), np.ones(3))
    cases["onecell"] = (rng.uniform(0.0, 2.0, (50, 3)), 5.0, np.zeros(3), np.full(3, 2.0))
    for name, (pts, rc, lo, hi) in cases.items():
        c = ref_r.build_cell_list(pts, rc, (lo, hi))
        out.update({f"{name}_pts": pts, f"{name}_rc": rc, f"{name}_lo": lo, f"{name}_hi": hi,
                    f"{name}_order": c.order, f"{name}_start": c.start, f"{name}_dims": c.dims,
                    f"{name}_edge": c.edge})
    np.savez_compressed(os.path.join(HERE, "cell_lists.npz"), names=np.array(list(cases)), **out)


def real_space():
    out = {}
    for kind in KINDS:
        for geom, n in (("half", 80), ("free", 60)):
            s = hsewald.generate_system(n, 2.0, kind, geom, seed=5)
            p = ref_r.RealSpaceParams(xi=3.0, rc=0.9)
            r = ref_r.real_space_sum(s, p)
            key = f"{kind}_{geom}"
            for k, v in sys_arrays(s).items():
                out[f"{key}_{k}"] = v
            out[f"{key}_u"] = r.velocities
            out[f"{key}_uk"] = r.parts["kernel"]
            out[f"{key}_uc"] = r.parts["correction"]
        # separate targets, no target indices (no self skip / self term)
        s = hsewald.generate_system(80, 2.0, kind, "half", seed=5)
        tg = np.random.default_rng(9).uniform([0, 0, 0.05], [2, 2, 1.9], (30, 3))
        r = ref_r.real_space_sum(s, ref_r.RealSpaceParams(xi=3.0, rc=0.9), targets=tg)
        out[f"{kind}_targets_tg"] = tg
        out[f"{kind}_targets_u"] = r.velocities
    np.savez_compressed(os.path.join(HERE, "real_space.npz"), **out)


def gridding():
    out = {}
    rng = np.random.default_rng(11)
    for geom, (L, M, P, xi) in (("free", (2.0, 12, 8, 3.0)), ("half", (2.0, 10, 8, 3.0))):
        g = ref_f.GridSpec(L=L, M=M, P=P, xi=xi, geometry=geom)
        lo = [0.3, 0.3, -1.6] if geom == "half" else [0.3] * 3
        pts = rng.uniform(lo, [1.7, 1.7, 1.7], (9, 3))
        w = rng.normal(size=(9, 2))
        grids = ref_f.spread(pts, w, g)
        F = rng.normal(size=(3,) + g.dims)
        gat = ref_f.gather(F, pts, g)
        out.update({f"{geom}_pts": pts, f"{geom}_w": w, f"{geom}_grids": grids, f"{geom}_F": F,
                    f"{geom}_gather": gat, f"{geom}_grid": np.array([L, M, P, xi])})
    np.savez_compressed(os.path.join(HERE, "gridding.npz"), **out)


def tables():
    out = {}
    for geom in ("half", "free"):
        g = ref_f.GridSpec(L=1.0, M=6, P=6, xi=4.0, geometry=geom)
        for kind in ("harmonic", "biharmonic"):
            t = ref_f.precompute_greens(kind, g)
            s = t.samples
            out[f"{geom}_{kind}_sub"] = s[::3, ::3, ::3]
            out[f"{geom}_{kind}_sum"] = np.array([s.sum(), (s * s).sum(), np.abs(s).max()])
            out[f"{geom}_{kind}_shape"] = np.array(s.shape)
    np.savez_compressed(os.path.join(HERE, "tables.npz"), **out)


def fourier():
    out = {}
    for kind in KINDS:
        for geom in ("half", "free"):
            s = hsewald.generate_system(30, 2.0, kind, geom, seed=13)
            g = ref_f.GridSpec(L=2.0, M=12, P=8, xi=3.0, geometry=geom)
            r = ref_f.fourier_space_sum(s, g)
            key = f"{kind}_{geom}"
            for k, v in sys_arrays(s).items():
                out[f"{key}_{k}"] = v
            out[f"{key}_u"] = r.velocities
            out[f"{key}_counts"] = np.array([r.meta["fft_count"], r.meta["ifft_count"]])
    np.savez_compressed(os.path.join(HERE, "fourier.npz"), **out)


def ewald():
    out = {}
    # BASELINE configs[0] (cfg1): N=1000 stokeslet, xi=12, rc=0.35, M=64, P=24
    s, _ = make_system("cfg1")
    params = EwaldParams(xi=12.0, rc=0.35, M=64, P=24)
    r = ewald_sum(s, params)
    out.update({"cfg1_pos": s.positions, "cfg1_f": s.f, "cfg1_u": r.velocities, "cfg1_ureal": r.parts["real"],
                "cfg1_ufourier": r.parts["fourier"]})
    # the two other kernels at a smaller configuration
    for kind in ("stresslet", "rotlet"):
        s = hsewald.generate_system(200, 1.0, kind, "half", seed=17)
        params = EwaldParams(xi=8.0, rc=0.45, M=24, P=16)
        r = ewald_sum(s, params)
        for k, v in sys_arrays(s).items():
            out[f"{kind}_{k}"] = v
        out[f"{kind}_u"] = r.velocities
    # separate targets with target indices (mixed semantics)
    s = hsewald.generate_system(150, 1.0, "stokeslet", "half", seed=19)
    tg = np.vstack([s.positions[:20], np.random.default_rng(3).uniform([0, 0, 0.02], [1, 1, 0.98], (20, 3))])
    ti = np.concatenate([np.arange(20), np.full(20, -1)])
    r = ewald_sum(s, EwaldParams(xi=8.0, rc=0.45, M=24, P=16), targets=tg, target_indices=ti)
    out.update({"mixed_pos": s.positions, "mixed_f": s.f, "mixed_tg": tg, "mixed_ti": ti, "mixed_u": r.velocities})
    np.savez_compressed(os.path.join(HERE, "ewald.npz"), **out)


def direct():
    out = {}
    for kind in KINDS:
        s = hsewald.generate_system(50, 2.0, kind, "half", seed=21)
        wall = np.column_stack([np.random.default_rng(22).uniform(0, 2, (20, 2)), np.zeros(20)])
        for k, v in sys_arrays(s).items():
            out[f"{kind}_{k}"] = v
        out[f"{kind}_u"] = direct_sum_half(s).velocities
        out[f"{kind}_wall"] = wall
        out[f"{kind}_uwall"] = direct_sum_half(s, targets=wall).velocities
        sf = hsewald.generate_system(40, 2.0, kind, "free", seed=23)
        for k, v in sys_arrays(sf).items():
            out[f"{kind}_free_{k}"] = v
        out[f"{kind}_free_u"] = direct_sum_free(sf).velocities
    np.savez_compressed(os.path.join(HERE, "direct.npz"), **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["cell_lists", "real_space", "gridding", "tables", "fourier", "ewald", "direct"]
    for w in which:
        print("generating", w, flush=True)
        globals()[w]()
