"""Full-size golden vectors for the configurations whose full complex spectra do not fit the
build container (cfg4: rotlet N=1e6, M=320; cfg5: stokeslet + stresslet N=4e6 with 4e6 separate
targets, L=2, M=384), from the memory-lean CPU oracle (oracle/hsoracle.py ewald_sum_lean: R2C
transforms of one channel at a time, Hermitian part of each output spectrum; tables from
precompute_greens_half).  The lean oracle is pinned to the REFERENCE's own full-size outputs at
HL / cfg2 / cfg3 (tests/test_oracle_golden.py::test_lean_oracle_vs_reference_fullsize).

Run on a host with >= 128 GB of memory (the GPU box: 196 GB, 16 cores; no GPU is used):
    python tests/golden/make_lean_golden.py cfg4 cfg5
cfg5 is BASELINE's mixed case: its reference answer is the sum of two ewald_sum calls, one per
kind (ref:ewald.py:46-80), which is what is stored.  Writes tests/golden/fullsize_<cfg>.npz
(subset indices + velocities; inputs are regenerated from the seeds).
"""

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.join(HERE, "..", "..")
sys.path.insert(0, ROOT)

from oracle import hsoracle as H  # noqa: E402  (test infrastructure)
from paper_1802_07844_b200.configs import WORKLOADS, make_system  # noqa: E402  (seeded generators only)


def subset(n, k=2000, seed=7):
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(n, size=min(k, n), replace=False)).astype(np.int64)


def run(name, workers):
    w = WORKLOADS[name]
    s, tg = make_system(w)
    grid = H.Grid(w.L, w.M, w.P, w.xi)
    nt = s.n if tg is None else tg.shape[0]
    idx = subset(nt)
    t0 = time.perf_counter()
    kinds = ["stokeslet", "stresslet"] if w.kind == "mixed" else [w.kind]
    tabs = {k: H.precompute_greens_half(k, grid, workers=workers) for k in ("biharmonic", "harmonic")
            if k in set(sum((H.table_kinds_for(kk, "half") for kk in kinds), []))}
    t_tab = time.perf_counter() - t0
    u = np.zeros((idx.size, 3))
    ur = np.zeros_like(u)
    uf = np.zeros_like(u)
    info = {}
    for kind in kinds:
        ps = s.stokeslet if kind == "stokeslet" and w.kind == "mixed" else (s.stresslet if w.kind == "mixed" else s)
        kw = {"f": ps.f} if kind == "stokeslet" else {"g": ps.g, "q": ps.q}
        targets = ps.positions[idx] if tg is None else tg[idx]
        tix = idx if tg is None else None
        tm = {}
        t1 = time.perf_counter()
        a, b, c = H.ewald_sum_lean(kind, "half", w.L, ps.positions, w.xi, w.rc, w.M, w.P, tabs, targets=targets,
                                   target_indices=tix, workers=workers, timings=tm, **kw)
        info[kind] = {"s": round(time.perf_counter() - t1, 1), **{k: round(v, 1) for k, v in tm.items()}}
        u += a
        ur += b
        uf += c
    # the reference's own goldens (make_fullsize_golden.py) are never overwritten: other names are
    # written as lean_<cfg>.npz (cross-checks only)
    out = f"fullsize_{name}.npz" if name in ("cfg4", "cfg5") else f"lean_{name}.npz"
    np.savez_compressed(os.path.join(HERE, out), idx=idx, u=u, u_real=ur, u_fourier=uf,
                        params=np.array([w.xi, w.rc, w.M, w.P, w.L]), padded=np.array(grid.padded_dims))
    print(json.dumps({"workload": name, "kinds": kinds, "n": s.n, "n_targets": nt, "subset": int(idx.size),
                      "padded": grid.padded_dims, "tables_s": round(t_tab, 1), "phases_s": info,
                      "threads": H.num_threads()}), flush=True)


if __name__ == "__main__":
    workers = os.cpu_count()
    H.set_threads(workers)
    for name in (sys.argv[1:] or ["cfg4", "cfg5"]):
        run(name, workers)
