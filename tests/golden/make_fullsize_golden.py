"""Full-size golden vectors from the REFERENCE implementation itself (build container only).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_golden \
        python tests/golden/make_fullsize_golden.py [HL cfg2 cfg3 cfg1]

For each BASELINE workload that the reference can hold in this container's 62 GB (HL at
N = 1e6 / M = 192, cfg2 and cfg3 at N = 1e5 / M = 128, cfg1), the reference's own
`ewald_sum` (ref:ewald.py:46-80) is run on the FULL system (every source spread, the full
grid transformed) and gathered at a seeded subset of 2000 targets that are sources
(`targets=pos[idx], target_indices=idx`, so the self-skip and the stokeslet self term apply
exactly as for targets=None).  Inputs are regenerated from the seeds (configs.make_system),
so only indices and outputs are stored: tests/golden/fullsize_<cfg>.npz.

Per-target neighbour audits (`nbr_count`, `nbr_img`, `nbr_hash`) restate the candidate
traversal of ref:ewald_real.py:277-299 in NumPy on the reference's own cell list
(`build_cell_list(src, 0.5 rc, (lo, hi))`, ref:ewald_real.py:428-430): 5x5x5 half-cells
around the target's cell, skip `ids == tcol`, accept `r2 <= rc^2` with
r2 = d0*d0 + d1*d1 + d2*d2 evaluated left to right.  `nbr_hash` = sum of splitmix64(id)
mod 2^64 over the accepted combined source ids (id >= n: image of id - n).  At cfg1 the
counts are cross-checked against the reference's CellList.neighbors_within.
"""

import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))

from hsewald import ewald_fourier as ref_f  # noqa: E402  (the reference, from PYTHONPATH)
from hsewald import ewald_real as ref_r  # noqa: E402
from hsewald.ewald import EwaldParams, ewald_sum  # noqa: E402
from hsewald.system import PointSystem, reflect  # noqa: E402

from paper_1802_07844_b200.configs import WORKLOADS, make_system  # noqa: E402  (seeded generators only)

M64 = (1 << 64) - 1


def splitmix64(x):
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    z = (np.asarray(x, np.uint64) + np.uint64(0x9E3779B97F4A7C15))
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def subset(n, k=2000, seed=7):
    rng = np.random.default_rng(seed)
    if n <= k:
        return np.arange(n, dtype=np.int64)
    return np.sort(rng.choice(n, size=k, replace=False)).astype(np.int64)


def ref_system(s):
    kw = {"f": s.f} if s.kind == "stokeslet" else {"g": s.g, "q": s.q}
    return PointSystem(kind=s.kind, geometry="half", box_length=s.box_length, positions=s.positions, **kw)


def neighbour_audit(rs, rc, targets, tcols):
    """NumPy restatement of the reference traversal (ref:ewald_real.py:277-299)."""
    L = rs.box_length
    img = reflect(rs)
    src = img.combined_positions
    cl = ref_r.build_cell_list(src, 0.5 * rc, (np.array([0.0, 0.0, -L]), np.array([L, L, L])))
    nx, ny, nz = (int(v) for v in cl.dims)
    rc2 = rc * rc
    n = rs.n
    cnt = np.zeros(len(targets), np.int64)
    nimg = np.zeros(len(targets), np.int64)
    hsh = np.zeros(len(targets), np.uint64)
    ids_sorted = cl.order
    for t, (x, tc) in enumerate(zip(targets, tcols)):
        c = [min(max(int((x[k] - cl.origin[k]) / cl.edge[k]), 0), int(cl.dims[k]) - 1) for k in range(3)]
        cand = []
        for ix in range(max(c[0] - 2, 0), min(c[0] + 3, nx)):
            for iy in range(max(c[1] - 2, 0), min(c[1] + 3, ny)):
                f0 = (ix * ny + iy) * nz
                z0, z1 = max(c[2] - 2, 0), min(c[2] + 3, nz)
                cand.append(ids_sorted[cl.start[f0 + z0]:cl.start[f0 + z1]])
        cand = np.concatenate(cand)
        cand = cand[cand != tc]
        d = x[None, :] - src[cand]
        r2 = d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1] + d[:, 2] * d[:, 2]
        acc = cand[r2 <= rc2]
        cnt[t] = acc.size
        nimg[t] = int(np.sum(acc >= n))
        hsh[t] = np.sum(splitmix64(acc), dtype=np.uint64)
    return cnt, nimg, hsh


def run(name):
    w = WORKLOADS[name]
    s, tg = make_system(w)
    assert tg is None, "separate-target workloads are generated on the GPU box (oracle lean mode)"
    rs = ref_system(s)
    idx = subset(s.n)
    params = EwaldParams(xi=w.xi, rc=w.rc, M=w.M, P=w.P)
    grid = params.grid(w.L, "half")
    t0 = time.perf_counter()
    tables = {k: ref_f.precompute_greens(k, grid, max_bytes=1e12) for k in ref_f.table_kinds_for(w.kind, "half")}
    t_tab = time.perf_counter() - t0
    t0 = time.perf_counter()
    res = ewald_sum(rs, params, tables=tables, threads=os.cpu_count(), targets=s.positions[idx], target_indices=idx)
    t_eval = time.perf_counter() - t0
    del tables
    t0 = time.perf_counter()
    cnt, nimg, hsh = neighbour_audit(rs, w.rc, s.positions[idx], idx)
    t_aud = time.perf_counter() - t0
    out = {"idx": idx, "u": res.velocities, "u_real": res.parts["real"], "u_fourier": res.parts["fourier"],
           "nbr_count": cnt, "nbr_img": nimg, "nbr_hash": hsh,
           "params": np.array([w.xi, w.rc, w.M, w.P, w.L]), "padded": np.array(grid.padded_dims),
           "fft_counts": np.array([res.meta["fft_count"], res.meta["ifft_count"]])}
    if name == "cfg1":
        # cross-check the traversal restatement with the reference's own closed-ball query
        img = reflect(rs)
        L = w.L
        cl = ref_r.build_cell_list(img.combined_positions, w.rc, (np.array([0.0, 0.0, -L]), np.array([L, L, L])))
        q = np.array([np.sum(cl.neighbors_within(x) != i) for i, x in zip(idx, s.positions[idx])])
        assert np.array_equal(q, cnt), "traversal restatement disagrees with CellList.neighbors_within"
    np.savez_compressed(os.path.join(HERE, f"fullsize_{name}.npz"), **out)
    print(f"{name}: N={s.n} subset={idx.size} padded={grid.padded_dims} tables {t_tab:.1f}s eval {t_eval:.1f}s "
          f"audit {t_aud:.1f}s mean pairs {cnt.mean():.1f} (images {nimg.mean():.2f}) times "
          f"{ {k: round(v, 2) for k, v in res.meta['times'].items()} }", flush=True)


if __name__ == "__main__":
    for name in (sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "HL"]):
        run(name)
