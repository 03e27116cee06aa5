"""North-star parity at the BASELINE configurations' FULL sizes, and bit-exact neighbour sets.

* Velocities: the GPU evaluates the whole system (targets = all sources, as the metric does);
  the values at a seeded 2000-target subset must match, to relative L2 <= 1e-10
  (BASELINE.json north star), the REFERENCE's own ewald_sum (ref:ewald.py:46-80) run on the
  same full system in the build container (tests/golden/make_fullsize_golden.py: HL N=1e6
  M=192, cfg2 N=1e5, cfg3 stresslet N=1e5, cfg1) or -- for the configurations whose full
  complex spectra exceed that container's memory (cfg4 rotlet N=1e6 M=320, cfg5 mixed 4e6 + 4e6
  targets M=384) -- the memory-lean CPU oracle (oracle/hsoracle.py ewald_sum_lean, pinned to the
  reference goldens in tests/test_oracle_golden.py; tests/golden/make_lean_golden.py).
* Neighbour sets: per-target [accepted pairs, accepted image pairs, sum of splitmix64(id)] of the
  CUDA pair pass (hs_plan_pair_audit) must equal the reference traversal's
  (ref:ewald_real.py:277-299, closed ball r2 <= rc^2, self skipped by index) exactly: against the
  reference-derived goldens, the oracle at the clustered cfg4, and a constructed case with
  source-target distances at r_c and one ulp either side.
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN, golden, rel_l2

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _workload(name):
    from paper_1802_07844_b200.configs import WORKLOADS, make_system
    w = WORKLOADS[name]
    s, tg = make_system(w)
    return w, s, tg


def _evaluator(gpu, w, s, nt=None, tas=True):
    from paper_1802_07844_b200._plan import get_evaluator
    p = gpu.EwaldParams(xi=w.xi, rc=w.rc, M=w.M, P=w.P)
    grid = p.grid(w.L, "half")
    ev = get_evaluator(s.kind, "half", w.L, w.xi, w.rc, grid, s.n, s.n if nt is None else nt, tas)
    if not ev.tables_ready:
        ev.build_tables()
    return ev


def _strengths(s):
    return (s.f, None) if s.kind == "stokeslet" else (s.g, s.q)


@pytest.mark.parametrize("name", ("cfg1", "cfg2", "cfg3", "HL"))
def test_fullsize_vs_reference(gpu, name):
    d = golden(f"fullsize_{name}")
    w, s, _ = _workload(name)
    idx = d["idx"]
    r = gpu.ewald_sum(s, gpu.EwaldParams(xi=w.xi, rc=w.rc, M=w.M, P=w.P))
    e_u = rel_l2(r.velocities[idx], d["u"])
    e_r = rel_l2(r.parts["real"][idx], d["u_real"])
    e_f = rel_l2(r.parts["fourier"][idx], d["u_fourier"])
    print(f"{name}: rel L2 u {e_u:.2e} real {e_r:.2e} fourier {e_f:.2e}")
    assert e_r < 1e-12
    assert e_u < TOL and e_f < TOL
    # the reference's own FFT counts (ref:ewald_fourier.py:522-531) are reported unchanged
    assert (r.meta["fft_count"], r.meta["ifft_count"]) == tuple(int(v) for v in d["fft_counts"])


@pytest.mark.parametrize("name", ("cfg1", "cfg2", "cfg3", "HL"))
def test_neighbour_sets_vs_reference(gpu, name):
    d = golden(f"fullsize_{name}")
    w, s, _ = _workload(name)
    ev = _evaluator(gpu, w, s)
    sa, sb = _strengths(s)
    aud = ev.pair_audit(s.positions, sa, sb)
    idx = d["idx"]
    np.testing.assert_array_equal(aud[idx, 0].astype(np.int64), d["nbr_count"])
    np.testing.assert_array_equal(aud[idx, 1].astype(np.int64), d["nbr_img"])
    np.testing.assert_array_equal(aud[idx, 2], d["nbr_hash"])


def test_neighbour_sets_clustered_cfg4_vs_oracle(gpu, oracle):
    """Wall-clustered rotlet at full size (1e6): dense image neighbourhoods near z = 0."""
    w, s, _ = _workload("cfg4")
    ev = _evaluator(gpu, w, s)
    aud = ev.pair_audit(s.positions, s.g, s.q)
    rng = np.random.default_rng(11)
    # bias the subset toward the wall, where image pairs are most numerous
    near = np.nonzero(s.positions[:, 2] < 2 * w.rc)[0]
    idx = np.unique(np.concatenate([rng.choice(near, 1500, replace=False), rng.choice(s.n, 1500, replace=False)]))
    ref = np.zeros((idx.size, 3), np.uint64)
    oracle.real_space_sum("rotlet", "half", w.L, s.positions, w.xi, w.rc, g=s.g, q=s.q,
                          targets=s.positions[idx], target_indices=idx, audit=ref)
    np.testing.assert_array_equal(aud[idx], ref)
    assert ref[:, 1].mean() > 10    # the subset really exercises image pairs


def _shell_case(rc=0.101, L=1.0, n_pairs=300, seed=5):
    """Targets with sources at exactly r2 == rc*rc (as the reference rounds it) and one ulp of
    the source coordinate either side, in random directions, plus their images near the wall."""
    rng = np.random.default_rng(seed)
    rc2 = rc * rc
    tg, src = [], []
    for _ in range(n_pairs):
        t = np.array([rng.uniform(0.2, 0.8), rng.uniform(0.2, 0.8), rng.uniform(0.02, 0.9)])
        v = rng.normal(size=3)
        v /= np.linalg.norm(v)
        if t[2] + rc * v[2] <= 1e-3 or t[2] + rc * v[2] >= 0.999:
            v[2] = -v[2]
        ax = int(np.argmax(np.abs(v)))
        y = t + rc * v
        # walk the dominant coordinate by ulps until r2 (reference rounding) crosses rc2
        def r2(yy):
            d = t - yy
            return d[0] * d[0] + d[1] * d[1] + d[2] * d[2]
        step = np.sign(v[ax])
        for _ in range(200):
            if r2(y) > rc2:
                y[ax] = np.nextafter(y[ax], y[ax] - step)
            else:
                nxt = y.copy()
                nxt[ax] = np.nextafter(y[ax], y[ax] + step)
                if r2(nxt) <= rc2:
                    y = nxt
                else:
                    break
        # y: last inside (r2 <= rc2); its neighbour one ulp outward is outside
        out = y.copy()
        out[ax] = np.nextafter(y[ax], y[ax] + step)
        inn = y.copy()
        inn[ax] = np.nextafter(y[ax], y[ax] - step)
        assert r2(y) <= rc2 < r2(out) and r2(inn) <= rc2
        tg.append(t)
        src += [y, out, inn]
    pos = np.vstack([np.array(tg), np.array(src)])
    pos[:, :2] = np.clip(pos[:, :2], 0.0, np.nextafter(L, 0))
    return pos


def test_neighbour_sets_rc_shell_exact(gpu, oracle):
    """Sources at r2 == rc^2 (accepted: closed ball) and one ulp outside / inside."""
    rc, xi, L = 0.101, 49.92, 1.0
    pos = _shell_case(rc, L)
    n = pos.shape[0]
    f = np.random.default_rng(1).normal(size=(n, 3))
    s = gpu.PointSystem(kind="stokeslet", geometry="half", box_length=L, positions=pos, f=f)
    from paper_1802_07844_b200._plan import get_evaluator
    grid = gpu.GridSpec(L=L, M=64, P=16, xi=xi, geometry="half")
    ev = get_evaluator("stokeslet", "half", L, xi, rc, grid, n, n, True)
    aud = ev.pair_audit(pos, f)
    ref = np.zeros((n, 3), np.uint64)
    oracle.real_space_sum("stokeslet", "half", L, pos, xi, rc, f=f, audit=ref)
    np.testing.assert_array_equal(aud, ref)
    # every constructed target keeps its r2 == rc^2 and inner partners and drops the outer one
    assert ref[:300, 0].min() >= 2


@pytest.mark.parametrize("name", ("cfg4", "cfg5"))
def test_fullsize_vs_lean_oracle(gpu, oracle, name):
    """cfg4 / cfg5 at full size vs the lean oracle's fixture.  Both sides use the ORACLE's
    Green's tables (ewald_sum(tables=...), as the reference's API takes them): the two sides'
    independently computed tables agree to ~5e-16 of their maximum (checked here), but this
    configuration amplifies that round-off to ~1e-10 in u (tools/table_sensitivity.py,
    DESIGN.md section 2.2), so the evaluation itself is compared on identical tables."""
    import os as _os
    from paper_1802_07844_b200 import _plan
    path = os.path.join(GOLDEN, f"fullsize_{name}.npz")
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: generate it with tests/golden/make_lean_golden.py on a large-memory host")
    d = np.load(path)
    w, s, tg = _workload(name)
    idx = d["idx"]
    p = gpu.EwaldParams(xi=w.xi, rc=w.rc, M=w.M, P=w.P)
    grid = p.grid(w.L, "half")
    go = oracle.Grid(w.L, w.M, w.P, w.xi)
    oracle.set_threads(_os.cpu_count())
    tables = {}
    for k in gpu.table_kinds_for(s.kind, "half"):
        half = oracle.precompute_greens_half(k, go, workers=_os.cpu_count())
        mine = gpu.precompute_greens(k, grid, max_bytes=None).samples[..., : half.shape[2]]
        assert np.abs(mine - half).max() < 1e-14 * np.abs(half).max()
        del mine
        tables[k] = gpu.GreensTable(kind=k, R=grid.R, Ltilde=grid.Ltilde, dims=tuple(grid.padded_dims),
                                    samples=oracle.expand_half_table(half, grid.padded_dims))
        del half
    _plan.clear_cache()
    try:
        if name == "cfg5":
            from paper_1802_07844_b200.ewald import ewald_sum_mixed
            r = ewald_sum_mixed(s, p, tables=tables, targets=tg)
        else:
            r = gpu.ewald_sum(s, p, tables=tables)
    finally:
        del tables
    e_u = rel_l2(r.velocities[idx], d["u"])
    e_r = rel_l2(r.parts["real"][idx], d["u_real"])
    e_f = rel_l2(r.parts["fourier"][idx], d["u_fourier"])
    print(f"{name}: rel L2 u {e_u:.2e} real {e_r:.2e} fourier {e_f:.2e}")
    _plan.clear_cache()
    assert e_r < 1e-12
    assert e_u < TOL and e_f < TOL
