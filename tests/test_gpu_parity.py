"""Parity of the CUDA path (through the C ABI) against the reference's golden
vectors and the CPU oracle.  Tolerances: bit-exact for cell lists (integer
work); relative L2 <= 1e-10 for FP64 velocities (BASELINE.json north star)."""

import numpy as np
import pytest

from conftest import golden, rel_l2

pytestmark = pytest.mark.gpu
KINDS = ("stokeslet", "stresslet", "rotlet")
TOL = 1e-10


def _system(hs, d, key, L, geom="half"):
    kw = dict(kind=None, geometry=geom, box_length=L, positions=d[f"{key}_pos"])
    if f"{key}_f" in d:
        kw.update(kind="stokeslet", f=d[f"{key}_f"])
    else:
        kw.update(g=d[f"{key}_g"], q=d[f"{key}_q"])
    return kw


def _mk(hs, kind, d, key, L, geom="half"):
    kw = _system(hs, d, key, L, geom)
    kw["kind"] = kind
    return hs.PointSystem(**kw)


def test_cell_lists_bit_exact(gpu):
    d = golden("cell_lists")
    for name in d["names"]:
        c = gpu.build_cell_list(d[f"{name}_pts"], float(d[f"{name}_rc"]), (d[f"{name}_lo"], d[f"{name}_hi"]))
        np.testing.assert_array_equal(c.dims, d[f"{name}_dims"])
        np.testing.assert_array_equal(c.edge, d[f"{name}_edge"])
        np.testing.assert_array_equal(c.order, d[f"{name}_order"], err_msg=name)
        np.testing.assert_array_equal(c.start, d[f"{name}_start"], err_msg=name)


def test_cell_list_large_vs_oracle(gpu, oracle):
    from paper_1802_07844_b200.configs import make_system
    s, _ = make_system("cfg4", n=200_000)     # wall-clustered: long segments
    zz = np.vstack([s.positions, s.positions * [1, 1, -1]])
    for rc in (0.0466, 0.02, 0.3):
        c = gpu.build_cell_list(zz, 0.5 * rc, (np.array([0, 0, -1.0]), np.ones(3)))
        dims, edge, order, start = oracle.build_cell_list(zz, 0.5 * rc, np.array([0, 0, -1.0]), np.ones(3))
        np.testing.assert_array_equal(c.order, order)
        np.testing.assert_array_equal(c.start, start)


def test_cell_list_bounds_error(gpu):
    with pytest.raises(gpu.GeometryError):
        gpu.build_cell_list(np.array([[0.5, 0.5, 1.5]]), 0.2, (np.zeros(3), np.ones(3)))


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("geom", ("half", "free"))
def test_real_space_golden(gpu, kind, geom):
    d = golden("real_space")
    key = f"{kind}_{geom}"
    s = _mk(gpu, kind, d, key, 2.0, geom)
    r = gpu.real_space_sum(s, gpu.RealSpaceParams(xi=3.0, rc=0.9))
    assert rel_l2(r.velocities, d[f"{key}_u"]) < 1e-12
    assert rel_l2(r.parts["kernel"], d[f"{key}_uk"]) < 1e-12
    if geom == "half":
        assert rel_l2(r.parts["correction"], d[f"{key}_uc"]) < 1e-11


@pytest.mark.parametrize("kind", KINDS)
def test_real_space_separate_targets(gpu, kind):
    d = golden("real_space")
    s = _mk(gpu, kind, d, f"{kind}_half", 2.0)
    r = gpu.real_space_sum(s, gpu.RealSpaceParams(xi=3.0, rc=0.9), targets=d[f"{kind}_targets_tg"])
    assert rel_l2(r.velocities, d[f"{kind}_targets_u"]) < 1e-12


@pytest.mark.parametrize("kind", KINDS)
def test_real_space_vs_oracle_cfg_scale(gpu, oracle, kind):
    from paper_1802_07844_b200.configs import make_system
    name = {"stokeslet": "cfg2", "stresslet": "cfg3", "rotlet": "cfg4"}[kind]
    s, _ = make_system(name, n=20_000)
    xi, rc = 20.0, 0.2
    r = gpu.real_space_sum(s, gpu.RealSpaceParams(xi=xi, rc=rc))
    kw = {"f": s.f} if kind == "stokeslet" else {"g": s.g, "q": s.q}
    u, uk, uc = oracle.real_space_sum(kind, "half", 1.0, s.positions, xi, rc, **kw)
    assert rel_l2(r.velocities, u) < 1e-11
    assert rel_l2(r.parts["correction"], uc) < 1e-10


def test_real_space_singular(gpu):
    pos = np.array([[0.5, 0.5, 0.5], [0.5, 0.5, 0.5], [0.2, 0.3, 0.4]])
    s = gpu.PointSystem(kind="stokeslet", geometry="half", box_length=1.0, positions=pos, f=np.ones((3, 3)))
    with pytest.raises(gpu.SingularityError):
        gpu.real_space_sum(s, gpu.RealSpaceParams(xi=3.0, rc=0.4))


def test_real_space_rc_zero_self_term(gpu):
    d = golden("real_space")
    s = _mk(gpu, "stokeslet", d, "stokeslet_half", 2.0)
    r = gpu.real_space_sum(s, gpu.RealSpaceParams(xi=3.0, rc=0.0))
    expect = -(4.0 * 3.0 / np.sqrt(np.pi)) * s.f / (8 * np.pi)
    np.testing.assert_allclose(r.velocities, expect, rtol=1e-14)


@pytest.mark.parametrize("geom", ("half", "free"))
def test_spread_gather_golden(gpu, geom):
    d = golden("gridding")
    L, M, P, xi = d[f"{geom}_grid"]
    g = gpu.GridSpec(L=L, M=int(M), P=int(P), xi=xi, geometry=geom)
    grids = gpu.spread(d[f"{geom}_pts"], d[f"{geom}_w"], g)
    assert rel_l2(grids, d[f"{geom}_grids"]) < 1e-13
    out = gpu.gather(d[f"{geom}_F"], d[f"{geom}_pts"], g)
    assert rel_l2(out, d[f"{geom}_gather"]) < 1e-13


def test_spread_gather_adjoint_and_mass(gpu):
    rng = np.random.default_rng(5)
    g = gpu.GridSpec(L=2.0, M=40, P=24, xi=8.0, geometry="half")
    pts = rng.uniform([0.2, 0.2, -1.8], [1.8, 1.8, 1.8], (500, 3))
    w = rng.normal(size=(500, 3))
    grids = gpu.spread(pts, w, g)
    np.testing.assert_allclose(grids.sum(axis=(1, 2, 3)) * g.h**3, w.sum(axis=0), rtol=1e-7)
    F = rng.normal(size=(3,) + g.dims)
    lhs = np.sum(grids * F) * g.h**3
    rhs = np.sum(w * gpu.gather(F, pts, g))
    np.testing.assert_allclose(lhs, rhs, rtol=1e-12)


def test_spread_out_of_grid(gpu):
    g = gpu.GridSpec(L=1.0, M=16, P=8, xi=4.0, geometry="free")
    with pytest.raises(gpu.GeometryError):
        gpu.spread(np.array([[2.5, 0.5, 0.5]]), np.ones((1, 1)), g)


@pytest.mark.parametrize("tg", ([[0.25, np.nextafter(1.0, 0.0), 0.5]],
                                [[0.5, 0.5, 0.5], [0.25, np.nextafter(1.0, 0.0), 0.5]]))
def test_gather_target_window_leaving_grid_raises(gpu, tg):
    """A target whose window leaves the grid (y = 1 - ulp rounds to the top node) raises
    GeometryError like the reference's gather (_gridding.py:50-52) -- also when it is alone in
    its work item (regression: an all-inactive item must not touch memory)."""
    from paper_1802_07844_b200.configs import make_system
    s, _ = make_system("cfg3", n=3000)
    p = gpu.EwaldParams(xi=33.28, rc=0.12, M=128, P=24)
    with pytest.raises(gpu.GeometryError):
        gpu.ewald_sum(s, p, targets=np.array(tg))
    # the context stays usable
    r = gpu.ewald_sum(s, p, targets=np.array([[0.5, 0.5, 0.5]]))
    assert np.all(np.isfinite(r.velocities))


@pytest.mark.parametrize("geom", ("half", "free"))
@pytest.mark.parametrize("kind", ("harmonic", "biharmonic"))
def test_tables_golden(gpu, geom, kind):
    d = golden("tables")
    g = gpu.GridSpec(L=1.0, M=6, P=6, xi=4.0, geometry=geom)
    s = gpu.precompute_greens(kind, g).samples
    np.testing.assert_array_equal(s.shape, d[f"{geom}_{kind}_shape"])
    assert rel_l2(s[::3, ::3, ::3], d[f"{geom}_{kind}_sub"]) < 1e-12
    np.testing.assert_allclose([s.sum(), (s * s).sum(), np.abs(s).max()], d[f"{geom}_{kind}_sum"], rtol=1e-11)


def test_tables_vs_oracle_cfg1(gpu, oracle):
    g = gpu.GridSpec(L=1.0, M=64, P=24, xi=12.0)
    og = oracle.Grid(1.0, 64, 24, 12.0)
    for kind in ("harmonic", "biharmonic"):
        s = gpu.precompute_greens(kind, g, max_bytes=None).samples
        assert rel_l2(s, oracle.precompute_greens(kind, og, workers=8)) < 1e-12


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("geom", ("half", "free"))
def test_fourier_golden(gpu, kind, geom):
    d = golden("fourier")
    key = f"{kind}_{geom}"
    s = _mk(gpu, kind, d, key, 2.0, geom)
    g = gpu.GridSpec(L=2.0, M=12, P=8, xi=3.0, geometry=geom)
    r = gpu.fourier_space_sum(s, g)
    assert rel_l2(r.velocities, d[f"{key}_u"]) < TOL
    assert (r.meta["fft_count"], r.meta["ifft_count"]) == tuple(d[f"{key}_counts"])


def test_ewald_cfg1_golden(gpu):
    """BASELINE configs[0] through ewald_sum vs the reference's own output (rel L2 <= 1e-10)."""
    d = golden("ewald")
    s = gpu.PointSystem(kind="stokeslet", geometry="half", box_length=1.0, positions=d["cfg1_pos"], f=d["cfg1_f"])
    r = gpu.ewald_sum(s, gpu.EwaldParams(xi=12.0, rc=0.35, M=64, P=24))
    assert rel_l2(r.parts["real"], d["cfg1_ureal"]) < 1e-12
    assert rel_l2(r.parts["fourier"], d["cfg1_ufourier"]) < TOL
    assert rel_l2(r.velocities, d["cfg1_u"]) < TOL


@pytest.mark.parametrize("kind", ("stresslet", "rotlet"))
def test_ewald_kinds_golden(gpu, kind):
    d = golden("ewald")
    s = _mk(gpu, kind, d, kind, 1.0)
    r = gpu.ewald_sum(s, gpu.EwaldParams(xi=8.0, rc=0.45, M=24, P=16))
    assert rel_l2(r.velocities, d[f"{kind}_u"]) < TOL


def test_ewald_mixed_targets_golden(gpu):
    d = golden("ewald")
    s = gpu.PointSystem(kind="stokeslet", geometry="half", box_length=1.0, positions=d["mixed_pos"], f=d["mixed_f"])
    r = gpu.ewald_sum(s, gpu.EwaldParams(xi=8.0, rc=0.45, M=24, P=16), targets=d["mixed_tg"],
                      target_indices=d["mixed_ti"])
    assert rel_l2(r.velocities, d["mixed_u"]) < TOL


@pytest.mark.parametrize("kind", KINDS)
def test_direct_golden(gpu, kind):
    d = golden("direct")
    s = _mk(gpu, kind, d, kind, 2.0)
    assert rel_l2(gpu.direct_sum_half(s).velocities, d[f"{kind}_u"]) < 1e-13
    uw = gpu.direct_sum_half(s, targets=d[f"{kind}_wall"]).velocities
    assert np.abs(uw).max() <= 1e-12 * np.abs(d[f"{kind}_u"]).max()   # no-slip at the wall
    sf = _mk(gpu, kind, d, f"{kind}_free", 2.0, "free")
    assert rel_l2(gpu.direct_sum_free(sf).velocities, d[f"{kind}_free_u"]) < 1e-13


@pytest.mark.parametrize("kind", KINDS)
def test_ewald_vs_direct_and_oracle_2e4(gpu, oracle, kind):
    """Moderate size: GPU ewald vs CPU oracle (same algorithm) and vs direct sum."""
    from paper_1802_07844_b200.configs import make_system
    name = {"stokeslet": "cfg2", "stresslet": "cfg3", "rotlet": "cfg4"}[kind]
    s, _ = make_system(name, n=20_000)
    xi, rc, M, P = 20.8, 0.17, 80, 24
    r = gpu.ewald_sum(s, gpu.EwaldParams(xi=xi, rc=rc, M=M, P=P))
    g = oracle.Grid(1.0, M, P, xi)
    tabs = {t: oracle.precompute_greens(t, g, workers=8) for t in oracle.table_kinds_for(kind, "half")}
    kw = {"f": s.f} if kind == "stokeslet" else {"g": s.g, "q": s.q}
    sub = np.arange(0, s.n, 97)
    u_or, _, _ = oracle.ewald_sum(kind, "half", 1.0, s.positions, xi, rc, M, P, tabs, targets=s.positions[sub],
                                  target_indices=sub, workers=8, **kw)
    assert rel_l2(r.velocities[sub], u_or) < TOL
    ud = gpu.direct_sum_half(s, targets=s.positions[sub], target_indices=sub).velocities
    assert rel_l2(r.velocities[sub], ud) < 2e-5   # truncation error at xi*rc = 3.5


def test_fourier_linearity_full_size(gpu):
    """Size-independent property at the headline grid: Fourier part is linear in the strengths."""
    from paper_1802_07844_b200.configs import make_system
    s, _ = make_system("HL", n=200_000)
    g = gpu.GridSpec(L=1.0, M=192, P=24, xi=49.92)
    u1 = gpu.fourier_space_sum(s, g).velocities
    u3 = gpu.fourier_space_sum(s.scaled(-3.0), g).velocities
    assert rel_l2(u3, -3.0 * u1) < 1e-13


def test_ewald_deterministic(gpu):
    from paper_1802_07844_b200.configs import make_system
    s, _ = make_system("cfg2", n=30_000)
    p = gpu.EwaldParams(xi=20.8, rc=0.17, M=80, P=24)
    a = gpu.ewald_sum(s, p).velocities
    b = gpu.ewald_sum(s, p).velocities
    np.testing.assert_array_equal(a, b)


def test_concurrent_pipelines_bitwise_equal_serial(gpu):
    """The default evaluation runs the real-space pipeline on a second stream concurrently with
    the Fourier pipeline; serialised (what bit 2) it must give the same bits, parts included."""
    from paper_1802_07844_b200._plan import get_evaluator
    from paper_1802_07844_b200.configs import make_system
    from paper_1802_07844_b200.ewald_fourier import prepare_tables
    s, _ = make_system("cfg3", n=30_000)
    p = gpu.EwaldParams(xi=20.8, rc=0.17, M=80, P=24)
    g = p.grid(1.0, "half")
    ev = get_evaluator(s.kind, s.geometry, 1.0, p.xi, p.rc, g, s.n, s.n, True)
    prepare_tables(ev, s, g, None, None)
    u1, r1, f1, _ = ev.execute(s.positions, s.g, s.q, what=3)
    u2, r2, f2, _ = ev.execute(s.positions, s.g, s.q, what=7)
    for x, y in ((u1, u2), (r1, r2), (f1, f2)):
        np.testing.assert_array_equal(x, y)


def test_missing_table_rejected(gpu):
    d = golden("fourier")
    s = _mk(gpu, "rotlet", d, "rotlet_half", 2.0)
    g1 = gpu.GridSpec(L=2.0, M=12, P=8, xi=3.0)
    g2 = gpu.GridSpec(L=2.0, M=16, P=8, xi=3.0)
    tabs = gpu.get_tables("rotlet", g1)
    with pytest.raises(gpu.ConfigError):
        gpu.fourier_space_sum(s, g2, tables=tabs)


def _subset_direct_check(gpu, s, targets, p, nsub=400, tol=1e-6):
    sub = np.arange(0, s.n if targets is None else targets.shape[0], max(1, (s.n if targets is None else targets.shape[0]) // nsub))
    ew = gpu.ewald_sum
    if s.kind == "mixed":
        from paper_1802_07844_b200.ewald import ewald_sum_mixed as ew
    if targets is None:
        r = ew(s, p)
        ud = gpu.direct_sum_half(s, targets=s.positions[sub], target_indices=sub).velocities
        return rel_l2(r.velocities[sub], ud)
    r = ew(s, p, targets=targets)
    ud = gpu.direct_sum_half(s, targets=targets[sub]).velocities
    return rel_l2(r.velocities[sub], ud)


def test_cfg2_full_vs_oracle_subset(gpu, oracle):
    """BASELINE configs[1] (N=1e5 stokeslet, balanced parameters) against the CPU oracle
    on a 2000-target subset (full-size spreading and FFTs on the oracle side)."""
    from paper_1802_07844_b200.configs import WORKLOADS, make_system
    w = WORKLOADS["cfg2"]
    s, _ = make_system(w)
    r = gpu.ewald_sum(s, gpu.EwaldParams(xi=w.xi, rc=w.rc, M=w.M, P=w.P))
    g = oracle.Grid(w.L, w.M, w.P, w.xi)
    tabs = {t: oracle.precompute_greens(t, g, workers=16) for t in oracle.table_kinds_for("stokeslet", "half")}
    sub = np.arange(0, s.n, 50)
    u, _, _ = oracle.ewald_sum("stokeslet", "half", w.L, s.positions, w.xi, w.rc, w.M, w.P, tabs, f=s.f,
                               targets=s.positions[sub], target_indices=sub, workers=16)
    assert rel_l2(r.velocities[sub], u) < TOL


@pytest.mark.parametrize("name", ("cfg3", "cfg4"))
def test_configs_vs_direct_subset(gpu, name):
    """BASELINE configs[2] (stresslet 1e5) and configs[3] (wall-clustered rotlet 1e6) at full size:
    Ewald vs the O(N Nt) direct half-space sum on a target subset (truncation-level agreement)."""
    from paper_1802_07844_b200.configs import WORKLOADS, make_system
    w = WORKLOADS[name]
    s, _ = make_system(w)
    err = _subset_direct_check(gpu, s, None, gpu.EwaldParams(xi=w.xi, rc=w.rc, M=w.M, P=w.P), nsub=300)
    # the method's truncation error at these parameters (measured 1.0e-11 cfg3, 1.9e-10 cfg4);
    # parity with the reference itself is tests/test_fullsize_parity.py
    assert err < 5e-10, err


def test_target_sharded_matches_unsharded(gpu):
    """Single-device emulation of the target-sharded multi-GPU evaluation (sharding.py):
    the shards' slices, evaluated independently, reassemble the unsharded result."""
    from paper_1802_07844_b200.configs import make_system
    from paper_1802_07844_b200.sharding import shard_bounds
    s, _ = make_system("cfg2", n=40_000)
    p = gpu.EwaldParams(xi=20.8, rc=0.17, M=80, P=24)
    full = gpu.ewald_sum(s, p).velocities
    parts = []
    for r in range(3):
        lo, hi = shard_bounds(s.n, 3, r)
        parts.append(gpu.ewald_sum(s, p, targets=s.positions[lo:hi], target_indices=np.arange(lo, hi)).velocities)
    assert rel_l2(np.concatenate(parts), full) < 1e-13


def _stress_targets(rng, L, h, n_rand=50):
    """Target layouts that exercise the gather's run / item cutting: a z line with gaps
    (single-target runs), a dense cluster (full runs and items), points at the wall and
    near the top, two targets far apart in one 4x4 block, and a ragged random tail."""
    line = np.column_stack([np.full(40, 0.31 * L), np.full(40, 0.47 * L),
                            np.linspace(0.01 * L, 0.99 * L, 40) ** 1.7 / L ** 0.7])
    cluster = np.array([0.6 * L, 0.2 * L, 0.5 * L]) + 1e-3 * h * rng.standard_normal((137, 3))
    wall = np.column_stack([rng.uniform(0, L, (9, 2)), np.zeros(9)])
    top = np.column_stack([rng.uniform(0, L, (5, 2)), np.full(5, L * (1 - 1e-9))])
    far = np.array([[0.5 * L, 0.5 * L, 0.02 * L], [0.5 * L + 0.5 * h, 0.5 * L, 0.97 * L]])
    rand = rng.uniform(0, L, (n_rand, 3))
    return np.vstack([line, cluster, wall, top, far, rand])


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("nt", (1, 7, 33, None))
def test_fourier_gather_layouts_vs_oracle(gpu, oracle, kind, nt):
    """Fourier part at separate targets of awkward layouts vs the CPU oracle (and the
    target-set independence of the per-target result)."""
    from paper_1802_07844_b200.configs import make_system
    name = {"stokeslet": "cfg2", "stresslet": "cfg3", "rotlet": "cfg4"}[kind]
    s, _ = make_system(name, n=3000)
    M, P, xi = 40, 24, 10.0
    rng = np.random.default_rng(11)
    tg = _stress_targets(rng, 1.0, 1.0 / M)
    if nt is not None:
        tg = tg[rng.permutation(len(tg))[:nt]]
    r = gpu.fourier_space_sum(s, gpu.GridSpec(L=1.0, M=M, P=P, xi=xi), targets=tg)
    g = oracle.Grid(1.0, M, P, xi)
    tabs = {t: oracle.precompute_greens(t, g, workers=8) for t in oracle.table_kinds_for(kind, "half")}
    kw = {"f": s.f} if kind == "stokeslet" else {"g": s.g, "q": s.q}
    u_or = oracle.fourier_space_sum(kind, "half", s.positions, g, tabs, targets=tg, workers=8, **kw)
    u_or = u_or[0] if isinstance(u_or, tuple) else u_or
    assert rel_l2(r.velocities, u_or) < TOL
    if nt is None:   # per-target results do not depend on the rest of the target set
        sub = np.arange(0, len(tg), 3)
        r2 = gpu.fourier_space_sum(s, gpu.GridSpec(L=1.0, M=M, P=P, xi=xi), targets=tg[sub])
        assert rel_l2(r2.velocities, r.velocities[sub]) < 1e-13


@pytest.mark.parametrize("kind,M", [(k, m) for k in KINDS for m in (192, 128)] + [("stokeslet", 384),
                                                                                  ("rotlet", 320), ("stresslet", 320)])
@pytest.mark.parametrize("alt", ("HS_XSTAGE_STOCKHAM", "HS_YSTAGE_CUFFT", "HS_ZSTAGE_CUFFT"))
def test_register_fft_stages_match_alternatives(tmp_path, kind, M, alt):
    """The register-FFT x stage and y stage (N = 480 = 15 x 32 at M=192, 352 = 11 x 32 at
    M=128, 864 = 27 x 32 at M=384, 750 = 30 x 25 at M=320) against the shared-memory Stockham x stage / the cuFFT y stage on the same input
    (each selected in its own process); the register z stage (924 = 2 x 22 x 21 real points at
    M=192, 660 = 2 x 22 x 15 at M=128, 1440 = 2 x 30 x 24 at M=320, 1680 = 2 x 30 x 28 at M=384, with
    the fused reflection and channel interleave) against the cuFFT D2Z / Z2D with the mirror and
    interleave passes."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    tool = os.path.join(root, "tools", "xstage_ab.py")
    a, b = tmp_path / "reg.npy", tmp_path / "stockham.npy"
    subprocess.run([sys.executable, tool, str(a), kind, str(M)], check=True)
    env = dict(os.environ, **{alt: "1"})
    subprocess.run([sys.executable, tool, str(b), kind, str(M)], check=True, env=env)
    ua, ub = np.load(a), np.load(b)
    assert rel_l2(ua, ub) < 1e-12


def test_register_z_stage_free_space_matches_cufft(tmp_path):
    """The register z stage with 3 output channels (free space: pitch-4 interleave) and nz = 428 < 432
    (M = 404 -> padded z length 924) against the cuFFT z stage + interleave pass."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    tool = os.path.join(root, "tools", "xstage_ab.py")
    a, b = tmp_path / "reg.npy", tmp_path / "cufft.npy"
    subprocess.run([sys.executable, tool, str(a), "free", "404"], check=True)
    subprocess.run([sys.executable, tool, str(b), "free", "404"], check=True, env=dict(os.environ, HS_ZSTAGE_CUFFT="1"))
    ua, ub = np.load(a), np.load(b)
    assert np.isfinite(ua).all() and rel_l2(ua, ub) < 1e-12


@pytest.mark.parametrize("kind", ("harmonic", "biharmonic"))
def test_separable_tables_match_full_grid(tmp_path, kind):
    """The separable pruned table precompute against the 3-D big-grid transform (each selected
    in its own process) on a moderate grid."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    tool = os.path.join(root, "tools", "table_ab.py")
    a, b = tmp_path / "sep.npy", tmp_path / "full.npy"
    subprocess.run([sys.executable, tool, str(a), kind, "64"], check=True)
    subprocess.run([sys.executable, tool, str(b), kind, "64"], check=True, env=dict(os.environ, HS_TABLE_FULL="1"))
    ta, tb = np.load(a), np.load(b)
    assert rel_l2(ta, tb) < 1e-12


def test_cfg5_full_size_vs_direct_subset(gpu):
    """BASELINE configs[4] (4e6 stokeslet + stresslet sources, 4e6 separate targets, L=2, M=384:
    padded grid (864,864,1680), one mixed plan, separable table precompute) at full size against
    the direct half-space sums of both kinds on a target subset."""
    from paper_1802_07844_b200.configs import WORKLOADS, make_system
    from paper_1802_07844_b200 import _plan
    _plan.clear_cache()
    w = WORKLOADS["cfg5"]
    s, tg = make_system(w)
    try:
        err = _subset_direct_check(gpu, s, tg, gpu.EwaldParams(xi=w.xi, rc=w.rc, M=w.M, P=w.P), nsub=200)
    finally:
        _plan.clear_cache()   # release the ~150 GB plan
    assert err < 5e-10, err


@pytest.mark.parametrize("geom", ("half", "free"))
@pytest.mark.parametrize("sep", (False, True))
def test_mixed_plan_equals_sum_of_kinds(gpu, oracle, geom, sep):
    """One mixed plan (both kinds' pairs in one pass, kernel + shared wall channels summed in
    k-space, one gather) == the reference's two ewald_sum calls (oracle) and the two single-kind
    GPU plans."""
    from paper_1802_07844_b200.ewald import MixedSystem, ewald_sum_mixed
    rng = np.random.default_rng(21)
    n, L = 3000, 1.0
    pos = np.column_stack([rng.uniform(0, L, n), rng.uniform(0, L, n), rng.uniform(0.01, 0.99, n)])
    f, g = rng.normal(size=(n, 3)), rng.normal(size=(n, 3))
    q = rng.normal(size=(n, 3))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    a = gpu.PointSystem(kind="stokeslet", geometry=geom, box_length=L, positions=pos, f=f)
    b = gpu.PointSystem(kind="stresslet", geometry=geom, box_length=L, positions=pos, g=g, q=q)
    m = MixedSystem(a, b)
    p = gpu.EwaldParams(xi=14.0, rc=0.3, M=48, P=16)
    tg = np.column_stack([rng.uniform(0, L, 500), rng.uniform(0, L, 500), rng.uniform(0.01, 0.99, 500)]) if sep \
        else None
    r = ewald_sum_mixed(m, p, targets=tg)
    ra, rb = gpu.ewald_sum(a, p, targets=tg), gpu.ewald_sum(b, p, targets=tg)
    assert rel_l2(r.velocities, ra.velocities + rb.velocities) < 1e-12
    assert rel_l2(r.parts["real"], ra.parts["real"] + rb.parts["real"]) < 1e-13
    assert (r.meta["fft_count"], r.meta["ifft_count"]) == ((28, 12) if geom == "half" else (12, 6))
    assert r.meta["fft_count_executed"] == ((19, 6) if geom == "half" else (9, 3))
    go = oracle.Grid(L, p.M, p.P, p.xi, geom)
    tabs = {k: oracle.precompute_greens(k, go) for k in ("biharmonic", "harmonic")}
    ua, _, _ = oracle.ewald_sum("stokeslet", geom, L, pos, p.xi, p.rc, p.M, p.P, tabs, f=f, targets=tg)
    ub, _, _ = oracle.ewald_sum("stresslet", geom, L, pos, p.xi, p.rc, p.M, p.P, tabs, g=g, q=q, targets=tg)
    assert rel_l2(r.velocities, ua + ub) < TOL


@pytest.mark.parametrize("P", (28, 30, 32))
def test_fourier_wide_window_support_vs_oracle(gpu, oracle, P):
    """Window supports up to P = 32 (GridSpec accepts them): P <= 29 runs the tensor-pipe gather
    (an item's x / y union, P + 3 nodes, fits its 32-wide tables), P = 30 .. 32 the warp-per-
    target gather; both against the oracle (no silent skips)."""
    s = gpu.generate_system(400, 1.0, "stokeslet", "half", seed=3)
    g = gpu.GridSpec(L=1.0, M=36, P=P, xi=9.0, geometry="half")
    r = gpu.fourier_space_sum(s, g)
    go = oracle.Grid(1.0, g.M, P, 9.0)
    tabs = {k: oracle.precompute_greens(k, go) for k in ("biharmonic", "harmonic")}
    u, _ = oracle.fourier_space_sum("stokeslet", "half", s.positions, go, tabs, f=s.f)
    assert rel_l2(r.velocities, u) < TOL
