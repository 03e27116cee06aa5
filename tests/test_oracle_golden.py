"""Pin the CPU oracle against golden vectors produced by the reference itself."""

import numpy as np
import pytest

from conftest import golden, rel_l2

KINDS = ("stokeslet", "stresslet", "rotlet")


def _sys(d, key):
    kw = {"pos": d[f"{key}_pos"]}
    if f"{key}_f" in d:
        kw["f"] = d[f"{key}_f"]
    else:
        kw["g"], kw["q"] = d[f"{key}_g"], d[f"{key}_q"]
    return kw


def test_cell_lists_bit_exact(oracle):
    d = golden("cell_lists")
    for name in d["names"]:
        dims, edge, order, start = oracle.build_cell_list(d[f"{name}_pts"], float(d[f"{name}_rc"]),
                                                          d[f"{name}_lo"], d[f"{name}_hi"])
        np.testing.assert_array_equal(dims, d[f"{name}_dims"])
        np.testing.assert_array_equal(edge, d[f"{name}_edge"])
        np.testing.assert_array_equal(order, d[f"{name}_order"])
        np.testing.assert_array_equal(start, d[f"{name}_start"])


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("geom", ("half", "free"))
def test_real_space(oracle, kind, geom):
    d = golden("real_space")
    key = f"{kind}_{geom}"
    s = _sys(d, key)
    u, uk, uc = oracle.real_space_sum(kind, geom, 2.0, s["pos"], 3.0, 0.9, f=s.get("f"), g=s.get("g"),
                                      q=s.get("q"))
    assert rel_l2(u, d[f"{key}_u"]) < 1e-13
    assert rel_l2(uk, d[f"{key}_uk"]) < 1e-13
    if geom == "half":
        assert rel_l2(uc, d[f"{key}_uc"]) < 1e-13


@pytest.mark.parametrize("kind", KINDS)
def test_real_space_separate_targets(oracle, kind):
    d = golden("real_space")
    s = _sys(d, f"{kind}_half")
    u, _, _ = oracle.real_space_sum(kind, "half", 2.0, s["pos"], 3.0, 0.9, f=s.get("f"), g=s.get("g"),
                                    q=s.get("q"), targets=d[f"{kind}_targets_tg"])
    assert rel_l2(u, d[f"{kind}_targets_u"]) < 1e-13


@pytest.mark.parametrize("geom", ("half", "free"))
def test_spread_gather(oracle, geom):
    d = golden("gridding")
    L, M, P, xi = d[f"{geom}_grid"]
    g = oracle.Grid(L, int(M), int(P), xi, geom)
    grids = oracle.spread(d[f"{geom}_pts"], d[f"{geom}_w"], g)
    assert rel_l2(grids, d[f"{geom}_grids"]) < 1e-14
    out = oracle.gather(d[f"{geom}_F"], d[f"{geom}_pts"], g)
    assert rel_l2(out, d[f"{geom}_gather"]) < 1e-14


@pytest.mark.parametrize("geom", ("half", "free"))
@pytest.mark.parametrize("kind", ("harmonic", "biharmonic"))
def test_tables(oracle, geom, kind):
    d = golden("tables")
    g = oracle.Grid(1.0, 6, 6, 4.0, geom)
    s = oracle.precompute_greens(kind, g)
    np.testing.assert_array_equal(s.shape, d[f"{geom}_{kind}_shape"])
    assert rel_l2(s[::3, ::3, ::3], d[f"{geom}_{kind}_sub"]) < 1e-13
    ref = d[f"{geom}_{kind}_sum"]
    np.testing.assert_allclose([s.sum(), (s * s).sum(), np.abs(s).max()], ref, rtol=1e-12)


def _tables(oracle, kind, grid):
    return {t: oracle.precompute_greens(t, grid) for t in oracle.table_kinds_for(kind, grid.geometry)}


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("geom", ("half", "free"))
def test_fourier(oracle, kind, geom):
    d = golden("fourier")
    key = f"{kind}_{geom}"
    s = _sys(d, key)
    g = oracle.Grid(2.0, 12, 8, 3.0, geom)
    u, counts = oracle.fourier_space_sum(kind, geom, s["pos"], g, _tables(oracle, kind, g), f=s.get("f"),
                                         g=s.get("g"), q=s.get("q"))
    assert rel_l2(u, d[f"{key}_u"]) < 1e-12
    assert tuple(counts) == tuple(d[f"{key}_counts"])


def test_ewald_cfg1(oracle):
    """BASELINE configs[0] end to end against the reference's own ewald_sum."""
    d = golden("ewald")
    g = oracle.Grid(1.0, 64, 24, 12.0, "half")
    u, ur, uf = oracle.ewald_sum("stokeslet", "half", 1.0, d["cfg1_pos"], 12.0, 0.35, 64, 24,
                                 _tables(oracle, "stokeslet", g), f=d["cfg1_f"], workers=8)
    assert rel_l2(ur, d["cfg1_ureal"]) < 1e-13
    assert rel_l2(uf, d["cfg1_ufourier"]) < 1e-12
    assert rel_l2(u, d["cfg1_u"]) < 1e-12


@pytest.mark.parametrize("kind", KINDS)
def test_direct(oracle, kind):
    d = golden("direct")
    s = _sys(d, kind)
    u = oracle.direct_sum(kind, "half", s["pos"], f=s.get("f"), g=s.get("g"), q=s.get("q"))
    assert rel_l2(u, d[f"{kind}_u"]) < 1e-13
    uw = oracle.direct_sum(kind, "half", s["pos"], f=s.get("f"), g=s.get("g"), q=s.get("q"), targets=d[f"{kind}_wall"])
    np.testing.assert_allclose(uw, d[f"{kind}_uwall"], atol=1e-12 * np.abs(d[f"{kind}_u"]).max())
    sf = _sys(d, f"{kind}_free")
    uf = oracle.direct_sum(kind, "free", sf["pos"], f=sf.get("f"), g=sf.get("g"), q=sf.get("q"))
    assert rel_l2(uf, d[f"{kind}_free_u"]) < 1e-13


# ---------------------------------------------------------------------------
# Full-size reference goldens (tests/golden/make_fullsize_golden.py: the reference's own ewald_sum
# on the whole HL / cfg2 / cfg3 / cfg1 systems, 2000-target subsets)

def _full(name):
    from paper_1802_07844_b200.configs import WORKLOADS, make_system
    w = WORKLOADS[name]
    s, _ = make_system(w)
    kw = {"f": s.f} if s.kind == "stokeslet" else {"g": s.g, "q": s.q}
    return w, s, kw, golden(f"fullsize_{name}")


@pytest.mark.parametrize("name", ("cfg1", "cfg2", "cfg3", "HL"))
def test_neighbour_audit_vs_reference(oracle, name):
    """The oracle's per-target neighbour sets (count, image count, id hash) equal the reference
    traversal's (ref:ewald_real.py:277-299) bit for bit."""
    w, s, kw, d = _full(name)
    idx = d["idx"]
    aud = np.zeros((idx.size, 3), np.uint64)
    u, _, _ = oracle.real_space_sum(s.kind, "half", w.L, s.positions, w.xi, w.rc, targets=s.positions[idx],
                                    target_indices=idx, audit=aud, **kw)
    np.testing.assert_array_equal(aud[:, 0].astype(np.int64), d["nbr_count"])
    np.testing.assert_array_equal(aud[:, 1].astype(np.int64), d["nbr_img"])
    np.testing.assert_array_equal(aud[:, 2], d["nbr_hash"])
    assert rel_l2(u, d["u_real"]) < 1e-13


def _lean_vs_reference(oracle, name):
    w, s, kw, d = _full(name)
    idx = d["idx"]
    g = oracle.Grid(w.L, w.M, w.P, w.xi)
    tabs = {k: oracle.precompute_greens_half(k, g) for k in oracle.table_kinds_for(s.kind, "half")}
    u, ur, uf = oracle.ewald_sum_lean(s.kind, "half", w.L, s.positions, w.xi, w.rc, w.M, w.P, tabs,
                                      targets=s.positions[idx], target_indices=idx, **kw)
    print(f"lean oracle vs reference {name}: u {rel_l2(u, d['u']):.2e} fourier {rel_l2(uf, d['u_fourier']):.2e}")
    assert rel_l2(ur, d["u_real"]) < 1e-13
    assert rel_l2(u, d["u"]) < 1e-10 and rel_l2(uf, d["u_fourier"]) < 1e-10


def test_lean_oracle_vs_reference_cfg2(oracle):
    """The memory-lean oracle (R2C, one channel at a time; used for the cfg4 / cfg5 goldens) against
    the reference's full-size cfg2 evaluation."""
    _lean_vs_reference(oracle, "cfg2")


@pytest.mark.slow
@pytest.mark.parametrize("name", ("cfg3", "HL"))
def test_lean_oracle_vs_reference_fullsize(oracle, name):
    _lean_vs_reference(oracle, name)


def test_lean_tables_match_full_precompute(oracle):
    """precompute_greens_half (separable cosine transforms) == the reference-layout big-grid
    irfftn path, on the R2C half grid."""
    for geom in ("half", "free"):
        g = oracle.Grid(1.0, 48, 16, 10.0, geom)
        nzh = g.padded_dims[2] // 2 + 1
        for kind in ("harmonic", "biharmonic"):
            a = oracle.precompute_greens(kind, g)[..., :nzh]
            b = oracle.precompute_greens_half(kind, g)
            assert np.abs(a - b).max() < 1e-14 * np.abs(a).max()
