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
